"""PHG strand-vertex steps/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config Cx]

One step = one trace of this rank's seed batch: every seed
integrated to termination through the field, kept vertices scanned and
gathered into the CSR payload (K1 + K2), plus -- at N > 1 -- the final
all-gather of per-rank (strands, vertices) that yields global CSR offsets.
Steps are counted as the reference counts them: sum over returned strands of
(len(vertices) - 1), summed over every rank.

Workload: C3 (512^3 curly field, 1M seeds) at one GPU, the config BASELINE.json's
metric is quoted on; at N > 1 the default is C4, BASELINE's scaling sweep: 4M
global seeds split over the ranks ("strong" scaling).  --config C3 at N > 1 fixes
1M seeds per GPU ("weak").  One process per GPU (torchrun), field replicated,
contiguous rank slices of the seed list.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_STEP = 2 * 8 * 16 + 1 + 24  # 2 samples x 8 float4 corners + cap probe + f64 vertex
METRIC = "PHG strand-vertex steps/sec at 1/2/4/8 B200 (512³ field, 1M seeds)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="C1..C5 (default: C3 at one GPU, C4's 4M-seed strong split at N > 1)")
    ap.add_argument("--dist-backend", default="auto", choices=["auto", "nccl", "gloo"],
                    help="auto: NCCL when every rank has its own GPU, else gloo (ranks sharing a "
                         "device: code-path validation only, not a scaling measurement)")
    ap.add_argument("--seeds", type=int, default=0, help="override seeds per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-root-gather", action="store_true",
                    help="N > 1: skip the peer-memory gather of every rank's CSR to rank 0")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="seeds in the CPU sample")
    ap.add_argument("--sweep", action="store_true", help="time every trace-kernel variant")
    ap.add_argument("--no-driver", action="store_true", help="skip the batch-driver leg")
    ap.add_argument("--sweep-sizes", default=None, metavar="V,V,...",
                    help="time the given trace-kernel variants across launch sizes")
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="seeds per chunk of the pipelined host path (0: library default)")
    return ap.parse_args()


def _native_variants():
    from paper_2604_05794_b200 import _native

    return int(_native.load().phg_num_variants())


def resolve_config(args, ws):
    """BASELINE.json: the metric is quoted on C3 (512^3, 1M seeds) at one GPU; its scaling
    sweep is C4 (512^3, 4M seeds partitioned across 2/4/8 GPUs)."""
    if args.config is None:
        args.config = "C3" if ws == 1 else "C4"
    return args.config


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML polled
    every 2 ms on a thread (a 5-step C3 region lasts ~65 ms), nvidia-smi at 200 ms otherwise."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop_evt = threading.Event()
        self.nvml = None
        self.proc = None

    def _handle(self, nv):
        try:
            import torch

            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop_evt.is_set():
                    try:
                        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                             nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.002)

            self.nvml = nv
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:  # fallback: nvidia-smi loop
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                mask = sum(1 << i for i, v in enumerate(parts[2:6])
                           if v.lower() in ("active", "1", "yes"))
                self.samples.append((float(parts[0]), float(parts[1]), mask))
            except ValueError:
                continue

    def stop(self):
        self.stop_evt.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
            bits = self.bits
        elif self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            bits = {n: 1 << i for i, n in enumerate(self.NAMES)}
        else:
            return None
        if not self.samples:
            return None
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for s in self.samples for n, b in bits.items() if s[2] & b})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)),
                "sm_max_mhz": float(max(s[1] for s in self.samples)), "reasons": reasons,
                "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def cpu_host_info():
    cores = len(os.sched_getaffinity(0))
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:  # noqa: BLE001
        pass
    return cores, model


CPU_SUBSET = 16384  # C2-C5 are timed on the first 16384 seeds, C1 on all


def cpu_sample_seeds(cfg, args, ori_t=None, occ_t=None):
    """The CPU legs' seeds: the first 16384 of the config's own seed list (all of C1's 10k),
    BASELINE.md 2; --cpu-sample overrides."""
    from paper_2604_05794_b200 import synth

    n = args.cpu_sample or (cfg.seeds if cfg.name == "C1" else CPU_SUBSET)
    n = min(n, cfg.seeds)
    seeds, dirs = synth.config_seeds(cfg, cfg.seeds, ori_t, occ_t)  # the workload's own list
    return np.ascontiguousarray(seeds[:n]), np.ascontiguousarray(dirs[:n])


def cpu_sample_note(cfg, n):
    return (f"all {n} seeds of {cfg.name}" if n >= cfg.seeds
            else f"first {n} seeds of {cfg.name}")


def cpu_legs(cfg, ori, occ, seeds, dirs, cores, model, one_core=True, c_port=True):
    """BASELINE.md 2's CPU baseline on this host, on the config's CPU sample:
      * value: the numpy restatement of trace_batch (bit-exact to the reference, the same
        numpy dispatch pattern) in a persistent `cores`-process fork pool -- the most
        CPU-favourable form of the reference's own multi-core path;
      * init_guide_strands: the reference's multi-core path as `strandkit bench` times it
        (cli.py:233-237): init_guide_strands(workers=cores, field_seeds=0), pool made per
        call, serial commit loop (phg.py:210-260);
      * one_core: trace_batch in one process;
      * c_port: our scalar C restatement on all threads (not the reference; context only)."""
    from types import SimpleNamespace

    from oracle import phg_oracle_np as onp  # CPU baseline legs only

    from paper_2604_05794_b200 import synth
    from paper_2604_05794_b200.phg import PhgParams

    params = PhgParams(field_seeds=0, batch_size=max(len(seeds), 1))
    f = onp.Field(np.zeros(3), synth.VOXEL_MM, occ.shape, occ, ori)
    out = {"unit": "steps/s", "cores": cores, "kind": "port"}
    pool = onp.TracePool(f, cores)
    try:
        pool.steps(seeds[: cores * 64], dirs[: cores * 64], params)  # warm the workers
        t0 = time.perf_counter()
        st = pool.steps(seeds, dirs, params)
        out["value"] = st / (time.perf_counter() - t0)
    finally:
        pool.close()
    out["sample"] = (f"{cpu_sample_note(cfg, len(seeds))}: numpy restatement of trace_batch "
                     f"(bit-exact to the reference) in a persistent {cores}-process fork pool, "
                     f"{len(seeds) // cores} seeds per worker (phg.py:201 slicing); host {model}")
    counts = np.zeros(occ.shape, np.uint16)
    ig = PhgParams(field_seeds=0)  # reference defaults: batch 16384, cap 16
    t0 = time.perf_counter()
    segs, st = onp.init_guide_strands_scalp(f, counts, seeds, dirs, ig, cores)
    dt = time.perf_counter() - t0
    out["init_guide_strands"] = {
        "value": st / dt, "seconds": dt, "steps": int(st), "segments": len(segs),
        "what": f"port of init_guide_strands(workers={cores}, field_seeds=0) as strandkit "
                "bench times it (cli.py:233-237): pool made per call, batch 16384, serial "
                "per-segment commit loop"}
    if one_core:
        t0 = time.perf_counter()
        _, keep, _ = onp.trace(f, seeds, dirs, params)
        dt = time.perf_counter() - t0
        out["one_core"] = {"value": int((keep - 1).sum()) / dt, "seconds": dt,
                           "what": "trace_batch port in one process (BASELINE.md 2 (i))"}
    if c_port:
        from oracle import phg_oracle_c as oc  # CPU baseline legs only

        t0 = time.perf_counter()
        _, keep, _ = oc.trace(np.zeros(3), synth.VOXEL_MM, occ, ori, seeds, dirs, params,
                              threads=cores)
        out["c_port_value"] = int((keep - 1).sum()) / (time.perf_counter() - t0)
        out["c_port_sample"] = (f"same seeds, our scalar C restatement on {cores} OpenMP "
                                "threads (context: not the reference's code)")
    return out


def host_field(cfg):
    from paper_2604_05794_b200 import synth

    ori, occ = cfg.field("cpu")
    return ori.numpy(), occ.numpy()


def run_reference(args):
    """--impl reference: the reference CPU path (numpy port, all host cores) on rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2604_05794_b200 import synth
    from paper_2604_05794_b200.phg import PhgParams

    cfg = synth.CONFIGS[resolve_config(args, ws)]
    cores, model = cpu_host_info()
    params = PhgParams(field_seeds=0)
    ori_t, occ_t = cfg.field("cpu")
    seeds, dirs = cpu_sample_seeds(cfg, args, ori_t, occ_t)
    ori, occ = ori_t.numpy(), occ_t.numpy()
    del ori_t, occ_t
    from oracle import phg_oracle_np as onp  # the reference arm: the port, on host cores

    f = onp.Field(np.zeros(3), synth.VOXEL_MM, occ.shape, occ, ori)
    pool = onp.TracePool(f, cores)
    try:
        for _ in range(min(max(args.warmup, 0), 1)):
            pool.steps(seeds[: cores * 64], dirs[: cores * 64], params)
        tot_t, tot_s = 0.0, 0
        for _ in range(args.steps):
            t0 = time.perf_counter()
            tot_s += pool.steps(seeds, dirs, params)
            tot_t += time.perf_counter() - t0
    finally:
        pool.close()
    v = tot_s / tot_t
    # BASELINE.md 2's other CPU legs, once (not per step): the reference's own multi-core
    # path init_guide_strands(workers=W, field_seeds=0) and trace_batch on one core
    extra = {}
    if not args.no_cpu:
        counts = np.zeros(occ.shape, np.uint16)
        t0 = time.perf_counter()
        segs, st = onp.init_guide_strands_scalp(f, counts, seeds, dirs, params, cores)
        dt = time.perf_counter() - t0
        extra["init_guide_strands"] = {
            "value": st / dt, "seconds": dt, "segments": len(segs),
            "what": f"port of init_guide_strands(workers={cores}, field_seeds=0) as strandkit "
                    "bench times it (cli.py:233-237): pool made per call, serial commit loop"}
        t0 = time.perf_counter()
        _, keep, _ = onp.trace(f, seeds, dirs, params)
        dt = time.perf_counter() - t0
        extra["one_core"] = {"value": int((keep - 1).sum()) / dt, "seconds": dt,
                             "what": "trace_batch port in one process (BASELINE.md 2 (i))"}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "steps/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "sample_seeds": int(len(seeds)),
                   "field": f"{cfg.n}^3 {cfg.kind}",
                   "seeds_per_worker": int(len(seeds)) // cores},
        "cpu_baseline": {"value": v, "unit": "steps/s", "cores": cores, "kind": "port",
                         "sample": f"{cpu_sample_note(cfg, len(seeds))} per step, numpy "
                                   f"restatement of trace_batch (pinned bit-exact to the "
                                   f"reference) in a persistent {cores}-process fork pool, "
                                   f"{len(seeds) // cores} seeds per worker (phg.py:184-207 "
                                   f"slicing); host {model}", **extra},
        "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def touched_footprint(cfg, off, verts):
    """How much of the field a trace actually visits (decides whether the gathers are served
    from L2 or HBM): distinct voxels holding a vertex, and the percentiles of each strand's
    top z (in voxels).  Computed on the device from the warm-up trace's CSR."""
    import torch

    from paper_2604_05794_b200 import synth

    n = cfg.n
    ijk = torch.floor(verts / synth.VOXEL_MM).to(torch.int64).clamp_(0, n - 1)
    lin = (ijk[:, 0] * n + ijk[:, 1]) * n + ijk[:, 2]
    plane = torch.zeros(n ** 3, dtype=torch.uint8, device=verts.device)
    plane[lin] = 1
    distinct = int(plane.sum(dtype=torch.int64).item())
    del plane, lin
    ends = off[1:] - 1
    z = ijk[ends.clamp(min=0), 2].double()
    q = torch.quantile(z[torch.randperm(z.numel(), device=z.device)[: 1 << 20]],
                       torch.tensor([0.5, 0.9, 0.99], dtype=torch.float64, device=z.device))
    return {"distinct_voxels_with_vertices": distinct,
            "frac_of_field_voxels": distinct / n ** 3,
            "vertex_voxel_bytes": distinct * 16,
            "strand_end_z_vox_p50_p90_p99": [float(v) for v in q.tolist()],
            "note": "the corner gathers read these voxels and their +1 neighbours (<= 8x); "
                    "compare with the 126 MB L2"}


def roofline_block(cfg, accepted, kernel_ms):
    """The trace kernel's roofline from its OWN config's ncu capture
    (profiles/ncu_<cfg>_trace.json; C4 runs C3's kernel on C3's field).  The kernel is bound
    by instruction issue (its 2x8 corner gathers are served mostly on chip), so the primary
    fraction is issue-based: warp instructions per step (ncu) x accepted steps / kernel time,
    against 148 SMs x 4 schedulers x 1 warp-instruction/clock at the max SM clock.  HBM (the
    SURVEY 8(d) algorithmic 281 B/step and the ncu DRAM bytes), L1 and L2 fractions sit
    beside it."""
    name = "C3" if cfg.name == "C4" else cfg.name
    path = os.path.join(ROOT, "profiles", f"ncu_{name}_trace.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except Exception:  # noqa: BLE001
        d = None
    peak_hbm, peak_kind = measured_peak()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:  # noqa: BLE001
        mhz = 1965.0
    sec = kernel_ms / 1e3
    algo_gbs = accepted * BYTES_PER_STEP / sec / 1e9
    out = {"bound": "issue", "kernel": "trace_kernel", "kernel_ms": kernel_ms,
           "unit": "Gwarp-inst/s", "peak": 148 * 4 * mhz * 1e6 / 1e9,
           "peak_source": f"148 SMs x 4 schedulers x 1 warp-inst/clk x {mhz:.0f} MHz "
                          "(MEASURED_PEAKS.json sm_max_mhz)",
           "achieved": None, "frac": None, "traffic": None,
           "hbm": {"algorithmic_bytes_per_step": BYTES_PER_STEP,
                   "algorithmic_gbs": algo_gbs, "peak_gbs": peak_hbm,
                   "peak_source": peak_kind},
           "source": os.path.relpath(path, ROOT) if d else None}
    if not d:
        out["note"] = f"no ncu capture for {name}: issue fraction unavailable"
        return out
    m = d.get("metrics", {})

    def num(k):
        try:
            return float(m[k][0])
        except Exception:  # noqa: BLE001
            return None

    steps_cap = float(d["steps_per_launch"])
    winst_step = num("smsp__inst_executed.sum") / steps_cap
    achieved = winst_step * accepted / sec / 1e9
    traffic = d["dram_bytes_per_launch"] * accepted / steps_cap
    out.update({"achieved": achieved, "frac": achieved / out["peak"], "traffic": traffic,
                "warp_inst_per_step": winst_step, "inst_per_step": winst_step * 32})
    out["hbm"].update({"dram_bytes_per_step": d["dram_bytes_per_step"],
                       "dram_gbs": traffic / sec / 1e9,
                       "dram_frac": traffic / sec / 1e9 / peak_hbm})
    pct = lambda k: (num(k) / 100.0 if num(k) is not None else None)  # noqa: E731
    out["ncu"] = {"issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                  "fp64_pipe": pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                  "xu_pipe": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                  "l1_frac": pct("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                  "l2_frac": pct("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                  "dram_frac": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                  "l1_hit": pct("l1tex__t_sector_hit_rate.pct"),
                  "l2_hit": pct("lts__t_sector_hit_rate.pct"),
                  "warps_per_sm": num("sm__warps_active.avg.per_cycle_active"),
                  "registers": num("launch__registers_per_thread"),
                  "kernel_ms_under_ncu": num("gpu__time_duration.sum"),
                  "stalls_per_issue": d.get("stalls_per_issue"),
                  "gather_gbs": d.get("gather_gbs")}
    return out


def init_dist(args, ws, local):
    """One process per GPU.  NCCL when every local rank has its own device (the driver's
    multi-GPU runs); gloo when ranks share a device (--dist-backend auto on a box with fewer
    GPUs than ranks: exercises the N > 1 code path through the real kernel for correctness,
    its timings are not a scaling measurement).  Returns (device, collective device, backend,
    shared)."""
    import torch
    import torch.distributed as dist

    ndev = max(torch.cuda.device_count(), 1)
    lws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    backend = args.dist_backend
    if backend == "auto":
        backend = "nccl" if ndev >= lws else "gloo"
    index = local % ndev
    torch.cuda.set_device(index)
    dev = torch.device("cuda", index)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    coll = dev if backend == "nccl" else torch.device("cpu")
    return dev, coll, backend, ws > 1 and ndev < lws


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2604_05794_b200 import dist as pdist
    from paper_2604_05794_b200 import phg, synth
    from paper_2604_05794_b200.volume import DeviceField

    ws, rank, local = dist_env()
    dev, coll, backend, shared = init_dist(args, ws, local)
    cfg = synth.CONFIGS[resolve_config(args, ws)]
    # C4 is BASELINE's scaling sweep: 4M global seeds split over the ranks (strong scaling);
    # every other config fixes the seeds per GPU (weak scaling)
    strong = cfg.name == "C4" and not args.seeds
    per_rank = args.seeds or (cfg.seeds // ws if strong else cfg.seeds)
    params = phg.PhgParams(field_seeds=0, batch_size=per_rank * ws)

    # field generated directly in HBM and packed once; at N > 1 rank 0 packs it and the packed
    # buffer is broadcast to the other ranks (dist.replicate_field: NCCL over NVLink), which
    # generate the field themselves only when the config's seeds need it (C5's interior seeds)
    setup = None
    need_field = ws == 1 or rank == 0 or cfg.kind == "sparse"
    ori, occ = cfg.field(dev) if need_field else (None, None)
    torch.cuda.empty_cache()  # the generator's temporaries (the C5 smoothing: tens of GB)
    ori_host = occ_host = None
    if ws == 1 and not args.no_cpu:
        ori_host, occ_host = ori.cpu().numpy(), occ.cpu().numpy()
    all_seeds, all_dirs = synth.config_seeds(cfg, per_rank * ws, ori, occ)  # disk: no field
    cpu_seeds = None
    if ori_host is not None:  # C1 all seeds, C2-C5 the first 16384
        k = min(args.cpu_sample or (cfg.seeds if cfg.name == "C1" else CPU_SUBSET), len(all_seeds))
        cpu_seeds = (np.ascontiguousarray(all_seeds[:k]), np.ascontiguousarray(all_dirs[:k]))
    if ws == 1:
        field = DeviceField(np.zeros(3), synth.VOXEL_MM, occ, ori,
                            torch.cuda.current_stream(dev).cuda_stream)
    else:
        from types import SimpleNamespace

        if rank != 0:  # only rank 0's copy feeds the field
            ori = occ = None
            torch.cuda.empty_cache()
        src = SimpleNamespace(origin=np.zeros(3), voxel_size=synth.VOXEL_MM, occ=occ, ori=ori)
        dist.barrier()
        t0 = time.perf_counter()
        field = pdist.replicate_field(src if rank == 0 else None, src=0, device=coll)
        dist.barrier()
        setup = {"field_replicate_s": time.perf_counter() - t0,
                 "field_bytes": field.packed()[1],
                 "how": "rank 0 packs, dist.replicate_field broadcasts the packed buffer"}
    del ori, occ
    torch.cuda.empty_cache()

    s_host = np.ascontiguousarray(all_seeds[rank * per_rank:(rank + 1) * per_rank])
    d_host = np.ascontiguousarray(all_dirs[rank * per_rank:(rank + 1) * per_rank])
    del all_seeds, all_dirs
    s_dev = torch.from_numpy(s_host).to(dev)
    d_dev = torch.from_numpy(d_host).to(dev)
    stream = torch.cuda.current_stream(dev)
    tracer = phg.Tracer()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    n_t = torch.tensor([per_rank], dtype=torch.int64, device=dev)

    def step_csr():
        off, verts, ent = phg.trace_device(field, s_dev, d_dev, params, tracer=tracer,
                                           stream=stream)
        if ws > 1:  # the one collective: global CSR placement of this rank's strands
            pdist.exchange_counts(per_rank, int(verts.shape[0]), device=coll)
        return off, verts

    def step():
        # the device-resident result: strand rows = the reference's buf[i, :keep[i]]
        # (phg.py:159-162), no host synchronisation inside the step
        rs = phg.trace_device_rows(field, s_dev, d_dev, params, tracer=tracer, stream=stream)
        if ws > 1:  # the one collective: (strands, vertices) of every rank -> CSR placement
            pdist.exchange_counts_device(n_t, rs.counters[1:2], device=coll)
        return rs

    if args.sweep:
        sweep_variants(args, step_csr, tracer, flush)
        return
    if args.sweep_sizes:
        sweep_launch_sizes(field, s_dev, d_dev, params, tracer, stream,
                           [int(v) for v in args.sweep_sizes.split(",")])
        return

    # warm-up, and the reference's step count from the CSR path (checked against the rows')
    for _ in range(args.warmup):
        flush.zero_()
        off, verts = step_csr()
    torch.cuda.synchronize()
    my_steps = int(verts.shape[0]) - per_rank  # sum(len - 1) over this rank's strands
    footprint = touched_footprint(cfg, off, verts) if rank == 0 else None
    del off, verts
    for _ in range(args.warmup):
        flush.zero_()
        rs = step()
    torch.cuda.synchronize()
    rows_steps = rs.steps
    accepted = tracer.last_steps()
    kernel_variant = {"variant": tracer.last_variant(), "sampler": tracer.last_sampler()}
    del rs
    if rows_steps != my_steps:
        raise RuntimeError(f"rows path steps {rows_steps} != CSR path steps {my_steps}")
    # whole-job steps: every rank's own count (ranks trace different seeds)
    tot = torch.tensor([my_steps], dtype=torch.int64, device=coll)
    if ws > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    total_steps = int(tot.item())

    def timed(fn, kern):
        """K steps between CUDA events on the launching stream, barrier + synchronize on
        both sides; max over ranks."""
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            flush.zero_()
            r = fn()
            if kern is not None:
                kern.append(tracer.last_kernel_ms()[0])
            del r
        e1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=coll)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(dev.index)
    clocks.start()
    kern_ms = []
    ms_max = timed(step, None)  # no host sync inside the timed rows steps
    clk = clocks.stop()
    ms_csr = timed(step_csr, kern_ms)  # kernel durations read per step (host sync per step)
    value = total_steps / (ms_max / 1e3)
    value_csr = total_steps / (ms_csr / 1e3)

    # e2e: host (pinned) buffers through the C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(args, tracer, field, params, s_host, d_host, per_rank, ws, coll,
                      total_steps)

    # N > 1: the rank-order concatenation on rank 0, fused into each rank's CSR gather kernel
    # writing over peer memory (dist.gather_csr_to_root_p2p; NVLink between GPUs)
    root_gather = None
    if ws > 1 and not args.no_root_gather:
        root_gather = root_gather_leg(args, tracer, field, params, s_dev, d_dev, per_rank, stream,
                                      coll)

    # the remaining legs run on their own contexts: release the timed context's slab and CSR
    # scratch first (C4's 4M seeds hold ~77 GB there)
    tracer.close()
    torch.cuda.empty_cache()
    driver = a9 = dropin = None
    if not args.no_driver and ws == 1:
        # the reference defaults on (at most) the first 1M seeds of the workload
        driver = driver_leg(cfg, field, s_host[:1_000_000], d_host[:1_000_000], dev)
        a9 = a9_leg()
    if not args.no_e2e and ws == 1 and ori_host is not None:
        dropin = dropin_leg(ori_host, occ_host, s_host, d_host, params)

    kernel_ms = float(np.mean(kern_ms))
    cpu = None
    if ws == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure (rank 0 only)
        cores, model = cpu_host_info()
        cpu = cpu_legs(cfg, ori_host, occ_host, cpu_seeds[0], cpu_seeds[1], cores, model)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "field": f"{cfg.n}^3 {cfg.kind}",
                       "seeds_per_gpu": per_rank, "global_seeds": per_rank * ws,
                       "max_vertices": params.max_vertices, "step_mm": params.step_mm,
                       "batch_size": per_rank * ws, "parallelism": f"seed-partition x{ws}",
                       "dist_backend": backend if ws > 1 else None,
                       "ranks_share_gpu": shared,
                       "l2": "256 MiB flush write between timed steps",
                       "field_bytes": (cfg.n + 2) ** 3 * 16, "touched_footprint": footprint},
            "steps_per_trace": total_steps, "accepted_steps_per_trace": accepted,
            "output": "device-resident strand rows (phg_trace_rows: the reference's buf[i, "
                      ":keep[i]], phg.py:159-162); value_csr adds the CSR scan + gather (K2)",
            "value_csr": value_csr, "ms_per_step_csr": ms_csr,
            "roofline": roofline_block(cfg, accepted, kernel_ms),
            "trace_kernel": kernel_variant,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "driver": driver, "a9": a9,
            "dropin": dropin, "setup": setup, "root_gather": root_gather,
            "gpu_launches": args.steps * phg.LAUNCHES_PER_TRACE_ROWS,
        }
        if shared:
            line["note"] = ("ranks share one GPU (gloo): validates the N > 1 code path through "
                            "the real kernel; not a scaling measurement")
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def root_gather_leg(args, tracer, field, params, s_dev, d_dev, per_rank, stream, coll):
    """Every rank's CSR written straight into rank 0's global CSR by its own gather kernel over
    peer memory (CUDA IPC; NVLink P2P between GPUs): time from the first barrier to the last,
    max over ranks (not part of the timed region of `value`)."""
    import torch
    import torch.distributed as dist

    from paper_2604_05794_b200 import dist as pdist

    off = torch.empty(per_rank + 1, dtype=torch.int64, device=s_dev.device)
    ent = torch.empty(max(per_rank, 1), dtype=torch.uint8, device=s_dev.device)
    m = tracer.trace(field, params, s_dev.data_ptr(), d_dev.data_ptr(), per_rank,
                     off.data_ptr(), ent.data_ptr(), None, stream.cuda_stream)
    info = pdist.exchange_counts(per_rank, m, device=coll)
    dist.barrier()
    t0 = time.perf_counter()
    err = None
    try:  # the root's allocation is agreed on inside (a failure raises on every rank)
        res = pdist.gather_csr_to_root_p2p(tracer, info, return_result=False)
    except Exception as exc:  # noqa: BLE001
        err, res = str(exc).splitlines()[0][:200], None
    dt = time.perf_counter() - t0
    if err is not None:
        return {"error": err}
    t = torch.tensor([dt], dtype=torch.float64, device=coll)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    if res is None:
        return None
    return {"seconds": dt, "bytes": res["bytes"], "gbs": res["bytes"] / dt / 1e9,
            "what": "dist.gather_csr_to_root_p2p: rank-order CSR on rank 0, each rank's gather "
                    "kernel writing into it over peer memory (IPC handles, NVLink P2P)"}


def driver_leg(cfg, field, s_host, d_host, dev, repeats=2):
    """init_guide_strands on the device (csrc/phg_grow.cu) with the reference's defaults:
    deferred-commit batches of 16384 seeds, occupancy_cap 16, 30000 field seeds; host seeds
    in, host CSR + updated counts out (wall clock, includes all copies)."""
    import ctypes

    import torch

    from paper_2604_05794_b200 import _native, grow
    from paper_2604_05794_b200.phg import PhgParams, _tracer

    params = PhgParams()
    lib = _native.load()
    tr = _tracer()
    counts = np.zeros(field.dims, np.uint16)
    p = _native.params_struct(params)
    g = grow.GrowParams(params.batch_size, params.occupancy_cap, params.field_seeds, 0)
    nseg, nv = ctypes.c_int64(), ctypes.c_int64()
    rep = (ctypes.c_int64 * 4)()
    times, dev_ms = [], []
    for _ in range(repeats):
        counts[:] = 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _native.check(lib.phg_grow_init(tr.handle, field.handle, ctypes.byref(p), ctypes.byref(g),
                                        s_host.ctypes.data, d_host.ctypes.data, len(s_host),
                                        counts.ctypes.data, ctypes.byref(nseg), ctypes.byref(nv),
                                        rep, None), "phg_grow_init")
        offsets = np.empty(nseg.value + 1, np.int64)
        verts = np.empty((nv.value, 3))
        rooted = np.empty(nseg.value, np.uint8)
        _native.check(lib.phg_grow_fetch(tr.handle, offsets.ctypes.data, verts.ctypes.data,
                                         rooted.ctypes.data, None), "phg_grow_fetch")
        times.append(time.perf_counter() - t0)
        dev_ms.append(tr.last_kernel_ms()[1])
    t = min(times)
    steps = int(nv.value - nseg.value)
    return {"what": "init_guide_strands (phg.py:210-303) on device, reference defaults",
            "seeds": int(len(s_host)), "batch_size": params.batch_size,
            "batches": int((len(s_host) + params.batch_size - 1) // params.batch_size),
            "field_seeds_traced": int(rep[2]), "segments": int(nseg.value),
            "scalp_segments": int(rep[1]), "vertices": int(nv.value), "seconds": t,
            "segment_steps_per_s": steps / t, "all_times_s": times,
            "device_ms": min(dev_ms),
            "note": "seconds = wall clock incl. vol.counts H2D/D2H and the pageable host CSR "
                    "copy; device_ms = CUDA-event window of the device work alone"}


def dropin_leg(ori_host, occ_host, s_host, d_host, params, repeats=2):
    """The reference-facing call itself: phg.trace_batch_csr / phg.trace_batch with pageable
    numpy arrays in and out (what strandkit callers get after install())."""
    from types import SimpleNamespace

    from paper_2604_05794_b200 import phg, synth

    vol = SimpleNamespace(origin=np.zeros(3), voxel_size=synth.VOXEL_MM, dims=occ_host.shape,
                          occ=occ_host, ori=ori_host)
    off, verts, ent = phg.trace_batch_csr(vol, s_host[:1000], d_host[:1000], params)  # warm
    t_csr, t_list = [], []
    for _ in range(repeats):
        t0 = time.perf_counter()
        off, verts, ent = phg.trace_batch_csr(vol, s_host, d_host, params)
        t_csr.append(time.perf_counter() - t0)
    steps = int(len(verts) - len(ent))
    del off, verts, ent
    t0 = time.perf_counter()
    out = phg.trace_batch(vol, s_host, d_host, params)
    t_list.append(time.perf_counter() - t0)
    del out
    return {"what": "phg.trace_batch_csr / trace_batch (drop-in), pageable numpy in and out",
            "csr_s": min(t_csr), "csr_steps_per_s": steps / min(t_csr),
            "list_s": t_list[0], "list_steps_per_s": steps / t_list[0],
            "note": "list_s includes building the reference's list of (vertices, entered) "
                    "tuples (one numpy view per strand)"}


def a9_leg(repeats=3):
    """The reference's A9 scene (tests/golden/a9_scene.npz, written by the reference's own scene
    pipeline): init_guide_strands and the full grow() on the device, host numpy in and out,
    against the only published PHG timing (init_guide_strands, 1 worker: 2.70 s,
    pkg/test_output.txt:28-34)."""
    from types import SimpleNamespace

    from paper_2604_05794_b200 import grow, link
    from paper_2604_05794_b200.phg import PhgParams
    from paper_2604_05794_b200.volume import OOVolume

    z = np.load(os.path.join(ROOT, "tests", "golden", "a9_scene.npz"))
    p = json.loads(str(z["params"]))
    p.update(json.loads(str(z["link_params"])))
    params = PhgParams(**{k: v for k, v in p.items() if k in PhgParams.__dataclass_fields__})
    vol = OOVolume.empty(z["origin"], float(z["voxel_size"]), z["occ"].shape)
    vol.occ, vol.ori = z["occ"], z["ori"]
    scalp = SimpleNamespace(seeds=z["seeds"], seed_normals=z["dirs"],
                            vertices=z["scalp_vertices"])
    t_init, t_grow = [], []
    for _ in range(repeats):
        vol.counts[:] = 0
        t0 = time.perf_counter()
        segs, _ = grow.init_guide_strands(scalp, vol, params)
        t_init.append(time.perf_counter() - t0)
        vol.counts[:] = 0
        t0 = time.perf_counter()
        sset, _ = link.grow(scalp, vol, params)
        t_grow.append(time.perf_counter() - t0)
    ref_here = z["reference_seconds_here"].tolist()
    return {"what": "reference A9 scene (4000 scalp + 4000 field seeds), host arrays in/out",
            "init_guide_strands_s": min(t_init), "grow_s": min(t_grow),
            "segments": len(segs), "strands": len(sset),
            "published_reference_init_s": 2.70,
            "reference_in_build_container_s": {"init_guide_strands": ref_here[0],
                                               "grow": ref_here[1]},
            "speedup_vs_published_init": 2.70 / min(t_init)}


def sweep_launch_sizes(field, s_dev, d_dev, params, tracer, stream, variants):
    """Trace-kernel time vs launch size for the given variants (small-batch regime: the
    reference's default deferred-commit batches are 16384 seeds); checks byte-identity."""
    import torch

    from paper_2604_05794_b200 import phg

    for n in (1024, 4096, 16384, 32768, 65536, 131072, 262144):
        ref = None
        row = {"seeds": n}
        for v in variants:
            os.environ["PHG_VARIANT"] = str(v)
            for _ in range(2):
                off, verts, _ = phg.trace_device(field, s_dev[:n], d_dev[:n], params,
                                                 tracer=tracer, stream=stream)
            ms = []
            for _ in range(3):
                off, verts, _ = phg.trace_device(field, s_dev[:n], d_dev[:n], params,
                                                 tracer=tracer, stream=stream)
                ms.append(tracer.last_kernel_ms()[0])
            torch.cuda.synchronize()
            same = ref is None or (torch.equal(ref[0], off) and torch.equal(ref[1], verts))
            if ref is None:
                ref = (off.clone(), verts.clone())
            row[tracer.last_variant()] = {"kernel_ms": min(ms), "identical": bool(same)}
        print(json.dumps(row), flush=True)
    os.environ.pop("PHG_VARIANT", None)


def sweep_variants(args, step, tracer, flush):
    """Time every compiled trace-kernel variant on this workload; check bit-identity."""
    import torch

    from paper_2604_05794_b200 import _native

    ref = None
    for v in range(_native.load().phg_num_variants()):
        os.environ["PHG_VARIANT"] = str(v)
        for _ in range(2):
            flush.zero_()
            off, verts = step()
        ms = []
        for _ in range(max(args.steps, 1)):
            flush.zero_()
            off, verts = step()
            ms.append(tracer.last_kernel_ms()[0])
        torch.cuda.synchronize()
        if ref is None:
            ref = (off.clone(), verts.clone())
            same = True
        else:
            same = bool(torch.equal(ref[0], off) and torch.equal(ref[1], verts))
        acc = tracer.last_steps()
        print(json.dumps({"variant": v, "name": tracer.last_variant(),
                          "sampler": tracer.last_sampler(), "kernel_ms": min(ms),
                          "kernel_ms_all": ms, "gsteps_per_s": acc / min(ms) / 1e6,
                          "identical_to_variant0": same}), flush=True)
        del off, verts
    os.environ.pop("PHG_VARIANT", None)


def e2e_leg(args, tracer, field, params, s_host, d_host, per_rank, ws, coll, total_steps):
    """Seeds from pinned host memory in, full CSR (offsets, entered, verts) out to pinned host."""
    import torch
    import torch.distributed as dist

    n = per_rank
    stream = torch.cuda.current_stream()
    err = None
    try:  # every rank pins ~24 B x its output vertices; agree on success before any collective
        pin_s = torch.from_numpy(s_host).pin_memory()
        pin_d = torch.from_numpy(d_host).pin_memory()
        out_off = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        out_ent = torch.empty(n, dtype=torch.uint8).pin_memory()
        total = tracer.trace(field, params, pin_s.data_ptr(), pin_d.data_ptr(), n,
                             out_off.data_ptr(), out_ent.data_ptr(), None, stream.cuda_stream)
        out_v = torch.empty((total, 3), dtype=torch.float64).pin_memory()
    except (RuntimeError, MemoryError) as exc:
        err = str(exc).splitlines()[0][:200] if str(exc) else type(exc).__name__
    if ws > 1:
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=coll)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not ok.item() and err is None:
            err = "another rank could not allocate its pinned host buffers"
    if err is not None:
        return {"value": None, "unit": "steps/s", "error": err}

    def one():
        # phg_trace_to_host: chunked, the D2H of chunk k overlaps the trace of chunk k+1
        return tracer.trace_to_host(field, params, pin_s.data_ptr(), pin_d.data_ptr(), n,
                                    out_off.data_ptr(), out_ent.data_ptr(), out_v.data_ptr(),
                                    int(out_v.shape[0]), args.e2e_chunk, stream.cuda_stream)

    for _ in range(max(1, args.warmup - 1)):
        one()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        total = one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.steps
    tt = torch.tensor([dt], dtype=torch.float64, device=coll)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt = float(tt.item())
    # the PCIe floor of this leg: a plain pinned D2H of the same payload size
    probe = torch.empty(min(total * 24, 2 << 30), dtype=torch.uint8, device="cuda")
    host = torch.empty(probe.numel(), dtype=torch.uint8).pin_memory()
    host.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    d2h_gbs = 0.0
    for _ in range(3):  # best of 3 rounds of 3 copies
        t0 = time.perf_counter()
        for _ in range(3):
            host.copy_(probe, non_blocking=True)
        torch.cuda.synchronize()
        d2h_gbs = max(d2h_gbs, 3 * probe.numel() / (time.perf_counter() - t0) / 1e9)
    del probe, host
    floor_ms = (total * 24 + (n + 1) * 8 + n) / d2h_gbs / 1e6
    return {"value": total_steps / dt, "unit": "steps/s",
            "pcie_d2h_gbs": d2h_gbs, "pcie_floor_ms": floor_ms,
            "frac_of_pcie_floor": floor_ms / (dt * 1e3), "chunk": args.e2e_chunk,
            "h2d_bytes_per_step": int(2 * n * 24), "d2h_bytes_per_step": int((n + 1) * 8 + n +
                                                                             total * 24),
            "ms_per_step": dt * 1e3,
            "path": "phg_trace_to_host (C ABI): pinned host seeds in, full host CSR out, "
                    "D2H of chunk k overlapped with the trace of chunk k+1"}


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
