"""Summarise an ncu --set full report of the trace kernel into profiles/*.json.

    python profiles/summarize_ncu.py <report.ncu-rep> <out.json> <label> <command> <steps_per_launch>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def _ratio(v, col, a, b):
    try:
        return float(v[col[a]].replace(",", "")) / float(v[col[b]].replace(",", ""))
    except (KeyError, ValueError, ZeroDivisionError):
        return None


def main(rep, out, label, cmd, steps):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    col = {k: i for i, k in enumerate(h)}
    m = {k: [v[col[k]], u[col[k]]] for k in KEYS if k in col}
    stalls = {}
    for k, i in col.items():
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                x = float(v[i])
            except ValueError:
                continue
            if x > 0.1:
                stalls[k.split("issue_stalled_")[1].split("_per")[0]] = x
    dr = float(v[col["dram__bytes_read.sum"]]) * SCALE[u[col["dram__bytes_read.sum"]]]
    dw = float(v[col["dram__bytes_write.sum"]]) * SCALE[u[col["dram__bytes_write.sum"]]]
    steps = int(steps)
    d = {"kernel": label, "command": cmd,
         "ncu": "--set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1",
         "steps_per_launch": steps, "dram_bytes_per_launch": dr + dw, "dram_read_bytes": dr,
         "dram_write_bytes": dw, "dram_bytes_per_step": (dr + dw) / steps,
         "inst_per_step": float(v[col["smsp__inst_executed.sum"]]) * 32 / steps,
         # sector efficiency: 32-B sectors touched per warp-level request.  A 16-B/lane corner
         # gather touches 16 sectors when the 32 lanes read 32 distinct contiguous voxels; fewer
         # means lanes share voxels (Morton-ordered neighbours); the staged vertex stores touch
         # 32 sectors per request (one row per lane) but always whole sectors
         "ld_sectors_per_request": _ratio(v, col, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                                          "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
         "st_sectors_per_request": _ratio(v, col, "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
                                          "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"),
         "stalls_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])), "metrics": m}
    # where the corner gathers are served: sectors x 32 B over the kernel duration
    try:
        t = float(v[col["gpu__time_duration.sum"]]) * {"ms": 1e-3, "us": 1e-6, "s": 1.0}[
            u[col["gpu__time_duration.sum"]]]
        l1 = float(v[col["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]]) * 32
        l2 = float(v[col["lts__t_sectors_srcunit_tex_op_read.sum"]]) * 32
        d["gather_gbs"] = {"l1_load_sectors": l1 / t / 1e9, "l2_read_from_l1": l2 / t / 1e9,
                           "dram_read": dr / t / 1e9, "dram_write": dw / t / 1e9}
    except (KeyError, ValueError):
        pass
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps({k: d[k] for k in ("dram_bytes_per_step", "inst_per_step",
                                        "stalls_per_issue")}, indent=1))
    for k in KEYS:
        if k in m:
            print(f"{k:70s} {m[k][0]:>18s} {m[k][1]}")


if __name__ == "__main__":
    main(*sys.argv[1:6])
