"""bench.py's JSON line keeps the driver's contract (keys, units, reference-arm shape).

CPU: the reference arm (`--impl reference`, the oracle port on host cores) on C1.
GPU: our arm on C1 with every leg, parsed and checked key by key.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1",
              "--cpu-sample", "600"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "steps/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] == "port"
    assert cb["value"] == d["value"] and d["e2e"]["value"] == d["value"]
    assert cb["init_guide_strands"]["value"] > 0 and cb["one_core"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--cpu-sample", "2000"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["value_csr"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] <= 1 and r["source"] == "profiles/ncu_C1_trace.json"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb)
    assert {"init_guide_strands", "one_core"} <= set(cb)
    assert d["clocks"] and d["clocks"]["samples"] > 0 and "reasons" in d["clocks"]
    assert d["gpu_launches"] == 3 * 8
    assert d["steps_per_trace"] == 1_260_000  # C1: 10k strands x 126 returned steps


def test_reference_arm_under_torchrun_prints_one_line():
    """The driver launches the reference arm like ours at N > 1 (torchrun); rank 0 alone runs
    it and prints ONE line, the other ranks exit 0 without work."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "1",
                        "--cpu-sample", "300", "--no-cpu"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
