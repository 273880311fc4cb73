"""Strict mode (phg.py:136-155): one cooperative launch vs max_vertices-1 launch pairs.

    python profiles/strict_ab.py [n_vox] [seeds]

Times phg.trace_batch_csr(strict=True) on a synthetic sparse field (host numpy in and out,
wall clock incl. the live_counts round trip), with PHG_STRICT_COOP=1 and =0, and checks the
outputs are identical.  Prints one JSON line per setting."""
import json
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_05794_b200 import phg, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
count = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
ori, occ = synth.make_field("sparse", n, "cpu")
ori, occ = ori.numpy(), occ.numpy()
s, d = synth.disk_seeds(n, count // 2, 3, radius_frac=0.45)
s2, d2 = synth.interior_seeds(occ, ori, count // 4, 4)
s, d = np.concatenate([s, s2, s2]), np.concatenate([d, d2, -d2])
vol = SimpleNamespace(origin=np.zeros(3), voxel_size=synth.VOXEL_MM, dims=occ.shape, occ=occ,
                      ori=ori)
p = phg.PhgParams(strict=True)
ref = None
for coop in ("1", "0", "1", "0"):
    os.environ["PHG_STRICT_COOP"] = coop
    counts = np.zeros(occ.shape, np.uint16)
    phg.trace_batch_csr(vol, s[:100], d[:100], p, live_counts=counts)  # warm
    counts[:] = 0
    t0 = time.perf_counter()
    off, v, e = phg.trace_batch_csr(vol, s, d, p, live_counts=counts)
    dt = time.perf_counter() - t0
    cur = (off, v, e, counts.copy())
    same = ref is None or all(np.array_equal(a, b) for a, b in zip(ref, cur))
    ref = ref or cur
    tr = phg._tracer()
    print(json.dumps({"coop": coop, "variant": tr.last_variant(), "seconds": dt,
                      "trace_ms": tr.last_kernel_ms()[0], "strands": len(s),
                      "steps": int(len(v) - len(s)), "max_len": int(np.diff(off).max()),
                      "identical": bool(same)}), flush=True)
