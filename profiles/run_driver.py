"""Profiling harness: run the device batch driver (init_guide_strands) once on a C3 field.

    python profiles/run_driver.py [n_seeds] [repeats]
"""
import os
import sys
import time
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_05794_b200 import grow, synth  # noqa: E402
from paper_2604_05794_b200.phg import PhgParams, _tracer  # noqa: E402
from paper_2604_05794_b200.volume import OOVolume  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.CONFIGS["C3"]
ori, occ = cfg.field("cuda")
vol = OOVolume.empty((0, 0, 0), synth.VOXEL_MM, occ.shape)
vol.ori, vol.occ = ori.cpu().numpy(), occ.cpu().numpy()
del ori, occ
seeds, dirs = synth.disk_seeds(cfg.n, n, cfg.key)
for r in range(reps):
    vol.counts[:] = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    off, verts, rooted, rep = grow.init_guide_strands_csr(seeds, dirs, vol, PhgParams())
    dev_ms = _tracer().last_kernel_ms()[1]
    print(f"run {r}: {time.perf_counter() - t0:.3f} s  device {dev_ms:.2f} ms  "
          f"segments={len(rooted)} verts={len(verts)} {rep}", flush=True)
