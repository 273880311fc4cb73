"""C5 (1024^3 sparse, 8M seeds): does warp coherence matter?  Times the trace kernel on
  * the config's seeds with the Morton locality order (default) and without (seed order),
  * the disk seeds and the interior seeds traced as two separate launches (mode-homogeneous
    warps: probing-from-the-bottom vs inside the blobs) against one mixed launch.
    python profiles/c5_coherence_probe.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_05794_b200 import phg, synth  # noqa: E402
from paper_2604_05794_b200.volume import DeviceField  # noqa: E402

cfg = synth.CONFIGS["C5"]
dev = torch.device("cuda", 0)
ori, occ = cfg.field(dev)
torch.cuda.empty_cache()
field = DeviceField(np.zeros(3), synth.VOXEL_MM, occ, ori)
s, d = synth.config_seeds(cfg, cfg.seeds, ori, occ)
del ori, occ
torch.cuda.empty_cache()
p = phg.PhgParams(field_seeds=0, batch_size=cfg.seeds)
tr = phg.Tracer()
disk = np.ones(len(s), bool)
disk[np.abs(s[:, 2] - 1.3) > 1e-9] = False  # disk seeds sit at z = 1.3 mm


def run(pos, dirs, order=True, reps=3):
    sp, sd = torch.from_numpy(np.ascontiguousarray(pos)).to(dev), torch.from_numpy(
        np.ascontiguousarray(dirs)).to(dev)
    ms = []
    for _ in range(reps + 1):
        phg.trace_device(field, sp, sd, p, tracer=tr, order=order)
        ms.append(tr.last_kernel_ms()[0])
    return min(ms[1:]), tr.last_steps()


out = {}
out["mixed_morton"] = run(s, d)
out["mixed_seed_order"] = run(s, d, order=False)
a = run(s[disk], d[disk])
b = run(s[~disk], d[~disk])
out["disk_only"] = a
out["interior_only"] = b
out["split_sum_ms"] = a[0] + b[0]
print(json.dumps({k: v for k, v in out.items()}))
