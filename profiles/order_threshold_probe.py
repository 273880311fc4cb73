"""Trace-call time (Morton sort + trace kernel, CUDA events) with and without the locality
order, on small launches: does the sort pay below the 1M-seed configs?
Usage: python profiles/order_threshold_probe.py C1 C2 [...]"""
import json
import sys

import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_05794_b200 import phg, synth
from paper_2604_05794_b200.volume import DeviceField


def main():
    for name in sys.argv[1:]:
        cfg = synth.CONFIGS[name]
        ori, occ = cfg.field("cuda")
        f = DeviceField(np.zeros(3), synth.VOXEL_MM, occ, ori)
        del ori, occ
        s, d = synth.config_seeds(cfg, cfg.seeds)
        s = torch.as_tensor(np.ascontiguousarray(s), device="cuda")
        d = torch.as_tensor(np.ascontiguousarray(d), device="cuda")
        p = phg.PhgParams(batch_size=len(s))
        for n in sorted({min(len(s), k) for k in (4096, 16384, 65536, len(s))}):
            row = {"config": name, "n": n}
            for order in (True, False):
                ms = []
                for _ in range(12):
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    torch.cuda.synchronize()
                    e0.record()
                    phg.trace_device(f, s[:n], d[:n], p, order=order)
                    e1.record()
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                row["ordered_ms" if order else "unordered_ms"] = float(np.median(ms[2:]))
            print(json.dumps(row), flush=True)
        f.close()


if __name__ == "__main__":
    main()
