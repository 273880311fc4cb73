"""Where the time of init_guide_strands goes on the reference's A9 scene (GPU box).

    python profiles/a9_breakdown.py

Prints the warm wall time of the device driver alone (CSR out: seeds H2D, device batches,
counts and CSR D2H) and of the full drop-in call (plus the reference's list of Strand
objects), then a cProfile of one call.
"""
import cProfile
import io
import json
import os
import pstats
import sys
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_05794_b200 import grow  # noqa: E402
from paper_2604_05794_b200.phg import PhgParams  # noqa: E402
from paper_2604_05794_b200.volume import OOVolume  # noqa: E402


def main():
    z = np.load(os.path.join(ROOT, "tests", "golden", "a9_scene.npz"))
    p = json.loads(str(z["params"]))
    p.update(json.loads(str(z["link_params"])))
    params = PhgParams(**{k: v for k, v in p.items() if k in PhgParams.__dataclass_fields__})
    vol = OOVolume.empty(z["origin"], float(z["voxel_size"]), z["occ"].shape)
    vol.occ, vol.ori = z["occ"], z["ori"]
    scalp = SimpleNamespace(seeds=z["seeds"], seed_normals=z["dirs"],
                            vertices=z["scalp_vertices"])

    def timed(fn, reps=5):
        best = float("inf")
        for _ in range(reps):
            vol.counts[:] = 0
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
        return best

    timed(lambda: grow.init_guide_strands(scalp, vol, params), reps=2)  # upload, warm-up
    print("device driver, CSR out [s]:",
          timed(lambda: grow.init_guide_strands_csr(scalp.seeds, scalp.seed_normals, vol, params)))
    print("init_guide_strands, Strand list out [s]:",
          timed(lambda: grow.init_guide_strands(scalp, vol, params)))
    vol.counts[:] = 0
    pr = cProfile.Profile()
    pr.enable()
    grow.init_guide_strands(scalp, vol, params)
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(15)
    print(s.getvalue())


if __name__ == "__main__":
    main()
