import cProfile, pstats, io, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from types import SimpleNamespace
from paper_2604_05794_b200 import grow
from paper_2604_05794_b200.phg import PhgParams
from paper_2604_05794_b200.volume import OOVolume
z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "a9_scene.npz"))
p = json.loads(str(z["params"])); p.update(json.loads(str(z["link_params"])))
params = PhgParams(**{k: v for k, v in p.items() if k in PhgParams.__dataclass_fields__})
vol = OOVolume.empty(z["origin"], float(z["voxel_size"]), z["occ"].shape)
vol.occ, vol.ori = z["occ"], z["ori"]
scalp = SimpleNamespace(seeds=z["seeds"], seed_normals=z["dirs"], vertices=z["scalp_vertices"])
for _ in range(3):
    vol.counts[:] = 0
    t0 = time.perf_counter(); segs, rep = grow.init_guide_strands(scalp, vol, params); print("init", time.perf_counter() - t0)
vol.counts[:] = 0
pr = cProfile.Profile(); pr.enable()
segs, rep = grow.init_guide_strands(scalp, vol, params)
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue()[:6000])
print(rep)
from paper_2604_05794_b200 import grow as G
ts = []
for _ in range(5):
    vol.counts[:] = 0
    t0 = time.perf_counter(); off, v, r, rp = G.init_guide_strands_csr(scalp.seeds, scalp.seed_normals, vol, params); t1 = time.perf_counter()
    ts.append(t1 - t0)
print("csr only", min(ts))
ts = []
for _ in range(5):
    vol.counts[:] = 0
    t0 = time.perf_counter(); segs, rep = grow.init_guide_strands(scalp, vol, params); ts.append(time.perf_counter() - t0)
print("full", min(ts))
