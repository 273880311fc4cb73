"""Generate the golden PHG fixtures by running the REFERENCE implementation.

Run in the build container only (it imports strandkit from /root/reference,
which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is one compressed .npz holding the exact inputs (field bytes,
seeds, params, cap / near-occupancy / counts planes) and the reference's
outputs in CSR form (offsets (n+1,), verts (M,3) f64, entered (n,)).  The
oracle (oracle/) is pinned bit-exact against these; the CUDA path is checked
against them in tests/test_gpu_parity.py.

Reference entry points exercised:
  strandkit.phg.trace_batch                 phg.py:67-163
  strandkit.volume.sample_orientation_batch volume.py:183-224
  strandkit.phg.init_guide_strands          phg.py:210-260 (incl. _trace_field_seeds :263-303)
  strandkit.phg.nearest_occupied_map        phg.py:57-64 (steer input)
Unit cases restate the inputs of the reference's own trace tests
(pkg/tests/test_phg.py:33-127, test_acceptance.py:224-262).
"""

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from strandkit import phg  # noqa: E402
from strandkit.scalp import ScalpMesh  # noqa: E402
from strandkit.strands import Strand  # noqa: E402
from strandkit.volume import OOVolume, sample_orientation_batch  # noqa: E402

from paper_2604_05794_b200 import synth  # noqa: E402

TRACE_KEYS = ("step_mm", "max_vertices", "min_support", "probe_steps", "coast_steps", "steer",
              "strict", "occupancy_cap", "batch_size", "field_seeds")


def params_json(p):
    return json.dumps({k: getattr(p, k) for k in TRACE_KEYS})


def to_csr(out):
    lens = np.array([len(v) for v, _ in out], dtype=np.int64)
    offsets = np.zeros(len(out) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    verts = np.concatenate([v for v, _ in out]) if out else np.zeros((0, 3))
    entered = np.array([e for _, e in out], dtype=bool)
    return offsets, verts, entered


def vol_of(origin, vs, occ, ori):
    vol = OOVolume.empty(origin, vs, occ.shape)
    vol.occ = occ.copy()
    vol.ori = ori.astype(np.float32).copy()
    return vol


def save(name, vol, seeds, dirs, params, out, at_cap=None, near_occ=None, counts_in=None,
         counts_out=None, extra=None):
    offsets, verts, entered = to_csr(out)
    d = dict(
        origin=np.asarray(vol.origin, np.float64), voxel_size=np.float64(vol.voxel_size),
        occ=vol.occ, ori=vol.ori, seeds=np.asarray(seeds, np.float64).reshape(-1, 3),
        dirs=np.asarray(dirs, np.float64).reshape(-1, 3), params=np.array(params_json(params)),
        offsets=offsets, verts=verts, entered=entered,
    )
    if at_cap is not None:
        d["at_cap"] = at_cap
    if near_occ is not None:
        d["near_occ"] = near_occ.astype(np.int64)
    if counts_in is not None:
        d["counts_in"] = counts_in
    if counts_out is not None:
        d["counts_out"] = counts_out
    if extra:
        d.update(extra)
    path = os.path.join(HERE, f"trace_{name}.npz")
    np.savez_compressed(path, **d)
    steps = int((np.diff(offsets) - 1).sum()) if len(out) else 0
    print(f"{name:24s} n={len(out):5d} M={len(verts):7d} steps={steps:7d} "
          f"{os.path.getsize(path) / 1e3:8.1f} kB")


def column(height=40, ori=(0.0, 0.0, 1.0)):
    """The reference tests' column volume (test_phg.py:14-19)."""
    vol = OOVolume.empty(origin=(-10.0, -10.0, 0.0), voxel_size=2.0, dims=(10, 10, height))
    vol.occ[:] = True
    vol.ori[:] = np.asarray(ori, dtype=np.float32)
    return vol


def unit_cases():
    P = phg.PhgParams
    up = [[0.0, 0.0, 1.0]]
    s0 = [[0.5, 0.5, 1.0]]
    vol = column()
    p = P(step_mm=1.0, max_vertices=30, probe_steps=0, coast_steps=0, field_seeds=0)
    save("unit_straight", vol, s0, up, p, phg.trace_batch(vol, s0, up, p))
    vol = column(height=5)
    p = P(step_mm=1.0, max_vertices=60, probe_steps=0, coast_steps=0, field_seeds=0)
    save("unit_slab_top", vol, s0, up, p, phg.trace_batch(vol, s0, up, p))
    for steps in (2, 15):
        vol = column()
        vol.occ[:, :, :6] = False
        p = P(step_mm=1.0, max_vertices=40, probe_steps=steps, coast_steps=0, field_seeds=0)
        save(f"unit_probe{steps}", vol, s0, up, p, phg.trace_batch(vol, s0, up, p))
    for coast in (0, 12):
        vol = column()
        vol.occ[:, :, 10:13] = False
        p = P(step_mm=1.0, max_vertices=90, probe_steps=0, field_seeds=0, coast_steps=coast)
        save(f"unit_coast{coast}", vol, s0, up, p, phg.trace_batch(vol, s0, up, p))
    vol = column(height=10)
    p = P(step_mm=1.0, max_vertices=80, probe_steps=0, coast_steps=10, field_seeds=0)
    save("unit_trim", vol, s0, up, p, phg.trace_batch(vol, s0, up, p))
    vol = column()
    p = P(step_mm=1.0, max_vertices=30, probe_steps=0, coast_steps=0, field_seeds=0, strict=True)
    seeds = np.array([[0.5, 0.5, 1.0], [0.5, 0.5, 0.2]])
    dirs = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    counts = np.zeros(vol.dims, np.uint16)
    c0 = counts.copy()
    out = phg.trace_batch(vol, seeds, dirs, p, live_counts=counts)
    save("unit_strict", vol, seeds, dirs, p, out, counts_in=c0, counts_out=counts)
    vol = column()
    p = P(step_mm=1.0, max_vertices=30, probe_steps=0, coast_steps=0, field_seeds=0,
          occupancy_cap=1)
    seeds = np.tile([[0.5, 0.5, 1.0]], (4, 1))
    dirs = np.tile([[0.0, 0.0, 1.0]], (4, 1))
    cap = np.zeros(vol.dims, dtype=bool)
    save("unit_deferred", vol, seeds, dirs, p, phg.trace_batch(vol, seeds, dirs, p, at_cap=cap),
         at_cap=cap)
    vol = column()
    p = P(step_mm=1.0, max_vertices=30, probe_steps=0, coast_steps=0, field_seeds=0)
    cap = np.zeros(vol.dims, dtype=bool)
    cap[:, :, 8:] = True
    save("unit_at_cap", vol, s0, up, p, phg.trace_batch(vol, s0, up, p, at_cap=cap), at_cap=cap)
    # max_vertices edge cases and a seed far outside the volume
    vol = column()
    for mv in (1, 2):
        p = P(max_vertices=mv, field_seeds=0)
        save(f"unit_maxv{mv}", vol, s0 + [[100.0, 0, 0]], up + up, p,
             phg.trace_batch(vol, s0 + [[100.0, 0, 0]], up + up, p))
    seeds = np.array([[500.0, 500.0, 500.0], [-3.0, 2.0, -30.0], [0.5, 0.5, 79.9], [0.0, 0.0, 40.0]])
    dirs = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [1e-14, 0.0, 0.0]])
    p = P(field_seeds=0)
    save("unit_outside", vol, seeds, dirs, p, phg.trace_batch(vol, seeds, dirs, p))
    # zero seeds
    p = P(field_seeds=0)
    save("unit_empty", vol, np.zeros((0, 3)), np.zeros((0, 3)), p,
         phg.trace_batch(vol, np.zeros((0, 3)), np.zeros((0, 3)), p))


def helix_case():
    """A8 helix field (test_acceptance.py:224-262), nearest-helix-point orientation."""
    from scipy.spatial import cKDTree

    r, pitch, vs = 20.0, 40.0, 2.0
    b = pitch / (2 * np.pi)
    speed = np.hypot(r, b)

    def helix(t):
        return np.stack([r * np.cos(t), r * np.sin(t), b * t], axis=-1)

    def helix_tan(t):
        v = np.stack([-r * np.sin(t), r * np.cos(t), np.full_like(t, b)], axis=-1)
        return v / np.linalg.norm(v, axis=-1, keepdims=True)

    tmax = 180.0 / speed
    origin = np.array([-r - 10.0, -r - 10.0, -10.0])
    dims = (int((2 * r + 20) / vs) + 1, int((2 * r + 20) / vs) + 1, int((b * tmax + 20) / vs) + 1)
    vol = OOVolume.empty(origin, vs, dims)
    grid = np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"), axis=-1).reshape(-1, 3)
    centers = vol.centers(grid)
    ts = np.linspace(0, tmax, 4000)
    d, i = cKDTree(helix(ts)).query(centers)
    occ = d < 6.0
    vol.occ = occ.reshape(dims)
    ori = np.zeros((len(centers), 3))
    ori[occ] = helix_tan(ts[i[occ]])
    vol.ori = ori.reshape(*dims, 3).astype(np.float32)
    p = phg.PhgParams(step_mm=1.0, max_vertices=101, probe_steps=0, coast_steps=0, field_seeds=0)
    ts0 = np.linspace(0.2, 0.6, 40)
    seeds, dirs = helix(ts0), helix_tan(ts0)
    save("helix", vol, seeds, dirs, p, phg.trace_batch(vol, seeds, dirs, p))


def field_np(kind, n, **kw):
    ori, occ = synth.make_field(kind, n, "cpu", **kw)
    return ori.numpy(), occ.numpy()


def analytic_cases():
    P = phg.PhgParams
    for kind, n, count, key in (("straight", 48, 600, 21), ("wavy", 48, 600, 22),
                                ("curly", 48, 150, 23)):
        ori, occ = field_np(kind, n)
        vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
        seeds, dirs = synth.disk_seeds(n, count, key)
        p = P(field_seeds=0, batch_size=count)
        save(f"{kind}{n}", vol, seeds, dirs, p,
             phg.trace_batch(vol, seeds, dirs, p, at_cap=np.zeros(occ.shape, bool)))
    # sparse field: scalp seeds + interior seeds in both directions
    n = 48
    ori, occ = field_np("sparse", n, sparse_sigma=2.0)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    s1, d1 = synth.disk_seeds(n, 400, 24, radius_frac=0.45)
    s2, d2 = synth.interior_seeds(occ, ori, 400, 25)
    seeds = np.concatenate([s1, s2, s2])
    dirs = np.concatenate([d1, d2, -d2])
    p = P(field_seeds=0)
    save("sparse48", vol, seeds, dirs, p, phg.trace_batch(vol, seeds, dirs, p))
    # non-empty cap plane on the curly field (caps must be covered)
    ori, occ = field_np("curly", 40)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    rng = np.random.Generator(np.random.Philox(key=26))
    cap = rng.random(occ.shape) < 0.04
    seeds, dirs = synth.disk_seeds(40, 500, 27)
    p = P(field_seeds=0, probe_steps=5, coast_steps=3)
    save("curly40_cap", vol, seeds, dirs, p, phg.trace_batch(vol, seeds, dirs, p, at_cap=cap),
         at_cap=cap)
    # non power-of-two voxel size and a shifted origin
    ori, occ = field_np("curly", 32)
    vol = vol_of((-31.7, 12.25, -3.0), 1.7, occ, ori)
    s, d = synth.disk_seeds(32, 100, 28)
    s = (s / synth.VOXEL_MM) * 1.7 + vol.origin
    p = P(field_seeds=0, step_mm=0.85, min_support=0.2)
    save("curly32_vs17", vol, s, d, p, phg.trace_batch(vol, s, d, p))
    # steer: sparse field, coasting strands pulled toward occupied voxels
    ori, occ = field_np("sparse", 40, sparse_sigma=2.0, sparse_key=9)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    near = phg.nearest_occupied_map(vol)
    s1, d1 = synth.disk_seeds(40, 300, 29, radius_frac=0.45)
    s2, d2 = synth.interior_seeds(occ, ori, 200, 30)
    seeds, dirs = np.concatenate([s1, s2]), np.concatenate([d1, d2])
    p = P(field_seeds=0, steer=0.5, coast_steps=8)
    save("sparse40_steer", vol, seeds, dirs, p,
         phg.trace_batch(vol, seeds, dirs, p, near_occ=near), near_occ=near)
    # strict mode with many interacting strands
    ori, occ = field_np("curly", 32)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    seeds, dirs = synth.disk_seeds(32, 300, 31)
    counts = np.zeros(occ.shape, np.uint16)
    counts[rng.random(occ.shape) < 0.01] = 1
    c0 = counts.copy()
    p = P(field_seeds=0, strict=True)
    out = phg.trace_batch(vol, seeds, dirs, p, live_counts=counts)
    save("curly32_strict", vol, seeds, dirs, p, out, counts_in=c0, counts_out=counts)


def nonfinite_case():
    """Non-finite orientations: NaN/inf in some unoccupied voxels, on occupied border voxels and
    in a few occupied interior voxels.  The reference's masked weights still multiply them
    (0 * NaN = NaN), so strands touching them change; the device must take its exact sampler."""
    ori, occ = field_np("curly", 24)
    rng = np.random.Generator(np.random.Philox(key=41))
    ori = ori.copy()
    empty = np.argwhere(~occ)
    for i in rng.choice(len(empty), size=min(40, len(empty)), replace=False):
        ori[tuple(empty[i])] = (np.nan, 0.5, -np.inf)
    full = np.argwhere(occ)
    border = full[(full == 0).any(axis=1) | (full == 23).any(axis=1)]
    for i in rng.choice(len(border), size=min(10, len(border)), replace=False):
        ori[tuple(border[i])] = (np.inf, np.nan, 0.0)
    for i in rng.choice(len(full), size=5, replace=False):
        ori[tuple(full[i])] = (np.nan, np.nan, np.nan)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    seeds, dirs = synth.disk_seeds(24, 300, 42, radius_frac=0.48)
    p = phg.PhgParams(field_seeds=0, max_vertices=120)
    save("curly24_nonfinite", vol, seeds, dirs, p, phg.trace_batch(vol, seeds, dirs, p))


def sampler_case():
    ori, occ = field_np("sparse", 24, sparse_sigma=1.5)
    vol = vol_of((-5.0, 3.0, 1.0), 1.5, occ, ori)
    rng = np.random.Generator(np.random.Philox(key=33))
    lo, hi = vol.origin - 3.0, vol.origin + np.array(vol.dims) * 1.5 + 3.0
    pts = rng.uniform(lo, hi, size=(4000, 3))
    prev = rng.normal(size=(4000, 3))
    prev /= np.linalg.norm(prev, axis=1, keepdims=True)
    dirs, has, sup = sample_orientation_batch(vol, pts, prev)
    np.savez_compressed(os.path.join(HERE, "sample_sparse24.npz"), origin=vol.origin,
                        voxel_size=np.float64(vol.voxel_size), occ=vol.occ, ori=vol.ori, pts=pts,
                        prev=prev, dirs=dirs, has=has, support=sup)
    print("sample_sparse24 ok")


def _driver(name, vol, seeds, dirs, p):
    scalp = ScalpMesh(vertices=np.zeros((3, 3)), faces=np.zeros((1, 3), int),
                      vertex_normals=np.zeros((3, 3)), seeds=seeds, seed_normals=dirs)
    segs, report = phg.init_guide_strands(scalp, vol, p, workers=1)
    out = [(s.vertices, s.rooted) for s in segs]
    offsets, verts, rooted = to_csr(out)
    np.savez_compressed(
        os.path.join(HERE, f"driver_{name}.npz"), origin=vol.origin,
        voxel_size=np.float64(vol.voxel_size), occ=vol.occ, ori=vol.ori, seeds=seeds, dirs=dirs,
        params=np.array(params_json(p)), offsets=offsets, verts=verts, rooted=rooted,
        counts_out=vol.counts, report=np.array(json.dumps(report)))
    print(f"driver_{name:18s} segments={len(segs)} report={report}")


def driver_cases():
    """init_guide_strands with several deferred-commit batches and a field pass."""
    n = 40
    ori, occ = field_np("sparse", n, sparse_sigma=2.0, sparse_key=7)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    seeds, dirs = synth.disk_seeds(n, 1500, 34, radius_frac=0.45)
    _driver("sparse40", vol, seeds, dirs,
            phg.PhgParams(batch_size=256, occupancy_cap=2, field_seeds=600, n_root=1500))
    # curly field, cap 1, many batches; field_seeds larger than the unvisited set (no striding)
    ori, occ = field_np("curly", 32)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    seeds, dirs = synth.disk_seeds(32, 800, 35)
    _driver("curly32_cap1", vol, seeds, dirs,
            phg.PhgParams(batch_size=100, occupancy_cap=1, field_seeds=100000, max_vertices=120))
    # strict mode: per-step commits in both passes, no segment commits
    ori, occ = field_np("sparse", 32, sparse_sigma=2.0, sparse_key=8)
    vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
    seeds, dirs = synth.disk_seeds(32, 400, 36, radius_frac=0.45)
    _driver("sparse32_strict", vol, seeds, dirs,
            phg.PhgParams(batch_size=128, field_seeds=300, strict=True))
    # steering + a non-power-of-two voxel size and shifted origin
    ori, occ = field_np("sparse", 32, sparse_sigma=2.0, sparse_key=9)
    vol = vol_of((-7.5, 3.25, 1.0), 1.7, occ, ori)
    seeds, dirs = synth.disk_seeds(32, 400, 37, radius_frac=0.45)
    seeds = (seeds / synth.VOXEL_MM) * 1.7 + vol.origin
    _driver("sparse32_steer_vs17", vol, seeds, dirs,
            phg.PhgParams(batch_size=150, occupancy_cap=3, field_seeds=250, steer=0.5,
                          step_mm=0.85))


def _strands_npz(path, strands, **extra):
    src_code = {"traced": 0, "field": 1, "linked": 2, "attached": 3}
    off = np.zeros(len(strands) + 1, np.int64)
    off[1:] = np.cumsum([len(s.vertices) for s in strands])
    verts = np.concatenate([s.vertices for s in strands]) if strands else np.zeros((0, 3))
    tang = (np.concatenate([s.tangents for s in strands])
            if strands and strands[0].tangents is not None else np.zeros((0, 3)))
    np.savez_compressed(path, offsets=off, verts=verts, tangents=tang,
                        rooted=np.array([s.rooted for s in strands], bool),
                        source=np.array([src_code[s.source] for s in strands], np.uint8), **extra)


def link_cases():
    """compute_links / connect_segments (phg.py:337-413), attach_to_scalp (:419-439), grow (:445)."""
    rng = np.random.Generator(np.random.Philox(key=62))
    # the reference's own random-segment linking setup (test_phg.py:130-179)
    segs = []
    for _ in range(400):
        a = rng.uniform(-60.0, 60.0, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        k = int(rng.integers(3, 7))
        segs.append(Strand(vertices=a + np.outer(np.linspace(0, 6.0, k), d)))
    p = phg.PhgParams(link_dist_mm=8.0, link_angle_deg=45.0)
    links = np.array(phg.compute_links(segs, p), np.int64).reshape(-1, 2)
    seg_off = np.zeros(len(segs) + 1, np.int64)
    seg_off[1:] = np.cumsum([len(s.vertices) for s in segs])
    strands = phg.connect_segments(segs, p)
    _strands_npz(os.path.join(HERE, "link_random400.npz"), strands, links=links,
                 seg_offsets=seg_off, seg_verts=np.concatenate([s.vertices for s in segs]),
                 seg_rooted=np.zeros(len(segs), bool), seg_source=np.zeros(len(segs), np.uint8),
                 params=np.array(json.dumps({"link_dist_mm": 8.0, "link_angle_deg": 45.0,
                                             "tangent_window": 3, "smooth": True,
                                             "smooth_strength": 0.25, "smooth_iters": 2,
                                             "step_mm": 1.0})))
    print(f"link_random400 links={len(links)} strands={len(strands)}")
    # full grow() on driver scenes, with a planar scalp grid under the seeds
    for name, n, kind, kw, nseeds, key, pkw in (
            ("sparse40", 40, "sparse", dict(sparse_sigma=2.0, sparse_key=7), 1500, 34,
             dict(batch_size=256, occupancy_cap=2, field_seeds=600)),
            ("curly32", 32, "curly", {}, 800, 35,
             dict(batch_size=100, occupancy_cap=1, field_seeds=100000, max_vertices=120,
                  link_dist_mm=3.0, link_angle_deg=60.0))):
        ori, occ = field_np(kind, n, **kw)
        vol = vol_of((0, 0, 0), synth.VOXEL_MM, occ, ori)
        seeds, dirs = synth.disk_seeds(n, nseeds, key, radius_frac=0.45)
        L = n * synth.VOXEL_MM
        g = np.arange(1.0, L, 2.0)
        gx, gy = np.meshgrid(g, g, indexing="ij")
        keep = (gx - L / 2) ** 2 + (gy - L / 2) ** 2 < (0.47 * L) ** 2
        sv = np.stack([gx[keep], gy[keep], np.full(keep.sum(), 0.5)], axis=1)
        scalp = ScalpMesh(vertices=sv, faces=np.zeros((1, 3), int),
                          vertex_normals=np.tile([0.0, 0.0, 1.0], (len(sv), 1)), seeds=seeds,
                          seed_normals=dirs)
        p = phg.PhgParams(**pkw)
        sset, report = phg.grow(scalp, vol, p, workers=1)
        rep = {k: v for k, v in report.items() if not k.startswith("t_")}
        _strands_npz(os.path.join(HERE, f"grow_{name}.npz"), sset.strands, origin=vol.origin,
                     voxel_size=np.float64(vol.voxel_size), occ=vol.occ, ori=vol.ori,
                     seeds=seeds, dirs=dirs, scalp_vertices=sv,
                     params=np.array(params_json(p)),
                     link_params=np.array(json.dumps({k: getattr(p, k) for k in (
                         "link_dist_mm", "link_angle_deg", "tangent_window", "smooth",
                         "smooth_strength", "smooth_iters", "step_mm", "attach_radius_mm")})),
                     report=np.array(json.dumps(rep)))
        print(f"grow_{name} strands={len(sset)} report={rep}")


def _digest(*arrays):
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def a9_case():
    """The reference's A9 scene (test_acceptance.py:302-334, conftest.small_config): the only
    published PHG timing (pkg/test_output.txt:28-34, 2.70 s at 1 worker).  Inputs are stored;
    outputs as digests (the full result is ~14 MB)."""
    import time

    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import small_config  # the reference's own test configuration
    from strandkit import pipeline
    from strandkit import volume as vol_mod
    from strandkit.scalp import sample_seeds

    cfg = small_config()
    _, gt, scalp, _ = pipeline.scene_from_config(cfg)
    verts, tans = gt.all_vertices_tangents()
    vol = vol_mod.voxelize(verts, tans, voxel_size=2.0)
    vol_mod.fill_interior(vol, scalp, max_depth_mm=6.0)
    params = phg.PhgParams(n_root=4000, field_seeds=4000)
    sample_seeds(scalp, params.n_root, seed=7)
    vol.counts[:] = 0
    t0 = time.perf_counter()
    segs, rep = phg.init_guide_strands(scalp, vol, params, workers=1)
    t_init = time.perf_counter() - t0
    seg_off = np.zeros(len(segs) + 1, np.int64)
    seg_off[1:] = np.cumsum([len(s.vertices) for s in segs])
    seg_v = np.concatenate([s.vertices for s in segs])
    seg_r = np.array([s.rooted for s in segs], bool)
    counts_after_init = vol.counts.copy()
    vol.counts[:] = 0
    t0 = time.perf_counter()
    sset, grep = phg.grow(scalp, vol, params, workers=1)
    t_grow = time.perf_counter() - t0
    st = list(sset)
    off = np.zeros(len(st) + 1, np.int64)
    off[1:] = np.cumsum([len(s.vertices) for s in st])
    src_code = {"traced": 0, "field": 1, "linked": 2, "attached": 3}
    np.savez_compressed(
        os.path.join(HERE, "a9_scene.npz"), origin=vol.origin,
        voxel_size=np.float64(vol.voxel_size), occ=vol.occ, ori=vol.ori, seeds=scalp.seeds,
        dirs=scalp.seed_normals, scalp_vertices=scalp.vertices, params=np.array(params_json(p=params)),
        link_params=np.array(json.dumps({k: getattr(params, k) for k in (
            "link_dist_mm", "link_angle_deg", "tangent_window", "smooth", "smooth_strength",
            "smooth_iters", "step_mm", "attach_radius_mm")})),
        init_digest=np.array(_digest(seg_off, seg_v, seg_r, counts_after_init)),
        init_report=np.array(json.dumps(rep)),
        init_steps=np.int64(len(seg_v) - len(segs)),
        grow_digest=np.array(_digest(off, np.concatenate([s.vertices for s in st]),
                                     np.concatenate([s.tangents for s in st]),
                                     np.array([s.rooted for s in st], bool),
                                     np.array([src_code[s.source] for s in st], np.uint8))),
        grow_report=np.array(json.dumps({k: v for k, v in grep.items() if not k.startswith("t_")})),
        reference_seconds_here=np.array([t_init, t_grow]))
    print(f"a9: dims={vol.dims} segments={len(segs)} init {t_init:.2f}s grow {t_grow:.2f}s "
          f"report={rep}")


def io_cases():
    """Reference wire formats: STND (strands.py:63-69) and OOVL (volume.py:236-246)."""
    from strandkit.strands import StrandSet, write_strands
    from strandkit.volume import write_volume

    z = np.load(os.path.join(HERE, "driver_sparse40.npz"))
    off, verts = z["offsets"], z["verts"]
    segs = [Strand(vertices=verts[off[i]:off[i + 1]]) for i in range(len(off) - 1)]
    write_strands(os.path.join(HERE, "io_driver_sparse40.stnd"), StrandSet(segs))
    ori, occ = field_np("sparse", 24, sparse_sigma=1.5)
    vol = vol_of((-5.0, 3.0, 1.0), 1.5, occ, ori)
    write_volume(os.path.join(HERE, "io_sparse24.oovl"), vol)
    print("io fixtures written")


if __name__ == "__main__":
    only = sys.argv[1:]  # e.g. `driver` to regenerate only the driver fixtures
    for fn in (unit_cases, helix_case, analytic_cases, nonfinite_case, sampler_case, driver_cases,
               io_cases, link_cases, a9_case):
        if not only or any(o in fn.__name__ for o in only):
            fn()
