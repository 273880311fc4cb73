"""Parity of the CUDA path (through the C ABI) with the reference and the oracle.

Bar: bit-exact.  The kernel computes in IEEE binary64 in the reference's
evaluation order (csrc/phg_trace.cu), so every vertex of every strand must be
identical to the reference's (golden fixtures) and to the oracle's at larger
sizes; the north_star tolerance (counts exact >= 99.9 %, positions <= 1e-3
voxel) is reported alongside as the weaker, stated bar.
"""

import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, csr_equal, load_case, trace_cases

pytestmark = pytest.mark.gpu

CASES = trace_cases()


@pytest.fixture(scope="module")
def gpu():
    import torch

    from paper_2604_05794_b200 import _native, build

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    build.build()
    _native.load()
    from paper_2604_05794_b200 import phg, volume

    return SimpleNamespace(phg=phg, volume=volume, torch=torch)


def run_gpu(gpu, c, live_counts=None):
    return gpu.phg.trace_batch_csr(c.vol, c.seeds, c.dirs, c.params,
                                   at_cap=getattr(c, "at_cap", None), live_counts=live_counts,
                                   near_occ=getattr(c, "near_occ", None))


def tolerance_report(off_a, v_a, off_b, v_b, vs):
    la, lb = np.diff(off_a), np.diff(off_b)
    same = la == lb
    err = 0.0
    for i in np.flatnonzero(same)[:: max(1, int(same.sum()) // 2000)]:
        a = v_a[off_a[i]:off_a[i + 1]]
        b = v_b[off_b[i]:off_b[i + 1]]
        if len(a):
            err = max(err, float(np.abs(a - b).max()) / vs)
    return float(same.mean()) if len(same) else 1.0, err


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[6:-4])
def test_cuda_matches_reference_golden(gpu, path):
    c = load_case(path)
    counts = c.counts_in.copy() if hasattr(c, "counts_in") else None
    off, v, ent = run_gpu(gpu, c, live_counts=counts)
    assert np.array_equal(ent, c.entered)
    assert csr_equal(off, v, c.offsets, c.verts), tolerance_report(off, v, c.offsets, c.verts,
                                                                   float(c.voxel_size))
    if counts is not None:
        assert np.array_equal(counts, c.counts_out)


def test_cuda_list_output_is_reference_shaped(gpu):
    c = load_case(os.path.join(GOLDEN, "trace_sparse48.npz"))
    out = gpu.phg.trace_batch(c.vol, c.seeds, c.dirs, c.params)
    assert len(out) == len(c.entered)
    for i, (v, e) in enumerate(out):
        assert v.dtype == np.float64 and v.ndim == 2 and v.shape[1] == 3
        assert v.flags.c_contiguous
        assert e is bool(c.entered[i])
        assert np.array_equal(v, c.verts[c.offsets[i]:c.offsets[i + 1]])


def test_cuda_sampler_matches_reference_golden(gpu):
    c = load_case(os.path.join(GOLDEN, "sample_sparse24.npz"))
    d, h, s = gpu.volume.sample_orientation_batch(c.vol, c.pts, c.prev)
    assert np.array_equal(h, c.has)
    assert np.array_equal(s, c.support)
    assert np.array_equal(d, c.dirs)


def test_sampler_sign_follows_query(gpu):
    """test_volume.py:58-67 analog: flipping prev flips the sampled direction."""
    c = load_case(os.path.join(GOLDEN, "sample_sparse24.npz"))
    d1, h1, _ = gpu.volume.sample_orientation_batch(c.vol, c.pts, c.prev)
    d2, h2, _ = gpu.volume.sample_orientation_batch(c.vol, c.pts, -c.prev)
    assert np.array_equal(h1, h2)
    assert np.allclose(d1[h1], -d2[h1], atol=1e-12)


# ---- larger sizes: GPU vs the C oracle on the BASELINE configs ----------------------
def _config_case(kind, n, count, key, params=None, seeds=None, interior=0):
    from paper_2604_05794_b200 import synth

    ori, occ = synth.make_field(kind, n, "cpu")
    ori, occ = ori.numpy(), occ.numpy()
    if seeds is None:
        s, d = synth.disk_seeds(n, count, key)
    else:
        s, d = seeds
    if interior:
        s2, d2 = synth.interior_seeds(occ, ori, interior, key + 100)
        s, d = np.concatenate([s, s2, s2]), np.concatenate([d, d2, -d2])
    p = params or SimpleNamespace(step_mm=1.0, max_vertices=400, min_support=0.05,
                                  probe_steps=24, coast_steps=25, steer=0.0, strict=False)
    vol = SimpleNamespace(origin=np.zeros(3), voxel_size=synth.VOXEL_MM, dims=occ.shape, occ=occ,
                          ori=ori)
    return vol, s, d, p


def _compare_with_oracle(gpu, oracle_c, vol, s, d, p, at_cap=None):
    off, v, ent = gpu.phg.trace_batch_csr(vol, s, d, p, at_cap=at_cap)
    slab, keep, ent_o = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s, d, p,
                                       at_cap=at_cap)
    off_o, v_o = oracle_c.to_csr(slab, keep)
    frac, err = tolerance_report(off, v, off_o, v_o, vol.voxel_size)
    assert frac >= 0.999 and err <= 1e-3, (frac, err)  # north_star bar
    assert np.array_equal(ent, ent_o)
    assert csr_equal(off, v, off_o, v_o)  # our bar: bit-exact
    return off


def test_c1_straight_full_10k_bit_exact(gpu, oracle_c):
    vol, s, d, p = _config_case("straight", 64, 10_000, 11)
    off = _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    assert (np.diff(off) - 1).sum() > 1_000_000


def test_c2_wavy_256_subset_bit_exact(gpu, oracle_c):
    vol, s, d, p = _config_case("wavy", 256, 2_000, 12)
    _compare_with_oracle(gpu, oracle_c, vol, s, d, p)


def test_c3_curly_512_subset_bit_exact(gpu, oracle_c):
    vol, s, d, p = _config_case("curly", 512, 1_000, 13)
    off = _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    assert np.all(np.diff(off) >= 300)


def test_c3_steep_helix_subset_bit_exact(gpu, oracle_c):
    """C3s (the steep variant, W = 4 pi / L: strands climb ~6x higher than C3's) on 1000 seeds
    of the 512^3 field, bit-exact against the oracle; the strands really do climb."""
    from paper_2604_05794_b200 import synth

    cfg = synth.CONFIGS["C3s"]
    ori, occ = cfg.field("cpu")
    ori, occ = ori.numpy(), occ.numpy()
    s, d = synth.disk_seeds(cfg.n, 1_000, cfg.key)
    p = SimpleNamespace(step_mm=1.0, max_vertices=400, min_support=0.05, probe_steps=24,
                        coast_steps=25, steer=0.0, strict=False)
    vol = SimpleNamespace(origin=np.zeros(3), voxel_size=synth.VOXEL_MM, dims=occ.shape,
                          occ=occ, ori=ori)
    off = _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    v = gpu.phg.trace_batch_csr(vol, s, d, p)[1]
    assert np.percentile(v[off[1:] - 1][:, 2], 50) > 40 * synth.VOXEL_MM  # C3: ~9 voxels


def test_c5_sparse_divergent_lengths_bit_exact(gpu, oracle_c):
    vol, s, d, p = _config_case("sparse", 96, 3_000, 15, interior=3_000)
    off = _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    lens = np.diff(off)
    assert lens.max() > 4 * np.median(lens)  # the stress case really is divergent


def test_nonempty_cap_plane_bit_exact(gpu, oracle_c):
    vol, s, d, p = _config_case("curly", 64, 5_000, 16)
    rng = np.random.Generator(np.random.Philox(key=3))
    cap = rng.random(vol.occ.shape) < 0.02
    _compare_with_oracle(gpu, oracle_c, vol, s, d, p, at_cap=cap)


def test_every_kernel_variant_bit_exact(gpu, oracle_c, monkeypatch):
    """Each compiled trace-kernel variant (PHG_VARIANT) against the oracle, with and
    without an at_cap plane, on the divergent sparse field."""
    from paper_2604_05794_b200 import _native

    vol, s, d, p = _config_case("sparse", 64, 1_500, 21, interior=1_500)
    cap = np.random.Generator(np.random.Philox(key=5)).random(vol.occ.shape) < 0.02
    tracer = gpu.phg._tracer()
    names, samplers = [], set()
    nv = _native.load().phg_num_variants()
    for v in range(nv):
        # variant 0 (block signs) needs a field with block bounds, the last variant (bare
        # occupancy flags) one without: forced here, as this sparse field would pick the latter
        if v in (0, nv - 1):
            monkeypatch.setenv("PHG_BLOCK_SIGN", "1" if v == 0 else "0")
            gpu.volume.invalidate()
        monkeypatch.setenv("PHG_VARIANT", str(v))
        for plane in (None, cap):
            _compare_with_oracle(gpu, oracle_c, vol, s, d, p, at_cap=plane)
        names.append(tracer.last_variant())
        samplers.add(tracer.last_sampler())
    assert len(set(names)) == len(names), names
    assert samplers == {"exact", "fast-pow2"}, samplers
    gpu.volume.invalidate()


def _packed_block_bounds(gpu, f, dims):
    """(occupancy flags, block bound floats) of a device field's padded voxels."""
    torch = gpu.torch
    ptr, nbytes, zeroed, _ = f.packed()
    assert zeroed
    arr = gpu.phg._CudaArray(ptr, (nbytes // 4,), "<u4")
    w = torch.as_tensor(arr, device="cuda").view(-1, 4)[:, 3].cpu().numpy()
    nx, ny, nz = dims
    w = w.reshape(nx + 2, ny + 2, nz + 2)
    live = (w & np.uint32(0xFFF00000)) == np.uint32(0x3FF00000)
    dead_ok = (w & np.uint32(0xFFF00000)) == 0
    assert np.all(live | dead_ok)
    # the top 20 bits of a double's high word (low word 0)
    t = ((w & np.uint32(0xFFFFF)).astype(np.uint64) << np.uint64(44)).view(np.float64)
    return live, t


@pytest.mark.parametrize("kind,fill", [("curly", None), ("sparse", None), ("fuzz", 0.5)])
def test_block_bounds_cover_corner_spread(gpu, monkeypatch, kind, fill):
    """The packed field's block bounds (csrc/phg_core.cuh block_bound): for every fully
    occupied block, t >= max over its corners of |o_k - o_base|_1 (computed here in exact
    fp64); +inf for every other block.  These bounds are what lets one fp32 dot decide all
    eight corner signs (and skip the occupancy tests), so an undershoot would be a parity
    bug."""
    if kind == "fuzz":
        rng = np.random.default_rng(7)
        dims = (23, 17, 29)
        occ, ori = _fuzz_field(rng, dims, fill, False)
    else:
        from paper_2604_05794_b200 import synth

        ori, occ = synth.make_field(kind, 48, "cpu")
        ori, occ = ori.numpy(), occ.numpy()
        dims = occ.shape
    monkeypatch.setenv("PHG_BLOCK_SIGN", "0")  # no bounds: .w is the bare occupancy flag
    f = gpu.volume.DeviceField(np.zeros(3), 2.0, occ, ori)
    try:
        live, t = _packed_block_bounds(gpu, f, dims)
    finally:
        f.close()
    assert np.all(t == 0)
    monkeypatch.setenv("PHG_BLOCK_SIGN", "1")  # bounds written whatever the field's sparsity
    f = gpu.volume.DeviceField(np.zeros(3), 2.0, occ, ori)
    try:
        live, t = _packed_block_bounds(gpu, f, dims)
    finally:
        f.close()
    nx, ny, nz = dims
    po = np.zeros((nx + 2, ny + 2, nz + 2), bool)
    po[1:-1, 1:-1, 1:-1] = occ
    pv = np.zeros((nx + 2, ny + 2, nz + 2, 3), np.float64)
    pv[1:-1, 1:-1, 1:-1] = np.where(occ[..., None], ori, 0.0)
    assert np.array_equal(live, po)
    base_v = pv[:-1, :-1, :-1]
    spread = np.zeros(base_v.shape[:3])
    full = np.ones(base_v.shape[:3], bool)
    for k in range(8):
        dx, dy, dz = k >> 2, (k >> 1) & 1, k & 1
        full &= po[dx:dx + nx + 1, dy:dy + ny + 1, dz:dz + nz + 1]
        ov = pv[dx:dx + nx + 1, dy:dy + ny + 1, dz:dz + nz + 1]
        spread = np.maximum(spread, np.abs(ov - base_v).sum(-1))
    tb = t[:-1, :-1, :-1]
    assert full.any()
    assert np.all(np.isfinite(tb[full]))
    assert np.all(tb[full] >= spread[full]), float((spread - tb)[full].max())
    assert np.all(np.isposinf(tb[~full]))
    assert np.all(np.isposinf(t[-1, :, :])) and np.all(np.isposinf(t[:, -1, :]))


@pytest.mark.parametrize("kind,interior", [("curly", 0), ("sparse", 1_500), ("fuzz", 0)])
def test_block_signs_forced_on_and_off_bit_exact(gpu, oracle_c, monkeypatch, kind, interior):
    """The trace kernel with one fp32 dot per certified corner block (Cfg::BSIGN) and with
    per-corner dots only, each forced on both a dense and a sparse field (the automatic
    choice takes the first on C3-like fields, the second on C5-like ones), equal the oracle
    bit for bit, with and without a cap plane."""
    if kind == "fuzz":
        rng = np.random.default_rng(11)
        dims = (31, 26, 35)
        occ, ori = _fuzz_field(rng, dims, 0.85, False)
        vol = SimpleNamespace(origin=np.zeros(3), voxel_size=2.0, dims=dims, occ=occ, ori=ori)
        s = _fuzz_points(rng, dims, 2.0, 4_000)[8:]
        d = rng.normal(size=s.shape)
        p = SimpleNamespace(step_mm=1.0, max_vertices=200, min_support=0.05, probe_steps=24,
                            coast_steps=25, steer=0.0, strict=False)
    else:
        vol, s, d, p = _config_case(kind, 48, 3_000, 61, interior=interior)
    cap = np.random.default_rng(3).random(vol.occ.shape) < 0.02
    tr = gpu.phg._tracer()
    try:
        for force in ("1", "0", None):
            if force is None:
                monkeypatch.delenv("PHG_BLOCK_SIGN", raising=False)
            else:
                monkeypatch.setenv("PHG_BLOCK_SIGN", force)
            gpu.volume.invalidate()
            # the angle-stop kernel always has the block test compiled in: on a field without
            # bounds it must fall through to the per-corner dots
            turn = SimpleNamespace(**vars(p), max_turn_deg=8.0)
            _compare_with_oracle(gpu, oracle_c, vol, s, d, turn, at_cap=cap)
            for plane in (None, cap):
                _compare_with_oracle(gpu, oracle_c, vol, s, d, p, at_cap=plane)
            on = tr.last_variant().endswith("+bsign")
            want = force == "1" if force is not None else {"curly": True, "sparse": False}.get(kind)
            assert want is None or on == want, (force, kind, tr.last_variant())
    finally:
        gpu.volume.invalidate()


@pytest.mark.parametrize("kind,vs,nan,want", [
    ("curly", 2.0, False, "fast-pow2"), ("curly", 1.7, False, "fast"),
    ("sparse", 0.5, False, "fast-pow2"), ("wavy", 2.0, True, "exact")])
def test_sampler_forms_bit_exact(gpu, oracle_c, kind, vs, nan, want):
    """The per-field sampler choice (exact / fast / fast-pow2) on fields of each kind and
    voxel size, against the oracle; one NaN ori anywhere selects the exact sampler."""
    vol, s, d, p = _config_case(kind, 48, 600, 31, interior=600 if kind == "sparse" else 0)
    ori = vol.ori.copy()
    if nan:
        ori[0, 0, 0] = (np.nan, 1.0, 0.0)
    vol.ori, vol.voxel_size = ori, vs
    s = s / synth_voxel() * vs
    _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    assert gpu.phg._tracer().last_sampler() == want


@pytest.mark.parametrize("case", ["orthogonal", "random-unit", "scaled-1e3", "scaled-1e-20"])
@pytest.mark.parametrize("force_fp64", [False, True])
def test_fp32_sign_fallback_bit_exact(gpu, oracle_c, case, force_fp64, monkeypatch):
    """Fields and seeds on which the fp32 corner-sign certificate (Cfg::SIGN32) is unsure:
    live corners exactly orthogonal to the query (d = +-0, incl. -0.0 components in ori and
    seed directions), occupied voxels with ori 0, random unit ori (many near-orthogonal
    corners), and ori far from unit length (the certificate scales with max|ori|).  Every
    case must still equal the oracle bit for bit."""
    n = 40
    vol, s, d, p = _config_case("straight", n, 800, 41)
    ori = vol.ori.copy()
    rng = np.random.Generator(np.random.Philox(key=41))
    if case == "orthogonal":
        # horizontal seed directions on a vertical field: d = +-0 at every live corner
        d = np.zeros_like(d)
        k = rng.integers(0, 4, len(d))
        d[k == 0] = (1.0, 0.0, 0.0)
        d[k == 1] = (-1.0, -0.0, -0.0)
        d[k == 2] = (0.0, -1.0, -0.0)
        d[k == 3] = rng.normal(size=(int((k == 3).sum()), 3))
        occ = vol.occ
        holes = occ & (rng.random(occ.shape) < 0.05)
        ori[holes] = 0.0                                   # occupied, ori exactly 0
        negz = occ & (rng.random(occ.shape) < 0.2)
        ori[negz] = np.array([-0.0, 0.0, 1.0], dtype=np.float32)  # -0.0 components
    elif case == "random-unit":
        r = rng.normal(size=ori.shape)
        r /= np.linalg.norm(r, axis=-1, keepdims=True)
        ori = np.where(vol.occ[..., None], r, 0.0).astype(np.float32)
        d = rng.normal(size=d.shape)
    else:
        scale = 1e3 if case == "scaled-1e3" else 1e-20
        tilt = rng.normal(scale=0.3, size=ori.shape).astype(np.float32)
        ori = np.where(vol.occ[..., None], (ori + tilt) * np.float32(scale), 0.0)
        ori = ori.astype(np.float32)
    vol.ori = ori
    if force_fp64:  # PHG_SIGN32=0: the fallback decides every sample's signs
        monkeypatch.setenv("PHG_SIGN32", "0")
    _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    assert gpu.phg._tracer().last_sampler() == "fast-pow2"


def synth_voxel():
    from paper_2604_05794_b200 import synth

    return synth.VOXEL_MM


def test_seed_order_does_not_change_results(gpu):
    """Locality ordering is scheduling only: seed i's strand is the same at any position."""
    vol, s, d, p = _config_case("sparse", 64, 6_000, 17, interior=1_000)
    off, v, e = gpu.phg.trace_batch_csr(vol, s, d, p)
    perm = np.random.Generator(np.random.Philox(key=4)).permutation(len(s))
    off2, v2, e2 = gpu.phg.trace_batch_csr(vol, s[perm], d[perm], p)
    for k, i in enumerate(perm[:500]):
        assert np.array_equal(v[off[i]:off[i + 1]], v2[off2[k]:off2[k + 1]])
        assert e[i] == e2[k]


def test_slab_budget_chunking_is_bit_identical(gpu, monkeypatch):
    """A seed set whose relaxed trace slab exceeds PHG_SLAB_BUDGET_GB is traced in seed-order
    chunks; offsets, vertices and entered flags equal the single-call result."""
    vol, s, d, p = _config_case("sparse", 64, 6_000, 18, interior=1_000)
    off, v, e = gpu.phg.trace_batch_csr(vol, s, d, p)
    row = gpu.phg.slab_row_bytes(p)
    monkeypatch.setenv("PHG_SLAB_BUDGET_GB", str(1_777 * row / (1 << 30)))  # 4 ragged chunks
    off2, v2, e2 = gpu.phg.trace_batch_csr(vol, s, d, p)
    assert np.array_equal(off, off2) and np.array_equal(v, v2) and np.array_equal(e, e2)
    monkeypatch.setattr(gpu.phg, "_CHUNK_HEADROOM", 0.01)  # host array regrown mid-call
    off3, v3, e3 = gpu.phg.trace_batch_csr(vol, s, d, p)
    assert np.array_equal(off, off3) and np.array_equal(v, v3) and np.array_equal(e, e3)


# ---- the reference's own trace tests, run against the GPU drop-in ---------------------
def _column(height=40):
    from paper_2604_05794_b200.volume import OOVolume

    vol = OOVolume.empty(origin=(-10.0, -10.0, 0.0), voxel_size=2.0, dims=(10, 10, height))
    vol.occ[:] = True
    vol.ori[:] = np.asarray((0.0, 0.0, 1.0), dtype=np.float32)
    return vol


def test_reference_unit_tests_on_gpu(gpu):
    """test_phg.py:33-127 restated against the GPU trace_batch."""
    P = gpu.phg.PhgParams
    tb = gpu.phg.trace_batch
    up, s0 = [[0.0, 0.0, 1.0]], [[0.5, 0.5, 1.0]]
    (v, e), = tb(_column(), s0, up, P(max_vertices=30, probe_steps=0, coast_steps=0))
    assert e and len(v) >= 29 and np.allclose(v[:, :2], [0.5, 0.5], atol=1e-9)
    assert np.allclose(np.diff(v[:, 2]), 1.0)
    (v, e), = tb(_column(5), s0, up, P(max_vertices=60, probe_steps=0, coast_steps=0))
    assert e and len(v) < 20
    vol = _column()
    vol.occ[:, :, :6] = False
    (_, e1), = tb(vol, s0, up, P(max_vertices=40, probe_steps=2, coast_steps=0))
    (v, e2), = tb(vol, s0, up, P(max_vertices=40, probe_steps=15, coast_steps=0))
    assert not e1 and e2 and len(v) > 20
    vol = _column()
    vol.occ[:, :, 10:13] = False
    (vn, _), = tb(vol, s0, up, P(max_vertices=90, probe_steps=0, coast_steps=0))
    (vy, _), = tb(vol, s0, up, P(max_vertices=90, probe_steps=0, coast_steps=12))
    assert vy[-1, 2] > 40.0 and vn[-1, 2] < 25.0
    (v, e), = tb(_column(10), s0, up, P(max_vertices=80, probe_steps=0, coast_steps=10))
    assert e and v[-1, 2] < 22.5
    counts = np.zeros((10, 10, 40), np.uint16)
    out = tb(_column(), [[0.5, 0.5, 1.0], [0.5, 0.5, 0.2]], up + up,
             P(max_vertices=30, probe_steps=0, coast_steps=0, strict=True), live_counts=counts)
    assert len(out[0][0]) >= 29 and len(out[1][0]) < 5 and counts.sum() > 0
    cap = np.zeros((10, 10, 40), bool)
    out = tb(_column(), np.tile(s0, (4, 1)), np.tile(up, (4, 1)),
             P(max_vertices=30, probe_steps=0, coast_steps=0, occupancy_cap=1), at_cap=cap)
    assert all(len(v) >= 29 for v, _ in out)
    cap[:, :, 8:] = True
    (v, e), = tb(_column(), s0, up, P(max_vertices=30, probe_steps=0, coast_steps=0), at_cap=cap)
    assert e and v[-1, 2] < 17.0


def test_errors_map_to_reference_types(gpu):
    from paper_2604_05794_b200.errors import ConfigError, DataError

    vol = _column()
    P = gpu.phg.PhgParams
    with pytest.raises(DataError):
        gpu.phg.trace_batch(vol, np.zeros((3, 3)), np.zeros((2, 3)), P())
    with pytest.raises(ConfigError):
        gpu.phg.trace_batch(vol, np.zeros((1, 3)), np.ones((1, 3)), P(max_vertices=0))
    with pytest.raises(DataError):
        gpu.phg.trace_batch(vol, np.zeros((1, 3)), np.ones((1, 3)), P(), at_cap=np.zeros((2, 2, 2)))
    assert gpu.phg.trace_batch(vol, np.zeros((0, 3)), np.zeros((0, 3)), P()) == []


def test_field_with_border_beyond_32bit_index_is_rejected(gpu):
    """The padded field ((nx+2)(ny+2)(nz+2) voxels) must index in 32 bits: 1626^3 fits
    unpadded but not with its border; the check runs before any array is read."""
    import ctypes

    from paper_2604_05794_b200 import _native

    lib = _native.load()
    f = ctypes.c_void_p()
    tiny = np.zeros(3, np.float32)
    org = np.zeros(3)
    rc = lib.phg_field_create(ctypes.byref(f), tiny.ctypes.data, tiny.ctypes.data, 1626, 1626,
                              1626, org.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              ctypes.c_double(2.0), None)
    assert rc == _native.PHG_ERR_INVALID and not f.value
    assert b"border" in lib.phg_last_error()


@pytest.mark.parametrize("dims", [(1, 1, 40), (2, 1, 3), (1, 7, 1), (3, 3, 3)])
def test_degenerate_dims_bit_exact(gpu, oracle_c, dims):
    """Fields one or two voxels thick on some axis (every corner block touches the border)."""
    rng = np.random.Generator(np.random.Philox(key=sum(dims)))
    occ = rng.random(dims) < 0.7
    ori = rng.normal(size=dims + (3,)).astype(np.float32)
    ori[..., 2] = np.abs(ori[..., 2]) + 0.5
    vol = SimpleNamespace(origin=np.array([-0.3, 0.2, 0.1]), voxel_size=2.0, dims=dims, occ=occ,
                          ori=ori)
    ext = np.array(dims) * 2.0
    s = vol.origin + rng.random((300, 3)) * ext * 1.2 - 0.1 * ext
    d = rng.normal(size=(300, 3))
    p = SimpleNamespace(step_mm=0.7, max_vertices=60, min_support=0.05, probe_steps=4,
                        coast_steps=3, steer=0.0, strict=False)
    _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    assert gpu.phg._tracer().last_sampler() == "fast-pow2"


def test_install_reroutes_module_global(gpu):
    """install() replaces trace_batch on a reference-shaped module and disables the fork pool."""
    import types

    mod = types.ModuleType("fake_phg")
    mod.trace_batch = lambda *a, **k: "cpu"
    mod._make_pool = lambda *a, **k: "pool"
    gpu.phg.install(mod)
    try:
        assert mod.trace_batch is gpu.phg.trace_batch
        assert mod._make_pool(None, None, None, 8) is None
    finally:
        gpu.phg.uninstall(mod)
    assert mod.trace_batch() == "cpu"
    mod.grow = mod.init_guide_strands = mod.connect_segments = lambda *a, **k: "cpu"
    gpu.phg.install(mod, full=True)
    try:
        from paper_2604_05794_b200 import grow, link

        assert mod.init_guide_strands is grow.init_guide_strands
        assert mod.connect_segments is link.connect_segments
        assert mod.grow is link.grow
    finally:
        gpu.phg.uninstall(mod)
    assert mod.grow() == "cpu" and mod._make_pool() == "pool"


def test_device_api_matches_host_api(gpu):
    torch = gpu.torch
    vol, s, d, p = _config_case("wavy", 64, 3_000, 18)
    off, v, e = gpu.phg.trace_batch_csr(vol, s, d, p)
    f = gpu.volume.field_for(vol)
    f.set_cap(None)
    f.set_near(None)
    o2, v2, e2 = gpu.phg.trace_device(f, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), p)
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy(), off)
    assert np.array_equal(v2.cpu().numpy(), v)
    assert np.array_equal(e2.cpu().numpy().astype(bool), e)


def test_pipelined_host_path_matches(gpu):
    """phg_trace_to_host (chunked, overlapped D2H) == phg_trace + phg_gather, any chunking."""
    torch = gpu.torch
    vol, s, d, p = _config_case("sparse", 64, 9_000, 19, interior=2_000)
    off, v, e = gpu.phg.trace_batch_csr(vol, s, d, p)
    f = gpu.volume.field_for(vol)
    f.set_cap(None)
    f.set_near(None)
    tr = gpu.phg.Tracer()
    n = len(s)
    for chunk in (0, 1000, 4096, n):
        o2 = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        e2 = torch.empty(n, dtype=torch.uint8).pin_memory()
        v2 = torch.empty((len(v) + 5, 3), dtype=torch.float64).pin_memory()
        total = tr.trace_to_host(f, p, s.ctypes.data, d.ctypes.data, n, o2.data_ptr(),
                                 e2.data_ptr(), v2.data_ptr(), v2.shape[0], chunk)
        assert total == len(v)
        assert np.array_equal(o2.numpy(), off)
        assert np.array_equal(e2.numpy().astype(bool), e)
        assert np.array_equal(v2.numpy()[:total], v)
    from paper_2604_05794_b200.errors import PipelineError

    small = torch.empty((10, 3), dtype=torch.float64).pin_memory()
    with pytest.raises(PipelineError):
        tr.trace_to_host(f, p, s.ctypes.data, d.ctypes.data, n, o2.data_ptr(), e2.data_ptr(),
                         small.data_ptr(), 10, 0)


def test_shared_reciprocal_division_matches_ieee_division(gpu):
    """csrc div_by(x, d, div_recip(d)) == x / d bitwise over 8M random + edge operands."""
    import ctypes

    from paper_2604_05794_b200 import _native

    lib = _native.load()
    bad = ctypes.c_int64(-1)
    _native.check(lib.phg_selftest(8_000_000, 12345, ctypes.byref(bad), None), "selftest")
    assert bad.value == 0


def test_c3_full_size_properties(gpu, oracle_c):
    """BASELINE C3 at full size (512^3 curly field, 1M disk seeds), device-resident:
    * a random sample of 2000 strands of the full trace equals the oracle bit for bit;
    * the trace does not depend on seed order (all 1M lengths and the sampled strands are
      identical when the seeds are reversed);
    * accepted steps = sum(len - 1) over strands, as the bench counts them."""
    from paper_2604_05794_b200 import phg, synth
    from paper_2604_05794_b200.volume import DeviceField

    torch = gpu.torch
    dev = torch.device("cuda", 0)
    cfg = synth.CONFIGS["C3"]
    ori, occ = cfg.field(dev)
    field = DeviceField(np.zeros(3), synth.VOXEL_MM, occ, ori,
                        torch.cuda.current_stream(dev).cuda_stream)
    s, d = synth.config_seeds(cfg, cfg.seeds, ori, occ)
    params = phg.PhgParams(field_seeds=0, batch_size=len(s))
    s_dev, d_dev = torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)
    off, verts, ent = phg.trace_device(field, s_dev, d_dev, params)
    lens = torch.diff(off)
    off_r, verts_r, ent_r = phg.trace_device(field, s_dev.flip(0), d_dev.flip(0), params)
    assert torch.equal(torch.diff(off_r).flip(0), lens)
    assert torch.equal(ent_r.flip(0), ent)
    assert int((lens - 1).sum()) == int(verts.shape[0]) - len(s)

    pick = np.sort(np.random.Generator(np.random.Philox(key=77)).choice(len(s), 2000,
                                                                        replace=False))
    off_h, ent_h = off.cpu().numpy(), ent.cpu().numpy()
    offr_h = off_r.cpu().numpy()
    vol = SimpleNamespace(origin=np.zeros(3), voxel_size=synth.VOXEL_MM, dims=occ.shape,
                          occ=occ.cpu().numpy(), ori=ori.cpu().numpy())
    slab, keep, ent_o = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s[pick],
                                       d[pick], params)
    off_o, v_o = oracle_c.to_csr(slab, keep)
    n = len(s)
    for k, i in enumerate(pick):
        got = verts[off_h[i]:off_h[i + 1]].cpu().numpy()
        assert np.array_equal(got, v_o[off_o[k]:off_o[k + 1]]), i
        assert bool(ent_h[i]) == bool(ent_o[k])
        j = n - 1 - i  # position of seed i in the reversed launch
        assert np.array_equal(got, verts_r[offr_h[j]:offr_h[j + 1]].cpu().numpy())


def test_c5_full_size_properties(gpu, oracle_c):
    """BASELINE C5 at full field size (1024^3, 10% fill; 1M seeds: half disk, half interior
    traced both ways), device-resident: order independence of all lengths, and a random
    sample of 1000 strands bit-exact against the oracle on the host copy of the field."""
    from paper_2604_05794_b200 import phg, synth
    from paper_2604_05794_b200.volume import DeviceField

    torch = gpu.torch
    dev = torch.device("cuda", 0)
    cfg = synth.CONFIGS["C5"]
    ori, occ = cfg.field(dev)
    field = DeviceField(np.zeros(3), synth.VOXEL_MM, occ, ori,
                        torch.cuda.current_stream(dev).cuda_stream)
    s, d = synth.config_seeds(cfg, 1_000_000, ori, occ)
    params = phg.PhgParams(field_seeds=0, batch_size=len(s))
    s_dev, d_dev = torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)
    off, verts, ent = phg.trace_device(field, s_dev, d_dev, params)
    lens = torch.diff(off)
    assert int(lens.max()) > 4 * float(lens.float().median())  # divergent lengths
    off_r, _, ent_r = phg.trace_device(field, s_dev.flip(0), d_dev.flip(0), params)
    assert torch.equal(torch.diff(off_r).flip(0), lens)
    assert torch.equal(ent_r.flip(0), ent)

    pick = np.sort(np.random.Generator(np.random.Philox(key=78)).choice(len(s), 1000,
                                                                        replace=False))
    off_h, ent_h = off.cpu().numpy(), ent.cpu().numpy()
    occ_h, ori_h = occ.cpu().numpy(), ori.cpu().numpy()
    del ori, occ
    slab, keep, ent_o = oracle_c.trace(np.zeros(3), synth.VOXEL_MM, occ_h, ori_h, s[pick],
                                       d[pick], params)
    off_o, v_o = oracle_c.to_csr(slab, keep)
    for k, i in enumerate(pick):
        got = verts[off_h[i]:off_h[i + 1]].cpu().numpy()
        assert np.array_equal(got, v_o[off_o[k]:off_o[k + 1]]), i
        assert bool(ent_h[i]) == bool(ent_o[k])


@pytest.mark.parametrize("count,cap", [(3_000, False), (30_000, False), (30_000, True)])
def test_rows_api_equals_csr_and_oracle(gpu, oracle_c, count, cap):
    """phg_trace_rows (device-resident strand rows, no CSR copy) holds exactly the strands of
    the CSR path and of the oracle: strand(i) == buf[i, :keep[i]] (phg.py:159-162), with and
    without the queue-order row map (launches beyond half a wave of resident lanes, SMs x 4 x
    128 / 2, sort the seeds) and a cap plane."""
    torch = gpu.torch
    min_sorted = torch.cuda.get_device_properties(0).multi_processor_count * 4 * 128 // 2
    vol, s, d, p = _config_case("sparse", 64, count, 31, interior=count // 4)
    at_cap = None
    if cap:
        rng = np.random.default_rng(5)
        at_cap = rng.random(vol.occ.shape) < 0.02
    off, v, ent = gpu.phg.trace_batch_csr(vol, s, d, p, at_cap=at_cap)
    f = gpu.volume.field_for(vol)
    f.set_cap(at_cap)
    f.set_near(None)
    tr = gpu.phg.Tracer()
    rs = gpu.phg.trace_device_rows(f, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(),
                                   p, tracer=tr)
    assert (rs.rowmap is not None) == (len(s) >= min_sorted)
    o2, v2, e2 = rs.to_csr()
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy(), off)
    assert np.array_equal(v2.cpu().numpy(), v)
    assert np.array_equal(e2.cpu().numpy().astype(bool), ent)
    assert rs.steps == len(v) - len(s) and rs.kept == len(v)
    i = len(s) // 3
    assert np.array_equal(rs.strand(i).cpu().numpy(), v[off[i]:off[i + 1]])
    slab, keep, _ = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s, d, p,
                                   at_cap=at_cap)
    off_o, v_o = oracle_c.to_csr(slab, keep)
    assert np.array_equal(off_o, off) and np.array_equal(v_o, v)
    assert tr.last_steps() >= rs.steps  # accepted steps include trimmed trailing coasts


@pytest.mark.parametrize("kind,deg", [("curly", 4.0), ("sparse", 10.0), ("wavy", 2.0)])
def test_opt_in_turn_stop(gpu, oracle_c, kind, deg):
    """The opt-in angle stop (PhgParams.max_turn_deg, PHG_FLAG_TURN_STOP; not in the
    reference): off (0) leaves every output identical to the reference semantics; on, the
    CUDA path equals the C oracle's restatement of the same rule bit for bit and stops some
    strands earlier."""
    vol, s, d, p = _config_case(kind, 48, 6_000, 41, interior=1_000 if kind == "sparse" else 0)
    base = gpu.phg.trace_batch_csr(vol, s, d, p)
    off0 = gpu.phg.trace_batch_csr(vol, s, d, SimpleNamespace(**vars(p), max_turn_deg=0.0))
    assert all(np.array_equal(a, b) for a, b in zip(base, off0))
    pt = SimpleNamespace(**vars(p), max_turn_deg=deg)
    for cap in (None, np.random.default_rng(2).random(vol.occ.shape) < 0.02):
        off, v, ent = gpu.phg.trace_batch_csr(vol, s, d, pt, at_cap=cap)
        slab, keep, ent_o = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s, d, pt,
                                           at_cap=cap)
        off_o, v_o = oracle_c.to_csr(slab, keep)
        assert np.array_equal(off, off_o) and np.array_equal(v, v_o)
        assert np.array_equal(ent, ent_o)
    assert len(v) < len(base[1]), "the angle stop never fired"


@pytest.mark.parametrize("kind,n,dims", [("sparse", 64, None), ("curly", 48, None),
                                         ("sparse", 40, (37, 41, 43))])
def test_bricked_sampler_bit_exact(gpu, oracle_c, monkeypatch, kind, n, dims):
    """The bricked copy of a sparse field (4^3 bricks with a +1 apron, empty bricks aliased to
    one zero brick; kSmpBrick*) traces bit-identically to the oracle, with and without a cap
    plane and the angle stop, on dims that are not multiples of the brick edge."""
    vol, s, d, p = _config_case(kind, n, 5_000, 51, interior=1_500 if kind == "sparse" else 0)
    if dims is not None:  # crop to odd dims (seeds outside the crop die at once, as they should)
        vol.occ = np.ascontiguousarray(vol.occ[: dims[0], : dims[1], : dims[2]])
        vol.ori = np.ascontiguousarray(vol.ori[: dims[0], : dims[1], : dims[2]])
        vol.dims = vol.occ.shape
    monkeypatch.setenv("PHG_BRICKS", "1")
    gpu.volume.invalidate()
    tr = gpu.phg._tracer()
    cap = np.random.default_rng(9).random(vol.occ.shape) < 0.02
    for plane in (None, cap):
        for pp in (p, SimpleNamespace(**vars(p), max_turn_deg=8.0)):
            off, v, ent = gpu.phg.trace_batch_csr(vol, s, d, pp, at_cap=plane)
            assert tr.last_sampler().startswith("brick"), tr.last_sampler()
            slab, keep, ent_o = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s, d,
                                               pp, at_cap=plane)
            off_o, v_o = oracle_c.to_csr(slab, keep)
            assert np.array_equal(off, off_o) and np.array_equal(v, v_o)
            assert np.array_equal(ent, ent_o)
    monkeypatch.setenv("PHG_BRICKS", "0")
    gpu.volume.invalidate()
    gpu.phg.trace_batch_csr(vol, s[:10], d[:10], p)
    assert not tr.last_sampler().startswith("brick")
    gpu.volume.invalidate()


def test_bricked_driver_bit_exact(gpu, monkeypatch):
    """The device batch driver (speculative windows, recording traces) on a bricked field
    reproduces the reference's init_guide_strands fixtures."""
    from paper_2604_05794_b200 import grow
    from paper_2604_05794_b200.phg import PhgParams
    from paper_2604_05794_b200.volume import OOVolume

    monkeypatch.setenv("PHG_BRICKS", "1")
    gpu.volume.invalidate()
    for name in ("driver_sparse40", "driver_curly32_cap1"):
        c = load_case(os.path.join(GOLDEN, f"{name}.npz"))
        vol = OOVolume.empty(c.origin, float(c.voxel_size), c.occ.shape)
        vol.occ, vol.ori = c.occ, c.ori
        prm = PhgParams(**{k: v for k, v in vars(c.params).items()
                           if k in PhgParams.__dataclass_fields__})
        off, verts, rooted, rep = grow.init_guide_strands_csr(c.seeds, c.dirs, vol, prm)
        assert np.array_equal(off, c.offsets) and np.array_equal(verts, c.verts)
        assert np.array_equal(rooted, c.rooted) and np.array_equal(vol.counts, c.counts_out)
    gpu.volume.invalidate()


@pytest.mark.parametrize("kind,turn", [("sparse", 0.0), ("curly", 0.0), ("curly", 3.0)])
def test_strict_cooperative_equals_per_step_launches(gpu, oracle_c, monkeypatch, kind, turn):
    """Strict mode in one cooperative launch (grid barriers between each step and its
    commits, early exit) equals the per-step launch pairs and the C oracle bit for bit,
    including the in-place live_counts (phg.py:136-155)."""
    vol, s, d, p = _config_case(kind, 48, 3_000, 61, interior=800 if kind == "sparse" else 0)
    p = SimpleNamespace(**vars(p))
    p.strict = True
    p.max_turn_deg = turn  # the opt-in angle stop inside strict mode too
    outs = []
    for coop in ("1", "0"):
        monkeypatch.setenv("PHG_STRICT_COOP", coop)
        counts = np.zeros(vol.occ.shape, np.uint16)
        counts[::3, ::5, ::7] = 1
        res = gpu.phg.trace_batch_csr(vol, s, d, p, live_counts=counts)
        outs.append((res, counts))
        assert gpu.phg._tracer().last_variant() == ("strict/cooperative" if coop == "1"
                                                    else "strict")
    (a, ca), (b, cb) = outs
    assert all(np.array_equal(x, y) for x, y in zip(a, b)) and np.array_equal(ca, cb)
    counts = np.zeros(vol.occ.shape, np.uint16)
    counts[::3, ::5, ::7] = 1
    slab, keep, ent = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s, d, p,
                                     live_counts=counts)
    off_o, v_o = oracle_c.to_csr(slab, keep)
    assert np.array_equal(a[0], off_o) and np.array_equal(a[1], v_o)
    assert np.array_equal(counts, ca)


def _fuzz_field(rng, dims, fill, noise_ori):
    occ = rng.random(dims) < fill
    ori = rng.normal(size=dims + (3,)).astype(np.float32)
    ori /= np.linalg.norm(ori, axis=-1, keepdims=True).astype(np.float32)
    if noise_ori:  # unoccupied voxels with garbage (finite) orientations: the fast sampler
        ori[~occ] *= 7.5  # must still ignore them (packed as 0 where unoccupied)
    else:
        ori[~occ] = 0
    return occ, ori


def _fuzz_points(rng, dims, vs, m):
    hi = np.array(dims) * vs
    pts = rng.uniform(-0.3 * hi, 1.3 * hi, size=(m, 3))     # inside and around the field
    k = m // 4
    pts[:k] = np.round(pts[:k] / (vs / 2)) * (vs / 2)          # exactly on voxel faces/centres
    pts[k:k + 8] = [[0, 0, 0], hi, [hi[0], 0, 0], [0, hi[1], 0], [0, 0, hi[2]],
                    [-vs, -vs, -vs], [1e300, 0, 0], [-1e300, 5, 5]]
    return pts


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_fuzz_sampler_and_trace_bit_exact(gpu, oracle_c, seed):
    """Randomised fields (odd dims, non-power-of-two voxel sizes, occupied fractions from
    sparse to dense, garbage orientations in empty voxels) and points / seeds inside, outside,
    exactly on voxel faces and far away, with random and zero directions: the CUDA sampler
    equals the numpy restatement of sample_orientation_batch (volume.py:190-224) and the CUDA
    trace equals the C oracle, bit for bit, with and without a cap plane."""
    from oracle import phg_oracle_np as onp

    rng = np.random.default_rng(seed)
    dims = tuple(int(x) for x in rng.integers(5, 40, size=3))
    vs = float(rng.choice([0.5, 1.0, 1.3, 2.0, 2.7]))
    occ, ori = _fuzz_field(rng, dims, float(rng.uniform(0.1, 0.9)), seed % 2 == 1)
    origin = rng.uniform(-5, 5, size=3)
    vol = SimpleNamespace(origin=origin, voxel_size=vs, dims=dims, occ=occ, ori=ori)
    pts = _fuzz_points(rng, dims, vs, 20_000) + origin
    prev = rng.normal(size=pts.shape)
    prev[::7] = 0.0
    d, h, s = gpu.volume.sample_orientation_batch(vol, pts, prev)
    f = onp.Field(origin, vs, dims, occ, ori)
    d_o, h_o, s_o = onp.sample(f, pts, prev)
    assert np.array_equal(h, h_o) and np.array_equal(s, s_o) and np.array_equal(d, d_o)
    seeds = _fuzz_points(rng, dims, vs, 6_000)[8:] + origin  # finite seeds
    dirs = rng.normal(size=seeds.shape)
    dirs[::11] = 0.0
    p = SimpleNamespace(step_mm=float(rng.choice([0.4, 1.0, 1.7])), max_vertices=int(
        rng.choice([2, 57, 400])), min_support=float(rng.choice([0.0, 0.05, 0.3])),
        probe_steps=int(rng.integers(0, 30)), coast_steps=int(rng.integers(0, 30)), steer=0.0,
        strict=False)
    for cap in (None, rng.random(dims) < 0.05):
        off, v, ent = gpu.phg.trace_batch_csr(vol, seeds, dirs, p, at_cap=cap)
        slab, keep, ent_o = oracle_c.trace(origin, vs, occ, ori, seeds, dirs, p, at_cap=cap)
        off_o, v_o = oracle_c.to_csr(slab, keep)
        assert np.array_equal(off, off_o) and np.array_equal(v, v_o) and np.array_equal(ent, ent_o)


def test_steering_runs_on_the_fast_sampler(gpu, oracle_c):
    """Steering (near_occ, steer > 0, phg.py:108-117) on a finite field now samples with the
    fast (zeroed-field) sampler; it equals the C oracle bit for bit, with and without a cap
    plane."""
    from scipy.ndimage import distance_transform_edt

    vol, s, d, p = _config_case("sparse", 64, 4_000, 71, interior=1_000)
    _, inds = distance_transform_edt(~vol.occ, return_indices=True)
    near = np.ascontiguousarray(np.stack(inds, axis=-1).astype(np.int64))
    p = SimpleNamespace(**vars(p))
    p.steer = 0.35
    for cap in (None, np.random.default_rng(4).random(vol.occ.shape) < 0.02):
        off, v, ent = gpu.phg.trace_batch_csr(vol, s, d, p, at_cap=cap, near_occ=near)
        assert gpu.phg._tracer().last_sampler() == "fast-pow2"
        slab, keep, ent_o = oracle_c.trace(vol.origin, vol.voxel_size, vol.occ, vol.ori, s, d, p,
                                           at_cap=cap, near_occ=near)
        off_o, v_o = oracle_c.to_csr(slab, keep)
        assert np.array_equal(off, off_o) and np.array_equal(v, v_o)
        assert np.array_equal(ent, ent_o)


def test_rows_api_edge_cases(gpu):
    """phg_trace_rows: zero seeds give an empty RowSet; strict mode (which needs live_counts
    and per-step commits) is refused with the reference's DataError."""
    torch = gpu.torch
    from paper_2604_05794_b200.errors import DataError

    vol, s, d, p = _config_case("curly", 32, 100, 97)
    f = gpu.volume.field_for(vol)
    f.set_cap(None)
    f.set_near(None)
    tr = gpu.phg.Tracer()
    empty = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    rs = gpu.phg.trace_device_rows(f, empty, empty, p, tracer=tr)
    assert rs.n == 0 and rs.steps == 0 and rs.kept == 0
    off, v, e = rs.to_csr()
    assert off.shape == (1,) and v.shape == (0, 3) and e.shape == (0,)
    ps = SimpleNamespace(**vars(p))
    ps.strict = True
    with pytest.raises(DataError):
        gpu.phg.trace_device_rows(f, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), ps,
                                  tracer=tr)
    tr.close()


def test_device_api_validates_and_copies_strided_seeds(gpu):
    """The device APIs take any (n,3) float64 CUDA tensors: strided views are made contiguous
    (the C ABI reads plain arrays); wrong dtypes / lengths raise the reference's DataError."""
    torch = gpu.torch
    from paper_2604_05794_b200.errors import DataError

    vol, s, d, p = _config_case("curly", 32, 400, 99)
    f = gpu.volume.field_for(vol)
    f.set_cap(None)
    f.set_near(None)
    sp, sd = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
    ref = gpu.phg.trace_device(f, sp[::2], sd[::2], p)
    got = gpu.phg.trace_device(f, sp[::2].contiguous(), sd[::2].contiguous(), p)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(ref, got))
    rs = gpu.phg.trace_device_rows(f, sp[::2], sd[::2], p)
    o2, v2, e2 = rs.to_csr()
    assert torch.equal(o2, ref[0]) and torch.equal(v2, ref[1])
    with pytest.raises(DataError):
        gpu.phg.trace_device(f, sp.float(), sd.float(), p)
    with pytest.raises(DataError):
        gpu.phg.trace_device_rows(f, sp, sd[:10], p)


@pytest.mark.parametrize("kind", ["straight", "curly"])
def test_certified_blocks_against_the_field_bit_exact(gpu, oracle_c, kind):
    """Strands running against the field direction on a dense field: every certified block has
    the negative sign, so the unsigned block sums are flipped (0 + s*sum).  The straight field's
    x/y sums are exactly zero, which exercises the sign-of-zero argument of that flip.  Seeds
    start mid-height, with exact and tilted directions, plus exactly orthogonal ones (d0 = 0:
    never certified)."""
    vol, _, _, p = _config_case(kind, 40, 10, 71)
    rng = np.random.default_rng(71)
    n = 3000
    L = 40 * synth_voxel()
    r = 0.4 * L * np.sqrt(rng.random(n))
    th = 2 * np.pi * rng.random(n)
    s = np.stack([L / 2 + r * np.cos(th), L / 2 + r * np.sin(th), rng.uniform(0.3, 0.7, n) * L], 1)
    d = np.tile([0.0, 0.0, -1.0], (n, 1))
    d[n // 3: 2 * n // 3] += rng.normal(scale=0.2, size=(n // 3, 3))
    d[2 * n // 3:] = np.stack([np.cos(th[2 * n // 3:]), np.sin(th[2 * n // 3:]),
                               np.zeros(n - 2 * n // 3)], 1)
    gpu.volume.invalidate()
    _compare_with_oracle(gpu, oracle_c, vol, s, d, p)
    assert gpu.phg._tracer().last_variant().endswith("+bsign")


@pytest.mark.parametrize("scale", [1e3, 1.0, 1e-20, 1e-30])
def test_block_signs_on_scaled_and_noisy_fields_bit_exact(gpu, oracle_c, monkeypatch, scale):
    """Block sign certificates (forced on) on a dense field whose orientations are scaled far
    from unit length and carry per-voxel noise, so the bounds, sign_eps and the base dot all
    scale together and a share of the blocks fails the certificate: equal to the oracle."""
    vol, s, d, p = _config_case("curly", 32, 4_000, 83)
    rng = np.random.default_rng(83)
    noise = rng.normal(scale=0.05, size=vol.ori.shape).astype(np.float32)
    vol.ori = np.where(vol.occ[..., None], (vol.ori + noise) * np.float32(scale), 0.0)
    vol.ori = vol.ori.astype(np.float32)
    d = d + rng.normal(scale=0.3, size=d.shape)
    monkeypatch.setenv("PHG_BLOCK_SIGN", "1")
    gpu.volume.invalidate()
    try:
        for cap in (None, rng.random(vol.occ.shape) < 0.03):
            _compare_with_oracle(gpu, oracle_c, vol, s, d, p, at_cap=cap)
        assert gpu.phg._tracer().last_variant().endswith("+bsign")
    finally:
        gpu.volume.invalidate()
