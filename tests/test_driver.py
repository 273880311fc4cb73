"""Deferred-commit batch driver (init_guide_strands, phg.py:210-303): oracle pinned to the
reference's fixtures on CPU; the device driver (csrc/phg_grow.cu) checked bit-exact on GPU."""

import glob
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, load_case

DRIVER_CASES = sorted(glob.glob(os.path.join(GOLDEN, "driver_*.npz")))


def near_map(occ):
    from scipy.ndimage import distance_transform_edt

    _, inds = distance_transform_edt(~occ, return_indices=True)
    return np.stack(inds, axis=-1)


def _csr(out):
    off = np.zeros(len(out) + 1, np.int64)
    off[1:] = np.cumsum([len(v) for v, _ in out])
    verts = np.concatenate([v for v, _ in out]) if out else np.zeros((0, 3))
    return off, verts, np.array([r for _, r in out], bool)


def test_driver_fixtures_present():
    assert len(DRIVER_CASES) >= 4


@pytest.mark.parametrize("path", DRIVER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
def test_driver_oracle_matches_reference(path, oracle_c):
    from oracle import phg_driver_np as dn

    c = load_case(path)
    counts = np.zeros(c.occ.shape, np.uint16)
    near = near_map(c.occ) if c.params.steer > 0 else None
    out, rep = dn.init_guide(c.origin, float(c.voxel_size), c.occ, c.ori, counts, c.seeds, c.dirs,
                             c.params, near_occ=near)
    off, verts, rooted = _csr(out)
    assert np.array_equal(off, c.offsets)
    assert np.array_equal(verts, c.verts)
    assert np.array_equal(rooted, c.rooted)
    assert np.array_equal(counts, c.counts_out)
    assert rep == json.loads(str(c.report))


# ---- GPU ----------------------------------------------------------------------------------
def _params(d):
    from paper_2604_05794_b200.phg import PhgParams

    return PhgParams(**{k: d[k] for k in d if k in PhgParams.__dataclass_fields__})


@pytest.mark.gpu
@pytest.mark.parametrize("path", DRIVER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
def test_device_driver_matches_reference(path):
    from paper_2604_05794_b200 import grow
    from paper_2604_05794_b200.volume import OOVolume

    c = load_case(path)
    vol = OOVolume.empty(c.origin, float(c.voxel_size), c.occ.shape)
    vol.occ, vol.ori = c.occ, c.ori
    scalp = SimpleNamespace(seeds=c.seeds, seed_normals=c.dirs)
    segs, rep = grow.init_guide_strands(scalp, vol, _params(vars(c.params)))
    off, verts, rooted = _csr([(s.vertices, s.rooted) for s in segs])
    assert np.array_equal(off, c.offsets)
    assert np.array_equal(verts, c.verts)
    assert np.array_equal(rooted, c.rooted)
    assert [s.source for s in segs] == ["traced" if r else "field" for r in c.rooted]
    assert np.array_equal(vol.counts, c.counts_out)
    assert rep == json.loads(str(c.report))


@pytest.mark.gpu
def test_device_driver_prefilled_counts_and_uint16_wrap(oracle_c):
    """Pre-filled vol.counts (some at 65535 so commits wrap to 0 like numpy's uint16 +=):
    the incrementally maintained cap plane must match counts >= cap after every batch."""
    from oracle import phg_driver_np as dn
    from paper_2604_05794_b200 import grow, synth
    from paper_2604_05794_b200.volume import OOVolume

    ori, occ = synth.make_field("curly", 40, "cpu")
    ori, occ = ori.numpy(), occ.numpy()
    rng = np.random.Generator(np.random.Philox(key=77))
    init = rng.choice(np.array([0, 0, 0, 1, 2, 3, 65534, 65535], np.uint16), size=occ.shape)
    seeds, dirs = synth.disk_seeds(40, 3000, 42)
    params = _params(dict(batch_size=300, occupancy_cap=3, field_seeds=700, max_vertices=150))
    vol = OOVolume.empty((0, 0, 0), synth.VOXEL_MM, occ.shape)
    vol.occ, vol.ori, vol.counts = occ, ori, init.copy()
    segs, rep = grow.init_guide_strands(SimpleNamespace(seeds=seeds, seed_normals=dirs), vol,
                                        params)
    counts = init.copy()
    out, rep_o = dn.init_guide(np.zeros(3), synth.VOXEL_MM, occ, ori, counts, seeds, dirs, params)
    assert np.array_equal(vol.counts, counts)
    assert rep == rep_o
    off, verts, rooted = _csr([(s.vertices, s.rooted) for s in segs])
    off_o, verts_o, rooted_o = _csr(out)
    assert np.array_equal(off, off_o) and np.array_equal(verts, verts_o)
    assert np.array_equal(rooted, rooted_o)
    assert (counts < init).any()  # some voxel really wrapped


@pytest.mark.gpu
@pytest.mark.parametrize("scalp_inside", [False, True])
def test_device_driver_wrap_in_field_window(oracle_c, scalp_inside):
    """A uint16 wrap inside the field pass's optimistic window (and, with scalp seeds inside
    the volume, in both passes): the window is rolled back and redone batch by batch, and the
    result must still equal the oracle bit for bit (segments, counts, report).  The cap is
    unreachable for uint16 counts, so strands cross the pre-filled 65535 voxels and wrap them;
    scalp seeds below the volume never enter, so every commit comes from the field pass."""
    from oracle import phg_driver_np as dn
    from paper_2604_05794_b200 import grow, synth
    from paper_2604_05794_b200.volume import OOVolume

    ori, occ = synth.make_field("curly", 40, "cpu")
    ori, occ = ori.numpy(), occ.numpy()
    rng = np.random.Generator(np.random.Philox(key=91))
    init = rng.choice(np.array([0, 0, 0, 0, 1, 65535], np.uint16), size=occ.shape)
    seeds, dirs = synth.disk_seeds(40, 600, 43)
    if not scalp_inside:
        seeds = seeds - np.array([0.0, 0.0, 500.0])  # below the volume: never entered
    params = _params(dict(batch_size=64, occupancy_cap=100000, field_seeds=900, max_vertices=120))
    vol = OOVolume.empty((0, 0, 0), synth.VOXEL_MM, occ.shape)
    vol.occ, vol.ori, vol.counts = occ, ori, init.copy()
    segs, rep = grow.init_guide_strands(SimpleNamespace(seeds=seeds, seed_normals=dirs), vol,
                                        params)
    counts = init.copy()
    out, rep_o = dn.init_guide(np.zeros(3), synth.VOXEL_MM, occ, ori, counts, seeds, dirs, params)
    assert np.array_equal(vol.counts, counts)
    assert rep == rep_o
    off, verts, rooted = _csr([(s.vertices, s.rooted) for s in segs])
    off_o, verts_o, rooted_o = _csr(out)
    assert np.array_equal(off, off_o) and np.array_equal(verts, verts_o)
    assert np.array_equal(rooted, rooted_o)
    assert (counts < init).any()  # some voxel really wrapped
    assert (~rooted_o).sum() > 0  # the field pass produced segments


def _driver_vs_oracle(kind, n, nseeds, key, radius_frac=0.4, **pkw):
    from oracle import phg_driver_np as dn
    from paper_2604_05794_b200 import grow, synth
    from paper_2604_05794_b200.volume import OOVolume

    ori, occ = synth.make_field(kind, n, "cpu")
    ori, occ = ori.numpy(), occ.numpy()
    seeds, dirs = synth.disk_seeds(n, nseeds, key, radius_frac=radius_frac)
    params = _params(pkw)
    vol = OOVolume.empty((0, 0, 0), synth.VOXEL_MM, occ.shape)
    vol.occ, vol.ori = occ, ori
    segs, rep = grow.init_guide_strands(SimpleNamespace(seeds=seeds, seed_normals=dirs), vol,
                                        params)
    counts = np.zeros(occ.shape, np.uint16)
    near = near_map(occ) if params.steer > 0 else None
    out, rep_o = dn.init_guide(np.zeros(3), synth.VOXEL_MM, occ, ori, counts, seeds, dirs, params,
                               near_occ=near)
    assert rep == rep_o
    assert np.array_equal(vol.counts, counts)
    off, verts, rooted = _csr([(s.vertices, s.rooted) for s in segs])
    off_o, verts_o, rooted_o = _csr(out)
    assert np.array_equal(off, off_o) and np.array_equal(rooted, rooted_o)
    assert np.array_equal(verts, verts_o)
    return rep


@pytest.mark.gpu
def test_device_driver_long_segments_global_hash_tables(oracle_c):
    """max_vertices 2500 with small steps: joined field segments exceed the shared-memory
    hash table, exercising the global-memory commit path (csrc/phg_grow.cu)."""
    rep = _driver_vs_oracle("wavy", 48, 600, 51, step_mm=0.05, max_vertices=2500,
                            batch_size=200, occupancy_cap=3, field_seeds=300)
    assert rep["n_segments"] > rep["n_scalp_segments"] > 0


@pytest.mark.gpu
def test_device_driver_strict_at_scale(oracle_c):
    _driver_vs_oracle("curly", 48, 1500, 52, strict=True, batch_size=500, field_seeds=400,
                      max_vertices=150)


@pytest.mark.gpu
def test_device_driver_steer_at_scale(oracle_c):
    _driver_vs_oracle("sparse", 48, 2000, 53, radius_frac=0.45, steer=0.4, coast_steps=6,
                      batch_size=700, occupancy_cap=2, field_seeds=800)


@pytest.mark.gpu
def test_device_driver_matches_oracle_at_scale(oracle_c):
    """128^3 curly field, 20k scalp seeds in 5 batches with cap 4, 8k field seeds."""
    from oracle import phg_driver_np as dn
    from paper_2604_05794_b200 import grow, synth
    from paper_2604_05794_b200.volume import OOVolume

    ori, occ = synth.make_field("curly", 128, "cpu")
    ori, occ = ori.numpy(), occ.numpy()
    seeds, dirs = synth.disk_seeds(128, 20_000, 41)
    params = _params(dict(batch_size=4096, occupancy_cap=4, field_seeds=8000, max_vertices=200))
    vol = OOVolume.empty((0, 0, 0), synth.VOXEL_MM, occ.shape)
    vol.occ, vol.ori = occ, ori
    segs, rep = grow.init_guide_strands(SimpleNamespace(seeds=seeds, seed_normals=dirs), vol,
                                        params)
    counts = np.zeros(occ.shape, np.uint16)
    out, rep_o = dn.init_guide(np.zeros(3), synth.VOXEL_MM, occ, ori, counts, seeds, dirs, params)
    assert rep == rep_o
    assert np.array_equal(vol.counts, counts)
    off, verts, rooted = _csr([(s.vertices, s.rooted) for s in segs])
    off_o, verts_o, rooted_o = _csr(out)
    assert np.array_equal(off, off_o) and np.array_equal(rooted, rooted_o)
    assert np.array_equal(verts, verts_o)
    assert rep["n_scalp_segments"] > 1000 and rep["n_segments"] > rep["n_scalp_segments"]


@pytest.mark.gpu
@pytest.mark.parametrize("cap,kind,window", [(1, "curly", "0"), (1, "curly", "5"),
                                             (2, "sparse", "0"), (16, "wavy", "7")])
def test_speculative_driver_equals_sequential(monkeypatch, cap, kind, window):
    """phg_grow_init traces all batches of a phase in one launch against the plane at the start
    and truncates each batch to the plane it must see (csrc/phg_grow.cu, spec_truncate_kernel).
    With 24 batches and a low cap most later strands are cut; the result must equal the
    per-batch traces (PHG_DRIVER_SPEC=0) in segments, order and counts.  ``window`` batches
    per speculative launch (PHG_SPEC_WINDOW; 0 = the default, here the whole phase)."""
    from paper_2604_05794_b200 import grow, synth
    from paper_2604_05794_b200.volume import OOVolume

    ori, occ = synth.make_field(kind, 96, "cpu")
    ori, occ = ori.numpy(), occ.numpy()
    seeds, dirs = synth.disk_seeds(96, 24_000, 61, radius_frac=0.45)
    params = _params(dict(batch_size=1000, occupancy_cap=cap, field_seeds=6000, max_vertices=250))

    monkeypatch.setenv("PHG_SPEC_WINDOW", window)

    def run(spec):
        monkeypatch.setenv("PHG_DRIVER_SPEC", "1" if spec else "0")
        vol = OOVolume.empty((0, 0, 0), synth.VOXEL_MM, occ.shape)
        vol.occ, vol.ori = occ, ori
        segs, rep = grow.init_guide_strands(SimpleNamespace(seeds=seeds, seed_normals=dirs), vol,
                                            params)
        return _csr([(s.vertices, s.rooted) for s in segs]), vol.counts.copy(), rep

    (off_s, v_s, r_s), counts_s, rep_s = run(True)
    (off_q, v_q, r_q), counts_q, rep_q = run(False)
    assert rep_s == rep_q and rep_s["n_segments"] > 0
    assert np.array_equal(off_s, off_q) and np.array_equal(r_s, r_q)
    assert np.array_equal(v_s, v_q)
    assert np.array_equal(counts_s, counts_q)


@pytest.mark.gpu
@pytest.mark.parametrize("path", DRIVER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
def test_reference_batch_loop_over_dropin_trace_batch(path, oracle_c):
    """The reference's own init_guide_strands batch loop (restated in oracle/phg_driver_np.py:
    per-batch frozen at_cap plane, commits, field-seed pass with +d/-d joins, strict
    live_counts) calling the drop-in ``phg.trace_batch`` on the GPU -- what strandkit.phg runs
    after install() -- reproduces the reference's fixtures: per-batch set_cap uploads, the
    field cache reused across batches of one volume, strict mode's in-place live_counts."""
    from oracle import phg_driver_np as dn
    from paper_2604_05794_b200 import phg, volume

    c = load_case(path)
    counts = np.zeros(c.occ.shape, np.uint16)
    near = near_map(c.occ) if c.params.steer > 0 else None
    uploads = []
    real = volume.DeviceField

    class Counting(real):
        def __init__(self, *a, **k):
            uploads.append(1)
            super().__init__(*a, **k)

    volume.DeviceField = Counting
    try:
        out, rep = dn.init_guide(c.origin, float(c.voxel_size), c.occ, c.ori, counts, c.seeds,
                                 c.dirs, c.params, near_occ=near, trace_batch=phg.trace_batch)
    finally:
        volume.DeviceField = real
    off, verts, rooted = _csr(out)
    assert np.array_equal(off, c.offsets)
    assert np.array_equal(verts, c.verts)
    assert np.array_equal(rooted, c.rooted)
    assert np.array_equal(counts, c.counts_out)
    assert rep == json.loads(str(c.report))
    assert len(uploads) == 1  # one field upload for the whole loop (field cache)
