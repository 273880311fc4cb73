"""Pin the oracle (C and numpy restatements) bit-exact to the reference's golden outputs."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, csr_equal, load_case, trace_cases
from oracle import phg_oracle_np as onp

CASES = trace_cases()


def _run_c(oc, c):
    counts = c.counts_in.copy() if hasattr(c, "counts_in") else None
    slab, keep, ent = oc.trace(c.origin, c.voxel_size, c.occ, c.ori, c.seeds, c.dirs, c.params,
                               at_cap=getattr(c, "at_cap", None), live_counts=counts,
                               near_occ=getattr(c, "near_occ", None))
    off, v = oc.to_csr(slab, keep)
    return off, v, ent, counts


def test_golden_fixtures_present():
    assert len(CASES) >= 20


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[6:-4])
def test_c_oracle_matches_reference(oracle_c, path):
    c = load_case(path)
    off, v, ent, counts = _run_c(oracle_c, c)
    assert csr_equal(off, v, c.offsets, c.verts)
    assert np.array_equal(ent, c.entered)
    if counts is not None:
        assert np.array_equal(counts, c.counts_out)


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[6:-4])
def test_numpy_oracle_matches_reference(oracle_c, path):
    c = load_case(path)
    f = onp.Field(c.origin, c.voxel_size, c.occ.shape, c.occ, c.ori)
    counts = c.counts_in.copy() if hasattr(c, "counts_in") else None
    slab, keep, ent = onp.trace(f, c.seeds, c.dirs, c.params, at_cap=getattr(c, "at_cap", None),
                                live_counts=counts, near_occ=getattr(c, "near_occ", None))
    off, v = oracle_c.to_csr(slab, keep)
    assert csr_equal(off, v, c.offsets, c.verts)
    assert np.array_equal(ent, c.entered)
    if counts is not None:
        assert np.array_equal(counts, c.counts_out)


def test_oracle_sampler_matches_reference(oracle_c):
    c = load_case(os.path.join(GOLDEN, "sample_sparse24.npz"))
    d, h, s = oracle_c.sample(c.origin, c.voxel_size, c.occ, c.ori, c.pts, c.prev)
    assert np.array_equal(d, c.dirs) and np.array_equal(h, c.has) and np.array_equal(s, c.support)
    d2, h2, s2 = onp.sample(onp.Field(c.origin, c.voxel_size, c.occ.shape, c.occ, c.ori), c.pts,
                            c.prev)
    assert np.array_equal(d2, c.dirs) and np.array_equal(h2, c.has)
    assert np.array_equal(s2, c.support)


def test_oracle_threads_do_not_change_results(oracle_c):
    c = load_case(os.path.join(GOLDEN, "trace_sparse48.npz"))
    outs = [oracle_c.trace(c.origin, c.voxel_size, c.occ, c.ori, c.seeds, c.dirs, c.params,
                           threads=t) for t in (1, 4)]
    assert np.array_equal(outs[0][1], outs[1][1])
    for i, k in enumerate(outs[0][1]):
        assert np.array_equal(outs[0][0][i, :k], outs[1][0][i, :k])


def test_golden_properties_match_reference_tests():
    """The fixtures reproduce the reference's own trace assertions (test_phg.py:33-127)."""
    def strands(name):
        c = load_case(os.path.join(GOLDEN, f"trace_{name}.npz"))
        return [c.verts[c.offsets[i]:c.offsets[i + 1]] for i in range(len(c.entered))], c.entered

    (v,), (e,) = strands("unit_straight")
    assert e and len(v) >= 29 and np.allclose(np.diff(v[:, 2]), 1.0)
    (v,), _ = strands("unit_slab_top")
    assert len(v) < 20
    _, (e,) = strands("unit_probe2")
    assert not e
    (v,), (e,) = strands("unit_probe15")
    assert e and len(v) > 20
    (v,), _ = strands("unit_coast12")
    assert v[-1, 2] > 40.0
    (v,), _ = strands("unit_coast0")
    assert v[-1, 2] < 25.0
    (v,), _ = strands("unit_trim")
    assert v[-1, 2] < 22.5
    vs, _ = strands("unit_strict")
    assert len(vs[0]) >= 29 and len(vs[1]) < 5
    vs, _ = strands("unit_deferred")
    assert all(len(v) >= 29 for v in vs)
    (v,), _ = strands("unit_at_cap")
    assert v[-1, 2] < 17.0


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_c_and_numpy_oracles_agree_on_fuzz(seed, oracle_c):
    """The two restatements (scalar C, vectorised numpy; each pinned to the reference's
    fixtures) agree bit for bit on randomised fields and seeds: odd dims, non-power-of-two
    voxel sizes, seeds on voxel faces / outside / far away, zero directions."""
    from types import SimpleNamespace

    from oracle import phg_oracle_np as onp

    rng = np.random.default_rng(100 + seed)
    dims = tuple(int(x) for x in rng.integers(5, 30, size=3))
    vs = float(rng.choice([0.5, 1.3, 2.0, 2.7]))
    occ = rng.random(dims) < rng.uniform(0.1, 0.9)
    ori = rng.normal(size=dims + (3,)).astype(np.float32)
    ori /= np.linalg.norm(ori, axis=-1, keepdims=True).astype(np.float32)
    ori[~occ] = 0
    origin = rng.uniform(-5, 5, size=3)
    hi = np.array(dims) * vs
    seeds = rng.uniform(-0.3 * hi, 1.3 * hi, size=(3000, 3))
    seeds[:700] = np.round(seeds[:700] / (vs / 2)) * (vs / 2)
    seeds += origin
    dirs = rng.normal(size=seeds.shape)
    dirs[::11] = 0.0
    p = SimpleNamespace(step_mm=float(rng.choice([0.4, 1.0, 1.7])), max_vertices=57,
                        min_support=float(rng.choice([0.0, 0.05, 0.3])), probe_steps=12,
                        coast_steps=6, steer=0.0, strict=False)
    cap = rng.random(dims) < 0.05
    f = onp.Field(origin, vs, dims, occ, ori)
    for plane in (None, cap):
        slab, keep, ent = oracle_c.trace(origin, vs, occ, ori, seeds, dirs, p, at_cap=plane)
        slab2, keep2, ent2 = onp.trace(f, seeds, dirs, p, at_cap=plane)
        assert np.array_equal(keep, keep2) and np.array_equal(ent, ent2)
        for i in range(len(keep)):
            assert np.array_equal(slab[i, :keep[i]], slab2[i, :keep[i]])
