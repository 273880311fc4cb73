"""Segment linking / chain assembly / scalp attachment / grow (phg.py:337-469): the oracle
pinned to reference fixtures on CPU, the device implementation bit-exact on GPU."""

import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, load_case

LINK = os.path.join(GOLDEN, "link_random400.npz")
GROW = [os.path.join(GOLDEN, f"grow_{n}.npz") for n in ("sparse40", "curly32")]


def _csr(rows):
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(v) for v in rows])
    return off, (np.concatenate(rows) if rows else np.zeros((0, 3)))


def _segments(c):
    return [c.seg_verts[c.seg_offsets[i]:c.seg_offsets[i + 1]] for i in range(len(c.seg_offsets) - 1)]


# ---- CPU: oracle vs the reference's outputs ----------------------------------------------
def test_link_oracle_matches_reference():
    from oracle import phg_link_np as L

    c = load_case(LINK)
    out, lk = L.connect(_segments(c), c.seg_rooted, c.seg_source, vars(c.params))
    assert np.array_equal(np.array(lk, np.int64).reshape(-1, 2), c.links)
    off, v = _csr([s[0] for s in out])
    assert np.array_equal(off, c.offsets) and np.array_equal(v, c.verts)
    assert np.array_equal([s[2] for s in out], c.source)


@pytest.mark.parametrize("path", GROW, ids=lambda p: os.path.basename(p)[:-4])
def test_grow_oracle_matches_reference(path, oracle_c):
    from oracle import phg_driver_np as dn
    from oracle import phg_link_np as L

    g = load_case(path)
    lp = json.loads(str(g.link_params))
    counts = np.zeros(g.occ.shape, np.uint16)
    segs, _ = dn.init_guide(g.origin, float(g.voxel_size), g.occ, g.ori, counts, g.seeds, g.dirs,
                            g.params)
    st, _ = L.connect([v for v, _ in segs], [r for _, r in segs], [0 if r else 1 for _, r in segs],
                      lp)
    st, unrooted = L.attach(st, g.scalp_vertices, lp["attach_radius_mm"])
    off, v = _csr([s[0] for s in st])
    assert np.array_equal(off, g.offsets) and np.array_equal(v, g.verts)
    assert np.array_equal(np.concatenate([L.tangents(s[0]) for s in st]), g.tangents)
    assert np.array_equal([s[1] for s in st], g.rooted)
    assert np.array_equal([s[2] for s in st], g.source)
    assert unrooted == json.loads(str(g.report))["n_unrooted"]


# ---- GPU ------------------------------------------------------------------------------------
def _params(**kw):
    from paper_2604_05794_b200.phg import PhgParams

    return PhgParams(**{k: v for k, v in kw.items() if k in PhgParams.__dataclass_fields__})


@pytest.mark.gpu
def test_device_link_matches_reference():
    from paper_2604_05794_b200 import link

    c = load_case(LINK)
    res = link.connect_segments_csr(c.seg_offsets, c.seg_verts, c.seg_rooted, c.seg_source,
                                    _params(**vars(c.params)))
    assert np.array_equal(res["links"], c.links)
    assert np.array_equal(res["offsets"], c.offsets)
    assert np.array_equal(res["verts"], c.verts)
    assert np.array_equal(res["source"], c.source)
    assert np.array_equal(res["rooted"], c.rooted)


@pytest.mark.gpu
def test_device_connect_segments_dropin():
    from paper_2604_05794_b200 import link
    from paper_2604_05794_b200.grow import Strand

    c = load_case(LINK)
    segs = [Strand(vertices=v) for v in _segments(c)]
    out = link.connect_segments(segs, _params(**vars(c.params)))
    off, v = _csr([s.vertices for s in out])
    assert np.array_equal(off, c.offsets) and np.array_equal(v, c.verts)
    assert [s.source for s in out] == [("traced", "field", "linked", "attached")[k]
                                       for k in c.source]
    assert link.connect_segments([], _params()) == []


@pytest.mark.gpu
@pytest.mark.parametrize("path", GROW, ids=lambda p: os.path.basename(p)[:-4])
def test_device_grow_matches_reference(path):
    from paper_2604_05794_b200 import link
    from paper_2604_05794_b200.volume import OOVolume

    g = load_case(path)
    lp = json.loads(str(g.link_params))
    params = _params(**{**vars(g.params), **lp})
    vol = OOVolume.empty(g.origin, float(g.voxel_size), g.occ.shape)
    vol.occ, vol.ori = g.occ, g.ori
    scalp = SimpleNamespace(seeds=g.seeds, seed_normals=g.dirs, vertices=g.scalp_vertices)
    sset, rep = link.grow(scalp, vol, params)
    strands = list(sset)
    off, v = _csr([s.vertices for s in strands])
    assert np.array_equal(off, g.offsets) and np.array_equal(v, g.verts)
    assert np.array_equal(np.concatenate([s.tangents for s in strands]), g.tangents)
    assert np.array_equal([s.rooted for s in strands], g.rooted)
    assert [s.source for s in strands] == [link.SOURCES[k] for k in g.source]
    ref = json.loads(str(g.report))
    assert rep["guide_init"] == ref["guide_init"]
    assert rep["n_after_link"] == ref["n_after_link"]
    assert rep["n_unrooted"] == ref["n_unrooted"]


@pytest.mark.gpu
def test_device_link_matches_oracle_random_large():
    """4000 random short segments in a 200 mm box, mixed rooted/source flags: exact."""
    from oracle import phg_link_np as L
    from paper_2604_05794_b200 import link

    rng = np.random.Generator(np.random.Philox(key=90))
    segs = []
    for _ in range(4000):
        a = rng.uniform(-100, 100, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        segs.append(a + np.outer(np.linspace(0, 5.0, int(rng.integers(2, 9))), d))
    lp = dict(link_dist_mm=6.0, link_angle_deg=50.0, tangent_window=3, smooth=True,
              smooth_strength=0.3, smooth_iters=3, step_mm=0.7)
    off, v = _csr(segs)
    rooted = (rng.random(len(segs)) < 0.3).astype(np.uint8)
    source = rng.integers(0, 2, len(segs)).astype(np.uint8)
    res = link.connect_segments_csr(off, v, rooted, source, _params(**lp))
    out, lk = L.connect(segs, rooted, source, lp)
    assert np.array_equal(res["links"], np.array(lk, np.int64).reshape(-1, 2))
    o2, v2 = _csr([s[0] for s in out])
    assert np.array_equal(res["offsets"], o2) and np.array_equal(res["verts"], v2)
    assert np.array_equal(res["source"], [s[2] for s in out])
    assert len(lk) > 100
