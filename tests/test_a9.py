"""The reference's A9 scene (test_acceptance.py:302-334): the scene behind the only published
PHG timing (2.70 s, pkg/test_output.txt:28-34).  Inputs come from tests/golden/a9_scene.npz
(written by the reference's own scene pipeline); the outputs of init_guide_strands and of
the full grow() are compared with the reference's by SHA-256 digest (bit-exact)."""

import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, load_case

A9 = os.path.join(GOLDEN, "a9_scene.npz")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def a9_inputs():
    from paper_2604_05794_b200.phg import PhgParams
    from paper_2604_05794_b200.volume import OOVolume

    c = load_case(A9)
    lp = json.loads(str(c.link_params))
    params = PhgParams(**{**{k: v for k, v in vars(c.params).items()
                             if k in PhgParams.__dataclass_fields__}, **lp})
    vol = OOVolume.empty(c.origin, float(c.voxel_size), c.occ.shape)
    vol.occ, vol.ori = c.occ, c.ori
    scalp = SimpleNamespace(seeds=c.seeds, seed_normals=c.dirs, vertices=c.scalp_vertices)
    return c, vol, scalp, params


def test_a9_fixture_is_the_reference_scene():
    c = load_case(A9)
    assert c.occ.shape == (115, 116, 80) and len(c.seeds) == 4000
    assert json.loads(str(c.init_report))["n_segments"] == 7925


@pytest.mark.gpu
def test_a9_init_guide_strands_bit_exact():
    from paper_2604_05794_b200 import grow

    c, vol, scalp, params = a9_inputs()
    segs, rep = grow.init_guide_strands(scalp, vol, params)
    off = np.zeros(len(segs) + 1, np.int64)
    off[1:] = np.cumsum([len(s.vertices) for s in segs])
    got = digest(off, np.concatenate([s.vertices for s in segs]),
                 np.array([s.rooted for s in segs], bool), vol.counts)
    assert rep == json.loads(str(c.init_report))
    assert got == str(c.init_digest)


@pytest.mark.gpu
def test_a9_grow_bit_exact():
    from paper_2604_05794_b200 import link

    c, vol, scalp, params = a9_inputs()
    sset, rep = link.grow(scalp, vol, params)
    st = list(sset)
    off = np.zeros(len(st) + 1, np.int64)
    off[1:] = np.cumsum([len(s.vertices) for s in st])
    got = digest(off, np.concatenate([s.vertices for s in st]),
                 np.concatenate([s.tangents for s in st]),
                 np.array([s.rooted for s in st], bool),
                 np.array([link.SOURCES.index(s.source) for s in st], np.uint8))
    ref = json.loads(str(c.grow_report))
    assert {k: rep[k] for k in ref} == ref
    assert got == str(c.grow_digest)
