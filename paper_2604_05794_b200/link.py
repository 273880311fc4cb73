"""Segment linking, scalp attachment and the full ``grow`` stage on the GPU.

Drop-ins for strandkit.phg (phg.py):
  connect_segments(segments, params)         :389-413  (compute_links :337-377 inside)
  grow(scalp, vol, params=None, workers=1)   :445-469  init_guide_strands -> connect_segments
                                                       -> attach_to_scalp -> tangents
The arithmetic runs in libphg_b200.so (csrc/phg_link.cu): candidate pairs by a uniform-grid
radius search, (d, i, j) ordering by stable radix sorts, chain assembly / smoothing /
numpy-exact resampling / exact nearest-scalp-vertex attachment / tangents on the device; the
greedy union-find acceptance (sequential by definition) runs in the library's native host
code.  Results are bit-identical to the reference (tests/test_link.py).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DataError
from .grow import GrowParams, Strand, _nearest_occupied_map
from .phg import PhgParams, _tracer, split_rows
from .volume import field_for

try:  # the reference's container when importable
    from strandkit.strands import StrandSet  # type: ignore
except Exception:  # noqa: BLE001
    @dataclass
    class StrandSet:
        """Mirror of strandkit.strands.StrandSet (strands.py:30-37)."""

        strands: list

        def __len__(self):
            return len(self.strands)

        def __iter__(self):
            return iter(self.strands)

SOURCES = ("traced", "field", "linked", "attached")
_SRC_CODE = {s: i for i, s in enumerate(SOURCES)}


def link_params(params, attach=True) -> _native.LinkParams:
    # the gate is computed with numpy exactly as compute_links does (phg.py:351)
    gate = float(np.cos(np.deg2rad(params.link_angle_deg)))
    return _native.LinkParams(float(params.link_dist_mm), gate, float(params.smooth_strength),
                              float(params.step_mm), float(params.attach_radius_mm),
                              int(params.tangent_window), int(bool(params.smooth)),
                              int(params.smooth_iters), int(bool(attach)))


def _run_link(offsets, verts, rooted, source, n, params, scalp_vertices, attach):
    lib = _native.load()
    tr = _tracer()
    lp = link_params(params, attach=attach)
    out = (ctypes.c_int64 * 4)()
    sv = None
    ns = 0
    if attach:
        sv = np.ascontiguousarray(np.asarray(scalp_vertices, dtype=np.float64).reshape(-1, 3))
        ns = len(sv)
    _native.check(lib.phg_link(tr.handle, offsets, verts, rooted, source, n,
                               sv.ctypes.data if ns else None, ns, ctypes.byref(lp), out, None),
                  "phg_link")
    nstr, nv, nlinks, nunrooted = (int(x) for x in out)
    off = np.empty(nstr + 1, np.int64)
    v = np.empty((nv, 3))
    t = np.empty((nv, 3))
    r = np.empty(nstr, np.uint8)
    s = np.empty(nstr, np.uint8)
    links = np.empty((nlinks, 2), np.int64)
    _native.check(lib.phg_link_fetch(tr.handle, off.ctypes.data, v.ctypes.data if nv else None,
                                     t.ctypes.data if nv else None,
                                     r.ctypes.data if nstr else None,
                                     s.ctypes.data if nstr else None,
                                     links.ctypes.data if nlinks else None, None),
                  "phg_link_fetch")
    if attach and ns == 0 and not r.all():
        # attach_to_scalp queries SpatialIndex(scalp.vertices).nearest for unrooted strands
        raise DataError("nearest() on an empty index")
    return {"offsets": off, "verts": v, "tangents": t, "rooted": r.astype(bool), "source": s,
            "links": links, "n_unrooted": nunrooted}


def connect_segments_csr(offsets, verts, rooted, source, params, scalp_vertices=None):
    """CSR in, CSR out: linking (+ attachment when ``scalp_vertices`` is given)."""
    offsets = np.ascontiguousarray(offsets, np.int64)
    verts = np.ascontiguousarray(verts, np.float64).reshape(-1, 3)
    rooted = np.ascontiguousarray(rooted, np.uint8)
    source = np.ascontiguousarray(source, np.uint8)
    n = len(offsets) - 1
    return _run_link(offsets.ctypes.data, verts.ctypes.data if len(verts) else None,
                     rooted.ctypes.data if n else None, source.ctypes.data if n else None, n,
                     params, scalp_vertices, scalp_vertices is not None)


def _strands(res, with_tangents):
    off = res["offsets"]
    verts = split_rows(res["verts"], off)
    names = [SOURCES[c] for c in res["source"].tolist()]
    out = [Strand(vertices=v, rooted=r, source=s)
           for v, r, s in zip(verts, res["rooted"].tolist(), names)]
    if with_tangents:
        for s, t in zip(out, split_rows(res["tangents"], off)):
            s.tangents = t
    return out


def connect_segments(segments, params):
    """GPU drop-in for strandkit.phg.connect_segments (phg.py:389-413)."""
    if len(segments) == 0:
        return []
    lens = [len(s.vertices) for s in segments]
    off = np.zeros(len(segments) + 1, np.int64)
    off[1:] = np.cumsum(lens)
    verts = np.concatenate([np.asarray(s.vertices, np.float64).reshape(-1, 3) for s in segments])
    rooted = np.array([bool(s.rooted) for s in segments], np.uint8)
    source = np.array([_SRC_CODE.get(s.source, 0) for s in segments], np.uint8)
    return _strands(connect_segments_csr(off, verts, rooted, source, params), False)


def grow(scalp, vol, params=None, workers=1):
    """GPU drop-in for strandkit.phg.grow (phg.py:445-469): the whole PHG stage on the device.

    ``t_link`` covers linking and attachment (one device pass); ``t_attach`` is reported as 0.
    """
    if params is None:
        params = PhgParams()
    lib = _native.load()
    report = {}
    t0 = time.perf_counter()
    seeds = np.ascontiguousarray(np.asarray(scalp.seeds, np.float64).reshape(-1, 3))
    normals = np.ascontiguousarray(np.asarray(scalp.seed_normals, np.float64).reshape(-1, 3))
    init_report = {"n_seeds": int(len(seeds)), "n_segments": 0, "n_never_entered": 0}
    have_segments = False
    if len(seeds) == 0:
        init_report["warning"] = "no scalp seeds; nothing to trace"
    else:
        f = field_for(vol)
        counts = vol.counts
        if not (isinstance(counts, np.ndarray) and counts.dtype == np.uint16
                and counts.flags.c_contiguous and counts.shape == f.dims):
            raise DataError("vol.counts must be a C-contiguous uint16 array of the field dims")
        f.set_near(_nearest_occupied_map(vol) if float(params.steer) > 0 else None)
        tr = _tracer()
        p = _native.params_struct(params)
        g = GrowParams(int(params.batch_size), int(params.occupancy_cap), int(params.field_seeds), 0)
        nseg, nv = ctypes.c_int64(), ctypes.c_int64()
        rep = (ctypes.c_int64 * 4)()
        _native.check(lib.phg_grow_init(tr.handle, f.handle, ctypes.byref(p), ctypes.byref(g),
                                        seeds.ctypes.data, normals.ctypes.data, len(seeds),
                                        counts.ctypes.data, ctypes.byref(nseg), ctypes.byref(nv),
                                        rep, None), "phg_grow_init")
        init_report["n_never_entered"] = int(rep[0])
        init_report["n_scalp_segments"] = int(rep[1])
        init_report["n_segments"] = int(nseg.value)
        have_segments = nseg.value > 0
    report["guide_init"] = init_report
    report["t_guide_init"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    if have_segments:
        # link straight from the device-resident segments of phg_grow_init
        res = _run_link(None, None, None, None, 0, params, scalp.vertices, True)
        strands = _strands(res, True)
        n_unrooted = res["n_unrooted"]
    else:
        strands, n_unrooted = [], 0
    report["n_after_link"] = len(strands)
    report["t_link"] = time.perf_counter() - t1
    report["n_unrooted"] = n_unrooted
    report["t_attach"] = 0.0
    if not strands:
        report["warning"] = "empty volume or no traceable seeds; no strands grown"
    return StrandSet(strands), report
