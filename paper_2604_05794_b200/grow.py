"""Device batch driver: ``init_guide_strands`` with deferred commits on the GPU.

Drop-in for strandkit.phg.init_guide_strands (phg.py:210-260) including the
field-seed second pass _trace_field_seeds (phg.py:263-303).  The whole loop --
frozen at_cap plane per batch, trace, segment selection, per-segment unique-voxel
commits to ``vol.counts``, unvisited-voxel field seeds, bidirectional traces and
joins -- runs in libphg_b200.so (csrc/phg_grow.cu); Python only builds the
reference's ``Strand`` objects from the CSR result.  Outputs (segments, report,
and the in-place update of ``vol.counts``) are bit-identical to the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DataError
from .phg import _tracer, split_rows
from .volume import field_for

try:  # the reference's own container when it is importable (drop-in object identity)
    from strandkit.strands import Strand  # type: ignore
except Exception:  # noqa: BLE001
    @dataclass
    class Strand:
        """Mirror of strandkit.strands.Strand (strands.py:19-27)."""

        vertices: np.ndarray
        rooted: bool = False
        source: str = "traced"
        tangents: np.ndarray | None = field(default=None, repr=False)

        def __len__(self):
            return len(self.vertices)


class GrowParams(ctypes.Structure):
    """phg_grow_params_v1"""

    _fields_ = [("batch_size", ctypes.c_int32), ("occupancy_cap", ctypes.c_int32),
                ("field_seeds", ctypes.c_int32), ("reserved", ctypes.c_int32)]


def _nearest_occupied_map(vol):
    """phg.nearest_occupied_map (phg.py:57-64): EDT indices of the nearest occupied voxel."""
    from scipy.ndimage import distance_transform_edt

    if not vol.occ.any():
        return None
    _, inds = distance_transform_edt(~vol.occ, return_indices=True)
    return np.stack(inds, axis=-1)


def init_guide_strands_csr(seeds, normals, vol, params):
    """Run the device driver; returns (offsets, verts, rooted, report) and updates vol.counts."""
    lib = _native.load()
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.float64).reshape(-1, 3))
    normals = np.ascontiguousarray(np.asarray(normals, dtype=np.float64).reshape(-1, 3))
    if len(seeds) != len(normals):
        raise DataError("scalp seeds and seed_normals lengths differ")
    counts = vol.counts
    if not (isinstance(counts, np.ndarray) and counts.dtype == np.uint16
            and counts.flags.c_contiguous):
        raise DataError("vol.counts must be a C-contiguous uint16 array")
    f = field_for(vol)
    if counts.shape != f.dims:
        raise DataError(f"vol.counts shape {counts.shape} != field dims {f.dims}")
    near = _nearest_occupied_map(vol) if float(params.steer) > 0 else None
    f.set_near(near)
    tr = _tracer()
    p = _native.params_struct(params)
    g = GrowParams(int(params.batch_size), int(params.occupancy_cap), int(params.field_seeds), 0)
    nseg, nv = ctypes.c_int64(), ctypes.c_int64()
    rep = (ctypes.c_int64 * 4)()
    n = len(seeds)
    _native.check(lib.phg_grow_init(tr.handle, f.handle, ctypes.byref(p), ctypes.byref(g),
                                    seeds.ctypes.data if n else None,
                                    normals.ctypes.data if n else None, n, counts.ctypes.data,
                                    ctypes.byref(nseg), ctypes.byref(nv), rep, None),
                  "phg_grow_init")
    offsets = np.empty(nseg.value + 1, np.int64)
    verts = np.empty((nv.value, 3))
    rooted = np.empty(nseg.value, np.uint8)
    _native.check(lib.phg_grow_fetch(tr.handle, offsets.ctypes.data,
                                     verts.ctypes.data if nv.value else None,
                                     rooted.ctypes.data if nseg.value else None, None),
                  "phg_grow_fetch")
    report = {"n_never_entered": int(rep[0]), "n_scalp_segments": int(rep[1]),
              "n_field_seeds": int(rep[2]), "n_field_segments": int(rep[3])}
    return offsets, verts, rooted.astype(bool), report


class DeviceGrowSession:
    """Batch-level steps of the device driver (C ABI phg_grow_begin .. phg_grow_end).

    The backend of dist.init_guide_strands_multirank on a GPU: seeds in, exported commit
    ids out as CUDA tensors (for an NCCL all-gather), ids of every rank applied back in.
    """

    def __init__(self, vol, params, device=None):
        import torch

        self.torch = torch
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.lib = _native.load()
        self.vol = vol
        self.params = params
        self.field = field_for(vol)
        self.tracer = _tracer()
        self._p = _native.params_struct(params)
        self._g = GrowParams(int(params.batch_size), int(params.occupancy_cap),
                             int(params.field_seeds), 0)
        near = _nearest_occupied_map(vol) if float(params.steer) > 0 else None
        self.field.set_near(near)

    def _ck(self, rc, what):
        _native.check(rc, what)

    def begin(self, counts):
        self._ck(self.lib.phg_grow_begin(self.tracer.handle, self.field.handle,
                                         ctypes.byref(self._p), ctypes.byref(self._g),
                                         counts.ctypes.data, None), "phg_grow_begin")

    def _ids(self, n):
        ids = self.torch.empty(max(int(n), 1), dtype=self.torch.int32, device=self.device)[:n]
        self._ck(self.lib.phg_grow_commits(self.tracer.handle, ids.data_ptr() if n else None,
                                           None), "phg_grow_commits")
        return ids

    def scalp_batch(self, seeds, normals, export):
        seeds = np.ascontiguousarray(seeds, np.float64)
        normals = np.ascontiguousarray(normals, np.float64)
        out = (ctypes.c_int64 * 2)()
        n = len(seeds)
        self._ck(self.lib.phg_grow_scalp_batch(self.tracer.handle,
                                               seeds.ctypes.data if n else None,
                                               normals.ctypes.data if n else None, n,
                                               int(export), out, None), "phg_grow_scalp_batch")
        return int(out[0]), (self._ids(out[1]) if export else None)

    def field_begin(self):
        nf = ctypes.c_int64()
        self._ck(self.lib.phg_grow_field_begin(self.tracer.handle, ctypes.byref(nf), None),
                 "phg_grow_field_begin")
        return int(nf.value)

    def field_batch(self, first, nb, export):
        out = (ctypes.c_int64 * 2)()
        self._ck(self.lib.phg_grow_field_batch(self.tracer.handle, int(first), int(nb),
                                               int(export), out, None), "phg_grow_field_batch")
        return int(out[0]), (self._ids(out[1]) if export else None)

    def apply(self, ids):
        n = int(ids.numel())
        self._ck(self.lib.phg_grow_apply(self.tracer.handle, ids.data_ptr() if n else None, n,
                                         None), "phg_grow_apply")

    def end(self, counts):
        nseg, nv = ctypes.c_int64(), ctypes.c_int64()
        rep = (ctypes.c_int64 * 4)()
        self._ck(self.lib.phg_grow_end(self.tracer.handle, counts.ctypes.data, ctypes.byref(nseg),
                                       ctypes.byref(nv), rep, None), "phg_grow_end")
        offsets = np.empty(nseg.value + 1, np.int64)
        verts = np.empty((nv.value, 3))
        rooted = np.empty(nseg.value, np.uint8)
        self._ck(self.lib.phg_grow_fetch(self.tracer.handle, offsets.ctypes.data,
                                         verts.ctypes.data if nv.value else None,
                                         rooted.ctypes.data if nseg.value else None, None),
                 "phg_grow_fetch")
        return offsets, verts, rooted.astype(bool), int(rep[0])


def init_guide_strands(scalp, vol, params, workers=1):
    """GPU drop-in for strandkit.phg.init_guide_strands (phg.py:210-260).

    Returns (segments, report) with the reference's Strand objects and report keys;
    ``workers`` is accepted for signature compatibility (the GPU replaces the pool).
    """
    seeds, normals = scalp.seeds, scalp.seed_normals
    report = {"n_seeds": int(len(seeds)), "n_segments": 0, "n_never_entered": 0}
    if len(seeds) == 0:
        report["warning"] = "no scalp seeds; nothing to trace"
        return [], report
    offsets, verts, rooted, rep = init_guide_strands_csr(seeds, normals, vol, params)
    segments = [Strand(vertices=part, rooted=r, source="traced" if r else "field")
                for part, r in zip(split_rows(verts, offsets), rooted.tolist())]
    report["n_never_entered"] = rep["n_never_entered"]
    report["n_scalp_segments"] = rep["n_scalp_segments"]
    report["n_segments"] = len(segments)
    return segments, report
