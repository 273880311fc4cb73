"""Occupancy/orientation volume and its packed, HBM-resident device copy.

``OOVolume`` mirrors the reference container (strandkit/volume.py:21-56:
origin, voxel_size, dims, occ, ori, counts and the voxel_of / in_bounds /
centers index math) so the package runs without the reference installed; any
object with those attributes (including the reference's own OOVolume) is
accepted everywhere.

``DeviceField`` owns the device copy (K0: float4 (ori.xyz, occ) per voxel,
16 B/voxel, plus optional 1-bit at_cap plane and nearest-occupancy map).
``field_for(vol)`` caches it per volume so repeated ``trace_batch`` calls
from the deferred-commit batch loop (phg.py:229-251) upload the field once.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DataError


@dataclass
class OOVolume:
    origin: np.ndarray
    voxel_size: float
    dims: tuple
    occ: np.ndarray = field(repr=False)
    ori: np.ndarray = field(repr=False)
    counts: np.ndarray = field(repr=False)

    @classmethod
    def empty(cls, origin, voxel_size, dims):
        nx, ny, nz = (int(d) for d in dims)
        return cls(origin=np.asarray(origin, dtype=np.float64), voxel_size=float(voxel_size),
                   dims=(nx, ny, nz), occ=np.zeros((nx, ny, nz), dtype=bool),
                   ori=np.zeros((nx, ny, nz, 3), dtype=np.float32),
                   counts=np.zeros((nx, ny, nz), dtype=np.uint16))

    def voxel_of(self, pts):
        pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
        return np.floor((pts - self.origin) / self.voxel_size).astype(np.int64)

    def in_bounds(self, idx):
        idx = idx.reshape(-1, 3)
        return np.all((idx >= 0) & (idx < np.array(self.dims)), axis=1)

    def centers(self, idx):
        return self.origin + (np.asarray(idx, dtype=np.float64) + 0.5) * self.voxel_size


def _ptr(a):
    """Raw data pointer of a C-contiguous numpy array or torch tensor (host or cuda)."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _is_torch(a):
    return type(a).__module__.startswith("torch")


# Buffers up to this size are hashed in full on every lookup; larger ones are probed at
# _PROBE_POINTS strided elements (PHG_FIELD_VERIFY=full hashes every buffer in full).
_FULL_HASH_BYTES = 16 << 20
_PROBE_POINTS = 1 << 16


def _fingerprint(a):
    """Content probe of a field buffer: a full BLAKE2 hash of small buffers (or of every buffer
    with PHG_FIELD_VERIFY=full), else a hash of 65536 strided elements plus the last one."""
    if _is_torch(a):
        a = a.detach()
        if a.is_cuda:  # device buffers are probed on the device, then only the sample moves
            flat = a.reshape(-1)
            step = max(1, flat.numel() // _PROBE_POINTS)
            return hash(flat[::step].cpu().numpy().tobytes()) ^ hash(
                flat[-1:].cpu().numpy().tobytes())
        a = a.numpy()
    flat = np.ascontiguousarray(a).reshape(-1)
    full = os.environ.get("PHG_FIELD_VERIFY", "") == "full"
    if full or flat.nbytes <= _FULL_HASH_BYTES:
        return hashlib.blake2b(flat.view(np.uint8), digest_size=16).digest()
    step = max(1, flat.size // _PROBE_POINTS)
    return hash(flat[::step].tobytes()) ^ hash(flat[-1:].tobytes())


class DeviceField:
    """Packed field on the current CUDA device (phg_field in the C ABI)."""

    def __init__(self, origin, voxel_size, occ, ori, stream=0):
        lib = _native.load()
        if _is_torch(occ):
            import torch

            if occ.dtype.is_floating_point:
                raise DataError("occ must be a bool/uint8 plane")
            occ = occ.contiguous().to(torch.uint8)
            ori = ori.contiguous().float()
            dims = tuple(int(d) for d in occ.shape)
            oshape = tuple(int(d) for d in ori.shape)
        else:
            occ = np.ascontiguousarray(occ)
            if occ.dtype not in (np.bool_, np.uint8):
                occ = occ.astype(bool)
            ori = np.ascontiguousarray(ori, dtype=np.float32)
            dims = occ.shape
            oshape = ori.shape
        if len(dims) != 3 or oshape != dims + (3,):
            raise DataError(f"field shapes disagree: occ {dims}, ori {oshape}")
        self.dims = tuple(int(d) for d in dims)
        self.origin = np.ascontiguousarray(np.asarray(origin, dtype=np.float64).reshape(3))
        self.voxel_size = float(voxel_size)
        h = ctypes.c_void_p()
        _native.check(lib.phg_field_create(
            ctypes.byref(h), _ptr(ori), _ptr(occ), self.dims[0], self.dims[1], self.dims[2],
            self.origin.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), self.voxel_size,
            stream), "phg_field_create")
        self.handle = h
        self._lib = lib
        self._cap_key = None
        self._near_key = None

    @classmethod
    def from_handle(cls, handle, dims, origin, voxel_size):
        """Wrap a phg_field* created by another C entry point (e.g. phg_field_from_oovl)."""
        self = cls.__new__(cls)
        self.handle = handle
        self._lib = _native.load()
        self.dims = tuple(int(d) for d in dims)
        self.origin = np.ascontiguousarray(np.asarray(origin, dtype=np.float64).reshape(3))
        self.voxel_size = float(voxel_size)
        self._cap_key = None
        self._near_key = None
        return self

    @classmethod
    def create_packed(cls, dims, origin, voxel_size, zeroed, maxabs, stream=0):
        """A field whose packed buffer the caller fills (dist.replicate_field); finish with
        ``packed_done()``."""
        lib = _native.load()
        origin = np.ascontiguousarray(np.asarray(origin, dtype=np.float64).reshape(3))
        h = ctypes.c_void_p()
        _native.check(lib.phg_field_create_packed(
            ctypes.byref(h), int(dims[0]), int(dims[1]), int(dims[2]),
            origin.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(voxel_size),
            int(bool(zeroed)), float(maxabs), stream), "phg_field_create_packed")
        return cls.from_handle(h, dims, origin, voxel_size)

    def packed(self):
        """(device pointer, bytes, zeroed, maxabs) of the padded packed voxel buffer."""
        ptr, nb = ctypes.c_void_p(), ctypes.c_int64()
        z, m = ctypes.c_int32(), ctypes.c_float()
        _native.check(self._lib.phg_field_packed(self.handle, ctypes.byref(ptr), ctypes.byref(nb),
                                                 ctypes.byref(z), ctypes.byref(m)),
                      "phg_field_packed")
        return int(ptr.value or 0), int(nb.value), bool(z.value), float(m.value)

    def packed_done(self, stream=0):
        _native.check(self._lib.phg_field_packed_done(self.handle, stream), "phg_field_packed_done")

    def close(self):
        if self.handle:
            self._lib.phg_field_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def set_cap(self, at_cap, stream=0):
        """Freeze the at_cap plane of the current batch (phg.py:236) or clear it (None)."""
        if at_cap is None:
            _native.check(self._lib.phg_field_set_cap(self.handle, None, stream), "set_cap")
            self._cap_key = None
            return
        if _is_torch(at_cap):
            plane = at_cap.contiguous()
        else:
            plane = np.ascontiguousarray(at_cap)
            if plane.dtype not in (np.bool_, np.uint8):
                plane = plane.astype(bool)
        if tuple(plane.shape) != self.dims:
            raise DataError(f"at_cap shape {tuple(plane.shape)} != field dims {self.dims}")
        _native.check(self._lib.phg_field_set_cap(self.handle, _ptr(plane), stream), "set_cap")

    def set_near(self, near_occ, stream=0):
        if near_occ is None:
            _native.check(self._lib.phg_field_set_near(self.handle, None, stream), "set_near")
            self._near_key = None
            return
        key = (id(near_occ), _ptr(near_occ) if not _is_torch(near_occ) else near_occ.data_ptr())
        if key == self._near_key:
            return
        if _is_torch(near_occ):
            near = near_occ.contiguous().long()
        else:
            near = np.ascontiguousarray(near_occ, dtype=np.int64)
        if tuple(near.shape) != self.dims + (3,):
            raise DataError(f"near_occ shape {tuple(near.shape)} != {self.dims + (3,)}")
        _native.check(self._lib.phg_field_set_near(self.handle, _ptr(near), stream), "set_near")
        self._near_key = key


# id(vol) -> (key, DeviceField, strong ref or None, finalizer or None).  The entry of a weak-referenceable
# volume dies with it (weakref.finalize), so neither the ~2 GiB packed field nor a recycled
# id can outlive the volume; volumes that cannot be weakly referenced are held strongly in an
# LRU of _STRONG_MAX entries instead.
_CACHE: "OrderedDict[int, tuple]" = OrderedDict()
_STRONG_MAX = 2


def _drop(vid):
    hit = _CACHE.pop(vid, None)
    if hit is not None:
        hit[1].close()


def field_for(vol, stream=0) -> DeviceField:
    """Device field for ``vol``, cached while ``vol`` lives.

    The cache key covers the volume's identity, its occ/ori buffers (address, shape),
    geometry and a content probe (_fingerprint): a full hash of buffers up to 16 MiB, a
    65536-point strided probe of larger ones (PHG_FIELD_VERIFY=full hashes everything).  An
    in-place edit of a large buffer that the probe misses is not detected: call
    ``invalidate(vol)`` after editing a volume's occ/ori in place.
    """
    key = (id(vol), _ptr(vol.occ) if not _is_torch(vol.occ) else vol.occ.data_ptr(),
           _ptr(vol.ori) if not _is_torch(vol.ori) else vol.ori.data_ptr(),
           tuple(vol.occ.shape), tuple(np.asarray(vol.origin, dtype=np.float64).tolist()),
           float(vol.voxel_size), _fingerprint(vol.occ), _fingerprint(vol.ori))
    vid = id(vol)
    hit = _CACHE.get(vid)
    if hit is not None and hit[0] == key:
        _CACHE.move_to_end(vid)
        return hit[1]
    fin = hit[3] if hit is not None else None  # the same live volume: keep its finalizer
    _drop(vid)
    f = DeviceField(vol.origin, vol.voxel_size, vol.occ, vol.ori, stream)
    strong = None
    if fin is None or not fin.alive:
        try:
            fin = weakref.finalize(vol, _drop, vid)
            fin.atexit = False  # no device frees during interpreter shutdown
        except TypeError:  # not weak-referenceable: hold it, bounded LRU
            fin, strong = None, vol
            while sum(1 for e in _CACHE.values() if e[2] is not None) >= _STRONG_MAX:
                _drop(next(k for k, e in _CACHE.items() if e[2] is not None))
    _CACHE[vid] = (key, f, strong, fin)
    return f


def invalidate(vol=None):
    """Drop cached device fields (all, or the one of ``vol``)."""
    if vol is None:
        for vid in list(_CACHE):
            _drop(vid)
    else:
        _drop(id(vol))


def sample_orientation_batch(vol, pts, prev_dirs):
    """GPU drop-in for strandkit.volume.sample_orientation_batch (volume.py:183-224).

    Returns (dirs (N,3) f64, has (N,) bool, support (N,) f64), bit-identical.
    """
    lib = _native.load()
    f = field_for(vol)
    pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    prev = np.ascontiguousarray(np.asarray(prev_dirs, dtype=np.float64).reshape(-1, 3))
    n = len(pts)
    if len(prev) != n:
        raise DataError(f"pts ({n}) and prev_dirs ({len(prev)}) lengths differ")
    dirs = np.zeros((n, 3))
    has = np.zeros(n, np.uint8)
    sup = np.zeros(n)
    _native.check(lib.phg_sample(f.handle, pts.ctypes.data, prev.ctypes.data, n, dirs.ctypes.data,
                                 has.ctypes.data, sup.ctypes.data, 0), "phg_sample")
    return dirs, has.astype(bool), sup


def sample_orientation(vol, p, prev_dir):
    """Single-point lookup (volume.py:227-230); None outside occupied space."""
    d, has, _ = sample_orientation_batch(vol, np.reshape(p, (1, 3)), np.reshape(prev_dir, (1, 3)))
    return d[0] if has[0] else None
