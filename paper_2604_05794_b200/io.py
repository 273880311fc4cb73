"""Reference wire formats straight to / from the GPU.

* ``read_volume_device(path)`` -- OOVL file (volume.py:236-266) to a packed device field
  without materialising the host ``occ``/``ori`` arrays: the packbits occupancy and the
  occupied-voxel orientations are uploaded as they lie in the file and scattered on the GPU
  (csrc/phg_io.cu ``phg_field_from_oovl``).
* ``write_strands_device(path, offsets, verts)`` -- STND file (strands.py:63-69) encoded on
  the GPU from a CSR strand set (``phg_stnd_encode``) and written with one ``write``.
Both are byte-compatible with the reference (tests/test_io.py against reference-written files).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native
from .errors import DataError
from .volume import DeviceField

VOLUME_MAGIC = b"OOVL"
STRAND_MAGIC = 0x444E5453


def _ptr(a):
    return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data


def read_volume_device(path):
    """Returns (DeviceField, header dict {origin, voxel_size, dims}) for an OOVL file."""
    lib = _native.load()
    with open(path, "rb") as f:
        if f.read(4) != VOLUME_MAGIC:
            raise DataError(f"{path}: not a volume file (bad magic)")
        nx, ny, nz, vs = struct.unpack("<IIIf", f.read(16))
        origin = np.array(struct.unpack("<fff", f.read(12)), dtype=np.float64)
        nvox = nx * ny * nz
        nbytes = (nvox + 7) // 8
        bits = np.frombuffer(f.read(nbytes), dtype=np.uint8)
        if len(bits) != nbytes:
            raise DataError(f"{path}: truncated occupancy bitset")
        nocc = int(np.bitwise_count(bits).sum())
        if nvox % 8:
            nocc -= int(np.bitwise_count(bits[-1] & np.uint8((1 << (8 - nvox % 8)) - 1)))
        ori = np.frombuffer(f.read(nocc * 12), dtype="<f4")
        if len(ori) != nocc * 3:
            raise DataError(f"{path}: truncated orientation payload")
    ori = np.ascontiguousarray(ori)
    h = ctypes.c_void_p()
    _native.check(lib.phg_field_from_oovl(
        ctypes.byref(h), bits.ctypes.data, ori.ctypes.data if nocc else None, nocc, nx, ny, nz,
        origin.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(vs), None),
        "phg_field_from_oovl")
    dims = (nx, ny, nz)
    return DeviceField.from_handle(h, dims, origin, float(vs)), {
        "origin": origin, "voxel_size": float(vs), "dims": dims}


def stnd_bytes(offsets, verts) -> bytes:
    """STND image of a CSR strand set, encoded on the GPU (host or device inputs)."""
    lib = _native.load()
    offsets = offsets if hasattr(offsets, "data_ptr") else np.ascontiguousarray(offsets, np.int64)
    n = int(offsets.shape[0]) - 1
    total = int(offsets[-1])
    if not hasattr(verts, "data_ptr"):
        verts = np.ascontiguousarray(verts, np.float64)
    out = np.empty(8 + 4 * n + 12 * total, np.uint8)
    _native.check(lib.phg_stnd_encode(_ptr(offsets), _ptr(verts) if total else None, n,
                                      out.ctypes.data, None), "phg_stnd_encode")
    return out.tobytes()


def write_strands_device(path, offsets, verts):
    with open(path, "wb") as f:
        f.write(stnd_bytes(offsets, verts))
