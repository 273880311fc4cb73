"""ctypes binding of oracle/phg_oracle.c -- TEST INFRASTRUCTURE ONLY.

The C restatement is the large-size checker (bit-exact with the reference,
OpenMP over strands).  Only tests/, ``__graft_entry__`` and bench.py's CPU legs
may import this module.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libphg_oracle.so")


class _Params(ctypes.Structure):
    _fields_ = [("step_mm", ctypes.c_double), ("min_support", ctypes.c_double),
                ("steer", ctypes.c_double), ("max_vertices", ctypes.c_int32),
                ("probe_steps", ctypes.c_int32), ("coast_steps", ctypes.c_int32),
                ("strict", ctypes.c_int32), ("turn_cos", ctypes.c_double)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.phg_oracle_trace.restype = ctypes.c_int
        _lib.phg_oracle_max_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    return ctypes.c_void_p(0 if a is None else a.ctypes.data)


def _params(p):
    deg = float(getattr(p, "max_turn_deg", 0.0) or 0.0)
    turn = math.cos(math.radians(deg)) if 0.0 < deg < 180.0 else -2.0
    return _Params(float(p.step_mm), float(p.min_support), float(getattr(p, "steer", 0.0)),
                   int(p.max_vertices), int(p.probe_steps), int(p.coast_steps),
                   int(bool(getattr(p, "strict", False))), turn)


def trace(origin, voxel_size, occ, ori, seed_pos, seed_dir, params, at_cap=None,
          live_counts=None, near_occ=None, threads=0):
    """Returns (slab (n,max_vertices,3) f64, keep (n,) i64, entered (n,) bool).

    ``live_counts`` (strict mode) is updated in place like the reference.
    """
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    ori = np.ascontiguousarray(ori, dtype=np.float32)
    nx, ny, nz = occ.shape
    origin = np.ascontiguousarray(origin, dtype=np.float64)
    sp = np.ascontiguousarray(seed_pos, dtype=np.float64).reshape(-1, 3)
    sd = np.ascontiguousarray(seed_dir, dtype=np.float64).reshape(-1, 3)
    n = len(sp)
    mv = int(params.max_vertices)
    cap = None if at_cap is None else np.ascontiguousarray(at_cap, dtype=np.uint8)
    near = None if near_occ is None else np.ascontiguousarray(near_occ, dtype=np.int64)
    if near is not None and not (float(getattr(params, "steer", 0.0)) > 0):
        near = None
    counts = live_counts
    if counts is not None:
        assert counts.dtype == np.uint16 and counts.flags.c_contiguous
    slab = np.zeros((n, max(mv, 1), 3))
    keep = np.zeros(n, np.int64)
    entered = np.zeros(n, np.uint8)
    P = _params(params)
    rc = lib().phg_oracle_trace(
        _p(ori), _p(occ), ctypes.c_int64(nx), ctypes.c_int64(ny), ctypes.c_int64(nz), _p(origin),
        ctypes.c_double(float(voxel_size)), _p(cap), _p(near), _p(counts), ctypes.byref(P),
        _p(sp), _p(sd), ctypes.c_int64(n), _p(slab), _p(keep), _p(entered), ctypes.c_int(threads))
    if rc != 0:
        raise RuntimeError(f"phg_oracle_trace failed ({rc})")
    return slab, keep, entered.astype(bool)


def to_csr(slab, keep):
    offsets = np.zeros(len(keep) + 1, np.int64)
    np.cumsum(keep, out=offsets[1:])
    verts = np.concatenate([slab[i, : keep[i]] for i in range(len(keep))]) if len(keep) else \
        np.zeros((0, 3))
    return offsets, verts


def sample(origin, voxel_size, occ, ori, pts, prev):
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    ori = np.ascontiguousarray(ori, dtype=np.float32)
    nx, ny, nz = occ.shape
    origin = np.ascontiguousarray(origin, dtype=np.float64)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    prev = np.ascontiguousarray(prev, dtype=np.float64).reshape(-1, 3)
    n = len(pts)
    dirs = np.zeros((n, 3))
    has = np.zeros(n, np.uint8)
    sup = np.zeros(n)
    lib().phg_oracle_sample(_p(ori), _p(occ), ctypes.c_int64(nx), ctypes.c_int64(ny),
                            ctypes.c_int64(nz), _p(origin), ctypes.c_double(float(voxel_size)),
                            _p(pts), _p(prev), ctypes.c_int64(n), _p(dirs), _p(has), _p(sup))
    return dirs, has.astype(bool), sup


def max_threads():
    return int(lib().phg_oracle_max_threads())
