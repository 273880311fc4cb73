"""ctypes binding of libphg_b200.so (the C ABI declared in include/phg_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_2604_05794_b200.build``.  There is NO fallback: if the
library is missing or fails to load, every entry point raises
``PipelineError`` -- the product path never silently runs on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, DataError, PipelineError

HERE = os.path.dirname(os.path.abspath(__file__))
# PHG_CHECKED_LIB=1 loads the checked build (device index checks + allocation canaries, the
# stand-in for compute-sanitizer; see include/phg_b200.h phg_debug_checks)
CHECKED = os.environ.get("PHG_CHECKED_LIB", "") == "1"
LIB_PATH = os.path.join(HERE, "libphg_b200_checked.so" if CHECKED else "libphg_b200.so")
# PHG_LIB_PATH=<file>: load another build of the library (A/B timing of kernel changes on one
# box); symbols that build lacks are left undeclared
_OVERRIDE = os.environ.get("PHG_LIB_PATH", "")
if _OVERRIDE:
    LIB_PATH = os.path.abspath(_OVERRIDE)

PHG_OK, PHG_ERR_INVALID, PHG_ERR_CUDA, PHG_ERR_OOM, PHG_ERR_CAPACITY, PHG_ERR_STATE = range(6)
PHG_FLAG_STRICT = 0x1
PHG_FLAG_NO_ORDER = 0x2
PHG_FLAG_TURN_STOP = 0x4

# every symbol include/phg_b200.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "phg_field_create", "phg_field_set_cap", "phg_field_set_near", "phg_field_destroy",
    "phg_field_info", "phg_ctx_create", "phg_ctx_destroy", "phg_trace", "phg_gather",
    "phg_last_steps", "phg_sample", "phg_last_error", "phg_abi_version", "phg_last_kernel_ms",
    "phg_last_variant", "phg_last_sampler", "phg_num_variants", "phg_selftest", "phg_grow_init",
    "phg_grow_fetch",
    "phg_trace_to_host", "phg_stnd_encode", "phg_field_from_oovl", "phg_link", "phg_link_fetch",
    "phg_grow_begin", "phg_grow_scalp_batch", "phg_grow_field_begin", "phg_grow_field_batch",
    "phg_grow_commits", "phg_grow_apply", "phg_grow_end", "phg_trace_rows",
    "phg_debug_checks", "phg_is_checked_build", "phg_field_packed", "phg_field_create_packed",
    "phg_field_packed_done", "phg_gather_to", "phg_ipc_alloc", "phg_ipc_free", "phg_ipc_open",
    "phg_ipc_close",
)


class LinkParams(ctypes.Structure):
    """phg_link_params_v1"""

    _fields_ = [("link_dist_mm", ctypes.c_double), ("link_cos_gate", ctypes.c_double),
                ("smooth_strength", ctypes.c_double), ("step_mm", ctypes.c_double),
                ("attach_radius_mm", ctypes.c_double), ("tangent_window", ctypes.c_int32),
                ("smooth", ctypes.c_int32), ("smooth_iters", ctypes.c_int32),
                ("attach", ctypes.c_int32)]


class Params(ctypes.Structure):
    """phg_params_v1"""

    _fields_ = [
        ("step_mm", ctypes.c_double),
        ("min_support", ctypes.c_double),
        ("steer", ctypes.c_double),
        ("max_vertices", ctypes.c_int32),
        ("probe_steps", ctypes.c_int32),
        ("coast_steps", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("max_turn_cos", ctypes.c_double),
    ]


class Rows(ctypes.Structure):
    """phg_rows_v1: device-resident strand rows of the last phg_trace_rows"""

    _fields_ = [("rows", ctypes.c_void_p), ("rowmap", ctypes.c_void_p),
                ("lengths", ctypes.c_void_p), ("entered", ctypes.c_void_p),
                ("row_stride", ctypes.c_int64), ("n", ctypes.c_int64),
                ("counters", ctypes.c_void_p)]


_lib = None
_load_error = None

VP = ctypes.c_void_p
I64 = ctypes.c_int64


def _declare(lib):
    S = ctypes.c_int
    sig = {
        "phg_field_create": (S, [ctypes.POINTER(VP), VP, VP, I64, I64, I64,
                                 ctypes.POINTER(ctypes.c_double), ctypes.c_double, VP]),
        "phg_field_set_cap": (S, [VP, VP, VP]),
        "phg_field_set_near": (S, [VP, VP, VP]),
        "phg_field_destroy": (S, [VP]),
        "phg_field_info": (S, [VP, ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_int)]),
        "phg_ctx_create": (S, [ctypes.POINTER(VP)]),
        "phg_ctx_destroy": (S, [VP]),
        "phg_trace": (S, [VP, VP, ctypes.POINTER(Params), VP, VP, I64, VP, VP, VP,
                          ctypes.POINTER(I64), VP]),
        "phg_gather": (S, [VP, VP, I64, VP]),
        "phg_trace_rows": (S, [VP, VP, ctypes.POINTER(Params), VP, VP, I64,
                               ctypes.POINTER(Rows), VP]),
        "phg_trace_to_host": (S, [VP, VP, ctypes.POINTER(Params), VP, VP, I64, I64, VP, VP, VP,
                                  I64, ctypes.POINTER(I64), VP]),
        "phg_last_steps": (S, [VP, ctypes.POINTER(I64)]),
        "phg_sample": (S, [VP, VP, VP, I64, VP, VP, VP, VP]),
        "phg_last_error": (ctypes.c_char_p, []),
        "phg_abi_version": (ctypes.c_int, []),
        "phg_last_kernel_ms": (S, [VP, ctypes.POINTER(ctypes.c_float),
                                   ctypes.POINTER(ctypes.c_float)]),
        "phg_last_variant": (ctypes.c_char_p, [VP]),
        "phg_last_sampler": (ctypes.c_char_p, [VP]),
        "phg_num_variants": (ctypes.c_int, []),
        "phg_selftest": (S, [I64, ctypes.c_uint64, ctypes.POINTER(I64), VP]),
        "phg_grow_init": (S, [VP, VP, ctypes.POINTER(Params), VP, VP, VP, I64, VP,
                              ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64), VP]),
        "phg_grow_fetch": (S, [VP, VP, VP, VP, VP]),
        "phg_stnd_encode": (S, [VP, VP, I64, VP, VP]),
        "phg_grow_begin": (S, [VP, VP, ctypes.POINTER(Params), VP, VP, VP]),
        "phg_grow_scalp_batch": (S, [VP, VP, VP, I64, ctypes.c_int32, ctypes.POINTER(I64), VP]),
        "phg_grow_field_begin": (S, [VP, ctypes.POINTER(I64), VP]),
        "phg_grow_field_batch": (S, [VP, I64, I64, ctypes.c_int32, ctypes.POINTER(I64), VP]),
        "phg_grow_commits": (S, [VP, VP, VP]),
        "phg_grow_apply": (S, [VP, VP, I64, VP]),
        "phg_grow_end": (S, [VP, VP, ctypes.POINTER(I64), ctypes.POINTER(I64),
                             ctypes.POINTER(I64), VP]),
        "phg_link": (S, [VP, VP, VP, VP, VP, I64, VP, I64, ctypes.POINTER(LinkParams),
                         ctypes.POINTER(I64), VP]),
        "phg_link_fetch": (S, [VP, VP, VP, VP, VP, VP, VP, VP]),
        "phg_debug_checks": (S, [ctypes.POINTER(I64), ctypes.POINTER(I64),
                                 ctypes.POINTER(I64)]),
        "phg_is_checked_build": (ctypes.c_int, []),
        "phg_field_packed": (S, [VP, ctypes.POINTER(VP), ctypes.POINTER(I64),
                                 ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float)]),
        "phg_field_create_packed": (S, [ctypes.POINTER(VP), I64, I64, I64,
                                        ctypes.POINTER(ctypes.c_double), ctypes.c_double,
                                        ctypes.c_int32, ctypes.c_float, VP]),
        "phg_field_packed_done": (S, [VP, VP]),
        "phg_gather_to": (S, [VP, VP, VP, VP, I64, I64, VP]),
        "phg_ipc_alloc": (S, [I64, ctypes.POINTER(VP), VP]),
        "phg_ipc_free": (S, [VP]),
        "phg_ipc_open": (S, [VP, ctypes.POINTER(VP)]),
        "phg_ipc_close": (S, [VP]),
        "phg_field_from_oovl": (S, [ctypes.POINTER(VP), VP, VP, I64, I64, I64, I64,
                                    ctypes.POINTER(ctypes.c_double), ctypes.c_double, VP]),
    }
    for name, (res, args) in sig.items():
        if _OVERRIDE and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Load (once) and return the native library; raise PipelineError if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise PipelineError(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"native PHG library not built: {LIB_PATH} is missing "
                       "(run `python -m paper_2604_05794_b200.build`)")
        raise PipelineError(_load_error)
    try:
        lib = ctypes.CDLL(LIB_PATH)
        _declare(lib)
    except OSError as e:
        _load_error = f"cannot load {LIB_PATH}: {e}"
        raise PipelineError(_load_error) from e
    _lib = lib
    return lib


def check(status: int, what: str):
    if status == PHG_OK:
        return
    msg = f"{what}: {_lib.phg_last_error().decode(errors='replace')}"
    if status == PHG_ERR_INVALID:
        raise DataError(msg)
    if status in (PHG_ERR_CAPACITY, PHG_ERR_STATE):
        raise PipelineError(msg)
    raise PipelineError(msg)


def params_struct(p, strict=None, order=True) -> Params:
    mv = int(p.max_vertices)
    if mv < 1:
        raise ConfigError(f"max_vertices must be >= 1 (got {mv})")
    st = bool(p.strict) if strict is None else strict
    flags = (PHG_FLAG_STRICT if st else 0) | (0 if order else PHG_FLAG_NO_ORDER)
    turn_cos = turn_stop_cos(p)
    if turn_cos is not None:
        flags |= PHG_FLAG_TURN_STOP
    return Params(float(p.step_mm), float(p.min_support), float(getattr(p, "steer", 0.0)), mv,
                  int(p.probe_steps), int(p.coast_steps), flags,
                  turn_cos if turn_cos is not None else -2.0)


def turn_stop_cos(p):
    """cos of the opt-in angle stop's limit, or None when it is off: ``max_turn_deg`` (an
    extension of PhgParams, not a reference field) in (0, 180); 0 / absent = off."""
    import math

    deg = float(getattr(p, "max_turn_deg", 0.0) or 0.0)
    if deg <= 0.0 or deg >= 180.0:
        return None
    return math.cos(math.radians(deg))
