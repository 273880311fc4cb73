"""Drop-in PHG grow step on B200: ``trace_batch`` with the reference's signature.

Reference boundary (strandkit/phg.py:67-163)::

    trace_batch(vol, seed_pos, seed_dir, params, at_cap=None, live_counts=None,
                near_occ=None) -> [(vertices (k,3) float64, entered bool), ...]

Every caller in the reference (init_guide_strands phg.py:233,240;
_trace_field_seeds.run_dir phg.py:283,288; the fork worker phg.py:180)
resolves ``trace_batch`` as a module global at call time, so ``install()``
reroutes the whole grow stage through the GPU by attribute replacement.

The arithmetic runs in libphg_b200.so (csrc/phg_trace.cu) -- IEEE binary64
in the reference's evaluation order, bit-identical output.  All modes run on
the GPU: relaxed (frozen ``at_cap`` plane), strict (lockstep per-step commits
to ``live_counts``) and steering (``near_occ`` with ``steer > 0``).  There is
no CPU fallback: without the native library every call raises PipelineError.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigError, DataError
from .volume import field_for


@dataclass
class PhgParams:
    """Mirror of strandkit.phg.PhgParams (phg.py:24-51): same fields, defaults, checks."""

    step_mm: float = 1.0
    max_vertices: int = 400
    batch_size: int = 16384
    occupancy_cap: int = 16
    link_dist_mm: float = 2.0
    link_angle_deg: float = 30.0
    n_root: int = 30000
    attach_radius_mm: float = 10.0
    probe_steps: int = 24
    min_support: float = 0.05
    coast_steps: int = 25
    steer: float = 0.0
    field_seeds: int = 30000
    smooth: bool = True
    smooth_strength: float = 0.25
    smooth_iters: int = 2
    strict: bool = False
    tangent_window: int = 3
    # extension, not a reference field: opt-in angle stop (degrees; 0 = off, the reference's
    # behaviour).  A step turning by more than this from the previous step direction ends the
    # strand (PHG_FLAG_TURN_STOP in include/phg_b200.h).
    max_turn_deg: float = 0.0

    def __post_init__(self):
        if self.link_dist_mm <= 0:
            raise ConfigError("link_dist_mm must be positive")
        if not (0 < self.link_angle_deg < 90):
            raise ConfigError("link_angle_deg must be in (0, 90)")
        if self.step_mm <= 0 or self.batch_size < 1 or self.occupancy_cap < 1:
            raise ConfigError("invalid tracing parameters")
        if not (0.0 <= self.max_turn_deg <= 180.0):
            raise ConfigError("max_turn_deg must be in [0, 180] (0 = off)")


class Tracer:
    """Owns a native context (scratch + last result). One per thread/stream."""

    def __init__(self):
        self._lib = _native.load()
        h = ctypes.c_void_p()
        _native.check(self._lib.phg_ctx_create(ctypes.byref(h)), "phg_ctx_create")
        self.handle = h

    def close(self):
        if self.handle:
            self._lib.phg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def trace(self, field, params, seed_pos, seed_dir, n, offsets_ptr, entered_ptr,
              live_counts_ptr=None, stream=0, order=True):
        """Phase 1 (phg_trace). Pointers may be host or device. Returns total kept vertices."""
        p = _native.params_struct(params, order=order)
        total = ctypes.c_int64()
        _native.check(self._lib.phg_trace(self.handle, field.handle, ctypes.byref(p), seed_pos,
                                          seed_dir, n, live_counts_ptr, offsets_ptr, entered_ptr,
                                          ctypes.byref(total), stream), "phg_trace")
        return int(total.value)

    def trace_to_host(self, field, params, seed_pos, seed_dir, n, offsets_ptr, entered_ptr,
                      verts_ptr, verts_cap, chunk=0, stream=0):
        """phg_trace_to_host: host seeds -> host CSR, D2H overlapped with the next chunk."""
        p = _native.params_struct(params)
        total = ctypes.c_int64()
        _native.check(self._lib.phg_trace_to_host(self.handle, field.handle, ctypes.byref(p),
                                                  seed_pos, seed_dir, n, chunk, offsets_ptr,
                                                  entered_ptr, verts_ptr, verts_cap,
                                                  ctypes.byref(total), stream),
                      "phg_trace_to_host")
        return int(total.value)

    def trace_rows(self, field, params, seed_pos, seed_dir, n, stream=0):
        """phg_trace_rows: asynchronous trace into device-resident strand rows."""
        p = _native.params_struct(params)
        out = _native.Rows()
        _native.check(self._lib.phg_trace_rows(self.handle, field.handle, ctypes.byref(p),
                                               seed_pos, seed_dir, n, ctypes.byref(out), stream),
                      "phg_trace_rows")
        return out

    def gather(self, verts_ptr, cap, stream=0):
        _native.check(self._lib.phg_gather(self.handle, verts_ptr, cap, stream), "phg_gather")

    def last_steps(self):
        v = ctypes.c_int64()
        _native.check(self._lib.phg_last_steps(self.handle, ctypes.byref(v)), "phg_last_steps")
        return int(v.value)

    def last_variant(self):
        return self._lib.phg_last_variant(self.handle).decode()

    def last_sampler(self):
        """exact / fast / fast-pow2 / fast-pow2-s32 (chosen per field; all bit-identical)."""
        return self._lib.phg_last_sampler(self.handle).decode()

    def last_kernel_ms(self):
        a, b = ctypes.c_float(), ctypes.c_float()
        _native.check(self._lib.phg_last_kernel_ms(self.handle, ctypes.byref(a), ctypes.byref(b)),
                      "phg_last_kernel_ms")
        return float(a.value), float(b.value)


# Kernel launches of one relaxed-mode phg_trace + phg_gather from libphg_b200.so:
# morton keys, CUB radix sort (histogram, exclusive-sum, 4 onesweep passes), trace,
# CUB scan (init + scan), gather -- as listed by ncu (profiles/r01_v0_launches.csv).
LAUNCHES_PER_TRACE = 11
# phg_trace_rows: morton keys, the 6 CUB radix-sort launches, trace (no scan, no gather)
LAUNCHES_PER_TRACE_ROWS = 8

_TRACER = None


def _tracer():
    global _TRACER
    if _TRACER is None:
        _TRACER = Tracer()
    return _TRACER


def _seeds(a, name):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))
    return a


def trace_batch_csr(vol, seed_pos, seed_dir, params, at_cap=None, live_counts=None,
                    near_occ=None):
    """trace_batch with CSR output: (offsets (n+1,) i64, verts (M,3) f64, entered (n,) bool).

    Host numpy in, host numpy out; H2D/D2H staging happens inside the C ABI.
    """
    pos = _seeds(seed_pos, "seed_pos")
    dirs = _seeds(seed_dir, "seed_dir")
    n = len(pos)
    if len(dirs) != n:
        raise DataError(f"seed_pos ({n}) and seed_dir ({len(dirs)}) lengths differ")
    if int(params.max_vertices) < 1:
        raise ConfigError(f"max_vertices must be >= 1 (got {params.max_vertices})")
    field = field_for(vol)
    strict = bool(params.strict)
    counts_ptr = None
    if strict:
        if live_counts is not None:
            if not (isinstance(live_counts, np.ndarray) and live_counts.dtype == np.uint16
                    and live_counts.flags.c_contiguous and live_counts.shape == field.dims):
                raise DataError("live_counts must be a C-contiguous uint16 array of the field dims")
            counts_ptr = live_counts.ctypes.data
        field.set_cap(None)
    else:
        cap = at_cap
        if cap is not None and tuple(np.shape(cap)) != field.dims:
            raise DataError(f"at_cap shape {tuple(np.shape(cap))} != field dims {field.dims}")
        if cap is not None and isinstance(cap, np.ndarray) and not cap.any():
            cap = None  # an all-False plane never stops a strand (phg.py:139-142)
        field.set_cap(cap)
    steer = near_occ is not None and float(params.steer) > 0
    field.set_near(near_occ if steer else None)
    offsets = np.zeros(n + 1, np.int64)
    entered = np.zeros(n, np.uint8)
    tr = _tracer()
    chunk = n if strict else max(1, min(n, slab_budget_bytes() // slab_row_bytes(params)))
    if chunk >= n:
        total = tr.trace(field, params, pos.ctypes.data if n else None,
                         dirs.ctypes.data if n else None, n, offsets.ctypes.data,
                         entered.ctypes.data if n else None, counts_ptr)
        verts = np.empty((total, 3))
        if total:
            tr.gather(verts.ctypes.data, total)
        return offsets, verts, entered.astype(bool)
    # Relaxed strands are independent (the cap plane is fixed for the call), so a seed set
    # whose trace slab would not fit the budget is traced in seed-order chunks: bit-identical
    # to one call, with the slab bounded instead of n * max_vertices * 24 bytes.
    # Each chunk's vertices are gathered straight into their final rows of one host array,
    # sized from the first chunk's yield (+25%; untouched tail pages are never committed) and
    # regrown by copy only if a later chunk overruns it.
    verts, base = None, 0
    for s0 in range(0, n, chunk):
        s1 = min(n, s0 + chunk)
        off_k = np.zeros(s1 - s0 + 1, np.int64)
        mk = tr.trace(field, params, pos[s0:s1].ctypes.data, dirs[s0:s1].ctypes.data, s1 - s0,
                      off_k.ctypes.data, entered[s0:].ctypes.data, None)
        offsets[s0:s1 + 1] = off_k + base
        if verts is None:
            verts = np.empty((max(mk, int(mk * n / (s1 - s0) * _CHUNK_HEADROOM) + 1024), 3))
        elif base + mk > len(verts):
            grown = np.empty((max(base + mk, 2 * len(verts)), 3))
            grown[:base] = verts[:base]
            verts = grown
        if mk:
            tr.gather(verts[base:].ctypes.data, mk)
        base += mk
    return offsets, verts[:base], entered.astype(bool)


_CHUNK_HEADROOM = 1.25  # host CSR sizing factor over the first chunk's vertices per seed


def slab_row_bytes(params):
    """Bytes of one strand's trace-slab row (phg_core.cuh row_stride_doubles)."""
    return ((int(params.max_vertices) + 3) & ~3) * 24


def slab_budget_bytes():
    """Cap on the relaxed trace slab of one trace_batch call (PHG_SLAB_BUDGET_GB, default 24)."""
    return int(float(os.environ.get("PHG_SLAB_BUDGET_GB", "24")) * (1 << 30))


def trace_batch(vol, seed_pos, seed_dir, params, at_cap=None, live_counts=None, near_occ=None):
    """GPU drop-in for strandkit.phg.trace_batch (phg.py:67-163).

    Returns a list of ``(vertices (k,3) float64, entered bool)`` in seed order;
    each ``vertices`` is a C-contiguous row block of one CSR payload.
    """
    offsets, verts, entered = trace_batch_csr(vol, seed_pos, seed_dir, params, at_cap=at_cap,
                                              live_counts=live_counts, near_occ=near_occ)
    return list(zip(split_rows(verts, offsets), entered.tolist()))


def split_rows(verts, offsets):
    """[verts[offsets[i]:offsets[i+1]] for each i] as views, ~4x faster than np.split for
    ~1M rows (no per-piece swapaxes)."""
    o = offsets.tolist()
    return list(map(verts.__getitem__, map(slice, o[:-1], o[1:])))


def _device_seeds(seed_pos, seed_dir):
    """(n,3) float64 CUDA tensors, C-contiguous (the C ABI reads them as plain arrays)."""
    import torch

    out = []
    for name, t in (("seed_pos", seed_pos), ("seed_dir", seed_dir)):
        if not (torch.is_tensor(t) and t.is_cuda):
            raise DataError(f"{name} must be a CUDA tensor")
        if t.dtype != torch.float64:
            raise DataError(f"{name} must be float64 (got {t.dtype})")
        t = t.reshape(-1, 3).contiguous()
        out.append(t)
    if out[0].shape[0] != out[1].shape[0]:
        raise DataError(f"seed_pos ({out[0].shape[0]}) and seed_dir ({out[1].shape[0]}) "
                        "lengths differ")
    return out[0], out[1]


def trace_device(field, seed_pos, seed_dir, params, tracer=None, stream=None, order=True):
    """Zero-copy device API: torch CUDA tensors in, torch CUDA tensors out.

    ``field`` is a DeviceField (cap / near planes already set); seeds are (n,3)
    float64 CUDA tensors.  Returns (offsets (n+1,) i64, verts (M,3) f64,
    entered (n,) u8) on the same device, all produced on ``stream``.
    """
    import torch

    tr = tracer or _tracer()
    seed_pos, seed_dir = _device_seeds(seed_pos, seed_dir)
    n = int(seed_pos.shape[0])
    dev = seed_pos.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    entered = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)[:n]
    total = tr.trace(field, params, seed_pos.data_ptr() if n else None,
                     seed_dir.data_ptr() if n else None, n, offsets.data_ptr(),
                     entered.data_ptr() if n else None, None, st.cuda_stream, order=order)
    verts = torch.empty((total, 3), dtype=torch.float64, device=dev)
    if total:
        tr.gather(verts.data_ptr(), total, st.cuda_stream)
    return offsets, verts, entered


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr, shape, typestr):
        # no "stream": the producer is the caller's own stream (RowSet's contract)
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None}


class RowSet:
    """Device-resident result of ``trace_device_rows``: the reference's own trace buffer
    ``buf`` (phg.py:85) and ``keep`` (phg.py:159-161) -- strand i is ``strand(i)`` =
    buf[i, :keep[i]], the array trace_batch returns for seed i.  Views of the tracer's
    memory, valid until its next trace.  ``steps`` (the reference's sum(len - 1)) and
    ``kept`` synchronise on first use; everything else stays asynchronous."""

    def __init__(self, tracer, raw, device, stream):
        import torch

        self._tracer, self.n, self.row_stride = tracer, int(raw.n), int(raw.row_stride)
        self.stream = stream  # the rows are produced on this stream
        n = self.n
        nrows = n
        with torch.cuda.device(device):
            def view(ptr, shape, ts):
                if not ptr or not all(shape):
                    return torch.empty(shape, dtype={"<f8": torch.float64, "<i4": torch.int32,
                                                     "<i8": torch.int64, "|u1": torch.uint8}[ts],
                                       device=device)
                return torch.as_tensor(_CudaArray(ptr, shape, ts), device=device)

            self.rows = view(raw.rows, (nrows, self.row_stride), "<f8")
            self.rowmap = view(raw.rowmap, (n,), "<i4") if raw.rowmap else None
            self.lengths = view(raw.lengths, (n,), "<i8")
            self.entered = view(raw.entered, (n,), "|u1")
            self.counters = view(raw.counters, (2,), "<i8")  # u64 counters, < 2^63
        self._kept = None

    def row_of(self, i):
        return int(self.rowmap[i]) if self.rowmap is not None else int(i)

    def strand(self, i):
        """(len_i, 3) f64 device view of seed i's vertices."""
        k = int(self.lengths[i])
        return self.rows[self.row_of(i), : 3 * k].view(k, 3)

    @property
    def kept(self):
        if self._kept is None:
            self._kept = int(self.counters[1].item())
        return self._kept

    @property
    def steps(self):
        """sum over strands of (len(vertices) - 1): the reference's step count."""
        return self.kept - self.n

    def to_csr(self):
        """(offsets (n+1,), verts (M,3), entered (n,)) torch CUDA tensors, built with torch
        ops from the rows (validation / convenience; the library's CSR path is
        trace_device)."""
        import torch

        off = torch.zeros(self.n + 1, dtype=torch.int64, device=self.rows.device)
        torch.cumsum(self.lengths, 0, out=off[1:])
        rows = (self.rowmap.long() if self.rowmap is not None
                else torch.arange(self.n, device=self.rows.device))
        seg = torch.repeat_interleave(torch.arange(self.n, device=self.rows.device),
                                      self.lengths)
        j = torch.arange(int(off[-1]), device=self.rows.device) - off[seg]
        r3 = self.rows.view(self.rows.shape[0], self.row_stride // 3, 3)
        return off, r3[rows[seg], j], self.entered


def trace_device_rows(field, seed_pos, seed_dir, params, tracer=None, stream=None):
    """Device API without the CSR copy: torch CUDA seeds in, a ``RowSet`` of device-resident
    strand rows out (phg_trace_rows), enqueued on ``stream`` without a host synchronisation.
    Strand i is the reference's buf[i, :keep[i]] (phg.py:159-162)."""
    import torch

    tr = tracer or _tracer()
    seed_pos, seed_dir = _device_seeds(seed_pos, seed_dir)
    n = int(seed_pos.shape[0])
    dev = seed_pos.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    raw = tr.trace_rows(field, params, seed_pos.data_ptr() if n else None,
                        seed_dir.data_ptr() if n else None, n, st.cuda_stream)
    return RowSet(tr, raw, dev, st)


# ----------------------------------------------------------------------------------
# installation into the reference package
# ----------------------------------------------------------------------------------
_SAVED = {}


_REROUTED = ("trace_batch", "_make_pool", "init_guide_strands", "connect_segments", "grow")


def install(module=None, full=False):
    """Reroute the reference grow stage through the GPU.

    Always replaces ``strandkit.phg.trace_batch`` (resolved as a module global by
    every caller) and disables the fork pool (``_make_pool`` -> None,
    phg.py:184-196) because CUDA state must not be inherited by forked workers;
    the batch loop then calls trace_batch in-process (phg.py:239-241).
    ``full=True`` also replaces ``init_guide_strands`` (device batch driver,
    grow.py), ``connect_segments`` and ``grow`` (link.py), so the whole PHG stage
    -- tracing, deferred commits, field seeds, linking, attachment, tangents --
    runs on the GPU.
    """
    if module is None:
        import strandkit.phg as module  # type: ignore
    if module in _SAVED:
        return module
    _SAVED[module] = {k: getattr(module, k) for k in _REROUTED if hasattr(module, k)}
    module.trace_batch = trace_batch
    if hasattr(module, "_make_pool"):
        module._make_pool = lambda *a, **k: None
    if full:
        from . import grow as _grow
        from . import link as _link

        module.init_guide_strands = _grow.init_guide_strands
        module.connect_segments = _link.connect_segments
        module.grow = _link.grow
    return module


def uninstall(module=None):
    if module is None:
        import strandkit.phg as module  # type: ignore
    saved = _SAVED.pop(module, None)
    for k, v in (saved or {}).items():
        setattr(module, k, v)
