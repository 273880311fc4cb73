"""Multi-GPU PHG: seed partitioning, one process per GPU (torchrun), no collective
on the hot path.

Seeds of one deferred-commit batch are independent given the frozen at_cap
plane (phg.py:1-8), so each rank traces a contiguous slice of
the batch against its own replica of the field.  The slices are the
reference's own fork-pool split, ``np.linspace(0, n, world + 1)``
(phg.py:201), and concatenating rank outputs in rank order reproduces the
single-GPU CSR byte for byte -- the analogue of the reference's
"identical output for any worker count" contract (A9, test_acceptance.py:326).

The only communication on the trace path is one all-gather of per-rank (strands,
vertices) counts, from which every rank derives its global CSR offsets; payloads stay
rank-local unless asked for: ``gather_to_root`` moves each rank's payload to the root only
(point-to-point), never to every rank, and ``gather_csr_to_root_p2p`` has each rank's CSR
gather kernel write straight into the root's global CSR over peer memory.  Setup:
``replicate_field`` packs the field once and broadcasts the packed buffer.  The same code
runs over NCCL (CUDA tensors) and gloo (CPU tensors, used by the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def slice_bounds(n: int, world: int) -> np.ndarray:
    """Contiguous rank slices of n seeds (phg.py:201's split)."""
    return np.linspace(0, n, world + 1).astype(np.int64)


@dataclass
class ShardInfo:
    rank: int
    world: int
    seed_lo: int
    seed_hi: int
    counts: np.ndarray        # (world, 2): per-rank (strands, vertices)
    strand_start: int         # global index of this rank's first strand
    vert_start: int           # global CSR offset of this rank's first vertex
    n_strands: int            # global totals
    n_verts: int


def exchange_counts(n_strands: int, n_verts: int, group=None, device="cpu") -> ShardInfo:
    """All-gather (strands, vertices) of every rank -> this rank's global offsets."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = torch.tensor([n_strands, n_verts], dtype=torch.int64, device=device)
    allc = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    counts = torch.stack(allc).cpu().numpy()
    before = counts[:rank].sum(axis=0)
    return ShardInfo(rank, world, 0, 0, counts, int(before[0]), int(before[1]),
                     int(counts[:, 0].sum()), int(counts[:, 1].sum()))


def replicate_field(vol=None, src=0, group=None, device="cuda"):
    """The packed field on every rank from ONE rank's upload (multi-GPU setup).

    Rank ``src`` packs ``vol`` (occ/ori host arrays) once; the padded float4 buffer (2 GiB at
    512^3) and its geometry are broadcast to the other ranks -- NCCL over NVLink when
    ``device`` is "cuda", staged through host memory for gloo ("cpu") -- so no other rank
    reads or packs the host arrays.  Returns this rank's DeviceField (bit-identical buffers).
    """
    import torch
    import torch.distributed as dist

    from .phg import _CudaArray
    from .volume import DeviceField

    rank = dist.get_rank(group)
    glob_src = dist.get_global_rank(group, src) if group is not None else src
    f = None
    err = None
    meta = torch.zeros(9, dtype=torch.float64)  # dims[0] = -1: the source could not pack it
    if rank == src:
        try:
            f = DeviceField(vol.origin, vol.voxel_size, vol.occ, vol.ori)
            _, _, zeroed, maxabs = f.packed()
            meta[:] = torch.tensor([*f.dims, *f.origin.tolist(), f.voxel_size, float(zeroed),
                                    maxabs if np.isfinite(maxabs) else -1.0],
                                   dtype=torch.float64)
        except Exception as exc:  # noqa: BLE001 - every rank must learn it before going on
            err = exc
            meta[0] = -1.0
    meta = meta.to(device)
    dist.broadcast(meta, glob_src, group=group)
    m = meta.cpu().tolist()
    if m[0] < 0:
        from .errors import PipelineError

        raise PipelineError(f"replicate_field: the source rank could not pack the field "
                            f"({err if err is not None else 'see the source rank'})")
    if rank != src:
        f = DeviceField.create_packed([int(m[0]), int(m[1]), int(m[2])], m[3:6], m[6],
                                      m[7] != 0.0, m[8] if m[8] >= 0 else float("inf"))
    ptr, nbytes, _, _ = f.packed()
    buf = torch.as_tensor(_CudaArray(ptr, (nbytes,), "|u1"), device=torch.cuda.current_device())
    if str(device).startswith("cuda"):
        dist.broadcast(buf, glob_src, group=group)
    else:  # gloo: through host memory
        host = buf.cpu() if rank == src else torch.empty(nbytes, dtype=torch.uint8)
        dist.broadcast(host, glob_src, group=group)
        if rank != src:
            buf.copy_(host)
    torch.cuda.synchronize()
    if rank != src:
        f.packed_done()
    return f


def exchange_counts_device(n_strands_t, n_verts_t, group=None, device="cpu"):
    """exchange_counts without a host synchronisation (NCCL): the (strands, vertices) pair is
    built from device tensors (e.g. phg_trace_rows' kept-vertex counter) and all-gathered on
    the stream; returns the (world, 2) tensor of every rank's counts, in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = torch.cat([n_strands_t.reshape(1), n_verts_t.reshape(1)]).to(device=device,
                                                                        dtype=torch.int64)
    allc = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    return torch.stack(allc)


def trace_sharded(trace_fn, seed_pos, seed_dir, group=None, device="cpu"):
    """Trace this rank's slice of a batch and return it with global CSR placement.

    ``trace_fn(pos, dirs) -> (offsets (k+1,), verts (m,3), entered (k,))`` traces
    a slice (the GPU path passes a closure over ``phg.trace_device``).  Returns
    (global_offsets (k+1,), verts, entered, ShardInfo): ``global_offsets`` are
    this rank's CSR row starts in the concatenated all-rank payload.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b = slice_bounds(len(seed_pos), world)
    lo, hi = int(b[rank]), int(b[rank + 1])
    off, verts, ent = trace_fn(seed_pos[lo:hi], seed_dir[lo:hi])
    info = exchange_counts(hi - lo, int(verts.shape[0]), group=group, device=device)
    info.seed_lo, info.seed_hi = lo, hi
    return off + info.vert_start, verts, ent, info


def _allgather_v(t, group=None):
    """All-gather of 1-D tensors of different lengths (pad to the longest)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    sizes = [int(x.item()) for x in ns]
    pad = torch.zeros(max(max(sizes), 1), dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:s] for o, s in zip(outs, sizes)]


def _gather_v_to_root(t, group=None, root=0):
    """Gather 1-D tensors of different lengths on ``root`` (rank order) with point-to-point
    sends: only the lengths are all-gathered, and each payload crosses the fabric once, to
    root (NCCL on CUDA tensors, gloo on CPU tensors).  Returns the list on root, None
    elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = t.contiguous()
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    sizes = [int(x.item()) for x in ns]

    def glob(r):
        return dist.get_global_rank(group, r) if group is not None else r

    if rank != root:
        if t.numel():
            dist.send(t, dst=glob(root), group=group)
        return None
    out = []
    for r in range(world):
        if r == root:
            out.append(t)
            continue
        buf = torch.empty(sizes[r], dtype=t.dtype, device=t.device)
        if sizes[r]:
            dist.recv(buf, src=glob(r), group=group)
        out.append(buf)
    return out


def init_guide_strands_multirank(seeds, normals, counts, params, backend, group=None,
                                 device="cpu", force_export=False):
    """init_guide_strands (phg.py:210-303) over all ranks of ``group``, exactly.

    Every deferred-commit batch -- scalp batches of ``params.batch_size`` seeds, then the
    field-seed batches -- is split in contiguous rank slices (phg.py:201's split); each rank
    traces its slice against the SAME frozen cap plane (every rank holds an identical
    ``counts`` replica), exports its commits (one voxel id per segment and distinct voxel,
    phg.py:248-251), and all ranks apply the all-gathered union before the next batch.  This
    is the one collective per batch the deferred-commit semantics require.
    ``backend`` runs the batch steps: grow.DeviceGrowSession on a GPU (NCCL, CUDA ids) or an
    oracle session on the CPU (gloo tests).  ``counts`` (uint16, vol.counts) is updated in
    place on every rank.  ``device`` is where the collectives run ("cuda" for NCCL, "cpu"
    for gloo); ``force_export`` exercises the export/all-gather/apply path on one rank.

    Returns (offsets, verts, rooted, report) of the full segment set, in the reference's
    order, on rank 0 and None on the other ranks.
    """
    import torch
    import torch.distributed as dist

    if bool(params.strict):
        from .errors import ConfigError

        raise ConfigError("strict mode commits after every step of every strand; run it on one rank")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    export = world > 1 or force_export
    bs = int(params.batch_size)
    backend.begin(counts)
    log = []  # segments this rank added per batch

    def exchange(ids):
        if export:
            backend.apply(torch.cat(_allgather_v(ids.to(device), group)))

    n = len(seeds)
    for b0 in range(0, n, bs):
        nb = min(bs, n - b0)
        b = slice_bounds(nb, world)
        lo, hi = b0 + int(b[rank]), b0 + int(b[rank + 1])
        added, ids = backend.scalp_batch(seeds[lo:hi], normals[lo:hi], export)
        exchange(ids)
        log.append(added)
    n_scalp_batches = len(log)
    nf = backend.field_begin() if (n > 0 and params.field_seeds > 0) else 0
    for b0 in range(0, nf, bs):
        nb = min(bs, nf - b0)
        b = slice_bounds(nb, world)
        added, ids = backend.field_batch(b0 + int(b[rank]), int(b[rank + 1] - b[rank]), export)
        exchange(ids)
        log.append(added)
    offsets, verts, rooted, never = backend.end(counts)
    # ---- global order: batch by batch, rank by rank (each rank's slice is contiguous)
    logs = _allgather_v(torch.tensor(log, dtype=torch.int64, device=device), group)
    nev = torch.tensor([never], dtype=torch.int64, device=device)
    dist.all_reduce(nev, group=group)
    # the segment payloads travel to rank 0 only (the one rank that assembles the result)
    lens = torch.as_tensor(np.diff(offsets), dtype=torch.int64, device=device)
    all_lens = _gather_v_to_root(lens, group)
    all_verts = _gather_v_to_root(torch.as_tensor(verts.reshape(-1), device=device), group)
    all_root = _gather_v_to_root(torch.as_tensor(rooted.astype(np.uint8), device=device), group)
    if rank != 0:
        return None
    per_rank = []
    for r in range(world):
        ln = all_lens[r].cpu().numpy()
        off = np.zeros(len(ln) + 1, np.int64)
        np.cumsum(ln, out=off[1:])
        per_rank.append((off, all_verts[r].cpu().numpy().reshape(-1, 3),
                         all_root[r].cpu().numpy().astype(bool), logs[r].cpu().numpy()))
    cursor = [0] * world
    parts_v, parts_len, parts_root = [], [], []
    n_scalp_segs = 0
    for bi in range(len(log)):
        for r in range(world):
            off, v, ro, lg = per_rank[r]
            k0, k1 = cursor[r], cursor[r] + int(lg[bi])
            cursor[r] = k1
            parts_v.append(v[off[k0]:off[k1]])
            parts_len.append(np.diff(off[k0:k1 + 1]))
            parts_root.append(ro[k0:k1])
            if bi < n_scalp_batches:
                n_scalp_segs += k1 - k0
    lens_all = np.concatenate(parts_len) if parts_len else np.zeros(0, np.int64)
    offsets_all = np.zeros(len(lens_all) + 1, np.int64)
    np.cumsum(lens_all, out=offsets_all[1:])
    verts_all = np.concatenate(parts_v) if parts_v else np.zeros((0, 3))
    rooted_all = np.concatenate(parts_root) if parts_root else np.zeros(0, bool)
    report = {"n_seeds": int(n), "n_segments": int(len(lens_all)),
              "n_never_entered": int(nev.item())}
    if n == 0:
        report["warning"] = "no scalp seeds; nothing to trace"
    else:
        report["n_scalp_segments"] = int(n_scalp_segs)
    return offsets_all, verts_all, rooted_all, report


def gather_csr_to_root_p2p(tracer, info: ShardInfo, group=None, root=0, return_result=True):
    """The CSR of the last ``tracer.trace`` on every rank, concatenated in rank order on
    ``root``'s GPU by the gather kernel itself: root allocates the global CSR once
    (``phg_ipc_alloc``), every rank opens it as peer memory (CUDA IPC; NVLink P2P between GPUs)
    and ``phg_gather_to`` writes the rank's strands straight to their global places -- the
    gather and the "gather to root" collective are one kernel per rank, no NCCL payload
    transfer.  ``info`` is this rank's ``exchange_counts`` result.

    Returns (offsets (N+1,), verts (M,3), entered (N,)) as CUDA tensors on root, None elsewhere
    (``return_result=False``: the global buffers are freed after the gather, root returns
    their sizes -- the measurement leg of bench.py).
    """
    import ctypes

    import torch
    import torch.distributed as dist

    from . import _native
    from .phg import _CudaArray

    lib = _native.load()
    rank = dist.get_rank(group)
    glob_root = dist.get_global_rank(group, root) if group is not None else root
    N, M = int(info.n_strands), int(info.n_verts)
    sizes = (M * 24, (N + 1) * 8, max(N, 1))
    handles = torch.zeros(3 * 64 + 1, dtype=torch.uint8)  # + status byte: 1 = root allocated
    ptrs = [None] * 3
    err = None
    if rank == root:
        try:
            for k, nb in enumerate(sizes):
                p, hb = ctypes.c_void_p(), ctypes.create_string_buffer(64)
                _native.check(lib.phg_ipc_alloc(nb, ctypes.byref(p),
                                                ctypes.cast(hb, ctypes.c_void_p)), "phg_ipc_alloc")
                ptrs[k] = p.value
                handles[64 * k: 64 * (k + 1)] = torch.frombuffer(bytearray(hb.raw),
                                                                 dtype=torch.uint8)
            handles[-1] = 1
        except Exception as exc:  # noqa: BLE001 - every rank must learn it before going on
            err = exc
            for q in ptrs:
                if q:
                    lib.phg_ipc_free(q)
    dev = torch.device("cuda", torch.cuda.current_device())
    bcast_dev = "cpu" if dist.get_backend(group) == "gloo" else dev
    h = handles.to(bcast_dev)
    dist.broadcast(h, glob_root, group=group)
    if int(h[-1].item()) != 1:
        from .errors import PipelineError

        raise PipelineError(f"gather_csr_to_root_p2p: the root could not allocate the global CSR "
                            f"({err if err is not None else 'see the root rank'})")
    opened = []
    err = None
    try:
        if rank != root:
            raw = bytes(h[:-1].cpu().numpy().tobytes())
            for k in range(3):
                p = ctypes.c_void_p()
                hb = ctypes.create_string_buffer(raw[64 * k: 64 * (k + 1)], 64)
                _native.check(lib.phg_ipc_open(ctypes.cast(hb, ctypes.c_void_p), ctypes.byref(p)),
                              "phg_ipc_open")
                ptrs[k] = p.value
                opened.append(p.value)
        _native.check(lib.phg_gather_to(tracer.handle, ptrs[0], ptrs[1], ptrs[2],
                                        int(info.vert_start), int(info.strand_start), 0),
                      "phg_gather_to")
        torch.cuda.synchronize()
    except Exception as exc:  # noqa: BLE001 - reported to every rank below
        err = exc
    finally:
        for p in opened:
            lib.phg_ipc_close(p)
    # every rank's strands are in place -- or every rank learns that one failed
    ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=bcast_dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if not int(ok.item()):
        if rank == root:
            for p in ptrs:
                lib.phg_ipc_free(p)
        from .errors import PipelineError

        raise PipelineError(f"gather_csr_to_root_p2p failed on a rank ({err or 'another rank'})")
    if rank != root:
        return None
    if not return_result:
        for p in ptrs:
            lib.phg_ipc_free(p)
        return {"strands": N, "vertices": M, "bytes": int(sum(sizes))}
    try:
        off = torch.as_tensor(_CudaArray(ptrs[1], (N + 1,), "<i8"), device=dev).clone()
        off[N] = M
        verts = (torch.as_tensor(_CudaArray(ptrs[0], (M, 3), "<f8"), device=dev).clone()
                 if M else torch.empty((0, 3), dtype=torch.float64, device=dev))
        ent = (torch.as_tensor(_CudaArray(ptrs[2], (N,), "|u1"), device=dev).clone()
               if N else torch.empty(0, dtype=torch.uint8, device=dev))
        torch.cuda.synchronize()
    finally:
        for p in ptrs:
            lib.phg_ipc_free(p)
    return off, verts, ent


def gather_to_root(offsets_global, verts, entered, info: ShardInfo, group=None, device="cpu",
                   root=0):
    """Concatenate every rank's CSR on ``root``: each rank sends its payload straight to root
    (point-to-point; sizes are already known from ``exchange_counts``), so no rank receives
    any other rank's vertices except root.

    Returns (offsets (N+1,), verts (M,3), entered (N,)) as numpy on root, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    def as_t(a, dtype):
        t = a if torch.is_tensor(a) else torch.as_tensor(np.asarray(a))
        return t.to(device=device, dtype=dtype).contiguous()

    k = int(info.counts[info.rank, 0])
    v = as_t(verts, torch.float64).reshape(-1)
    e = as_t(entered, torch.uint8).reshape(-1)[:k]
    o = as_t(offsets_global, torch.int64).reshape(-1)[:k]

    def glob(r):
        return dist.get_global_rank(group, r) if group is not None else r

    if info.rank != root:
        for t in (v, e, o):
            if t.numel():
                dist.send(t, dst=glob(root), group=group)
        return None
    parts_v, parts_e, parts_o = [], [], []
    for r in range(info.world):
        kr, mr = int(info.counts[r, 0]), int(info.counts[r, 1])
        if r == root:
            bufs = (v, e, o)
        else:
            bufs = (torch.empty(3 * mr, dtype=torch.float64, device=device),
                    torch.empty(kr, dtype=torch.uint8, device=device),
                    torch.empty(kr, dtype=torch.int64, device=device))
            for t in bufs:
                if t.numel():
                    dist.recv(t, src=glob(r), group=group)
        parts_v.append(bufs[0].cpu().numpy().reshape(-1, 3))
        parts_e.append(bufs[1].cpu().numpy().astype(bool))
        parts_o.append(bufs[2].cpu().numpy())
    offsets = np.concatenate(parts_o + [np.array([info.n_verts], np.int64)])
    return offsets, np.concatenate(parts_v), np.concatenate(parts_e)
