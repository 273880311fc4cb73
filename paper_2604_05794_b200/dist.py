"""Multi-GPU PHG: seed partitioning, one process per GPU (torchrun), no collective
on the hot path.

Seeds of one deferred-commit batch are independent given the frozen at_cap
plane (phg.py:1-8), so each rank traces a contiguous slice of
the batch against its own replica of the field.  The slices are the
reference's own fork-pool split, ``np.linspace(0, n, world + 1)``
(phg.py:201), and concatenating rank outputs in rank order reproduces the
single-GPU CSR byte for byte -- the analogue of the reference's
"identical output for any worker count" contract (A9, test_acceptance.py:326).

The only communication is one all-gather of per-rank (strands, vertices)
counts, from which every rank derives its global CSR offsets; payloads stay
rank-local unless ``gather_to_root`` is asked for.  The same code runs over
NCCL (CUDA tensors) and gloo (CPU tensors, used by the CPU tests).
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


def gather_to_root(offsets_global, verts, entered, info: ShardInfo, group=None, device="cpu",
                   root=0):
    """Concatenate every rank's CSR on ``root`` (pad-to-max all-gather; NCCL has no gatherv).

    Returns (offsets (N+1,), verts (M,3), entered (N,)) as numpy on root, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    mx_s = int(info.counts[:, 0].max())
    mx_v = int(info.counts[:, 1].max())
    k = int(info.counts[info.rank, 0])
    m = int(info.counts[info.rank, 1])
    v = torch.zeros((max(mx_v, 1), 3), dtype=torch.float64, device=device)
    e = torch.zeros(max(mx_s, 1), dtype=torch.uint8, device=device)
    o = torch.zeros(max(mx_s, 1), dtype=torch.int64, device=device)
    v[:m] = torch.as_tensor(np.asarray(verts) if not torch.is_tensor(verts) else verts,
                            dtype=torch.float64, device=device).reshape(-1, 3)
    e[:k] = torch.as_tensor(np.asarray(entered) if not torch.is_tensor(entered) else entered,
                            device=device).to(torch.uint8)
    og = offsets_global if torch.is_tensor(offsets_global) else torch.as_tensor(
        np.asarray(offsets_global))
    o[:k] = og[:k].to(device=device, dtype=torch.int64)
    vs = [torch.empty_like(v) for _ in range(info.world)]
    es = [torch.empty_like(e) for _ in range(info.world)]
    os_ = [torch.empty_like(o) for _ in range(info.world)]
    dist.all_gather(vs, v, group=group)
    dist.all_gather(es, e, group=group)
    dist.all_gather(os_, o, group=group)
    if info.rank != root:
        return None
    parts_v, parts_e, parts_o = [], [], []
    for r in range(info.world):
        kr, mr = int(info.counts[r, 0]), int(info.counts[r, 1])
        parts_v.append(vs[r][:mr].cpu().numpy())
        parts_e.append(es[r][:kr].cpu().numpy().astype(bool))
        parts_o.append(os_[r][:kr].cpu().numpy())
    offsets = np.concatenate(parts_o + [np.array([info.n_verts], np.int64)])
    return offsets, np.concatenate(parts_v), np.concatenate(parts_e)
