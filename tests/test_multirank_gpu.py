"""World-size-2 runs of the multi-GPU paths THROUGH THE CUDA KERNEL (two processes on cuda:0).

The box has one GPU, so the two ranks share it and talk over gloo (CPU collectives); every
trace, commit and gather runs in libphg_b200.so exactly as it does with one GPU per rank
(only the collective transport differs from NCCL).  Contract, as the reference's A9
(test_acceptance.py:302-334): the rank-order result equals the single-process
result byte for byte, and equals the reference's own fixtures.

  * dist.trace_sharded over phg.trace_device + dist.gather_to_root (the bench's N > 1 path)
  * dist.init_guide_strands_multirank over grow.DeviceGrowSession (multi-batch driver, one
    commit exchange per deferred-commit batch)
"""

import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT, load_case

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return torch, dist


def _trace_worker(rank, world, port, case_path, out_path):
    torch, dist = _init(rank, world, port)
    try:
        from paper_2604_05794_b200 import dist as pdist
        from paper_2604_05794_b200 import phg
        from paper_2604_05794_b200.volume import field_for

        c = load_case(case_path)
        f = field_for(c.vol)
        cap = getattr(c, "at_cap", None)
        f.set_cap(cap if cap is not None and cap.any() else None)
        f.set_near(None)

        def trace_fn(pos, dirs):
            off, v, e = phg.trace_device(f, torch.from_numpy(np.ascontiguousarray(pos)).cuda(),
                                         torch.from_numpy(np.ascontiguousarray(dirs)).cuda(),
                                         c.params)
            torch.cuda.synchronize()
            return off, v, e

        off_g, verts, ent, info = pdist.trace_sharded(trace_fn, c.seeds, c.dirs)
        assert info.seed_hi - info.seed_lo == len(ent)
        # payload to rank 0 only (CPU tensors: gloo)
        res = pdist.gather_to_root(off_g[:-1].cpu(), verts.cpu(), ent.cpu(), info)
        if rank == 0:
            off, v, e = res
            np.savez(out_path, offsets=off, verts=v, entered=e, counts=info.counts)
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["trace_curly48", "trace_sparse48", "trace_curly40_cap"])
def test_two_ranks_on_device_equal_reference(tmp_path, name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    out = str(tmp_path / "out.npz")
    mp.start_processes(_trace_worker, args=(2, _free_port(), path, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    c = load_case(path)
    assert np.array_equal(got["offsets"], c.offsets)
    assert np.array_equal(got["verts"], c.verts)
    assert np.array_equal(got["entered"], c.entered)
    assert got["counts"][:, 0].sum() == len(c.entered)


def _driver_worker(rank, world, port, case_path, out_path):
    torch, dist = _init(rank, world, port)
    try:
        from paper_2604_05794_b200 import dist as pdist
        from paper_2604_05794_b200.grow import DeviceGrowSession
        from paper_2604_05794_b200.phg import PhgParams
        from paper_2604_05794_b200.volume import OOVolume

        c = load_case(case_path)
        vol = OOVolume.empty(c.origin, float(c.voxel_size), c.occ.shape)
        vol.occ, vol.ori = c.occ, c.ori
        p = PhgParams(**{k: v for k, v in vars(c.params).items()
                         if k in PhgParams.__dataclass_fields__})
        be = DeviceGrowSession(vol, p)
        res = pdist.init_guide_strands_multirank(c.seeds, c.dirs, vol.counts, p, be)
        if rank == 0:
            off, verts, rooted, rep = res
            np.savez(out_path, offsets=off, verts=verts, rooted=rooted, counts=vol.counts,
                     report=json.dumps(rep))
        else:
            assert res is None
            np.save(out_path + f".counts{rank}.npy", vol.counts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["driver_sparse40", "driver_curly32_cap1",
                                  "driver_sparse32_steer_vs17"])
def test_two_rank_device_driver_equals_reference(tmp_path, name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    out = str(tmp_path / "out.npz")
    mp.start_processes(_driver_worker, args=(2, _free_port(), path, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    c = load_case(path)
    assert np.array_equal(got["offsets"], c.offsets)
    assert np.array_equal(got["verts"], c.verts)
    assert np.array_equal(got["rooted"], c.rooted)
    assert np.array_equal(got["counts"], c.counts_out)
    assert np.array_equal(np.load(out + ".counts1.npy"), c.counts_out)  # replicas agree
    assert json.loads(str(got["report"])) == json.loads(str(c.report))


def _replicate_worker(rank, world, port, case_path, out_path):
    torch, dist = _init(rank, world, port)
    try:
        from paper_2604_05794_b200 import dist as pdist
        from paper_2604_05794_b200 import phg

        c = load_case(case_path)
        f = pdist.replicate_field(c.vol if rank == 0 else None, src=0, device="cpu")
        cap = getattr(c, "at_cap", None)
        f.set_cap(cap if cap is not None and cap.any() else None)
        off, v, e = phg.trace_device(f, torch.from_numpy(c.seeds).cuda(),
                                     torch.from_numpy(c.dirs).cuda(), c.params)
        ptr, nbytes, zeroed, maxabs = f.packed()
        np.savez(out_path + f".{rank}.npz", offsets=off.cpu().numpy(), verts=v.cpu().numpy(),
                 entered=e.cpu().numpy(), meta=np.array([nbytes, zeroed, maxabs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["trace_sparse48", "trace_curly40_cap"])
def test_field_replicated_from_one_rank(tmp_path, name):
    """dist.replicate_field: rank 0 packs the field once and broadcasts the packed buffer;
    rank 1, which never sees the host arrays, traces the reference fixture bit-exactly."""
    path = os.path.join(GOLDEN, f"{name}.npz")
    out = str(tmp_path / "out")
    mp.start_processes(_replicate_worker, args=(2, _free_port(), path, out), nprocs=2,
                       join=True, start_method="spawn")
    c = load_case(path)
    r0, r1 = np.load(out + ".0.npz"), np.load(out + ".1.npz")
    assert np.array_equal(r0["meta"], r1["meta"])
    for r in (r0, r1):
        assert np.array_equal(r["offsets"], c.offsets)
        assert np.array_equal(r["verts"], c.verts)
        assert np.array_equal(r["entered"].astype(bool), c.entered)


def _p2p_worker(rank, world, port, case_path, out_path, n=None):
    torch, dist = _init(rank, world, port)
    try:
        from paper_2604_05794_b200 import dist as pdist
        from paper_2604_05794_b200 import phg
        from paper_2604_05794_b200.volume import field_for

        c = load_case(case_path)
        if n is not None:  # fewer seeds than ranks: some ranks contribute nothing
            c.seeds, c.dirs = c.seeds[:n], c.dirs[:n]
        f = field_for(c.vol)
        cap = getattr(c, "at_cap", None)
        f.set_cap(cap if cap is not None and cap.any() else None)
        f.set_near(None)
        b = pdist.slice_bounds(len(c.seeds), world)
        lo, hi = int(b[rank]), int(b[rank + 1])
        tr = phg.Tracer()
        pos = np.ascontiguousarray(c.seeds[lo:hi])
        dirs = np.ascontiguousarray(c.dirs[lo:hi])
        off_l = np.zeros(hi - lo + 1, np.int64)
        ent_l = np.zeros(max(hi - lo, 1), np.uint8)
        m = tr.trace(f, c.params, pos.ctypes.data if hi > lo else None,
                     dirs.ctypes.data if hi > lo else None, hi - lo, off_l.ctypes.data,
                     ent_l.ctypes.data)
        info = pdist.exchange_counts(hi - lo, m)
        res = pdist.gather_csr_to_root_p2p(tr, info)
        if rank == 0:
            off, v, e = (t.cpu().numpy() for t in res)
            np.savez(out_path, offsets=off, verts=v, entered=e)
        else:
            assert res is None
        tr.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("trace_curly48", None), ("trace_curly40_cap", None),
                                    ("trace_curly48", 1)])
def test_gather_to_root_over_peer_memory(tmp_path, name, n):
    """dist.gather_csr_to_root_p2p: each rank's CSR gather kernel writes straight into the
    root's global CSR through CUDA IPC peer memory (NVLink between GPUs; the same device
    here) -- byte-identical to the reference's single-process output."""
    path = os.path.join(GOLDEN, f"{name}.npz")
    out = str(tmp_path / "out.npz")
    mp.start_processes(_p2p_worker, args=(2, _free_port(), path, out, n), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    c = load_case(path)
    k = len(c.entered) if n is None else n
    assert np.array_equal(got["offsets"], c.offsets[:k + 1])
    assert np.array_equal(got["verts"], c.verts[: c.offsets[k]])
    assert np.array_equal(got["entered"].astype(bool), c.entered[:k])
