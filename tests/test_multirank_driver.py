"""Multi-rank deferred-commit batch driver (dist.init_guide_strands_multirank).

CPU: world_size 2 over gloo with the oracle backend -- per batch each rank traces its slice,
commit ids are all-gathered and applied by every rank -- must reproduce the reference's
init_guide_strands output (tests/golden/driver_*.npz) exactly: segments, order, rooted flags,
vol.counts and the report.
GPU: the same orchestration with the device backend (grow.DeviceGrowSession), direct and
with the export/all-gather/apply path forced on a single rank.
"""

import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT, load_case

CASES = ["driver_sparse40", "driver_curly32_cap1", "driver_sparse32_steer_vs17"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, path, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle.phg_driver_np import OracleGrowSession
    from paper_2604_05794_b200 import dist as pdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = load_case(path)
        counts = np.zeros(c.occ.shape, np.uint16)
        be = OracleGrowSession(c.origin, float(c.voxel_size), c.occ, c.ori, c.params)
        res = pdist.init_guide_strands_multirank(c.seeds, c.dirs, counts, c.params, be)
        if rank == 0:
            off, verts, rooted, rep = res
            np.savez(out, offsets=off, verts=verts, rooted=rooted, counts=counts,
                     report=json.dumps(rep))
        else:
            np.save(out + f".counts{rank}.npy", counts)
    finally:
        dist.destroy_process_group()


def _check(c, off, verts, rooted, counts, rep):
    assert np.array_equal(off, c.offsets)
    assert np.array_equal(verts, c.verts)
    assert np.array_equal(rooted, c.rooted)
    assert np.array_equal(counts, c.counts_out)
    assert rep == json.loads(str(c.report))


@pytest.mark.parametrize("name", CASES)
def test_two_rank_driver_matches_reference(tmp_path, name, oracle_c):
    path = os.path.join(GOLDEN, f"{name}.npz")
    out = str(tmp_path / "out.npz")
    mp.start_processes(_worker, args=(2, _free_port(), path, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    c = load_case(path)
    _check(c, got["offsets"], got["verts"], got["rooted"], got["counts"],
           json.loads(str(got["report"])))
    assert np.array_equal(np.load(out + ".counts1.npy"), c.counts_out)  # replicas agree


@pytest.mark.gpu
@pytest.mark.parametrize("force_export", [False, True])
@pytest.mark.parametrize("name", CASES)
def test_device_multirank_driver_one_rank(name, force_export):
    import torch.distributed as dist

    from paper_2604_05794_b200 import dist as pdist
    from paper_2604_05794_b200.grow import DeviceGrowSession
    from paper_2604_05794_b200.phg import PhgParams
    from paper_2604_05794_b200.volume import OOVolume

    c = load_case(os.path.join(GOLDEN, f"{name}.npz"))
    vol = OOVolume.empty(c.origin, float(c.voxel_size), c.occ.shape)
    vol.occ, vol.ori = c.occ, c.ori
    p = PhgParams(**{k: v for k, v in vars(c.params).items()
                     if k in PhgParams.__dataclass_fields__})
    dist.init_process_group("gloo", rank=0, world_size=1,
                            init_method=f"tcp://127.0.0.1:{_free_port()}")
    try:
        be = DeviceGrowSession(vol, p)
        off, verts, rooted, rep = pdist.init_guide_strands_multirank(
            c.seeds, c.dirs, vol.counts, p, be, force_export=force_export)
    finally:
        dist.destroy_process_group()
    _check(c, off, verts, rooted, vol.counts, rep)
