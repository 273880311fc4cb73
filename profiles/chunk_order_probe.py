"""Probe: how much seed locality does the trace kernel lose when the Morton ordering is done
per contiguous seed-order chunk instead of over the whole launch?

Motivation ((f) next): a seed-order-chunked queue would let each chunk's CSR gather
start while later chunks are still tracing.  This measures the K1 cost of chunking alone.
Seeds are permuted on the host (chunk id, Morton code of the seed voxel) and traced with the
library's own ordering disabled, so the queue order is exactly the probed one.

    python profiles/chunk_order_probe.py [C3|C5] [chunks,...]
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_05794_b200 import phg, synth  # noqa: E402
from paper_2604_05794_b200.volume import DeviceField  # noqa: E402


def spread3(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    for s, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                 (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(s))) & np.uint64(m)
    return v


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    chunk_list = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,16").split(",")]
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ori, occ = cfg.field(dev)
    stream = torch.cuda.current_stream(dev)
    field = DeviceField(np.zeros(3), synth.VOXEL_MM, occ, ori, stream.cuda_stream)
    seeds, dirs = synth.config_seeds(cfg, 1_000_000, ori, occ)
    del ori, occ
    torch.cuda.empty_cache()
    n = len(seeds)
    params = phg.PhgParams(field_seeds=0, batch_size=n)
    tracer = phg.Tracer()
    vox = np.clip(np.floor(seeds / synth.VOXEL_MM).astype(np.int64), 0, cfg.n - 1)
    code = spread3(vox[:, 0]) << np.uint64(2) | spread3(vox[:, 1]) << np.uint64(1) | spread3(vox[:, 2])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(s, d, order, reps=3):
        s_dev = torch.from_numpy(np.ascontiguousarray(s)).to(dev)
        d_dev = torch.from_numpy(np.ascontiguousarray(d)).to(dev)
        ms = []
        for _ in range(reps + 1):
            flush.zero_()
            off, verts, _ = phg.trace_device(field, s_dev, d_dev, params, tracer=tracer,
                                             stream=stream, order=order)
            torch.cuda.synchronize()
            ms.append(tracer.last_kernel_ms()[0])
            steps = int(verts.shape[0]) - n
            del off, verts
        return min(ms[1:]), steps

    out = {"config": name, "seeds": n}
    out["library_morton_ms"], steps = timed(seeds, dirs, True)
    out["seed_order_ms"], _ = timed(seeds, dirs, False)
    for k in chunk_list:
        chunk = np.arange(n) * k // n
        perm = np.lexsort((code, chunk))  # by chunk, then Morton code
        out[f"chunked{k}_ms"], s2 = timed(seeds[perm], dirs[perm], False)
        assert s2 == steps
    out["steps"] = steps
    print(json.dumps(out))


if __name__ == "__main__":
    main()
