"""Synthetic PHG workloads (the BASELINE.json configs C1-C5).

Fields are analytic and saddle-free so the reference itself is well
conditioned on them: tiny input perturbations do not flip
strand lengths, which is what makes vertex-exact parity meaningful.

Geometry shared by every config: origin (0,0,0), voxel 2.0 mm
(config.py:60 default), L = 2n mm, fields evaluated at voxel centres
(``OOVolume.centers``, volume.py:51-53), unit fp32 ``ori`` with ``ori = 0``
where unoccupied (the layout of ``OOVolume``, volume.py:21-28).

Everything is generated with torch so the same code builds a 64^3 test field
on the CPU and a 512^3 / 1024^3 bench field directly in HBM.  Seeds come from
numpy Philox with rejection sampling in a disk (only +,*,< -- bit-reproducible
on any host).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

VOXEL_MM = 2.0


@dataclass(frozen=True)
class Config:
    name: str
    n: int              # field is n^3 voxels
    kind: str           # straight | wavy | curly | sparse
    seeds: int          # seeds per GPU (scalp disk; sparse adds interior seeds)
    key: int            # Philox key for the seeds
    note: str
    omega_turns: float = 24.0  # curly / sparse fields: vortex rate W = omega_turns * pi / L

    def field(self, device="cpu"):
        """(ori, occ) of this config (make_field with the config's parameters)."""
        return make_field(self.kind, self.n, device, omega_turns=self.omega_turns)


CONFIGS = {
    "C1": Config("C1", 64, "straight", 10_000, 11, "64^3 straight cylinder, 10k seeds"),
    "C2": Config("C2", 256, "wavy", 100_000, 12, "256^3 wavy cylinder, 100k seeds"),
    "C3": Config("C3", 512, "curly", 1_000_000, 13, "512^3 curly vortex cylinder, 1M seeds"),
    "C4": Config("C4", 512, "curly", 4_000_000, 14, "512^3 curly, 4M seeds split over ranks"),
    "C5": Config("C5", 1024, "sparse", 8_000_000, 15, "1024^3 10%-fill sparse, scalp+interior"),
    # not a BASELINE config: C3 with a 6x slower vortex (W = 4 pi / L), so the helices climb
    # ~6x higher instead of winding near the seed plane (strand tops p50: C3 ~9 voxels, C3s
    # ~56): a stress case with a larger field footprint, measured beside C3
    "C3s": Config("C3s", 512, "curly", 1_000_000, 13, "512^3 steep curly (W = 4 pi/L), 1M seeds",
                  omega_turns=4.0),
}


def _centers(n, device):
    return (torch.arange(n, device=device, dtype=torch.float64) + 0.5) * VOXEL_MM


def make_field(kind: str, n: int, device="cpu", omega_turns: float = 24.0, sparse_key: int = 5,
               sparse_sigma: float = 3.0, sparse_fill: float = 0.10):
    """Return (ori f32 (n,n,n,3), occ bool (n,n,n)) on ``device``.

    straight: (0,0,1)                               [SURVEY 8(d) C1]
    wavy:     (0.6 cos(k z + 0.05 y), 0, 1), k = 8 pi / L   [C2]
    curly:    (-W (y - L/2), W (x - L/2), 1), W = omega_turns * pi / L  [C3]
    All three live in the cylinder r < 0.45 L about the z axis through (L/2, L/2).
    sparse:   curly orientation inside {gaussian-smoothed noise > its (1-fill) quantile}  [C5]
    """
    L = n * VOXEL_MM
    c = _centers(n, device)
    x = c.view(n, 1, 1)
    y = c.view(1, n, 1)
    z = c.view(1, 1, n)
    if kind == "straight":
        vx = torch.zeros((n, n, n), dtype=torch.float64, device=device)
        vy = torch.zeros_like(vx)
        vz = torch.ones_like(vx)
    elif kind == "wavy":
        k = 2 * math.pi / (L / 4)
        vx = (0.6 * torch.cos(k * z + 0.05 * y)).expand(n, n, n)
        vy = torch.zeros((n, n, n), dtype=torch.float64, device=device)
        vz = torch.ones_like(vy)
    elif kind in ("curly", "sparse"):
        w = omega_turns * math.pi / L
        vx = (-w * (y - L / 2)).expand(n, n, n)
        vy = (w * (x - L / 2)).expand(n, n, n)
        vz = torch.ones((n, n, n), dtype=torch.float64, device=device)
    else:
        raise ValueError(f"unknown field kind {kind!r}")
    nrm = torch.sqrt((vx * vx + vy * vy) + vz * vz)
    ori = torch.stack([vx / nrm, vy / nrm, vz / nrm], dim=-1).to(torch.float32)
    if kind == "sparse":
        occ = _sparse_occupancy(n, device, sparse_key, sparse_sigma, sparse_fill)
    else:
        occ = ((x - L / 2) ** 2 + (y - L / 2) ** 2 < (0.45 * L) ** 2).expand(n, n, n).clone()
    ori = ori * occ.unsqueeze(-1)
    return ori.contiguous(), occ.contiguous()


def _sparse_occupancy(n, device, key, sigma, fill):
    g = torch.Generator(device=device)
    g.manual_seed(key)
    vol = torch.randn((n, n, n), generator=g, device=device, dtype=torch.float32)
    r = int(4 * sigma + 0.5)
    t = torch.arange(-r, r + 1, device=device, dtype=torch.float32)
    kern = torch.exp(-0.5 * (t / sigma) ** 2)
    kern = (kern / kern.sum()).view(1, 1, -1)
    for axis in range(3):
        v = vol.movedim(axis, -1).reshape(-1, 1, n)
        v = torch.nn.functional.pad(v, (r, r), mode="reflect")
        v = torch.nn.functional.conv1d(v, kern)
        shape = list(vol.movedim(axis, -1).shape)
        vol = v.reshape(shape).movedim(-1, axis).contiguous()
    flat = vol.reshape(-1)
    sub = flat[torch.randint(0, flat.numel(), (min(flat.numel(), 1 << 22),), generator=g,
                             device=device)]
    thr = torch.quantile(sub.double(), 1.0 - fill).float()
    return vol > thr


def disk_seeds(n_vox: int, count: int, key: int, z_mm: float = 1.3, radius_frac: float = 0.4):
    """Scalp-like seeds: uniform in the disk r < radius_frac*L at height z_mm, dir +z.

    Rejection sampling from the bounding square (exact arithmetic only).
    Returns (pos (count,3) f64, dir (count,3) f64) numpy arrays.
    """
    L = n_vox * VOXEL_MM
    R = radius_frac * L
    rng = np.random.Generator(np.random.Philox(key=key))
    out = np.empty((0, 2))
    while len(out) < count:
        m = int((count - len(out)) * 1.35) + 64
        uv = rng.random((m, 2)) * (2 * R) - R
        uv = uv[(uv * uv).sum(axis=1) < R * R]
        out = np.concatenate([out, uv])
    out = out[:count]
    pos = np.empty((count, 3))
    pos[:, 0] = out[:, 0] + L / 2
    pos[:, 1] = out[:, 1] + L / 2
    pos[:, 2] = z_mm
    d = np.zeros((count, 3))
    d[:, 2] = 1.0
    return pos, d


def interior_seeds_torch(occ, ori, count: int, key: int):
    """interior_seeds for (possibly CUDA) torch fields: random occupied voxel centres
    (with replacement), dir = normalised voxel ori.  Returns float64 numpy arrays."""
    dev = occ.device
    g = torch.Generator(device=dev)
    g.manual_seed(key)
    idx = torch.nonzero(occ.reshape(-1)).squeeze(1)
    pick = idx[torch.randint(0, idx.numel(), (count,), generator=g, device=dev)]
    _, ny, nz = occ.shape
    ijk = torch.stack([pick // (ny * nz), (pick // nz) % ny, pick % nz], dim=1)
    pos = (ijk.double() + 0.5) * VOXEL_MM
    d = ori.reshape(-1, 3)[pick].double()
    d = d / torch.clamp(torch.linalg.vector_norm(d, dim=1, keepdim=True), min=1e-12)
    return pos.cpu().numpy(), d.cpu().numpy()


def config_seeds(cfg: "Config", count: int, ori=None, occ=None):
    """Seeds of a bench config: the disk for C1-C4; for the sparse C5 half disk seeds and
    half interior seeds traced in both directions (+d then -d), as SURVEY.md 8(d) C5."""
    if cfg.kind != "sparse":
        return disk_seeds(cfg.n, count, cfg.key)
    nd = count // 2
    ni = (count - nd) // 2
    sd, dd = disk_seeds(cfg.n, nd, cfg.key, radius_frac=0.45)
    si, di = interior_seeds_torch(occ, ori, ni, cfg.key + 1)
    pos = np.concatenate([sd, si, si])
    dirs = np.concatenate([dd, di, -di])
    # interleave the three groups in proportion (disk, disk, +d, -d, ...): every contiguous
    # slice -- a rank's share, the CPU legs' first-16384 sample -- carries the config's mix
    grp = [np.arange(nd), nd + np.arange(ni), nd + ni + np.arange(ni)]
    key = np.concatenate([(g - g[0] + 0.5) / len(g) for g in grp if len(g)])
    perm = np.argsort(key, kind="stable")
    return pos[perm], dirs[perm]


def interior_seeds(occ: np.ndarray, ori: np.ndarray, count: int, key: int):
    """Field-style seeds at centres of random occupied voxels, dir = voxel ori.

    Mirrors the seeding of ``_trace_field_seeds`` (phg.py:266-275) but picks
    voxels at random (Philox) instead of a strided scan.
    """
    idx = np.argwhere(occ)
    rng = np.random.Generator(np.random.Philox(key=key))
    pick = idx[rng.choice(len(idx), size=min(count, len(idx)), replace=False)]
    pos = (pick.astype(np.float64) + 0.5) * VOXEL_MM
    d = ori[pick[:, 0], pick[:, 1], pick[:, 2]].astype(np.float64)
    d = d / np.maximum(np.linalg.norm(d, axis=1, keepdims=True), 1e-12)
    return pos, d
