"""CPU restatement of the reference's deferred-commit batch driver -- TEST INFRASTRUCTURE.

Restates strandkit.phg.init_guide_strands (/root/reference/pkg/src/strandkit/phg.py:210-260)
and _trace_field_seeds (phg.py:263-303) on top of the C trace oracle
(oracle/phg_oracle.c); pinned bit-exact against tests/golden/driver_sparse40.npz, which
the reference produced.  Only tests/ and bench CPU legs may import this module.
"""

from __future__ import annotations

import numpy as np

from . import phg_oracle_c as oc


def _unit(v):
    return v / np.maximum(np.linalg.norm(v, axis=-1, keepdims=True), 1e-12)


def _commit(counts, origin, vs, dims, v):
    """counts[unique in-bounds voxels of v] += 1 (phg.py:248-251)."""
    ijk = np.floor((v - origin) / vs).astype(np.int64)
    ok = np.all((ijk >= 0) & (ijk < np.asarray(dims)), axis=1)
    u = np.unique(ijk[ok], axis=0)
    counts[u[:, 0], u[:, 1], u[:, 2]] += 1


def init_guide(origin, vs, occ, ori, counts, seeds, normals, params, near_occ=None,
               trace_batch=None):
    """Returns ([(vertices, rooted), ...], report); updates ``counts`` (uint16) in place.

    ``trace_batch`` (optional): a function with the reference's trace_batch signature
    (vol, seed_pos, seed_dir, params, at_cap=None, live_counts=None, near_occ=None) ->
    [(vertices, entered), ...] that replaces the C oracle trace -- the GPU tests pass the
    drop-in ``paper_2604_05794_b200.phg.trace_batch`` to run the reference's batch loop
    (phg.py:229-251, 277-302) over it, exactly as strandkit.phg does after install()."""
    origin = np.asarray(origin, np.float64)
    dims = occ.shape
    strict = bool(params.strict)
    near = near_occ if float(params.steer) > 0 else None
    report = {"n_seeds": int(len(seeds)), "n_segments": 0, "n_never_entered": 0}
    if len(seeds) == 0:
        report["warning"] = "no scalp seeds; nothing to trace"
        return [], report
    out = []

    if trace_batch is not None:  # one volume object for the whole loop, as the reference has
        from types import SimpleNamespace

        vol = SimpleNamespace(origin=origin, voxel_size=vs, dims=occ.shape, occ=occ, ori=ori,
                              counts=counts)

    def run(pos, dirs):
        cap = None if strict else (counts >= params.occupancy_cap)
        if trace_batch is not None:
            return trace_batch(vol, pos, dirs, params, at_cap=None if strict else cap,
                               live_counts=counts if strict else None, near_occ=near)
        slab, keep, ent = oc.trace(origin, vs, occ, ori, pos, dirs, params, at_cap=cap,
                                   live_counts=counts if strict else None, near_occ=near)
        return [(slab[i, : keep[i]].copy(), bool(ent[i])) for i in range(len(keep))]

    bs = int(params.batch_size)
    for b0 in range(0, len(seeds), bs):
        for v, entered in run(seeds[b0:b0 + bs], normals[b0:b0 + bs]):
            if not entered or len(v) < 2:
                report["n_never_entered"] += int(not entered)
                continue
            out.append((v, True))
            if not strict:
                _commit(counts, origin, vs, dims, v)
    report["n_scalp_segments"] = len(out)
    if params.field_seeds > 0:
        unvisited = np.argwhere(occ & (counts == 0))
        if len(unvisited):
            if len(unvisited) > params.field_seeds:
                pick = np.linspace(0, len(unvisited) - 1, params.field_seeds).astype(np.int64)
                unvisited = unvisited[pick]
            centers = origin + (unvisited.astype(np.float64) + 0.5) * vs
            odir = ori[unvisited[:, 0], unvisited[:, 1], unvisited[:, 2]].astype(np.float64)
            ok = np.linalg.norm(odir, axis=1) > 1e-9
            centers, odir = centers[ok], _unit(odir[ok])
            for b0 in range(0, len(centers), bs):
                cb, db = centers[b0:b0 + bs], odir[b0:b0 + bs]
                fwd = run(cb, 1.0 * db)
                bwd = run(cb, -1.0 * db)
                for (vf, ef), (vb, eb) in zip(fwd, bwd):
                    v = np.concatenate([vb[::-1], vf[1:]]) if len(vb) > 1 else vf
                    if len(v) < 4 or not (ef or eb):
                        continue
                    out.append((v, False))
                    if not strict:
                        _commit(counts, origin, vs, dims, v)
    report["n_segments"] = len(out)
    return out, report


class OracleGrowSession:
    """Batch-level steps of the driver on the CPU oracle -- the test backend of
    paper_2604_05794_b200.dist.init_guide_strands_multirank (same API as
    grow.DeviceGrowSession; commit ids as int64 CPU tensors for gloo)."""

    def __init__(self, origin, vs, occ, ori, params):
        self.origin = np.asarray(origin, np.float64)
        self.vs = float(vs)
        self.occ, self.ori, self.params = occ, ori, params
        self.dims = occ.shape
        self.near = _near_map(occ) if float(params.steer) > 0 else None

    def begin(self, counts):
        self.counts = counts.copy()
        self.segs, self.never, self.field = [], 0, None

    def _trace(self, pos, dirs):
        cap = self.counts >= self.params.occupancy_cap
        slab, keep, ent = oc.trace(self.origin, self.vs, self.occ, self.ori, pos, dirs,
                                   self.params, at_cap=cap, near_occ=self.near)
        return [(slab[i, : keep[i]].copy(), bool(ent[i])) for i in range(len(keep))]

    def _ids(self, v):
        ijk = np.floor((v - self.origin) / self.vs).astype(np.int64)
        ok = np.all((ijk >= 0) & (ijk < np.asarray(self.dims)), axis=1)
        u = np.unique(ijk[ok], axis=0)
        return np.ravel_multi_index((u[:, 0], u[:, 1], u[:, 2]), self.dims)

    def _finish(self, kept, export):
        import torch

        ids = [self._ids(v) for v, _ in kept]
        ids = np.concatenate(ids) if ids else np.zeros(0, np.int64)
        self.segs += kept
        if not export:
            self.apply(ids)
            return len(kept), None
        return len(kept), torch.as_tensor(ids, dtype=torch.int64)

    def scalp_batch(self, seeds, normals, export):
        kept = []
        for v, e in self._trace(seeds, normals):
            if not e or len(v) < 2:
                self.never += int(not e)
                continue
            kept.append((v, True))
        return self._finish(kept, export)

    def field_begin(self):
        un = np.argwhere(self.occ & (self.counts == 0))
        if len(un) > self.params.field_seeds:
            un = un[np.linspace(0, len(un) - 1, self.params.field_seeds).astype(np.int64)]
        c = self.origin + (un.astype(np.float64) + 0.5) * self.vs
        d = self.ori[un[:, 0], un[:, 1], un[:, 2]].astype(np.float64)
        ok = np.linalg.norm(d, axis=1) > 1e-9
        self.field = (c[ok], _unit(d[ok]))
        return int(ok.sum())

    def field_batch(self, first, nb, export):
        c, d = self.field[0][first:first + nb], self.field[1][first:first + nb]
        kept = []
        for (vf, ef), (vb, eb) in zip(self._trace(c, 1.0 * d), self._trace(c, -1.0 * d)):
            v = np.concatenate([vb[::-1], vf[1:]]) if len(vb) > 1 else vf
            if len(v) >= 4 and (ef or eb):
                kept.append((v, False))
        return self._finish(kept, export)

    def apply(self, ids):
        ids = np.asarray(ids, np.int64)
        if len(ids):
            np.add.at(self.counts.reshape(-1), ids, 1)

    def end(self, counts):
        counts[...] = self.counts
        off = np.zeros(len(self.segs) + 1, np.int64)
        off[1:] = np.cumsum([len(v) for v, _ in self.segs])
        verts = np.concatenate([v for v, _ in self.segs]) if self.segs else np.zeros((0, 3))
        return off, verts, np.array([r for _, r in self.segs], bool), self.never


def _near_map(occ):
    from scipy.ndimage import distance_transform_edt

    _, inds = distance_transform_edt(~occ, return_indices=True)
    return np.stack(inds, axis=-1)
