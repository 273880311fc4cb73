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


def init_guide(origin, vs, occ, ori, counts, seeds, normals, params, near_occ=None):
    """Returns ([(vertices, rooted), ...], report); updates ``counts`` (uint16) in place."""
    origin = np.asarray(origin, np.float64)
    dims = occ.shape
    strict = bool(params.strict)
    near = near_occ if float(params.steer) > 0 else None
    report = {"n_seeds": int(len(seeds)), "n_segments": 0, "n_never_entered": 0}
    if len(seeds) == 0:
        report["warning"] = "no scalp seeds; nothing to trace"
        return [], report
    out = []

    def run(pos, dirs):
        cap = None if strict else (counts >= params.occupancy_cap)
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
