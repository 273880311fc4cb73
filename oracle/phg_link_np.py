"""CPU restatement of the reference's segment linking and scalp attachment -- TEST INFRASTRUCTURE.

Restates (results bit-exact; structure our own):
  compute_links           /root/reference/pkg/src/strandkit/phg.py:337-377
  _smooth / connect_segments                                     :380-413
  attach_to_scalp                                                :419-439
  grow (tangents)                                                :445-469
  geom.resample_polyline_uniform / polyline_lengths / polyline_tangents  geom.py:57-103
Candidate pairs come from an exact O(n^2) scan (the reference test's link oracle,
test_phg.py:141-179) instead of a KD-tree; nearest scalp vertex is a brute-force scan with
the reference's (distance, lowest id) tie rule (spatial.py:54-65).  Pinned against
tests/golden/link_*.npz and grow_*.npz.  Only tests/ may import this module.
"""

from __future__ import annotations

import numpy as np

TRACED, FIELD, LINKED, ATTACHED = 0, 1, 2, 3


def _unit(v):
    return v / np.maximum(np.linalg.norm(v, axis=-1, keepdims=True), 1e-12)


def end_tangent(v, window):
    k = min(window, len(v) - 1)
    return _unit(v[-1] - v[-1 - k])


def start_tangent(v, window):
    k = min(window, len(v) - 1)
    return _unit(v[k] - v[0])


def links(segs, link_dist, link_angle_deg, window):
    n = len(segs)
    if n == 0:
        return []
    starts = np.stack([s[0] for s in segs])
    st = np.stack([start_tangent(s, window) for s in segs])
    et = np.stack([end_tangent(s, window) for s in segs])
    gate = np.cos(np.deg2rad(link_angle_deg))
    cand = []
    for i, s in enumerate(segs):
        d = np.linalg.norm(starts - s[-1], axis=1)
        for j in np.flatnonzero(d < link_dist):
            if j != i and np.dot(et[i], st[j]) > gate:
                cand.append((float(d[j]), i, int(j)))
    cand.sort()
    root = list(range(n))

    def find(a):
        while root[a] != a:
            root[a] = root[root[a]]
            a = root[a]
        return a

    has_out, has_in, out = [False] * n, [False] * n, []
    for _, i, j in cand:
        if has_out[i] or has_in[j]:
            continue
        a, b = find(i), find(j)
        if a == b:
            continue
        root[b] = a
        has_out[i] = has_in[j] = True
        out.append((i, j))
    return out


def polyline_lengths(v):
    return np.concatenate([[0.0], np.cumsum(np.linalg.norm(np.diff(v, axis=0), axis=1))])


def resample_uniform(v, step):
    if len(v) < 2:
        return v.copy()
    s = polyline_lengths(v)
    n = max(1, int(round(s[-1] / step)))
    grid = np.linspace(0.0, s[-1], n + 1)
    return np.stack([np.interp(grid, s, v[:, k]) for k in range(3)], axis=1)


def smooth(v, strength, iters):
    v = v.copy()
    for _ in range(iters):
        if len(v) < 3:
            break
        v[1:-1] += strength * (0.5 * (v[:-2] + v[2:]) - v[1:-1])
    return v


def connect(segs, rooted, source, lp):
    """Returns (strands [(vertices, rooted, source)], links)."""
    lk = links(segs, lp["link_dist_mm"], lp["link_angle_deg"], lp["tangent_window"])
    nxt = dict(lk)
    has_prev = {j for _, j in lk}
    out = []
    for i in range(len(segs)):
        if i in has_prev:
            continue
        parts, j = [segs[i]], i
        while j in nxt:
            j = nxt[j]
            parts.append(segs[j])
        merged = len(parts) > 1
        v = np.concatenate(parts) if merged else parts[0]
        if merged and lp["smooth"]:
            v = smooth(v, lp["smooth_strength"], lp["smooth_iters"])
        v = resample_uniform(v, lp["step_mm"])
        if len(v) < 2:
            continue
        out.append((v, bool(rooted[i]), LINKED if merged else int(source[i])))
    return out, lk


def nearest(points, q):
    d = np.linalg.norm(points - q, axis=1)
    dmin = d.min()
    return int(np.flatnonzero(d == dmin).min()), float(dmin)


def attach(strands, scalp_vertices, radius):
    out, unrooted = [], 0
    for v, rooted, src in strands:
        if rooted:
            out.append((v, rooted, src))
            continue
        hid, hd = nearest(scalp_vertices, v[0])
        tid, td = nearest(scalp_vertices, v[-1])
        if min(hd, td) >= radius:
            unrooted += 1
            out.append((v, rooted, src))
        elif td < hd:
            out.append((np.concatenate([[scalp_vertices[tid]], v[::-1]]), True, ATTACHED))
        else:
            out.append((np.concatenate([[scalp_vertices[hid]], v]), True, ATTACHED))
    return out, unrooted


def tangents(v):
    d = _unit(np.diff(v, axis=0))
    return np.concatenate([d, d[-1:]], axis=0)
