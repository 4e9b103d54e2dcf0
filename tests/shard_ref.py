"""Reference for the sharded scoring step on tiny graphs -- test infrastructure.

Restates twc_score_shard's contract in plain numpy: the degree orientation u -> v iff
(deg u, u) < (deg v, v) (reading C9), the pivot ranges (rank r of P owns the vertices
whose oriented lists start in [r m / P, (r+1) m / P)), and, by brute force over all vertex
triples, each triangle credited to its lowest-key vertex's rank on its three edges.
"""
import numpy as np


def pivot_ranges(g, world):
    n, m = g.n, g.m
    deg = np.diff(g.rowptr.astype(np.int64))
    src = np.repeat(np.arange(n), deg)
    dst = g.colidx.astype(np.int64)
    out = (deg[src] < deg[dst]) | ((deg[src] == deg[dst]) & (src < dst))
    dplus = np.bincount(src[out], minlength=n)
    rp_or = np.concatenate([[0], np.cumsum(dplus)])
    bounds = []
    for r in range(world + 1):
        if r == 0:
            bounds.append(0)
        elif r == world:
            bounds.append(n)
        else:
            bounds.append(int(np.searchsorted(rp_or, m * r // world, side="left")))
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def partial_counts(g, world):
    """[world][m] int64: per rank, the triangles of its pivots counted on their three edges."""
    n = g.n
    deg = np.diff(g.rowptr.astype(np.int64))
    A = np.zeros((n, n), dtype=bool)
    A[np.repeat(np.arange(n), deg), g.colidx] = True
    cid = {}
    for u in range(n):
        for v in g.colidx[g.rowptr[u]:g.rowptr[u + 1]]:
            if v > u:
                cid[(u, int(v))] = len(cid)
    ranges = pivot_ranges(g, world)
    owner = np.empty(n, dtype=np.int64)
    for r, (lo, hi) in enumerate(ranges):
        owner[lo:hi] = r
    part = np.zeros((world, g.m), dtype=np.int64)
    for a in range(n):
        for b in range(a + 1, n):
            if not A[a, b]:
                continue
            for c in range(b + 1, n):
                if A[a, c] and A[b, c]:
                    p = min((a, b, c), key=lambda x: (deg[x], x))
                    r = owner[p]
                    part[r, cid[(a, b)]] += 1
                    part[r, cid[(a, c)]] += 1
                    part[r, cid[(b, c)]] += 1
    return part
