"""Brute-force motif enumeration on tiny graphs -- an independent pin for the oracle.

Works on a dense adjacency matrix and enumerates, for each edge (u,v), every third vertex w:
  * w adjacent to both u and v  -> the edge sits in the triangle {u,v,w}       (t,     P:337)
  * w adjacent to exactly one   -> the edge sits in an open wedge (path of 2) (wedge, P:337,
                                   reading C20: |N(u) u N(v)| - |N(u) n N(v)| - 2 counts
                                   exactly these w, the "-2" removing u and v themselves)
This is the motif-participation meaning of the definitions, O(n^3) total, not the set formula.
"""
import numpy as np


def adjacency(g):
    A = np.zeros((g.n, g.n), dtype=np.int64)
    deg = np.diff(g.rowptr.astype(np.int64))
    src = np.repeat(np.arange(g.n), deg)
    A[src, g.colidx] = 1
    return A


def edge_motifs(g):
    A = adjacency(g)
    out = {}
    for u in range(g.n):
        for v in range(u + 1, g.n):
            if not A[u, v]:
                continue
            tri = 0
            wed = 0
            for w in range(g.n):
                if w == u or w == v:
                    continue
                a, b = A[u, w], A[v, w]
                if a and b:
                    tri += 1
                elif a or b:
                    wed += 1
            out[(u, v)] = (tri, wed)
    return out


def triangles_total(g):
    A = adjacency(g)
    return int(np.trace(A @ A @ A)) // 6


def components_bfs(n, pairs):
    """Plain BFS labelling with min-id labels."""
    adj = [[] for _ in range(n)]
    for a, b in pairs:
        adj[a].append(b)
        adj[b].append(a)
    lab = [-1] * n
    for s in range(n):
        if lab[s] >= 0:
            continue
        lab[s] = s
        stack = [s]
        while stack:
            x = stack.pop()
            for y in adj[x]:
                if lab[y] < 0:
                    lab[y] = s
                    stack.append(y)
    return np.asarray(lab, dtype=np.int32)


def edge_k4(g):
    """4-cliques per edge by enumerating every 4-subset of vertices (tiny graphs only)."""
    import itertools
    A = adjacency(g)
    out = {}
    for u in range(g.n):
        for v in range(u + 1, g.n):
            if A[u, v]:
                out[(u, v)] = 0
    for q in itertools.combinations(range(g.n), 4):
        if all(A[a, b] for a, b in itertools.combinations(q, 2)):
            for a, b in itertools.combinations(q, 2):
                out[(a, b)] += 1
    return out
