"""Seeded synthetic graph generators shared by the oracle tests, the CUDA tests and bench.py.

This module holds NO arithmetic of the method: it never counts triangles or wedges, never
scores, thresholds or labels anything.  It only samples random graphs and assembles the
input CSR that the paper's method takes as given -- "we first sort the adjacency list by
node id" (Sec. 3.3): symmetric CSR, rows strictly
increasing, no self-loops, no duplicate edges.

All randomness is numpy PCG64 (`numpy.random.default_rng(seed)`); every generator is a
pure function of its arguments.  The recipes (and why they stand in for the paper's
workloads) are in DESIGN.md Sec. "Input recipe".
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Graph", "csr_from_pairs", "complete", "path", "cycle", "star", "complete_bipartite",
    "wheel", "bridge_triangles", "empty", "erdos_renyi", "two_block_sbm", "planted_partition",
    "dc_sbm", "rmat", "config_graph", "CONFIGS", "relabel",
]


@dataclass
class Graph:
    """Undirected simple graph in CSR form (SPEC S:23-33 layout).

    rowptr: (n+1,) int32 or int64; colidx: (2m,) int32; rows strictly increasing.
    """
    n: int
    rowptr: np.ndarray
    colidx: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.rowptr[-1]) // 2 if self.n > 0 else 0

    def with_rowptr_dtype(self, dt) -> "Graph":
        return Graph(self.n, self.rowptr.astype(dt), self.colidx, dict(self.meta))

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.int64(self.n).tobytes())
        h.update(np.ascontiguousarray(self.rowptr.astype(np.int64)).tobytes())
        h.update(np.ascontiguousarray(self.colidx).tobytes())
        return h.hexdigest()

    def canonical_pairs(self):
        """(u, v) with u < v in lexicographic order -- SPEC S:66-69 edge enumeration.

        Pure CSR bookkeeping (which slots are the upper triangle), used by tests only.
        """
        deg = np.diff(self.rowptr.astype(np.int64))
        src = np.repeat(np.arange(self.n, dtype=np.int64), deg)
        dst = self.colidx.astype(np.int64)
        up = dst > src
        return src[up], dst[up]


def _sorted_unique(x):
    x = np.sort(x)
    if x.size == 0:
        return x
    keep = np.empty(x.size, dtype=bool)
    keep[0] = True
    np.not_equal(x[1:], x[:-1], out=keep[1:])
    return x[keep]


def csr_from_pairs(n: int, a, b, rowptr_dtype=np.int32, meta=None) -> Graph:
    """Symmetric CSR from an undirected pair list: drops self-loops, collapses duplicates,
    sorts every row (P:618 pre-processing; SPEC S:46-49 load semantics)."""
    a = np.asarray(a, dtype=np.int64).ravel()
    b = np.asarray(b, dtype=np.int64).ravel()
    if n < 0 or n >= 2**31:
        raise ValueError("n out of range")
    keep = a != b
    lo = np.minimum(a, b)[keep]
    hi = np.maximum(a, b)[keep]
    if lo.size and (lo.min() < 0 or hi.max() >= n):
        raise ValueError("vertex id out of range")
    key = _sorted_unique(lo * np.int64(max(n, 1)) + hi)     # sorted by (lo, hi), unique
    lo = key // max(n, 1)
    hi = key - lo * max(n, 1)
    m = key.size
    deg_up = np.bincount(lo, minlength=n).astype(np.int64)  # entries v > u in row u
    deg_lo = np.bincount(hi, minlength=n).astype(np.int64)  # entries v < u in row u
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg_up + deg_lo, out=rowptr[1:])
    colidx = np.empty(2 * m, dtype=np.int32)
    # upper entries of row u: already ordered by (lo, hi)
    up_start = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg_up, out=up_start[1:])
    rank = np.arange(m, dtype=np.int64) - up_start[lo]
    colidx[rowptr[lo] + deg_lo[lo] + rank] = hi
    # lower entries of row u: the pairs (hi=u, lo) ordered by (hi, lo)
    rkey = np.sort(hi * np.int64(max(n, 1)) + lo)
    hs = rkey // max(n, 1)
    ls = rkey - hs * max(n, 1)
    del rkey
    lo_start = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg_lo, out=lo_start[1:])
    rank = np.arange(m, dtype=np.int64) - lo_start[hs]
    colidx[rowptr[hs] + rank] = ls
    if rowptr_dtype == np.int32 and 2 * m >= 2**31:
        raise ValueError("2m does not fit int32 rowptr")
    return Graph(n, rowptr.astype(rowptr_dtype), colidx, dict(meta or {}))


def relabel(g: Graph, perm: np.ndarray) -> Graph:
    """Graph with vertex u renamed perm[u] (relabelling-invariance pins)."""
    s, d = g.canonical_pairs()
    return csr_from_pairs(g.n, perm[s], perm[d], g.rowptr.dtype.type, g.meta)


# ---------------------------------------------------------------------------------------
# Closed-form families (SURVEY 8(c) pins).  Pure pair lists.
# ---------------------------------------------------------------------------------------

def empty(n: int) -> Graph:
    return csr_from_pairs(n, [], [])


def complete(n: int, rowptr_dtype=np.int32) -> Graph:
    a, b = np.triu_indices(n, 1)
    return csr_from_pairs(n, a, b, rowptr_dtype)


def path(n: int) -> Graph:
    a = np.arange(n - 1)
    return csr_from_pairs(n, a, a + 1)


def cycle(n: int) -> Graph:
    a = np.arange(n)
    return csr_from_pairs(n, a, (a + 1) % n)


def star(k: int, center: int = 0, rowptr_dtype=np.int32) -> Graph:
    """K_{1,k}; the hub gets id `center`, leaves the other ids."""
    ids = np.array([i for i in range(k + 1) if i != center], dtype=np.int64)
    return csr_from_pairs(k + 1, np.full(k, center), ids, rowptr_dtype)


def complete_bipartite(a: int, b: int, rowptr_dtype=np.int32) -> Graph:
    x, y = np.meshgrid(np.arange(a), np.arange(a, a + b), indexing="ij")
    return csr_from_pairs(a + b, x.ravel(), y.ravel(), rowptr_dtype)


def wheel(k: int) -> Graph:
    """Hub 0 joined to a rim cycle 1..k."""
    rim = np.arange(1, k + 1)
    a = np.concatenate([np.zeros(k, np.int64), rim])
    b = np.concatenate([rim, (rim % k) + 1])
    return csr_from_pairs(k + 1, a, b)


def bridge_triangles() -> Graph:
    """Triangles {0,1,2} and {3,4,5} joined by the bridge (2,3)."""
    a = [0, 0, 1, 3, 3, 4, 2]
    b = [1, 2, 2, 4, 5, 5, 3]
    return csr_from_pairs(6, a, b)


# ---------------------------------------------------------------------------------------
# Random families.
# ---------------------------------------------------------------------------------------

def erdos_renyi(n: int, p: float, seed: int) -> Graph:
    """G(n, p) by one Bernoulli draw per vertex pair: O(n^2) memory, so small n only."""
    if n > 20_000:
        raise ValueError("erdos_renyi enumerates all pairs; use gnm() for large n")
    rng = np.random.default_rng(seed)
    a, b = np.triu_indices(n, 1)
    keep = rng.random(a.size) < p
    return csr_from_pairs(n, a[keep], b[keep], meta={"kind": "er", "n": n, "p": p, "seed": seed})


def gnm(n: int, m: int, seed: int, rowptr_dtype=np.int32) -> Graph:
    """Sparse uniform random graph for large n: m uniformly drawn vertex pairs, loops and
    duplicates dropped (so the realised m is slightly below the request)."""
    rng = np.random.default_rng(seed)
    a = rng.integers(0, n, size=m, dtype=np.int64)
    b = rng.integers(0, n, size=m, dtype=np.int64)
    keep = a != b
    return csr_from_pairs(n, a[keep], b[keep], rowptr_dtype=rowptr_dtype,
                          meta={"kind": "gnm", "n": n, "m": m, "seed": seed})


def two_block_sbm(n: int, p1: float, p2: float, q: float, seed: int) -> Graph:
    """Inhomogeneous 2-block SBM of P:509 (B1 = ids 0..n-1 with p1, B2 = n..2n-1 with p2,
    across q); the Fig. 3 setting is n=50 per block, p1=.1, p2=.8, q=.05 (reading C14)."""
    rng = np.random.default_rng(seed)
    a, b = np.triu_indices(2 * n, 1)
    blk_a, blk_b = a >= n, b >= n
    prob = np.where(blk_a != blk_b, q, np.where(blk_a, p2, p1))
    keep = rng.random(a.size) < prob
    return csr_from_pairs(2 * n, a[keep], b[keep],
                          meta={"kind": "sbm2", "n": n, "p1": p1, "p2": p2, "q": q, "seed": seed})


def planted_partition(n_blocks: int, s: int, p_in: float, p_out: float, seed: int,
                      rowptr_dtype=np.int32) -> Graph:
    """Planted-partition SBM: blocks are contiguous id ranges [b*s, (b+1)*s).

    Intra-block: one Bernoulli(p_in) per pair.  Inter-block: M ~ Binomial(N_out, p_out)
    distinct pairs drawn uniformly by rejection -- exactly the SBM law."""
    rng = np.random.default_rng(seed)
    n = n_blocks * s
    ta, tb = np.triu_indices(s, 1)
    keep = rng.random((n_blocks, ta.size)) < p_in
    blk, pidx = np.nonzero(keep)
    ia = blk * s + ta[pidx]
    ib = blk * s + tb[pidx]
    n_out = n * (n - 1) // 2 - n_blocks * (s * (s - 1) // 2)
    M = int(rng.binomial(n_out, p_out)) if n_out > 0 else 0
    got = np.empty(0, dtype=np.int64)
    while got.size < M:
        need = M - got.size
        k = int(need * 1.1) + 16
        u = rng.integers(0, n, size=k)
        v = rng.integers(0, n, size=k)
        ok = (u // s) != (v // s)
        lo, hi = np.minimum(u[ok], v[ok]), np.maximum(u[ok], v[ok])
        keys = lo * n + hi
        # keep first occurrences in draw order (deterministic), then de-duplicate globally
        keys = np.concatenate([got, keys])
        _, first = np.unique(keys, return_index=True)
        got = keys[np.sort(first)][:M]
    oa, ob = got // n, got % n
    return csr_from_pairs(n, np.concatenate([ia, oa]), np.concatenate([ib, ob]), rowptr_dtype,
                          meta={"kind": "pp", "blocks": n_blocks, "s": s, "p_in": p_in,
                                "p_out": p_out, "seed": seed})


def _powerlaw_mean(tmin, tmax, g):
    a, b = 1.0 - g, 2.0 - g
    return (a / b) * (tmax ** b - tmin ** b) / (tmax ** a - tmin ** a)


def _solve_theta_min(target_mean, tmax, g):
    lo, hi = 1e-6, target_mean
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if _powerlaw_mean(mid, tmax, g) < target_mean:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _block_sizes(rng, n, smin, smax, expo):
    vals = np.arange(smin, smax + 1, dtype=np.int64)
    p = vals.astype(np.float64) ** (-expo)
    p /= p.sum()
    mean = float((vals * p).sum())
    draw = rng.choice(vals, size=int(1.5 * n / mean) + 64, p=p)
    cs = np.cumsum(draw)
    k = int(np.searchsorted(cs, n, side="left"))  # cs[k] >= n
    sizes = draw[:k].tolist()
    rem = n - (int(cs[k - 1]) if k > 0 else 0)
    if rem >= smin or not sizes:
        sizes.append(rem)
    else:
        sizes[-1] += rem
    return np.asarray(sizes, dtype=np.int64)


def dc_sbm(n: int, m_target: int, gamma: float, theta_max: float, smin: int, smax: int,
           mu: float, seed: int, eps: float = 0.0, block_exp: float = 1.5,
           rowptr_dtype=np.int32) -> Graph:
    """Degree-corrected SBM (SURVEY 8(d) "DC-SBM").

    Block sizes i.i.d. from P(s) ~ s^-block_exp on [smin, smax] until they cover n; blocks
    placed on a seeded random permutation of ids.  Vertex weights theta: continuous power law
    with exponent gamma on [theta_min, theta_max], theta_min solved so mean(theta) = 2m/n.
    round(mu*m*(1+eps)) intra draws (u ~ theta globally, v ~ theta inside block(u)) and
    round((1-mu)*m*(1+eps)) inter draws (u, v ~ theta, redrawn while in the same block);
    self-loops dropped and duplicates collapsed by csr_from_pairs.  eps and theta_max are
    calibrated per config (graphgen/calibrate.py) so the realised m / d_max hit the targets.
    """
    rng = np.random.default_rng(seed)
    sizes = _block_sizes(rng, n, smin, smax, block_exp)
    nb = sizes.size
    # position in block-sorted order -> vertex id
    perm = rng.permutation(n).astype(np.int64)
    blk_sorted = np.repeat(np.arange(nb, dtype=np.int64), sizes)
    bstart = np.zeros(nb + 1, dtype=np.int64)
    np.cumsum(sizes, out=bstart[1:])
    tmin = _solve_theta_min(2.0 * m_target / n, theta_max, gamma)
    a = 1.0 - gamma
    U = rng.random(n)
    theta = (tmin ** a + U * (theta_max ** a - tmin ** a)) ** (1.0 / a)
    cum = np.cumsum(theta)
    total = cum[-1]
    cum_b = np.concatenate([[0.0], cum])[bstart]          # cumulative weight at block starts
    mi = int(round(mu * m_target * (1.0 + eps)))
    mo = int(round((1.0 - mu) * m_target * (1.0 + eps)))

    def draw_global(k, shuffle):
        # sorted uniforms make the binary searches cache-friendly; a random shuffle of the
        # sorted sample restores an i.i.d. sequence where the pairing matters
        r = np.sort(rng.random(k)) * total
        idx = np.minimum(np.searchsorted(cum, r, side="right"), n - 1)
        return rng.permutation(idx) if shuffle else idx

    # intra-block
    u = draw_global(mi, False)
    bu = blk_sorted[u]
    lo_w, hi_w = cum_b[bu], cum_b[bu + 1]
    v = np.searchsorted(cum, lo_w + rng.random(mi) * (hi_w - lo_w), side="right")
    v = np.clip(v, bstart[bu], bstart[bu + 1] - 1)
    # inter-block, rejection on same block
    ou = np.empty(0, dtype=np.int64)
    ov = np.empty(0, dtype=np.int64)
    while ou.size < mo:
        k = mo - ou.size
        x, y = draw_global(k, False), draw_global(k, True)
        ok = blk_sorted[x] != blk_sorted[y]
        ou = np.concatenate([ou, x[ok]])
        ov = np.concatenate([ov, y[ok]])
        if nb == 1:
            break
    A = perm[np.concatenate([u, ou])]
    B = perm[np.concatenate([v, ov])]
    block_of = np.empty(n, dtype=np.int64)
    block_of[perm] = blk_sorted
    meta = {"kind": "dcsbm", "n": n, "m_target": m_target, "gamma": gamma, "theta_max": theta_max,
            "smin": smin, "smax": smax, "mu": mu, "seed": seed, "eps": eps, "blocks": int(nb)}
    g = csr_from_pairs(n, A, B, rowptr_dtype, meta)
    g.meta["block_of"] = block_of
    return g


def rmat(scale: int, m_req: int, seed: int, a=(0.45, 0.15, 0.15, 0.25),
         rowptr_dtype=np.int32, n: int | None = None, chunk: int = 1 << 24) -> Graph:
    """R-MAT (Chakrabarti et al.) with the paper's static seed matrix a = (a11, a12, a21, a22)
    = (0.45, 0.15, 0.15, 0.25), no noise.  Each of the m_req draws descends `scale`
    levels of the 2x2 recursion (one uniform per level picks the quadrant).  With n given
    (n <= 2^scale), draws with an endpoint >= n are redrawn, so ids cover exactly [0, n)
    (reading N3).  Self-loops and duplicate pairs are then dropped, so the realised
    m is at most m_req.  Draws are generated in chunks to bound memory."""
    rng = np.random.default_rng(seed)
    nv = (1 << scale) if n is None else int(n)
    if nv > (1 << scale):
        raise ValueError("n exceeds 2^scale")
    c1, c2, c3 = np.cumsum(np.asarray(a, dtype=np.float64))[:3]
    us, vs, got = [], [], 0
    while got < m_req:
        k = min(chunk, m_req - got)
        u = np.zeros(k, dtype=np.int64)
        v = np.zeros(k, dtype=np.int64)
        for lvl in range(scale):
            r = rng.random(k)
            q = (r >= c1).astype(np.int64) + (r >= c2) + (r >= c3)  # quadrant 0..3
            u |= (q >> 1) << lvl
            v |= (q & 1) << lvl
        if n is not None:
            ok = (u < nv) & (v < nv)
            u, v = u[ok], v[ok]
        us.append(u)
        vs.append(v)
        got += u.size
    return csr_from_pairs(nv, np.concatenate(us), np.concatenate(vs), rowptr_dtype,
                          meta={"kind": "rmat", "scale": scale, "n": nv, "m_req": m_req,
                                "seed": seed, "a": tuple(a)})


# R-MAT workloads of Table "tab:syn": densities very sparse
# m = 5n, sparse m = 50n, dense m = n^1.5, at 10^7 and 10^8 requested edges.  n is the paper's
# (rounded as printed; the dense n = m^(2/3)); the R-MAT scale is the smallest with 2^scale >= n.
RMAT_CONFIGS = {
    "vs-1e7": dict(n=2_000_000, m=10_000_000, paper_tw_s=1.77),
    "vs-1e8": dict(n=20_000_000, m=100_000_000, paper_tw_s=20.05),
    "s-1e7": dict(n=200_000, m=10_000_000, paper_tw_s=4.96),
    "s-1e8": dict(n=2_000_000, m=100_000_000, paper_tw_s=71.06),
    "d-1e7": dict(n=46_416, m=10_000_000, paper_tw_s=13.91),
    "d-1e8": dict(n=215_443, m=100_000_000, paper_tw_s=378.11),
}


def rmat_graph(name: str, seed: int = 11) -> Graph:
    c = RMAT_CONFIGS[name]
    n, m = c["n"], c["m"]
    scale = max(1, int(np.ceil(np.log2(n))))
    rp = np.int64 if 2 * m >= (1 << 31) else np.int32
    g = rmat(scale, m, seed, n=n, rowptr_dtype=rp)
    g.meta["config"] = "rmat-" + name
    return g


# ---------------------------------------------------------------------------------------
# BASELINE.json configs.  DC-SBM eps / theta_max come from calibrate.py.
# ---------------------------------------------------------------------------------------

CONFIGS = {
    1: dict(kind="pp", n_blocks=4, s=250, p_in=0.10, p_out=0.005, seed=0, rowptr=np.int32),
    2: dict(kind="pp", n_blocks=1000, s=100, p_in=0.06, p_out=2e-5, seed=1, rowptr=np.int32),
    3: dict(kind="dcsbm", n=335_000, m_target=925_000, gamma=2.5, theta_max=1400.451, smin=10,
            smax=500, mu=0.80, seed=2, eps=0.192600, rowptr=np.int32),
    4: dict(kind="dcsbm", n=1_130_000, m_target=3_000_000, gamma=2.1, theta_max=141070.427,
            smin=10, smax=3000, mu=0.70, seed=3, eps=0.529908, rowptr=np.int32),
    5: dict(kind="dcsbm", n=4_000_000, m_target=35_000_000, gamma=2.3, theta_max=38876.186,
            smin=20, smax=5000, mu=0.75, seed=4, eps=0.267084, rowptr=np.int64),
}


MANIFEST = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                        "golden", "graph_manifest.json")


def manifest() -> dict:
    """Realised statistics of the five workloads (scripts/make_manifest.py), keyed "1".."5"."""
    with open(MANIFEST) as f:
        return json.load(f)


def config_graph(k: int) -> Graph:
    """BASELINE.json workload k.  With TWC_GRAPH_CACHE=<dir> set, the CSR bytes are cached there
    as config<k>.npz and reused only when their sha256 equals the manifest's (numpy does not
    promise identical random streams across versions, SURVEY 8(d) "Conventions")."""
    cache = os.environ.get("TWC_GRAPH_CACHE")
    if cache:
        path = os.path.join(cache, f"config{k}.npz")
        want = manifest().get(str(k), {}).get("sha256")
        if os.path.exists(path):
            z = np.load(path)
            g = Graph(int(z["n"]), z["rowptr"], z["colidx"], {"config": k})
            if "block_of" in z:
                g.meta["block_of"] = z["block_of"]
            if g.sha256() == want:
                return g
        g = _generate_config(k)
        if g.sha256() == want:
            os.makedirs(cache, exist_ok=True)
            extra = {"block_of": g.meta["block_of"]} if "block_of" in g.meta else {}
            np.savez(path + ".tmp.npz", n=g.n, rowptr=g.rowptr, colidx=g.colidx, **extra)
            os.replace(path + ".tmp.npz", path)
        return g
    return _generate_config(k)


def _generate_config(k: int) -> Graph:
    c = dict(CONFIGS[k])
    kind = c.pop("kind")
    rp = c.pop("rowptr")
    if kind == "pp":
        g = planted_partition(c["n_blocks"], c["s"], c["p_in"], c["p_out"], c["seed"], rp)
    else:
        g = dc_sbm(c["n"], c["m_target"], c["gamma"], c["theta_max"], c["smin"], c["smax"],
                   c["mu"], c["seed"], eps=c["eps"], rowptr_dtype=rp)
    g.meta["config"] = k
    return g
