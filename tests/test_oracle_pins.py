"""Pins for the CPU oracle (oracle/), against things other than the oracle itself.

Each test names what pins it: brute-force motif enumeration (tests/brute.py), closed forms
(all derivable by hand from P:337 and Eq. 2), global invariants checked with
networkx / scipy, the worked examples in tests/golden/, relabelling invariance, and the
paper's expectation table by Monte Carlo with graph-level standard errors.
"""
import json
import math
import os

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

import brute
import graphgen as gg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def by_pair(g, arr):
    s, d = g.canonical_pairs()
    return {(int(a), int(b)): int(x) for a, b, x in zip(s, d, arr)}


def degrees(g):
    return np.diff(g.rowptr.astype(np.int64))


def canon_labels(lab):
    """Relabel an arbitrary component id vector to min-vertex-id labels."""
    lab = np.asarray(lab)
    k = lab.max() + 1 if lab.size else 0
    mins = np.full(k, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(mins, lab, np.arange(lab.size))
    return mins[lab].astype(np.int32)


def scipy_labels(g, tw, delta):
    s, d = g.canonical_pairs()
    keep = ~(tw.astype(np.float64) < delta)
    A = sp.coo_matrix((np.ones(int(keep.sum())), (s[keep], d[keep])), shape=(g.n, g.n))
    _, lab = connected_components(A, directed=False)
    return canon_labels(lab), int(keep.sum())


# ------------------------------------------------------------------ brute force

@pytest.mark.parametrize("p", [0.05, 0.1, 0.3])
def test_score_equals_brute_force_er60(oracle_mod, p):
    for seed in range(17):          # 3 x 17 = 51 graphs, n = 60 (SPEC acceptance #1)
        g = gg.erdos_renyi(60, p, seed=1000 * seed + int(p * 100))
        t, wedge, tw = oracle_mod.score(g)
        bf = brute.edge_motifs(g)
        s, d = g.canonical_pairs()
        assert len(bf) == g.m == t.size
        for i, (a, b) in enumerate(zip(s, d)):
            bt, bw = bf[(int(a), int(b))]
            assert (t[i], wedge[i], tw[i]) == (bt, bw, bt - bw), (seed, a, b)


def test_score_equals_brute_force_small_random(oracle_mod):
    rng = np.random.default_rng(7)
    for it in range(200):
        n = int(rng.integers(1, 41))
        p = float(rng.random())
        g = gg.erdos_renyi(n, p, seed=it)
        t, wedge, tw = oracle_mod.score(g)
        bf = brute.edge_motifs(g)
        s, d = g.canonical_pairs()
        got = {(int(a), int(b)): (int(x), int(y)) for a, b, x, y in zip(s, d, t, wedge)}
        assert got == bf
        assert np.array_equal(tw, t - wedge)


# ------------------------------------------------------------------ closed forms

def _all_equal(oracle_mod, g, expect_fn):
    t, wedge, tw = oracle_mod.score(g)
    s, d = g.canonical_pairs()
    for i, (a, b) in enumerate(zip(s, d)):
        assert (t[i], wedge[i], tw[i]) == expect_fn(int(a), int(b)), (a, b)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 60])
def test_complete_graph(oracle_mod, n):
    _all_equal(oracle_mod, gg.complete(n), lambda a, b: (n - 2, 0, n - 2))


@pytest.mark.parametrize("n", [2, 3, 5, 9])
def test_path(oracle_mod, n):
    g = gg.path(n)
    deg = degrees(g)
    _all_equal(oracle_mod, g, lambda a, b: (0, deg[a] + deg[b] - 2, 2 - deg[a] - deg[b]))


@pytest.mark.parametrize("n", [4, 5, 8, 31])
def test_cycle(oracle_mod, n):
    _all_equal(oracle_mod, gg.cycle(n), lambda a, b: (0, 2, -2))


def test_triangle_is_k3(oracle_mod):
    _all_equal(oracle_mod, gg.cycle(3), lambda a, b: (1, 0, 1))


@pytest.mark.parametrize("k,center", [(1, 0), (3, 0), (6, 3), (50, 50)])
def test_star(oracle_mod, k, center):
    _all_equal(oracle_mod, gg.star(k, center), lambda a, b: (0, k - 1, 1 - k))


@pytest.mark.parametrize("a,b", [(1, 1), (2, 3), (3, 3), (4, 2), (5, 9)])
def test_complete_bipartite(oracle_mod, a, b):
    _all_equal(oracle_mod, gg.complete_bipartite(a, b),
               lambda x, y: (0, a + b - 2, 2 - a - b))


@pytest.mark.parametrize("k", [4, 5, 8, 20])
def test_wheel(oracle_mod, k):
    # spoke (hub 0, rim r): (2, k-3, 5-k); rim edge: (1, 2, -1)
    _all_equal(oracle_mod, gg.wheel(k),
               lambda a, b: (2, k - 3, 5 - k) if a == 0 else (1, 2, -1))


def test_bridge_graph(oracle_mod):
    g = gg.bridge_triangles()
    t, wedge, tw = oracle_mod.score(g)
    got = {k: v for k, v in zip(zip(*[x.tolist() for x in g.canonical_pairs()]),
                                 zip(t.tolist(), wedge.tolist(), tw.tolist()))}
    assert got[(2, 3)] == (0, 4, -4)
    for e in [(0, 2), (1, 2), (3, 4), (3, 5)]:
        assert got[e] == (1, 1, 0)
    for e in [(0, 1), (4, 5)]:
        assert got[e] == (1, 0, 1)


def test_degenerate_inputs(oracle_mod):
    for n in [0, 1, 5]:
        g = gg.empty(n)
        t, w, tw = oracle_mod.score(g)
        assert t.size == 0
        lab, kept, ncomp = oracle_mod.cluster(g, tw, 0.0)
        assert kept == 0 and ncomp == n and np.array_equal(lab, np.arange(n))
    g = gg.path(2)                                  # single edge
    t, w, tw = oracle_mod.score(g)
    assert (t.tolist(), w.tolist(), tw.tolist()) == ([0], [0], [0])


# ------------------------------------------------------------------ golden worked examples

def test_golden_score_examples(oracle_mod):
    gold = json.load(open(GOLDEN))
    for case in gold["score"]:
        e = np.array(case["edges"]).reshape(-1, 2)
        g = gg.csr_from_pairs(case["n"], e[:, 0], e[:, 1])
        t, w, tw = oracle_mod.score(g)
        T, W, TW = by_pair(g, t), by_pair(g, w), by_pair(g, tw)
        for key, ex in case["expect"].items():
            a, b = map(int, key.split("-"))
            assert (T[(a, b)], W[(a, b)], TW[(a, b)]) == (ex["t"], ex["wedge"], ex["tw"]), case["cite"]


def test_golden_cluster_examples(oracle_mod):
    gold = json.load(open(GOLDEN))
    for case in gold["cluster"]:
        e = np.array(case["edges"], dtype=np.int64).reshape(-1, 2)
        g = gg.csr_from_pairs(case["n"], e[:, 0], e[:, 1])
        _, _, tw = oracle_mod.score(g)
        delta = float(case["delta"])
        lab, kept, _ = oracle_mod.cluster(g, tw, delta)
        assert kept == case["kept"], case["cite"]
        assert lab.tolist() == case["labels"], case["cite"]


# ------------------------------------------------------------------ invariants + libraries

def _check_invariants(oracle_mod, g, check_matrix=True):
    t, wedge, tw = oracle_mod.score(g)
    deg = degrees(g)
    s, d = g.canonical_pairs()
    G = nx.Graph()
    G.add_nodes_from(range(g.n))
    G.add_edges_from(zip(s.tolist(), d.tolist()))
    T = sum(nx.triangles(G).values()) // 3
    W = int((deg * (deg - 1) // 2).sum())
    assert int(t.sum()) == 3 * T                                   # sum t = 3T
    assert int(wedge.sum()) == int((deg ** 2).sum()) - 2 * g.m - 6 * T
    assert int(tw.sum()) == 9 * T - 2 * W
    assert np.array_equal(wedge, deg[s] + deg[d] - 2 * t - 2)      # union counted directly
    assert (t >= 0).all() and (t <= np.minimum(deg[s], deg[d]) - 1).all()
    assert (wedge >= 0).all() and (wedge <= deg[s] + deg[d] - 2).all()
    if check_matrix and g.m:                                       # t(u,v) = (A^2)_uv
        A = sp.csr_matrix((np.ones(g.colidx.size), g.colidx.astype(np.int64),
                           g.rowptr.astype(np.int64)), shape=(g.n, g.n))
        A2 = (A @ A).tocsr()
        assert np.array_equal(np.asarray(A2[s, d]).ravel().astype(np.int64), t.astype(np.int64))


def test_invariants_random(oracle_mod):
    for seed in range(30):
        rng = np.random.default_rng(seed)
        g = gg.erdos_renyi(int(rng.integers(5, 120)), float(rng.random() * 0.4), seed)
        _check_invariants(oracle_mod, g)


@pytest.mark.parametrize("k", [1, 2])
def test_invariants_configs(oracle_mod, k):
    _check_invariants(oracle_mod, gg.config_graph(k))


def test_invariants_config3(oracle_mod):
    _check_invariants(oracle_mod, gg.config_graph(3))


def test_relabel_invariance(oracle_mod):
    for seed in range(10):
        g = gg.erdos_renyi(80, 0.15, seed)
        perm = np.random.default_rng(100 + seed).permutation(g.n)
        h = gg.relabel(g, perm)
        t1, w1, tw1 = oracle_mod.score(g)
        t2, w2, tw2 = oracle_mod.score(h)
        m2 = by_pair(h, t2), by_pair(h, w2), by_pair(h, tw2)
        s, d = g.canonical_pairs()
        for i, (a, b) in enumerate(zip(s, d)):
            key = tuple(sorted((int(perm[a]), int(perm[b]))))
            assert (t1[i], w1[i], tw1[i]) == (m2[0][key], m2[1][key], m2[2][key])


def test_row_range_scoring_matches_full(oracle_mod):
    g = gg.config_graph(1)
    full = oracle_mod.score(g)
    part = [np.zeros_like(x) for x in full]
    for r0 in range(0, g.n, 137):
        seg = oracle_mod.score(g, rows=(r0, min(g.n, r0 + 137)))
        for acc, x in zip(part, seg):
            acc += x
    for a, b in zip(full, part):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ statistical

def _class_means(g, t, tw, block):
    s, d = g.canonical_pairs()
    deg = degrees(g)
    inside = block[s] == block[d]
    dsum = deg[s] + deg[d]
    return {cls: (t[mask].mean(), dsum[mask].mean(), tw[mask].mean())
            for cls, mask in (("in", inside), ("out", ~inside))}


def test_planted_partition_class_means(oracle_mod):
    """K blocks of s, n=Ks: inside E[t]=(s-2)p^2+(n-s)q^2, E[du+dv]=2+2(s-2)p+2(n-s)q;
    across E[t]=2(s-1)pq+(n-2s)q^2, E[du+dv]=2+2(s-1)p+2(n-s-1)q; E[TW]=3E[t]-E[dsum]+2.
    Graph-level standard errors over 30 seeds (reading C16)."""
    K, s_, p, q = 4, 250, 0.10, 0.005
    n = K * s_
    rows = []
    for seed in range(30):
        g = gg.planted_partition(K, s_, p, q, seed=500 + seed)
        t, _, tw = oracle_mod.score(g)
        block = np.arange(n) // s_
        cm = _class_means(g, t, tw, block)
        rows.append([*cm["in"], *cm["out"]])
    R = np.array(rows)
    mean, se = R.mean(0), R.std(0, ddof=1) / math.sqrt(len(R))
    et_in = (s_ - 2) * p * p + (n - s_) * q * q
    ed_in = 2 + 2 * (s_ - 2) * p + 2 * (n - s_) * q
    et_out = 2 * (s_ - 1) * p * q + (n - 2 * s_) * q * q
    ed_out = 2 + 2 * (s_ - 1) * p + 2 * (n - s_ - 1) * q
    expect = [et_in, ed_in, 3 * et_in - ed_in + 2, et_out, ed_out, 3 * et_out - ed_out + 2]
    z = (mean - np.array(expect)) / se
    assert np.all(np.abs(z) < 4.0), z


def test_two_block_sbm_matches_expectation_table(oracle_mod):
    """Inhomogeneous 2-block SBM.  Monte Carlo per-class means of t, d_u+d_v and TW,
    divided by n, against the paper's table -- the table drops O(1/n) terms
    ("n-2 ~ n"; reading C13), so the check allows |mean/n - table| <= 4 SE/n + 4/n."""
    n, p1, p2, q = 300, 0.1, 0.8, 0.05
    rows = []
    for seed in range(30):
        g = gg.two_block_sbm(n, p1, p2, q, seed=900 + seed)
        t, _, tw = oracle_mod.score(g)
        block = (np.arange(2 * n) >= n).astype(np.int64)
        s, d = g.canonical_pairs()
        deg = degrees(g)
        in1 = (block[s] == 0) & (block[d] == 0)
        acr = block[s] != block[d]
        dsum = deg[s] + deg[d]
        rows.append([t[in1].mean(), dsum[in1].mean(), tw[in1].mean(),
                     t[acr].mean(), dsum[acr].mean(), tw[acr].mean()])
    R = np.array(rows) / n
    mean, se = R.mean(0), R.std(0, ddof=1) / math.sqrt(len(R))
    table = [p1 ** 2 + q ** 2, 2 * (p1 + q), 3 * p1 ** 2 - 2 * p1 + 3 * q ** 2 - 2 * q,
             p1 * q + p2 * q, p1 + p2 + 2 * q, 3 * p1 * q + 3 * p2 * q - p1 - p2 - 2 * q]
    gold = json.load(open(GOLDEN))["expectation_table"][0]
    assert abs(table[2] - gold["inside_tw_over_n"]) < 1e-12
    assert np.all(np.abs(mean - np.array(table)) <= 4 * se + 4.0 / n), (mean, table, se)
    # TW separates the classes in expectation (the Theorem-1 gap is positive)
    gap = n * (p2 - p1) - 3 * n * (p1 * (q - p1) + q * (p2 - q))
    assert gap > 0


# ------------------------------------------------------------------ clustering (Alg. 1)

def test_cluster_matches_scipy_and_bfs(oracle_mod):
    rng = np.random.default_rng(3)
    for it in range(100):                       # SPEC acceptance #5: 100 graphs, n <= 500
        n = int(rng.integers(1, 501))
        p = float(rng.random() * 8.0 / max(n, 1))
        g = gg.erdos_renyi(n, min(p, 1.0), seed=it)
        _, _, tw = oracle_mod.score(g)
        delta = float(rng.integers(-6, 3)) if tw.size else 0.0
        lab, kept, ncomp = oracle_mod.cluster(g, tw, delta)
        ref, kref = scipy_labels(g, tw, delta)
        assert kept == kref
        assert np.array_equal(lab, ref)
        assert ncomp == len(np.unique(ref))
        s, d = g.canonical_pairs()
        keep = ~(tw < delta)
        assert np.array_equal(lab, brute.components_bfs(n, zip(s[keep], d[keep])))
        assert (lab <= np.arange(n)).all() and np.array_equal(lab[lab], lab)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_cluster_configs_match_scipy(oracle_mod, k):
    g = gg.config_graph(k)
    _, _, tw = oracle_mod.score(g)
    for delta in [float(np.median(tw)), float(tw.min()) - 1, float(tw.max()) + 1]:
        lab, kept, _ = oracle_mod.cluster(g, tw, delta)
        ref, kref = scipy_labels(g, tw, delta)
        assert kept == kref and np.array_equal(lab, ref)


def test_cluster_extremes_ties_and_nesting(oracle_mod):
    g = gg.config_graph(1)
    _, _, tw = oracle_mod.score(g)
    lab, kept, _ = oracle_mod.cluster(g, tw, -math.inf)       # keeps everything
    assert kept == g.m
    ref, _ = scipy_labels(g, tw, -math.inf)
    assert np.array_equal(lab, ref)
    lab, kept, ncomp = oracle_mod.cluster(g, tw, math.inf)    # keeps nothing
    assert kept == 0 and ncomp == g.n and np.array_equal(lab, np.arange(g.n))
    v = int(np.median(tw))                                    # equality is kept (reading C4)
    _, kept_eq, _ = oracle_mod.cluster(g, tw, float(v))
    _, kept_gt, _ = oracle_mod.cluster(g, tw, float(v) + 0.5)
    assert kept_eq - kept_gt == int((tw == v).sum())
    prev = None
    for delta in sorted(set(tw.tolist()))[::7]:               # monotone refinement
        lab, _, _ = oracle_mod.cluster(g, tw, float(delta))
        if prev is not None:
            # the partition at the larger delta refines the one at the smaller delta
            for c in np.unique(lab):
                assert len(np.unique(prev[lab == c])) == 1
        prev = lab


def test_cluster_relabel_invariance(oracle_mod):
    g = gg.erdos_renyi(300, 0.02, 11)
    perm = np.random.default_rng(5).permutation(g.n)
    h = gg.relabel(g, perm)
    _, _, tw1 = oracle_mod.score(g)
    _, _, tw2 = oracle_mod.score(h)
    l1, k1, c1 = oracle_mod.cluster(g, tw1, -1.0)
    l2, k2, c2 = oracle_mod.cluster(h, tw2, -1.0)
    assert (k1, c1) == (k2, c2)
    # same partition up to renaming: u~v in g  <=>  perm[u]~perm[v] in h
    same1 = l1[:, None] == l1[None, :]
    same2 = l2[perm][:, None] == l2[perm][None, :]
    assert np.array_equal(same1, same2)


def test_fig3_two_block_recovery(oracle_mod):
    """Fig. 3 setting (reading C14: 50 per block): whenever both blocks are internally
    connected, some TW threshold recovers exactly the two blocks (reading C15)."""
    n, p1, p2, q = 50, 0.1, 0.8, 0.05
    truth = (np.arange(2 * n) >= n).astype(np.int32) * n
    cond = rec = 0
    for seed in range(20):
        g = gg.two_block_sbm(n, p1, p2, q, seed=seed)
        s, d = g.canonical_pairs()
        inb = (s < n) == (d < n)
        A = sp.coo_matrix((np.ones(int(inb.sum())), (s[inb], d[inb])), shape=(2 * n, 2 * n))
        ncc, _ = connected_components(A, directed=False)
        if ncc != 2:
            continue
        cond += 1
        _, _, tw = oracle_mod.score(g)
        ok = False
        for delta in sorted(set(tw.tolist())):
            lab, _, _ = oracle_mod.cluster(g, tw, float(delta))
            if np.array_equal(lab, truth):
                ok = True
                break
        rec += ok
    assert cond >= 10
    assert rec == cond, (rec, cond)


