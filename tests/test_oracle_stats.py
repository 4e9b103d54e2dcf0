"""Pins for the oracle's sweep statistics and selection rules.

oracle.partition_stats is pinned against: the worked modularity examples of S:290-292
(tests/golden/), the literal double sum of P:350-352 evaluated in exact rational arithmetic
(fractions.Fraction, so the oracle's one-division form must equal its correctly rounded value),
networkx's modularity routine, the closed form Q = 1 - 1/k for k disjoint equal cliques, scipy's
connected components for the component count and size, and label-renaming invariance.
oracle.select is pinned against the synthetic reports of S:371-372 (golden) and hand-built
reports exercising every branch of the rule (reading C22).
"""
import json
import os
from fractions import Fraction

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

import graphgen as gg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def _graph(n, edges):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return gg.csr_from_pairs(n, e[:, 0], e[:, 1])


def literal_q(g, labels):
    """P:350-352 written out: (1/2m) sum over ALL ordered pairs (u, v), u = v included, of
    (A_uv - d_u d_v / 2m) [c_u = c_v], in exact rationals."""
    n = g.n
    m2 = int(g.rowptr[-1])
    A = np.zeros((n, n), dtype=np.int64)
    for u in range(n):
        A[u, g.colidx[g.rowptr[u]:g.rowptr[u + 1]]] = 1
    d = A.sum(1)
    tot = Fraction(0)
    for u in range(n):
        for v in range(n):
            if labels[u] == labels[v]:
                tot += Fraction(int(A[u, v])) - Fraction(int(d[u] * d[v]), m2)
    return tot / m2


def test_golden_modularity_examples(oracle_mod):
    for case in json.load(open(GOLDEN))["modularity"]:
        g = _graph(case["n"], case["edges"])
        nc, largest, intra, sd2, q = oracle_mod.partition_stats(g, np.array(case["labels"]))
        assert q == case["expect_q"], case["cite"]


@pytest.mark.parametrize("seed", range(12))
def test_modularity_equals_literal_double_sum(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 14))
    g = gg.erdos_renyi(n, float(rng.uniform(0.2, 0.8)), seed=seed)
    if g.m == 0:
        return
    labels = rng.integers(0, n, size=n).astype(np.int32)  # arbitrary labels, not canonical
    q = oracle_mod.partition_stats(g, labels)[4]
    assert q == float(literal_q(g, labels))


@pytest.mark.parametrize("seed", range(6))
def test_modularity_matches_networkx(oracle_mod, seed):
    g = gg.erdos_renyi(60, 0.1, seed=seed)
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 5, size=g.n).astype(np.int32)
    G = nx.Graph()
    G.add_nodes_from(range(g.n))
    s, d = g.canonical_pairs()
    G.add_edges_from(zip(s.tolist(), d.tolist()))
    comms = [set(np.flatnonzero(labels == c).tolist()) for c in np.unique(labels)]
    ref = nx.community.modularity(G, comms)
    q = oracle_mod.partition_stats(g, labels)[4]
    assert abs(q - ref) < 1e-12


@pytest.mark.parametrize("k,s", [(2, 3), (3, 4), (5, 6), (7, 2)])
def test_disjoint_cliques_closed_form(oracle_mod, k, s):
    # k disjoint K_s, partition = the cliques: E_in = m, D_c = 2m/k, Q = 1 - 1/k
    a, b = [], []
    for c in range(k):
        for i in range(s):
            for j in range(i + 1, s):
                a.append(c * s + i)
                b.append(c * s + j)
    g = gg.csr_from_pairs(k * s, np.array(a), np.array(b))
    labels = np.repeat(np.arange(k) * s, s).astype(np.int32)
    nc, largest, intra, sd2, q = oracle_mod.partition_stats(g, labels)
    assert (nc, largest, intra) == (k, s, g.m)
    assert sd2 == k * (2 * g.m // k) ** 2
    assert q == float(Fraction(1) - Fraction(1, k))


def test_stats_match_scipy_components(oracle_mod):
    for seed in range(4):
        g = gg.erdos_renyi(300, 0.006, seed=seed)
        t, w, tw = oracle_mod.score(g)
        for delta in (-3.0, -1.0, 0.0, 1.0):
            labels, kept, ncc = oracle_mod.cluster(g, tw, delta)
            nc, largest, intra, sd2, q = oracle_mod.partition_stats(g, labels)
            assert nc == ncc == len(np.unique(labels))
            assert largest == np.bincount(labels).max()
            s, d = g.canonical_pairs()
            assert intra == int(np.sum(labels[s] == labels[d]))
            assert intra >= kept  # every kept edge joins its own component
            deg = np.diff(g.rowptr.astype(np.int64))
            D = np.bincount(labels, weights=deg, minlength=g.n).astype(np.int64)
            assert sd2 == int(np.sum(D * D))
    # the components of the unfiltered graph are scipy's
    g = gg.erdos_renyi(300, 0.006, seed=9)
    A = sp.csr_matrix((np.ones(g.colidx.size), g.colidx, g.rowptr), shape=(g.n, g.n))
    ncc, _ = connected_components(A, directed=False)
    labels, _, _ = oracle_mod.cluster(g, oracle_mod.score(g)[2], -1e18)
    assert oracle_mod.partition_stats(g, labels)[0] == ncc


def test_label_renaming_invariance(oracle_mod):
    g = gg.two_block_sbm(60, 0.1, 0.8, 0.05, seed=3)
    rng = np.random.default_rng(0)
    labels = rng.integers(0, 6, size=g.n).astype(np.int32)
    perm = rng.permutation(g.n).astype(np.int32)
    a = oracle_mod.partition_stats(g, labels)
    b = oracle_mod.partition_stats(g, perm[labels])
    assert a == b


def test_stats_degenerate(oracle_mod):
    g = gg.empty(5)  # m = 0: Q undefined
    nc, largest, intra, sd2, q = oracle_mod.partition_stats(g, np.arange(5))
    assert (nc, largest, intra, sd2) == (5, 1, 0, 0) and np.isnan(q)
    g = gg.complete(4)
    assert oracle_mod.partition_stats(g, np.arange(4))[:4] == (4, 1, 0, 4 * 9)
    with pytest.raises(ValueError):
        oracle_mod.partition_stats(g, np.array([0, 1, 2, 4]))


def test_sweep_extremes_and_refinement(oracle_mod):
    # delta below every score keeps all edges; above every score isolates all vertices.
    # partitions refine as delta grows, so #CC is non-decreasing and largest
    # non-increasing along ascending delta.
    g = gg.planted_partition(6, 30, 0.4, 0.02, seed=1)
    t, w, tw = oracle_mod.score(g)
    deltas = [float(tw.min()) - 1] + list(range(-30, 1, 2)) + [float(tw.max()) + 1]
    pts = oracle_mod.sweep_report(g, tw, deltas)
    assert pts[0]["kept"] == g.m and pts[-1]["kept"] == 0
    assert pts[-1]["n_cc"] == g.n and pts[-1]["largest"] == 1
    ncc = [p["n_cc"] for p in pts]
    lg = [p["largest"] for p in pts]
    assert ncc == sorted(ncc) and lg == sorted(lg, reverse=True)
    assert all(p["intra"] >= p["kept"] for p in pts)


def _rule(r):
    return {0: "jump", 1: "modularity"}[r]


def test_golden_selection_examples(oracle_mod):
    for case in json.load(open(GOLDEN))["selection"]:
        i, r = oracle_mod.select(case["deltas"], case["largest"], case["n"], case["modularity"])
        assert case["deltas"][i] == case["expect_delta"], case["cite"]
        assert _rule(r) == case["expect_rule"], case["cite"]


def test_selection_branches(oracle_mod):
    sel = oracle_mod.select
    # input order does not matter: the scan is by decreasing delta
    d = [4, 0, 8, 2, 6]
    lg = [0, 9, 0, 9, 0]
    assert d[sel(d, lg, 10, [0.0] * 5)[0]] == 4
    # the largest of several jumps wins; it must reach jump_factor
    d = [10, 8, 6, 4, 2, 0]
    lg = [1, 2, 4, 5, 9, 10]        # increases on decreasing delta: .1 .2 .1 .4 .1 (n = 10)
    i, r = sel(d, lg, 10, [0.0] * 6)
    assert (d[i], r) == (4, 0)
    i, r = sel(d, lg, 10, [0, 0, 0, 0.5, 0, 0], jump_factor=0.5)   # .4 < .5 -> modularity
    assert (d[i], r) == (4, 1)
    # equal jumps: the first on the decreasing scan (the larger delta) wins
    i, r = sel([3, 2, 1, 0], [0, 5, 5, 10], 10, [0.0] * 4)
    assert (i, r) == (0, 0)
    # modularity ties -> larger delta; NaN never selected over a number
    i, r = sel([0, 1, 2, 3], [1, 1, 1, 1], 10, [0.3, 0.5, 0.5, float("nan")])
    assert (i, r) == (2, 1)
    # a jump exactly equal to jump_factor selects (>=); a decrease never counts
    i, r = sel([1, 0], [0, 1], 10, [0.0, 0.0], jump_factor=0.1)
    assert (i, r) == (0, 0)
    i, r = sel([1, 0], [5, 0], 10, [0.0, 0.7])
    assert (i, r) == (1, 1)
    # one point: modularity rule, index 0
    assert sel([3.0], [2], 10, [0.1]) == (0, 1)


def test_fig3_selection_recovers_two_blocks(oracle_mod):
    # on SBM(n=50 per block, p1=0.1, p2=0.8, q=0.05) (the Fig. 3 setting, reading C14)
    # with the TW grid, the selected delta removes every cross-block edge, so no community
    # mixes the blocks, and clustering at it recovers the two blocks (exactly, whenever the
    # sparse block stays internally connected at that delta).
    exact = 0
    n = 50
    truth = (np.arange(2 * n) >= n).astype(np.int32) * n
    deltas = [float(x) for x in range(-30, 1, 2)]
    for seed in range(20):
        g = gg.two_block_sbm(n, 0.1, 0.8, 0.05, seed=seed)
        t, w, tw = oracle_mod.score(g)
        pts = oracle_mod.sweep_report(g, tw, deltas)
        i, r = oracle_mod.select(deltas, [p["largest"] for p in pts], g.n,
                                 [p["modularity"] for p in pts])
        labels, _, _ = oracle_mod.cluster(g, tw, deltas[i])
        block = np.arange(g.n) >= n
        assert all(len(set(block[labels == c])) == 1 for c in np.unique(labels)), seed
        assert len(np.unique(labels[block])) == 1, seed          # the dense block is one
        exact += int(np.array_equal(labels, truth))
    assert exact >= 15
