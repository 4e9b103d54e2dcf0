"""Pins for oracle.k4 (kappa-clique participation, kappa = 4: Table 1):
brute-force enumeration of all 4-subsets on tiny graphs, closed forms (K_n -> C(n-2, 2) per
edge: K4 -> 1 and K5 -> 3 are S:133's worked examples; triangle-free and K4-free families -> 0),
the global identity sum_e K4(e) = 6 * #K4 with networkx's clique enumeration, the bound
K4(e) <= C(t(e), 2), and relabelling invariance."""
import math

import networkx as nx
import numpy as np
import pytest

import brute
import graphgen as gg


def by_pair(g, arr):
    s, d = g.canonical_pairs()
    return {(int(a), int(b)): int(x) for a, b, x in zip(s, d, arr)}


@pytest.mark.parametrize("seed", range(25))
def test_k4_equals_brute_force(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 14))
    g = gg.erdos_renyi(n, float(rng.uniform(0.3, 0.9)), seed=seed)
    assert by_pair(g, oracle_mod.k4(g)) == brute.edge_k4(g)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 9, 20])
def test_complete_graph_closed_form(oracle_mod, n):
    k = oracle_mod.k4(gg.complete(n))
    assert k.size == n * (n - 1) // 2 and (k == math.comb(n - 2, 2)).all()


def test_golden_k4_examples(oracle_mod):
    # "K4, any edge, with_k4 -> K4=1; K5, any edge -> K4=3"
    assert (oracle_mod.k4(gg.complete(4)) == 1).all()
    assert (oracle_mod.k4(gg.complete(5)) == 3).all()


@pytest.mark.parametrize("g", [gg.path(9), gg.cycle(12), gg.star(20, 3), gg.wheel(7),
                               gg.complete_bipartite(6, 7), gg.bridge_triangles()])
def test_k4_free_families(oracle_mod, g):
    assert (oracle_mod.k4(g) == 0).all()


@pytest.mark.parametrize("seed", range(5))
def test_global_identity_and_bound(oracle_mod, seed):
    g = gg.erdos_renyi(200, 0.15, seed=seed)
    k4 = oracle_mod.k4(g)
    t, _, _ = oracle_mod.score(g)
    G = nx.Graph()
    G.add_nodes_from(range(g.n))
    s, d = g.canonical_pairs()
    G.add_edges_from(zip(s.tolist(), d.tolist()))
    n4 = sum(1 for c in nx.enumerate_all_cliques(G) if len(c) == 4)
    assert int(k4.sum()) == 6 * n4
    assert np.all(k4 <= t.astype(np.int64) * (t.astype(np.int64) - 1) // 2)


def test_relabel_invariance(oracle_mod):
    g = gg.planted_partition(4, 30, 0.5, 0.02, seed=2)
    perm = np.random.default_rng(1).permutation(g.n)
    h = gg.relabel(g, perm)
    a = by_pair(g, oracle_mod.k4(g))
    b = by_pair(h, oracle_mod.k4(h))
    assert all(b[tuple(sorted((int(perm[u]), int(perm[v]))))] == x for (u, v), x in a.items())
