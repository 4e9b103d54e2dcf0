"""Pins for the oracle's Table-1 similarity kinds (NEXT(1) of SURVEY 8(f)): Tectonic, Jaccard,
K3, TW and the effective-resistance proxy, and Alg. 1 on real-valued scores.

Pinned by: the SPEC worked examples, closed forms on K_n, exact rational
arithmetic on brute-force triangle counts, and Proposition 1 (thresholding Jaccard
at delta removes exactly the edges that thresholding Tectonic at delta/(1+delta) removes)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import brute
import graphgen as gg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def exact_scores(g):
    """Exact rationals per canonical edge from brute-force t and the degrees."""
    bf = brute.edge_motifs(g)
    deg = np.diff(g.rowptr.astype(np.int64))
    s, d = g.canonical_pairs()
    out = {k: [] for k in ("tw", "tectonic", "jaccard", "k3", "effres")}
    for a, b in zip(s.tolist(), d.tolist()):
        t, w = bf[(a, b)]
        D = int(deg[a] + deg[b])
        out["tw"].append(Fraction(t - w))
        out["tectonic"].append(Fraction(t, D))
        out["jaccard"].append(Fraction(t, D - t))
        out["k3"].append(Fraction(t))
        out["effres"].append(Fraction(-2, 2 + t))
    return out


def test_golden_similarity(oracle_mod):
    gold = json.load(open(GOLDEN))
    for case in gold["similarity"]:
        e = np.array(case["edges"]).reshape(-1, 2)
        g = gg.csr_from_pairs(case["n"], e[:, 0], e[:, 1])
        t, _, _ = oracle_mod.score(g)
        s, d = g.canonical_pairs()
        a, b = map(int, case["edge"].split("-"))
        idx = [i for i, (x, y) in enumerate(zip(s, d)) if (x, y) == (a, b)][0]
        for kind, val in case["expect"].items():
            v = float(Fraction(*val)) if isinstance(val, list) else float(val)
            assert oracle_mod.similarity(g, t, kind)[idx] == v, (case["cite"], kind)


@pytest.mark.parametrize("n", [3, 4, 7, 30])
def test_complete_graph_closed_forms(oracle_mod, n):
    g = gg.complete(n)
    t, _, _ = oracle_mod.score(g)
    assert np.all(oracle_mod.similarity(g, t, "tectonic") == (n - 2) / (2 * (n - 1)))
    assert np.all(oracle_mod.similarity(g, t, "jaccard") == (n - 2) / n)
    assert np.all(oracle_mod.similarity(g, t, "k3") == n - 2)
    assert np.all(oracle_mod.similarity(g, t, "effres") == -2 / n)
    assert np.all(oracle_mod.similarity(g, t, "tw") == n - 2)


def test_scores_equal_exact_rationals_rounded(oracle_mod):
    """One correctly rounded IEEE division per score: fp64 == float(exact rational)."""
    for seed in range(20):
        g = gg.erdos_renyi(40, 0.25, seed=300 + seed)
        t, _, _ = oracle_mod.score(g)
        ex = exact_scores(g)
        for kind, vals in ex.items():
            got = oracle_mod.similarity(g, t, kind)
            assert got.tolist() == [float(x) for x in vals], kind


def test_jaccard_is_increasing_in_tectonic(oracle_mod):
    g = gg.config_graph(1)
    t, _, _ = oracle_mod.score(g)
    tec = oracle_mod.similarity(g, t, "tectonic")
    jac = oracle_mod.similarity(g, t, "jaccard")
    assert np.allclose(jac, tec / (1 - tec), rtol=1e-12, atol=0)   # J = T / (1 - T)
    order = np.argsort(tec, kind="stable")
    assert np.all(np.diff(jac[order]) >= 0)


def test_proposition_1_equivalence(oracle_mod):
    """P:434-448 / S:247: Jaccard at delta and Tectonic at delta/(1+delta) remove the same
    edges, for 20 random graphs and delta = k/20, k = 1..19.  Decided exactly on the oracle's
    integer t and degrees (t/(D-t) < d  <=>  t/D < d/(1+d)); the fp64 scores agree with the
    exact decision everywhere except at exact rational ties, where rounding delta/(1+delta) in
    floating point may flip it (reading N1 in DESIGN.md)."""
    for seed in range(20):
        g = gg.erdos_renyi(200, 0.05, seed=700 + seed)
        t, _, _ = oracle_mod.score(g)
        deg = np.diff(g.rowptr.astype(np.int64))
        s, d = g.canonical_pairs()
        D = deg[s] + deg[d]
        tt = t.astype(np.int64)
        jac = oracle_mod.similarity(g, t, "jaccard")
        tec = oracle_mod.similarity(g, t, "tectonic")
        for k in range(1, 20):
            keep_j = 20 * tt >= k * (D - tt)          # t/(D-t) >= k/20
            keep_t = (20 + k) * tt >= k * D           # t/D >= (k/20)/(1 + k/20) = k/(20+k)
            assert np.array_equal(keep_j, keep_t), (seed, k)
            dj = k / 20
            tie_j = 20 * tt == k * (D - tt)
            assert np.array_equal((jac >= dj)[~tie_j], keep_j[~tie_j])
            assert np.array_equal((tec >= dj / (1 + dj))[~tie_j], keep_t[~tie_j])
            lj, kj, cj = oracle_mod.cluster(g, keep_j.astype(np.int32), 0.5)
            lt, kt, ct = oracle_mod.cluster(g, keep_t.astype(np.int32), 0.5)
            assert (kj, cj) == (kt, ct) and np.array_equal(lj, lt)


def test_cluster_f64_matches_integer_cluster_on_tw(oracle_mod):
    g = gg.config_graph(2)
    _, _, tw = oracle_mod.score(g)
    twd = oracle_mod.similarity(g, oracle_mod.score(g)[0], "tw")
    assert np.array_equal(twd, tw.astype(np.float64))
    for delta in (-math.inf, -10.0, -3.5, 0.0, math.inf):
        a = oracle_mod.cluster(g, tw, delta)
        b = oracle_mod.cluster_f64(g, twd, delta)
        assert a[1:] == b[1:] and np.array_equal(a[0], b[0])
