"""GPU parity for the Table-1 similarity kinds and the fp64 sweep.

Bar (north_star): fp64 scores within 1e-12 relative of the oracle -- asserted here as exact
equality, since each score is one correctly rounded IEEE operation on identical integers -- and
bit-exact min-id labels for Alg. 1 on those scores."""
import math

import numpy as np
import pytest
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc
from paper_2412_12382_b200 import build as twc_build

pytestmark = pytest.mark.gpu
KINDS = ["tw", "tectonic", "jaccard", "k3", "effres"]


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests need a B200 (there is no CPU fallback)")
    twc_build.build()
    twc.load_library()


def check_graph(oracle_mod, g, deltas_by_kind):
    rp, ci = harness.to_device(g)
    t, _, _ = twc.twc_score(rp, ci)
    ot, _, _ = oracle_mod.score(g)
    assert np.array_equal(t.cpu().numpy(), ot)
    for kind in KINDS:
        gs = twc.twc_similarity(rp, ci, t, kind)
        os_ = oracle_mod.similarity(g, ot, kind)
        got = gs.cpu().numpy()
        np.testing.assert_allclose(got, os_, rtol=1e-12, atol=0)
        assert np.array_equal(got, os_), kind          # in fact bit-identical
        deltas = deltas_by_kind(kind, os_)
        lab, st = twc.twc_sweep_f64(rp, ci, gs, deltas)
        lab, st = lab.cpu().numpy(), st.cpu().numpy()
        for i, d in enumerate(deltas):
            ol, kept, ncomp = oracle_mod.cluster_f64(g, os_, d)
            assert np.array_equal(lab[i], ol), (kind, d)
            assert (int(st[i, 0]), int(st[i, 1])) == (kept, ncomp), (kind, d)


def _deltas(kind, score):
    if score.size == 0:
        return [0.0, -math.inf]
    qs = np.quantile(score, [0.1, 0.5, 0.9]).tolist()
    extra = {"tectonic": [0.05, 0.1, 1 / 6], "jaccard": [0.2, 0.25, 1 / 3],
             "effres": [-0.5, -0.25], "k3": [1.0, 3.0], "tw": [-4.0, 0.0]}[kind]
    return [-math.inf, math.inf] + qs + extra


def test_similarity_small_graphs(oracle_mod):
    for g in (gg.complete(12), gg.bridge_triangles(), gg.star(40, 5), gg.wheel(9), gg.empty(4)):
        check_graph(oracle_mod, g, _deltas)
    rng = np.random.default_rng(5)
    for it in range(10):
        n = int(rng.integers(5, 3000))
        g = gg.erdos_renyi(n, min(1.0, 25.0 / n), seed=40 + it)
        check_graph(oracle_mod, g, _deltas)


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_similarity_configs(oracle_mod, config):
    check_graph(oracle_mod, gg.config_graph(config), _deltas)


def test_similarity_int64_rowptr(oracle_mod):
    g = gg.erdos_renyi(1500, 0.02, seed=77).with_rowptr_dtype(np.int64)
    check_graph(oracle_mod, g, _deltas)


def test_proposition_1_on_gpu(oracle_mod):
    """Jaccard at delta vs Tectonic at delta/(1+delta): identical partitions
    whenever no edge sits exactly on the threshold (checked on the oracle's integers)."""
    g = gg.config_graph(1)
    rp, ci = harness.to_device(g)
    t, _, _ = twc.twc_score(rp, ci)
    jac = twc.twc_similarity(rp, ci, t, "jaccard")
    tec = twc.twc_similarity(rp, ci, t, "tectonic")
    ot, _, _ = oracle_mod.score(g)
    deg = np.diff(g.rowptr.astype(np.int64))
    s, d = g.canonical_pairs()
    D = deg[s] + deg[d]
    tt = ot.astype(np.int64)
    for k in range(1, 20):
        if np.any(20 * tt == k * (D - tt)):
            continue                                   # exact tie: fp rounding may differ
        dj = k / 20
        lj, sj = twc.twc_sweep_f64(rp, ci, jac, [dj])
        lt, st = twc.twc_sweep_f64(rp, ci, tec, [dj / (1 + dj)])
        assert torch.equal(lj, lt) and torch.equal(sj, st), k


def test_similarity_unaligned_buffers_and_ragged_tail(oracle_mod):
    """t and the score array need only their natural alignment (views shifted by one element,
    4 / 8 bytes off a 16-byte boundary), for the streaming kinds (K3, -R_eff: no CSR read) and
    the degree kinds alike; m not a multiple of the 1,024-edge tile exercises the ragged tail."""
    for n, p, seed in ((700, 0.03, 3), (2500, 0.004, 4), (1203, 0.011, 5)):
        g = gg.erdos_renyi(n, p, seed=seed)
        rp, ci = harness.to_device(g)
        t, _, _ = twc.twc_score(rp, ci)
        ot, _, _ = oracle_mod.score(g)
        m = int(t.numel())
        tbuf = torch.empty(m + 1, dtype=torch.int32, device=t.device)
        tbuf[1:].copy_(t)
        obuf = torch.empty(m + 1, dtype=torch.float64, device=t.device)
        for kind in KINDS:
            os_ = oracle_mod.similarity(g, ot, kind)
            got = twc.twc_similarity(rp, ci, tbuf[1:], kind, out=obuf[1:])
            assert got.data_ptr() % 16 == 8 and tbuf[1:].data_ptr() % 16 == 4
            assert np.array_equal(got.cpu().numpy(), os_), (kind, m)
            got = twc.twc_similarity(rp, ci, t, kind)
            assert np.array_equal(got.cpu().numpy(), os_), (kind, m)
