"""GPU parity of per-edge K4 participation (Table 1) through
twc_score_k4 against oracle.k4: bit-exact int64 counts per canonical edge, with t, wedge and TW
unchanged.  Covers closed forms (K_n -> C(n-2, 2) incl. S:133's K4/K5 examples, K4-free
families), random graphs over many tiles, the big-pivot path (|N+(a)| > 256: K_300 and dense
blocks), int64 rowptr, degenerate inputs and BASELINE configs 1-5 at full size."""
import math

import numpy as np
import pytest
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc
from paper_2412_12382_b200 import build as twc_build

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests need a B200 (there is no CPU fallback)")
    twc_build.build()
    twc.load_library()


def gpu_k4(g):
    rp, ci = harness.to_device(g)
    t, w, tw, k4 = twc.twc_score_k4(rp, ci)
    torch.cuda.synchronize()
    return t.cpu().numpy(), tw.cpu().numpy(), k4.cpu().numpy()


def assert_k4_parity(oracle_mod, g):
    t, tw, k4 = gpu_k4(g)
    ok4 = oracle_mod.k4(g)
    bad = np.nonzero(k4 != ok4)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: gpu {k4[bad[:5]]} oracle {ok4[bad[:5]]}"
    ot, _, otw = oracle_mod.score(g)
    assert np.array_equal(t, ot) and np.array_equal(tw, otw)


@pytest.mark.parametrize("n", [3, 4, 5, 6, 40, 300])
def test_complete_graphs(n):
    t, tw, k4 = gpu_k4(gg.complete(n))
    assert (k4 == math.comb(n - 2, 2)).all() and (t == n - 2).all()


@pytest.mark.parametrize("g", [gg.path(9), gg.cycle(12), gg.star(50, 3), gg.wheel(9),
                               gg.complete_bipartite(6, 70), gg.bridge_triangles()])
def test_k4_free(g):
    assert (gpu_k4(g)[2] == 0).all()


def test_random_graphs_many_tiles(oracle_mod):
    for seed in range(12):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(50, 3000))
        assert_k4_parity(oracle_mod, gg.erdos_renyi(n, float(rng.uniform(3, 60)) / n, seed=seed))


def test_dense_blocks_big_pivots(oracle_mod):
    # blocks of 300 at p = 0.9: pivots with |N+(a)| in (256, 300) take the big-pivot path
    oracle_mod.set_threads(oracle_mod.max_threads())
    assert_k4_parity(oracle_mod, gg.planted_partition(3, 300, 0.9, 0.01, seed=4))


def test_int64_rowptr_and_degenerate(oracle_mod):
    g = gg.planted_partition(20, 40, 0.5, 0.01, seed=6).with_rowptr_dtype(np.int64)
    assert_k4_parity(oracle_mod, g)
    for g in (gg.empty(5), gg.path(2), gg.complete(3)):
        t, tw, k4 = gpu_k4(g)
        assert k4.size == g.m and (k4 == 0).all()


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_configs_full_size(oracle_mod, config):
    oracle_mod.set_threads(oracle_mod.max_threads())
    assert_k4_parity(oracle_mod, gg.config_graph(config))
