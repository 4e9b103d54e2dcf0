"""GPU parity of the sharded scoring step: twc_score_shard's partial counts per
rank against the brute-force reference of the contract (tests/shard_ref.py), their sum against
the oracle's t, and twc_finish_scores against the oracle's wedge and TW -- all bit-exact."""
import numpy as np
import pytest
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc
from paper_2412_12382_b200 import build as twc_build

import shard_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    twc_build.build()
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _shards(g, world, rb=None):
    rp, ci = harness.to_device(g, "cuda")
    if rb is not None:
        rp = rp.to(rb)
    return rp, ci, [twc.twc_score_shard(rp, ci, r, world).cpu().numpy() for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_partials_match_contract_small(world):
    rng = np.random.default_rng(7 + world)
    for it in range(6):
        n = int(rng.integers(3, 60))
        g = gg.erdos_renyi(n, float(rng.uniform(0.05, 0.5)), seed=300 + 10 * world + it)
        _, _, parts = _shards(g, world)
        ref = shard_ref.partial_counts(g, world)
        for r in range(world):
            assert np.array_equal(parts[r], ref[r]), (world, it, r)


@pytest.mark.parametrize("world", [1, 2, 4, 7])
def test_sum_and_finish_match_oracle(oracle_mod, world):
    graphs = [gg.config_graph(1), gg.config_graph(2), gg.complete(300), gg.star(5000, 3),
              gg.erdos_renyi(2000, 0.02, seed=11)]
    for g in graphs:
        ot, ow, otw = oracle_mod.score(g)
        for rb in (torch.int32, torch.int64):
            rp, ci, parts = _shards(g, world, rb)
            assert all((p >= 0).all() for p in parts)
            t = np.sum(parts, axis=0)
            assert np.array_equal(t, ot)
            wedge, tw = twc.twc_finish_scores(rp, ci, torch.from_numpy(t.astype(np.int32)).cuda())
            assert np.array_equal(wedge.cpu().numpy(), ow)
            assert np.array_equal(tw.cpu().numpy(), otw)


def test_config3_four_shards(oracle_mod):
    g = gg.config_graph(3)
    ot, ow, otw = oracle_mod.score(g)
    _, _, parts = _shards(g, 4)
    assert np.array_equal(np.sum(parts, axis=0), ot)


def test_shard_argument_errors():
    g = gg.complete(5)
    rp, ci = harness.to_device(g, "cuda")
    for rank, world in [(-1, 2), (2, 2), (0, 0)]:
        with pytest.raises(twc.TwcError):
            twc.twc_score_shard(rp, ci, rank, world)
