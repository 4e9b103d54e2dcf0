"""GPU parity of the threshold-selection workflow: twc_partition_stats and
twc_select_threshold through the C ABI against oracle.partition_stats / oracle.select.

Bar: the four integer statistics bit-exact, the modularity bit-identical (both sides divide the
same two exact integers once, reading C21), the selected index and rule identical.  Each side
computes its own scores and labels from the same seeded graph: no oracle input comes from the
CUDA path."""
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


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.int64)


def oracle_report(oracle_mod, g, deltas):
    _, _, tw = oracle_mod.score(g)
    pts = oracle_mod.sweep_report(g, tw, deltas)
    sel = oracle_mod.select(deltas, [p["largest"] for p in pts], g.n,
                            [p["modularity"] for p in pts]) if g.n else None
    return pts, sel


def assert_report_parity(oracle_mod, g, deltas):
    rp, ci = harness.to_device(g)
    rep = twc.sweep_report(rp, ci, deltas)
    pts, sel = oracle_report(oracle_mod, g, deltas)
    for a, b in zip(rep["points"], pts):
        assert (a["n_cc"], a["largest"], a["intra_edges"], a["sum_deg_sq"], a["kept"]) == \
            (b["n_cc"], b["largest"], b["intra"], b["sum_d2"], b["kept"]), a["delta"]
        assert _bits(a["modularity"]) == _bits(b["modularity"]), (a, b)
    if g.n:
        assert (rep["selected_index"], rep["rule"]) == \
            (sel[0], {0: "largest_cc_jump", 1: "max_modularity"}[sel[1]])
    return rep


@pytest.mark.parametrize("seed", range(8))
def test_random_graphs(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(200, 5000))
    g = gg.erdos_renyi(n, float(rng.uniform(2, 40)) / n, seed=seed)
    assert_report_parity(oracle_mod, g, [float(x) for x in range(-30, 1, 2)])


def test_planted_partition_and_fig3(oracle_mod):
    assert_report_parity(oracle_mod, gg.planted_partition(40, 50, 0.3, 0.002, seed=2),
                         [float(x) for x in range(-30, 1, 2)])
    for seed in range(5):
        assert_report_parity(oracle_mod, gg.two_block_sbm(50, 0.1, 0.8, 0.05, seed=seed),
                             [float(x) for x in range(-30, 1, 2)])


def test_arbitrary_labels_many_groups(oracle_mod):
    # non-canonical labels; k = 21 partitions -> several k_part_edges groups with a ragged one
    g = gg.erdos_renyi(3000, 0.004, seed=5)
    rng = np.random.default_rng(7)
    labs = [rng.integers(0, c, size=g.n).astype(np.int32) for c in
            [1, 2, 3, 10, 50, 100, 1000, 3000] * 2 + [1, 7, 3000, 2999, 5]]
    L = torch.from_numpy(np.stack(labs)).cuda()
    rp, ci = harness.to_device(g)
    counts, q = twc.twc_partition_stats(rp, ci, L)
    counts, q = counts.cpu().numpy(), q.cpu().numpy()
    for j, lab in enumerate(labs):
        nc, lg, intra, sd2, qq = oracle_mod.partition_stats(g, lab)
        assert tuple(int(x) for x in counts[j]) == (nc, lg, intra, sd2), j
        assert _bits(q[j]) == _bits(qq), j


def test_int64_rowptr_and_giant_component(oracle_mod):
    # one label for all vertices: the run-length / warp-merge path of k_part_vertex
    g = gg.gnm(200_000, 2_000_000, seed=3)
    g64 = gg.gnm(200_000, 2_000_000, seed=3, rowptr_dtype=np.int64)
    for gr in (g, g64):
        rp, ci = harness.to_device(gr)
        lab = np.zeros((2, gr.n), dtype=np.int32)
        lab[1] = np.arange(gr.n) // 1000 * 1000
        counts, q = twc.twc_partition_stats(rp, ci, torch.from_numpy(lab).cuda())
        counts, q = counts.cpu().numpy(), q.cpu().numpy()
        for j in range(2):
            nc, lg, intra, sd2, qq = oracle_mod.partition_stats(gr, lab[j])
            assert tuple(int(x) for x in counts[j]) == (nc, lg, intra, sd2)
            assert _bits(q[j]) == _bits(qq)
        assert q[0] == 0.0   # one community: Q = 0


def test_degenerate_and_errors():
    g = gg.empty(7)                       # m = 0: Q undefined -> NaN
    rp, ci = harness.to_device(g)
    counts, q = twc.twc_partition_stats(rp, ci, torch.arange(7, dtype=torch.int32).cuda())
    assert counts.cpu().tolist() == [[7, 1, 0, 0]] and np.isnan(q.item())
    g = gg.complete(5)
    rp, ci = harness.to_device(g)
    with pytest.raises(twc.TwcError) as e:
        twc.twc_partition_stats(rp, ci, torch.tensor([0, 1, 2, 3, 5], dtype=torch.int32).cuda())
    assert e.value.status == twc.TWC_EINVAL
    with pytest.raises(twc.TwcError):
        twc.twc_partition_stats(rp, ci, torch.tensor([0, 1, -1, 3, 4], dtype=torch.int32).cuda())
    counts, q = twc.twc_partition_stats(rp, ci, torch.zeros(5, dtype=torch.int32).cuda())
    assert counts.cpu().tolist() == [[1, 5, 10, 400]] and q.item() == 0.0


def test_sweep_extremes(oracle_mod):
    # below every score -> all edges kept; above -> every vertex alone
    g = gg.planted_partition(10, 30, 0.4, 0.02, seed=1)
    rep = assert_report_parity(oracle_mod, g, [-1e9, 0.0, 1e9])
    lo, _, hi = rep["points"]
    assert lo["norm_edges"] == 1.0 and hi["norm_cc"] == 1.0 and hi["norm_largest_cc"] == 1 / g.n


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_config_reports_full_size(oracle_mod, config):
    oracle_mod.set_threads(oracle_mod.max_threads())
    g = gg.config_graph(config)
    deltas = [float(x) for x in range(-30, 1, 2)] if config == 5 else \
        harness.thresholds(config, oracle_mod.score(g)[2])
    assert_report_parity(oracle_mod, g, deltas)
