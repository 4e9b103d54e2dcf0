"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bar (north_star): t, wedge, TW bit-exact; labels bit-exact (both
sides emit min-vertex-id labels).  Sizes span many tiles with ragged tails; configs 1-5 run at
their full BASELINE.json sizes in the launch configuration bench.py times."""
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


def gpu_score(g):
    rp, ci = harness.to_device(g)
    t, w, tw = twc.twc_score(rp, ci)
    torch.cuda.synchronize()
    return t.cpu().numpy(), w.cpu().numpy(), tw.cpu().numpy()


def gpu_sweep(g, tw, deltas):
    rp, ci = harness.to_device(g)
    twd = torch.from_numpy(np.ascontiguousarray(tw)).cuda()
    lab, st = twc.twc_sweep(rp, ci, twd, deltas)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), st.cpu().numpy()


def assert_score_parity(oracle_mod, g):
    ot, ow, otw = oracle_mod.score(g)
    gt, gw, gtw = gpu_score(g)
    assert gt.shape == ot.shape
    bad = np.nonzero((gt != ot) | (gw != ow) | (gtw != otw))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: gpu t={gt[bad[:5]]} oracle t={ot[bad[:5]]}"
    return otw


def assert_cluster_parity(oracle_mod, g, tw, deltas):
    lab, st = gpu_sweep(g, tw, deltas)
    for i, d in enumerate(deltas):
        ol, kept, ncomp = oracle_mod.cluster(g, tw, d)
        assert np.array_equal(lab[i], ol), (d, np.nonzero(lab[i] != ol)[0][:5])
        assert (int(st[i, 0]), int(st[i, 1])) == (kept, ncomp), d


# ------------------------------------------------------------------ small / closed forms

@pytest.mark.parametrize("maker", [
    lambda: gg.complete(3), lambda: gg.complete(60), lambda: gg.path(2), lambda: gg.path(9),
    lambda: gg.cycle(31), lambda: gg.star(50, 25), lambda: gg.complete_bipartite(5, 9),
    lambda: gg.wheel(20), lambda: gg.bridge_triangles()])
def test_small_closed_forms(oracle_mod, maker):
    g = maker()
    tw = assert_score_parity(oracle_mod, g)
    assert_cluster_parity(oracle_mod, g, tw, [-math.inf, -2.0, 0.0, 0.5, math.inf])


def test_random_graphs_many_tiles(oracle_mod):
    rng = np.random.default_rng(11)
    for it in range(30):
        n = int(rng.integers(2, 3000))
        p = float(rng.random()) * min(1.0, 40.0 / n)
        g = gg.erdos_renyi(n, p, seed=it)
        tw = assert_score_parity(oracle_mod, g)
        if tw.size:
            ds = sorted({float(np.median(tw)), float(tw.min()), float(tw.max()) + 1, -math.inf})
            assert_cluster_parity(oracle_mod, g, tw, ds)


def test_dense_small_many_tiles(oracle_mod):
    g = gg.erdos_renyi(2000, 0.2, seed=5)          # ~400k edges, d+ up to ~200, ragged tail
    assert_score_parity(oracle_mod, g)


@pytest.mark.parametrize("rb", [np.int32, np.int64])
def test_hub_closed_forms(rb):
    """Closed forms, no oracle needed: K_3000 (every d+ beyond the smem staging capacity),
    star K_{1,200000}, K_{2,100000} (SURVEY 8(c) hub-bin stress)."""
    g = gg.complete(3000, rb)
    t, w, tw = gpu_score(g)
    assert t.size == 3000 * 2999 // 2
    assert (t == 2998).all() and (w == 0).all() and (tw == 2998).all()
    g = gg.star(200_000, 7, rb)
    t, w, tw = gpu_score(g)
    assert (t == 0).all() and (w == 199_999).all() and (tw == 1 - 200_000).all()
    g = gg.complete_bipartite(2, 100_000, rb)
    t, w, tw = gpu_score(g)
    assert (t == 0).all() and (w == 100_000).all() and (tw == -100_000).all()
    lab, st = gpu_sweep(g, tw, [-math.inf, -100_000.0, -99_999.5])
    assert (lab[0] == 0).all() and (lab[1] == 0).all() and np.array_equal(lab[2], np.arange(g.n))
    assert st.tolist() == [[g.m, 1], [g.m, 1], [0, g.n]]


def test_hub_beyond_smem_staging():
    """K_8300: the top pivots' oriented lists (up to 8,299) exceed the hub kernel's 2,048-entry
    smem staging, so their candidates are verified in global memory (closed form t = n - 2)."""
    g = gg.complete(8300, np.int64)
    t, w, tw = gpu_score(g)
    assert t.size == 8300 * 8299 // 2
    assert (t == 8298).all() and (w == 0).all() and (tw == 8298).all()


def test_hub_pivots_with_community_structure(oracle_mod):
    """Dense planted partition (blocks of 600, p_in 0.9): many pivots with |N+(u)| in
    (256, 600] -- the hub kernel's staged path -- against the oracle."""
    g = gg.planted_partition(3, 600, 0.9, 0.01, seed=9)
    assert_score_parity(oracle_mod, g)


def test_sparse_rows_uncached_tiles(oracle_mod):
    """Tiles spanning more rows than the smem row caches hold: a perfect matching on 3 of
    every 3k ids plus isolated vertices (every tile of canonical ids / CSR slots covers
    thousands of rows), with a few triangles and a hub mixed in."""
    k = 40_000
    a = np.arange(k) * 3
    hub = 3 * k + 1
    leaves = np.arange(0, 3 * k, 7)
    A = np.concatenate([a, [0, 0, 1], np.full(leaves.size, hub)])
    B = np.concatenate([a + 1, [2, 3, 3], leaves])
    for rb in (np.int32, np.int64):
        g = gg.csr_from_pairs(3 * k + 2, A, B, rb)
        tw = assert_score_parity(oracle_mod, g)
        assert_cluster_parity(oracle_mod, g, tw, [-math.inf, 0.0, float(np.median(tw))])


def test_int64_rowptr_small(oracle_mod):
    for seed in range(5):
        g = gg.erdos_renyi(700, 0.05, seed).with_rowptr_dtype(np.int64)
        tw = assert_score_parity(oracle_mod, g)
        assert_cluster_parity(oracle_mod, g, tw, [float(np.median(tw)), -math.inf])


def test_degenerate_inputs():
    for n in [1, 5]:
        g = gg.empty(n)
        rp, ci = harness.to_device(g)
        t, w, tw = twc.twc_score(rp, ci)
        assert t.numel() == 0
        lab, st = twc.twc_cluster(rp, ci, tw, 0.0)
        assert lab.cpu().tolist() == list(range(n)) and st.cpu().tolist() == [0, n]
    rp = torch.zeros(1, dtype=torch.int32, device="cuda")   # n = 0
    ci = torch.zeros(0, dtype=torch.int32, device="cuda")
    t, w, tw = twc.twc_score(rp, ci)
    lab, st = twc.twc_cluster(rp, ci, tw, 0.0)
    assert lab.numel() == 0 and st.cpu().tolist() == [0, 0]
    g = gg.path(2)                                          # single edge
    t, w, tw = gpu_score(g)
    assert (t.tolist(), w.tolist(), tw.tolist()) == ([0], [0], [0])
    g = gg.csr_from_pairs(10, [0, 5], [1, 9])               # isolated vertices
    t, w, tw = gpu_score(g)
    lab, st = gpu_sweep(g, tw, [0.0, 1.0])
    assert lab[0].tolist() == [0, 0, 2, 3, 4, 5, 6, 7, 8, 5]
    assert lab[1].tolist() == list(range(10))


def test_sweep_equals_independent_clusters_and_duplicates(oracle_mod):
    g = gg.config_graph(2)
    _, _, tw = oracle_mod.score(g)
    rp, ci = harness.to_device(g)
    twd = torch.from_numpy(tw).cuda()
    deltas = [-3.0, 0.0, -10.0, -3.0, math.inf, -math.inf, -7.5, 0.0]
    lab, st = twc.twc_sweep(rp, ci, twd, deltas)
    for i, d in enumerate(deltas):
        l1, s1 = twc.twc_cluster(rp, ci, twd, d)
        assert torch.equal(l1, lab[i]) and torch.equal(s1, st[i]), d


def test_determinism_repeated_runs():
    g = gg.config_graph(3)
    rp, ci = harness.to_device(g)
    ref = [x.clone() for x in twc.twc_score(rp, ci)]
    lab0, _ = twc.twc_sweep(rp, ci, ref[2], harness.SWEEP_GRID)
    for _ in range(3):
        out = twc.twc_score(rp, ci)
        for a, b in zip(ref, out):
            assert torch.equal(a, b)
        lab, _ = twc.twc_sweep(rp, ci, ref[2], harness.SWEEP_GRID)
        assert torch.equal(lab, lab0)


def test_pipeline_host_matches_device_path(oracle_mod):
    g = gg.config_graph(1)
    ot, ow, otw = oracle_mod.score(g)
    deltas = harness.thresholds(1, otw)
    out = twc.twc_pipeline_host(torch.from_numpy(g.rowptr).pin_memory(),
                                torch.from_numpy(g.colidx).pin_memory(), deltas)
    assert np.array_equal(out["t"].numpy(), ot)
    assert np.array_equal(out["wedge"].numpy(), ow)
    assert np.array_equal(out["tw"].numpy(), otw)
    for i, d in enumerate(deltas):
        ol, kept, ncomp = oracle_mod.cluster(g, otw, d)
        assert np.array_equal(out["labels"][i].numpy(), ol)
        assert out["stats"][i].tolist() == [kept, ncomp]


def test_pipeline_host_async_in_flight(oracle_mod):
    # three graphs in flight on three streams (different sizes, int32 and int64 rowptr, one
    # with duplicate and unsorted thresholds): every call's host outputs equal the oracle's
    graphs = [gg.config_graph(1), gg.erdos_renyi(3000, 0.01, seed=4),
              gg.planted_partition(30, 40, 0.3, 0.01, seed=5).with_rowptr_dtype(np.int64)]
    deltas = [[-1.0, 0.0, 2.0], [0.0, -3.0, 0.0, -1.0], [-30.0, -10.0, 0.0]]
    calls = []
    for g, d in zip(graphs, deltas):
        st = torch.cuda.Stream()
        out = twc.twc_pipeline_host(torch.from_numpy(g.rowptr).pin_memory(),
                                    torch.from_numpy(g.colidx).pin_memory(), d, stream=st,
                                    asynchronous=True)
        calls.append((g, d, st, out))
    for g, d, st, out in calls:
        st.synchronize()
        ot, ow, otw = oracle_mod.score(g)
        assert np.array_equal(out["tw"].numpy(), otw) and np.array_equal(out["t"].numpy(), ot)
        for i, x in enumerate(d):
            ol, kept, ncomp = oracle_mod.cluster(g, otw, x)
            assert np.array_equal(out["labels"][i].numpy(), ol)
            assert out["stats"][i].tolist() == [kept, ncomp]


def test_validate_csr():
    g = gg.config_graph(1)
    rp, ci = harness.to_device(g)
    twc.twc_validate_csr(rp, ci)
    twc.twc_validate_csr(rp.to(torch.int64), ci)
    bad = ci.clone()
    bad[5] = bad[4]                        # duplicate / unsorted entry
    with pytest.raises(twc.TwcError) as e:
        twc.twc_validate_csr(rp, bad)
    assert e.value.status == twc.TWC_EGRAPH
    h = gg.csr_from_pairs(4, [0, 1], [1, 2])
    rp, ci = harness.to_device(h)
    ci2 = ci.clone()
    ci2[0] = 3                             # 0's neighbour 1 -> 3: asymmetric
    with pytest.raises(twc.TwcError):
        twc.twc_validate_csr(rp, ci2)
    ci3 = ci.clone()
    ci3[0] = 0                             # self-loop
    with pytest.raises(twc.TwcError):
        twc.twc_validate_csr(rp, ci3)


def fused_parity(oracle_mod, g, deltas, ot=None):
    """twc_score_sweep (the fused path bench.py times) against the oracle."""
    if ot is None:
        ot = oracle_mod.score(g)
    rp, ci = harness.to_device(g)
    t, w, tw, lab, st = twc.twc_score_sweep(rp, ci, deltas)
    torch.cuda.synchronize()
    for a, b in zip((t, w, tw), ot):
        assert np.array_equal(a.cpu().numpy(), b)
    lab, st = lab.cpu().numpy(), st.cpu().numpy()
    for i, d in enumerate(deltas):
        ol, kept, ncomp = oracle_mod.cluster(g, ot[2], d)
        assert np.array_equal(lab[i], ol), (d, np.nonzero(lab[i] != ol)[0][:5])
        assert (int(st[i, 0]), int(st[i, 1])) == (kept, ncomp), d


def test_fused_score_sweep_small(oracle_mod):
    rng = np.random.default_rng(21)
    for it in range(12):
        n = int(rng.integers(2, 4000))
        g = gg.erdos_renyi(n, float(rng.random()) * min(1.0, 30.0 / n), seed=100 + it)
        ds = [-math.inf, 0.0, -3.0, -3.0, 2.5, math.inf, -1e300, 1e300]
        fused_parity(oracle_mod, g, ds)
    for g in (gg.empty(7), gg.path(2), gg.complete(40), gg.star(3000, 11)):
        fused_parity(oracle_mod, g, [-2.0, math.inf, -math.inf])
    fused_parity(oracle_mod, gg.complete(3000), [2998.0, 2999.0, 0.0])


def test_fused_call_in_cuda_graph(oracle_mod):
    # the fused call makes no host synchronisation and no host->device copy, so it can be
    # captured in a CUDA graph; replays (after the inputs change in place) match the oracle
    g = gg.config_graph(2)
    rp, ci = harness.to_device(g, "cuda")
    ot = oracle_mod.score(g)
    deltas = harness.thresholds(2, ot[2])
    k = len(deltas)
    t, w, tw = (torch.empty(g.m, dtype=torch.int32, device="cuda") for _ in range(3))
    labels = torch.empty((k, g.n), dtype=torch.int32, device="cuda")
    stats = torch.empty((k, 2), dtype=torch.int64, device="cuda")
    ws = torch.empty(twc.twc_score_sweep_workspace_bytes(g.n, g.m, rp.element_size()),
                     dtype=torch.uint8, device="cuda")

    def step():
        twc.twc_score_sweep(rp, ci, deltas, out=(t, w, tw), labels=labels, stats=stats,
                            workspace=ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(cg, stream=s):
            step()
    torch.cuda.synchronize()
    for _ in range(2):
        t.fill_(-7); labels.fill_(-7); stats.fill_(-7)
        cg.replay()
        torch.cuda.synchronize()
        assert np.array_equal(t.cpu().numpy(), ot[0])
        assert np.array_equal(w.cpu().numpy(), ot[1])
        assert np.array_equal(tw.cpu().numpy(), ot[2])
        lab, st = labels.cpu().numpy(), stats.cpu().numpy()
        for i, d in enumerate(deltas):
            ol, kept, ncomp = oracle_mod.cluster(g, ot[2], d)
            assert np.array_equal(lab[i], ol), d
            assert (int(st[i, 0]), int(st[i, 1])) == (kept, ncomp), d


# ------------------------------------------------------------------ the five configs, full size

@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_config_parity_full_size(oracle_mod, config):
    oracle_mod.set_threads(oracle_mod.max_threads())
    g = gg.config_graph(config)
    ot = oracle_mod.score(g)
    tw = assert_score_parity(oracle_mod, g)
    deltas = harness.thresholds(config, tw)
    assert_cluster_parity(oracle_mod, g, tw, deltas)
    fused_parity(oracle_mod, g, deltas, ot)


def test_misaligned_colidx_view_rejected():
    """a contiguous view with an odd storage offset must come back as TWC_EINVAL, not
    as a misaligned-address fault that poisons the context."""
    g = gg.complete(40)
    rp, ci = harness.to_device(g)
    buf = torch.empty(ci.numel() + 1, dtype=torch.int32, device=ci.device)
    buf[1:].copy_(ci)
    with pytest.raises(twc.TwcError) as ei:
        twc.twc_score(rp, buf[1:])
    assert ei.value.status == twc.TWC_EINVAL
    t, _, _ = twc.twc_score(rp, ci)        # the context is still healthy
    torch.cuda.synchronize()
    assert int(t.min()) == 38 and int(t.max()) == 38


def test_temporary_workspace_on_side_stream(oracle_mod):
    """a temporary workspace used on a non-current stream is tied to that stream, so
    allocations made on the current stream meanwhile cannot reuse it."""
    g = gg.erdos_renyi(2000, 0.02, seed=5)
    ot, ow, otw = oracle_mod.score(g)
    rp, ci = harness.to_device(g)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(4):
        t, w, tw = twc.twc_score(rp, ci, stream=side)      # no workspace: a temporary each call
        junk = torch.full((1 << 22,), -1, dtype=torch.int32, device=ci.device)  # current stream
        outs.append((t, w, tw, junk))
    torch.cuda.synchronize()
    for t, w, tw, _ in outs:
        assert np.array_equal(t.cpu().numpy(), ot) and np.array_equal(tw.cpu().numpy(), otw)
