"""GPU parity of the distributed step (include/twc.h twc_dist_*): one graph split
over P ranks.  Emulated (all ranks on this GPU, one after the other, the exchanges routed in
process): the union of the ranks' canonical slices must equal the oracle's t, wedge and TW
element by element, every rank's labels and stats must equal the oracle's (min-id labels), for
P = 1..8, including BASELINE config 5 at full size with its 16 thresholds.  Two real processes
(torch.distributed, gloo, both on cuda:0; the exchanges go through the host, no kernel waits on
another process) run the same library path through TorchComm."""
import math
import os
import socket

import numpy as np
import pytest
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc
from paper_2412_12382_b200 import build as twc_build
from paper_2412_12382_b200 import dist as tdist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests need a B200 (there is no CPU fallback)")
    twc_build.build()
    twc.load_library()


def check_emulated(oracle_mod, g, deltas, world, ref=None):
    ot, ow, otw = ref if ref is not None else oracle_mod.score(g)
    rp, ci = harness.to_device(g)
    ranks, info = tdist.score_sweep_emulated(rp, ci, deltas, world)
    torch.cuda.synchronize()
    rows, cb = tdist.slice_bounds(rp, ci, world)
    t = np.zeros(g.m, np.int32)
    w = np.zeros(g.m, np.int32)
    tw = np.zeros(g.m, np.int32)
    for r, rk in enumerate(ranks):
        c0, c1 = cb[r], cb[r + 1]
        t[c0:c1] = rk.t[c0:c1].cpu().numpy()
        w[c0:c1] = rk.wedge[c0:c1].cpu().numpy()
        tw[c0:c1] = rk.tw[c0:c1].cpu().numpy()
    for a, b, what in ((t, ot, "t"), (w, ow, "wedge"), (tw, otw, "tw")):
        bad = np.nonzero(a != b)[0]
        assert bad.size == 0, f"P={world} {what}: {bad.size} mismatches, first {bad[:5]}"
    lab0, st0 = ranks[0].labels.cpu().numpy(), ranks[0].stats.cpu().numpy()
    for i, d in enumerate(deltas):
        ol, kept, ncomp = oracle_mod.cluster(g, otw, d)
        assert np.array_equal(lab0[i], ol), (world, d)
        assert (int(st0[i, 0]), int(st0[i, 1])) == (kept, ncomp), (world, d)
    for rk in ranks[1:]:
        assert np.array_equal(rk.labels.cpu().numpy(), lab0)
        assert np.array_equal(rk.stats.cpu().numpy(), st0)
    return info


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
def test_emulated_small_graphs(oracle_mod, world):
    rng = np.random.default_rng(70 + world)
    graphs = [gg.complete(40), gg.star(300, 7), gg.bridge_triangles(), gg.path(50),
              gg.config_graph(1), gg.erdos_renyi(1500, 0.01, seed=3)]
    for it in range(4):
        n = int(rng.integers(2, 2500))
        graphs.append(gg.erdos_renyi(n, float(rng.random()) * min(1.0, 30.0 / n), seed=90 + it))
    for g in graphs:
        if g.m == 0:
            continue
        otw = oracle_mod.score(g)[2]
        deltas = sorted({-math.inf, float(np.median(otw)), float(otw.max()) + 1, 0.0, -3.0})
        check_emulated(oracle_mod, g, deltas, world)


def test_emulated_int64_rowptr_and_duplicate_thresholds(oracle_mod):
    g = gg.erdos_renyi(2000, 0.01, seed=8).with_rowptr_dtype(np.int64)
    check_emulated(oracle_mod, g, [-2.0, -2.0, 0.5, math.inf, -math.inf], 3)


@pytest.mark.parametrize("config", [2, 3, 4])
@pytest.mark.parametrize("world", [2, 4])
def test_emulated_configs(oracle_mod, config, world):
    g = gg.config_graph(config)
    ref = oracle_mod.score(g)
    info = check_emulated(oracle_mod, g, harness.thresholds(config, ref[2]), world, ref)
    assert sum(x["counts_pairs_in"] for x in info) > 0      # counts really crossed ranks


@pytest.mark.slow
def test_emulated_config5_full_size(oracle_mod):
    """BASELINE config 5 (35M edges, 16 thresholds) split over P = 2, 4, 8: scores and labels
    identical to the oracle's (the P partial count arrays sum to t exactly)."""
    oracle_mod.set_threads(oracle_mod.max_threads())
    g = gg.config_graph(5)
    ref = oracle_mod.score(g)
    for world in (2, 4, 8):
        check_emulated(oracle_mod, g, harness.SWEEP_GRID, world, ref)
        torch.cuda.empty_cache()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    twc.load_library()
    g = gg.config_graph(2)
    rp, ci = harness.to_device(g, "cuda:0")
    deltas = [-20.0, -15.0, -10.0]
    t, w, tw, lab, st, info = tdist.score_sweep_distributed(rp, ci, deltas)
    torch.cuda.synchronize()
    q.put((rank, t.cpu().numpy(), w.cpu().numpy(), tw.cpu().numpy(), lab.cpu().numpy(),
           st.cpu().numpy(), info))
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_gloo_library_path(oracle_mod):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = gg.config_graph(2)
    ot, ow, otw = oracle_mod.score(g)
    rp, ci = harness.to_device(g)
    _, cb = tdist.slice_bounds(rp, ci, world)
    t = np.concatenate([res[r][1][cb[r]:cb[r + 1]] for r in range(world)])
    tw = np.concatenate([res[r][3][cb[r]:cb[r + 1]] for r in range(world)])
    assert np.array_equal(t, ot) and np.array_equal(tw, otw)
    for i, d in enumerate([-20.0, -15.0, -10.0]):
        ol, kept, ncomp = oracle_mod.cluster(g, otw, d)
        for r in range(world):
            assert np.array_equal(res[r][4][i], ol)
            assert (int(res[r][5][i, 0]), int(res[r][5][i, 1])) == (kept, ncomp)
    assert res[0][6]["counts_pairs_in"] > 0 and res[1][6]["requests_in"] > 0
