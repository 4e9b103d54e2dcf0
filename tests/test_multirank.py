"""World-size-2 gloo tests of the N > 1 host logic: bench.py's replicas and max-over-ranks, and
the exchange step of the sharded scoring path (partial counts per rank, one
all-reduce, the sum is t).  The GPU kernels themselves are covered by tests/test_gpu_shard.py;
here each rank's partial comes from the reference of the shard contract (tests/shard_ref.py)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

import graphgen as gg
import harness


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
    g = gg.config_graph(1)                      # every rank builds the same replica
    local_s = 1.0 + rank                        # rank-dependent "device time"
    mx = harness.max_over_ranks(local_s)
    val = harness.weak_scaling_value(g.m * 10, world, mx)
    q.put((rank, g.sha256(), mx, val))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shas = {r[1] for r in res}
    assert len(shas) == 1                          # identical replicas on every rank
    assert all(r[2] == 2.0 for r in res)           # max over ranks, on every rank
    m = gg.config_graph(1).m
    assert np.isclose(res[0][3], 2 * m * 10 / 2.0)


def test_single_process_is_identity():
    assert harness.max_over_ranks(3.5) == 3.5
    assert harness.weak_scaling_value(100, 1, 2.0) == 50.0


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_2412_12382_b200 as twc
    import shard_ref
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = gg.erdos_renyi(45, 0.3, seed=5)
    part = shard_ref.partial_counts(g, world)[rank]
    t = torch.from_numpy(part.astype(np.int32))
    twc.allreduce_counts(t)                      # the exchange step (NCCL on the GPU nodes)
    q.put((rank, t.numpy().tolist(), int(part.sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_counts_gloo(oracle_mod):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ot = oracle_mod.score(gg.erdos_renyi(45, 0.3, seed=5))[0]
    for _, t, _ in res:
        assert np.array_equal(np.array(t), ot)       # every rank holds the full t
    assert all(r[2] > 0 for r in res)              # both ranks had triangles to count
