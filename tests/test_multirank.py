"""World-size-2 gloo test of the N > 1 host logic of bench.py (replicas, max-over-ranks)."""
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
