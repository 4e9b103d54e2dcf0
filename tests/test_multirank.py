"""World-size-2 gloo tests of the N > 1 host logic: max-over-ranks timing and the exchanges of the
distributed step (paper_2412_12382_b200/dist.py).  The library path itself runs in
tests/test_gpu_dist.py (emulated ranks and two real processes on one GPU)."""
import os
import socket

import numpy as np
import torch
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


def _comm_data(world, seed=3):
    """Per rank: an int32 send buffer of width-2 records grouped by destination, and the record
    counts per destination (some zero)."""
    rng = np.random.default_rng(seed)
    data = []
    for r in range(world):
        sizes = [int(x) for x in rng.integers(0, 5, size=world)]
        sizes[r] = 0
        buf = torch.from_numpy(rng.integers(0, 1000, size=max(2, 2 * sum(sizes))).astype(np.int32))
        data.append((buf, sizes))
    return data


def _comm_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2412_12382_b200 import dist as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = tdist.TorchComm()
    buf, sizes = _comm_data(world)[rank]
    recv, rsz = comm.all_to_all([buf], [sizes], 2)
    gathered = comm.all_gather([torch.tensor([rank, 10 * rank], dtype=torch.int64)])[0]
    mx = comm.max_int([7 * rank + 1])
    q.put((rank, recv[0][:2 * sum(rsz[0])].tolist(), rsz[0], gathered.tolist(), mx))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_exchanges_gloo():
    """The three exchanges of the distributed step (paper_2412_12382_b200/dist.py TorchComm:
    all-to-all of variable-size records, all-gather, max) over a real world-size-2 gloo group
    equal the in-process routing the emulated GPU tests use (dist.Emulated)."""
    from paper_2412_12382_b200 import dist as tdist
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = _comm_data(world)
    emu = tdist.Emulated(world)
    outs, rsz = emu.all_to_all([d[0] for d in data], [d[1] for d in data], 2)
    for r in range(world):
        assert res[r][1] == outs[r].tolist()
        assert res[r][2] == rsz[r]
        assert res[r][3] == [[q_, 10 * q_] for q_ in range(world)]
        assert res[r][4] == 7 * (world - 1) + 1
