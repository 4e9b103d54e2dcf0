#!/usr/bin/env python
"""Sharded scoring step: one graph split over P GPUs by pivot ranges.

    torchrun --nproc-per-node P scripts/bench_shard.py [--config 5] [--steps K]
        one process per GPU (NCCL): twc_score_shard on the rank's pivots, ONE all-reduce of the
        int32 partial counts, twc_finish_scores; device time max over ranks, "scaling": "strong"
    python scripts/bench_shard.py --emulate 2,4,8
        one GPU: each rank's shard call timed alone (ranks run one after another and never wait
        on each other), i.e. the per-rank compute of a P-GPU step; the all-reduce is NOT
        measured here (4m bytes per rank; reported as bytes only).  Not a multi-GPU number.
Prints one JSON line.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
import harness  # noqa: E402
import paper_2412_12382_b200 as twc  # noqa: E402


def timed(fn, reps, stream):
    evs = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--emulate", type=str, default="")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g = gg.config_graph(args.config)
    n, m = g.n, g.m
    rp, ci = harness.to_device(g, dev)
    ws_s = torch.empty(twc.twc_score_workspace_bytes(n, m, rp.element_size()), dtype=torch.uint8,
                       device=dev)
    ws_c = torch.empty(twc.twc_cluster_workspace_bytes(n, m, rp.element_size()),
                       dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    t_ref, _, _ = twc.twc_score(rp, ci)
    full_ms = timed(lambda: twc.twc_score(rp, ci, workspace=ws_s), args.steps, stream)
    out = {"config": args.config, "n": n, "m": m, "full_score_ms": full_ms}
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        t = torch.empty(m, dtype=torch.int32, device=dev)

        def step():
            twc.twc_score_shard(rp, ci, rank, world, out=t, workspace=ws_s)
            twc.allreduce_counts(t)
            twc.twc_finish_scores(rp, ci, t, workspace=ws_c)

        step()
        torch.cuda.synchronize()
        assert torch.equal(t, t_ref)
        dist.barrier()
        ms = timed(step, args.steps, stream)
        ms = harness.max_over_ranks(ms / 1000.0, dev) * 1000.0
        out.update({"mode": "sharded (NCCL all-reduce)", "n_gpus": world, "ms_per_step": ms,
                    "value": m / (ms / 1000.0), "unit": "edges/s", "scaling": "strong"})
        dist.destroy_process_group()
    else:
        res = {}
        t = torch.empty(m, dtype=torch.int32, device=dev)
        fin_ms = timed(lambda: twc.twc_finish_scores(rp, ci, t_ref, workspace=ws_c), args.steps,
                       stream)
        for P in [int(x) for x in args.emulate.split(",") if x]:
            acc = torch.zeros(m, dtype=torch.int32, device=dev)
            per = []
            for r in range(P):
                twc.twc_score_shard(rp, ci, r, P, out=t, workspace=ws_s)
                acc += t
                per.append(timed(lambda: twc.twc_score_shard(rp, ci, r, P, out=t, workspace=ws_s),
                                 args.steps, stream))
            torch.cuda.synchronize()
            assert torch.equal(acc, t_ref)
            res[P] = {"per_rank_shard_ms": per, "max_rank_ms": max(per),
                      "allreduce_bytes_per_rank": 4 * m}
        out.update({"mode": "one-GPU emulation of the per-rank compute (no collective measured)",
                    "finish_ms": fin_ms, "shards": res})
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
