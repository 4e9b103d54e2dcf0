#!/usr/bin/env python
"""Per-rank cost of the distributed step (paper_2412_12382_b200/dist.py) on ONE GPU.

    python scripts/bench_dist_emulated.py [--config 5] [--worlds 1,2,4,8] [--reps 5]

All P ranks of one graph run on this GPU one after the other (dist.Emulated: the exchanges are
routed in process), and every phase of every rank is timed alone with CUDA events (ranks never
wait on each other).  Reported per P: each phase's max over ranks, the per-rank compute of the
slowest rank, and the bytes each exchange moves per rank.  The exchanges themselves are NOT
measured here (one GPU): `model_ms` adds them at an assumed 400 GB/s per-rank NVLink rate plus
25 us per collective -- a model, not a multi-GPU measurement.  Prints one JSON line.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
import harness  # noqa: E402
import paper_2412_12382_b200 as twc  # noqa: E402
from paper_2412_12382_b200 import dist as tdist  # noqa: E402

NVLINK_GBS = 400.0
COLL_US = 25.0


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def run_timed(ranks, comm):
    """run_phases with per-rank, per-phase events."""
    T = {r.rank: {} for r in ranks}

    def tm(r, name, fn, *a):
        e0 = ev()
        out = fn(*a)
        e1 = ev()
        T[r.rank][name] = (e0, e1)
        return out

    sends, sizes = zip(*[tm(r, "A_count", r.count) for r in ranks])
    recvs, rsz = comm.all_to_all(list(sends), list(sizes), 2)
    for r, b, s in zip(ranks, recvs, rsz):
        tm(r, "B_apply", r.apply, b, sum(s))
    reqs, qsz = zip(*[tm(r, "C_epilogue", r.epilogue) for r in ranks])
    req_in, rin = comm.all_to_all(list(reqs), list(qsz), 1)
    outs = [tm(r, "D_serve", r.serve, b, sum(s)) for r, b, s in zip(ranks, req_in, rin)]
    replies, _ = comm.all_to_all(outs, rin, 1)
    nf = [tm(r, "E_forest", r.forest_phase, rep) for r, rep in zip(ranks, replies)]
    cap = max(1, comm.max_int(nf))
    forests = comm.all_gather([r.forest[:2 * cap] for r in ranks])
    fcum = comm.all_gather([r.forest_cum for r in ranks])
    kept = comm.all_gather([r.kept_sizes for r in ranks])
    for r, f, c, k in zip(ranks, forests, fcum, kept):
        tm(r, "F_sweep", r.sweep, f.contiguous(), cap, c.contiguous(), k.contiguous())
    torch.cuda.synchronize()
    ms = {rk: {k: a.elapsed_time(b) for k, (a, b) in d.items()} for rk, d in T.items()}
    vol = {"ex1_count_pairs_bytes": [8 * sum(s) for s in rsz],
           "ex2_request_bytes": [4 * sum(s) for s in rin],
           "ex2_reply_bytes": [4 * sum(s) for s in rin],
           "ex3_forest_bytes": [8 * cap * len(ranks)] * len(ranks)}
    return ms, vol


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    twc.load_library()
    g = gg.config_graph(a.config)
    rp, ci = harness.to_device(g)
    _, _, tw = twc.twc_score(rp, ci)
    deltas = harness.thresholds(a.config, tw.cpu().numpy())
    out = {"config": a.config, "n": g.n, "m": g.m, "k": len(deltas), "worlds": {}}
    for P in [int(x) for x in a.worlds.split(",")]:
        ranks = [tdist.DistRank(rp, ci, deltas, r, P) for r in range(P)]
        comm = tdist.Emulated(P)
        run_timed(ranks, comm)                       # warm
        reps = []
        for _ in range(a.reps):
            reps.append(run_timed(ranks, comm))
        phases = sorted(reps[0][0][0])
        per = {ph: statistics.median(max(ms[r][ph] for r in ms) for ms, _ in reps)
               for ph in phases}
        rank_ms = statistics.median(max(sum(ms[r].values()) for r in ms) for ms, _ in reps)
        vol = reps[0][1]
        ex_ms = sum(max(v) / (NVLINK_GBS * 1e6) for v in vol.values()) + 4 * COLL_US / 1000.0
        out["worlds"][P] = {"phase_ms_max_over_ranks": per, "slowest_rank_compute_ms": rank_ms,
                            "exchange_bytes_per_rank_max": {k: max(v) for k, v in vol.items()},
                            "model_ms": rank_ms + (ex_ms if P > 1 else 0.0),
                            "model_edges_per_s": g.m / ((rank_ms + (ex_ms if P > 1 else 0.0)) / 1e3)}
        print(P, json.dumps(out["worlds"][P]), file=sys.stderr, flush=True)
        del ranks
        torch.cuda.empty_cache()
    out["note"] = ("one GPU, ranks timed one after the other; model_ms = slowest rank's compute + "
                   f"exchange bytes at {NVLINK_GBS:g} GB/s + {COLL_US:g} us per collective (a "
                   "model, not a multi-GPU measurement)")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
