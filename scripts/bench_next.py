#!/usr/bin/env python
"""Measurements of the NEXT rows beside the headline bench:

* K4 participation (NEXT(4)): twc_score_k4 vs twc_score on config 5 and R-MAT graphs (CUDA
  events, L2 flushed, median of 5); the K4 share = the difference.  The CPU oracle's K4 on the
  same graph is timed beside it (OpenMP, all host cores) as the reported baseline.
* Table-1 fp64 scores (NEXT(1)): twc_similarity per kind on config 5.

Writes profiles/next_<tag>.json and prints one JSON line per measurement.

    python scripts/bench_next.py [--tag r1] [--graphs 5,rmat-s-1e7,rmat-vs-1e7] [--no-oracle]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc


def graph(name):
    return gg.rmat_graph(name[5:]) if name.startswith("rmat-") else gg.config_graph(int(name))


def timed(fn, flush, reps=5):
    out = []
    for i in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--graphs", default="5,rmat-s-1e7,rmat-vs-1e7")
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    twc.load_library()
    dev = torch.device("cuda")
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev)
    res = []
    for name in args.graphs.split(","):
        g = graph(name)
        n, m = g.n, g.m
        rp, ci = harness.to_device(g, dev)
        rb = rp.element_size()
        ws = torch.empty(twc.twc_score_k4_workspace_bytes(n, m, rb), dtype=torch.uint8, device=dev)
        out = tuple(torch.empty(m, dtype=torch.int32, device=dev) for _ in range(3)) + (
            torch.empty(m, dtype=torch.int64, device=dev),)
        score_ms = timed(lambda: twc.twc_score(rp, ci, out=out[:3], workspace=ws), flush)
        k4_ms = timed(lambda: twc.twc_score_k4(rp, ci, out=out, workspace=ws), flush)
        k4 = out[3]
        line = {"what": "k4", "graph": name, "n": n, "m": m,
                "k4_total": int(k4.sum().item()) // 6,
                "score_ms": score_ms, "score_k4_ms": k4_ms, "k4_ms": k4_ms - score_ms,
                "k4_edges_per_s": m / ((k4_ms - score_ms) / 1e3)}
        if not args.no_oracle:
            import oracle
            oracle.set_threads(oracle.max_threads())
            t0 = time.perf_counter()
            ok4 = oracle.k4(g)
            dt = time.perf_counter() - t0
            assert np.array_equal(ok4, k4.cpu().numpy())
            line["oracle_k4_s"] = dt
            line["oracle_cores"] = oracle.max_threads()
            line["oracle_k4_edges_per_s"] = m / dt
        print(json.dumps(line), flush=True)
        res.append(line)
        if name == "5":
            t = out[0]
            score = torch.empty(m, dtype=torch.float64, device=dev)
            wsc = torch.empty(twc.twc_cluster_workspace_bytes(n, m, rb), dtype=torch.uint8,
                              device=dev)
            for kind in twc.SIM_KINDS:
                ms = timed(lambda: twc.twc_similarity(rp, ci, t, kind, out=score, workspace=wsc),
                           flush)
                # degree kinds: t, colidx, deg(u) + deg(v), the 8-byte score; K3 / -R_eff read t only
                bpe = 4 + 8 if kind in ("k3", "effres") else 4 + 8 + 8 + 4
                line = {"what": "similarity", "graph": name, "kind": kind, "ms": ms,
                        "edges_per_s": m / (ms / 1e3),
                        "bytes_per_edge_model": bpe,
                        "achieved_gbs_model": m * bpe / (ms / 1e3) / 1e9}
                print(json.dumps(line), flush=True)
                res.append(line)
        del rp, ci, ws, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"next_{args.tag}.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
