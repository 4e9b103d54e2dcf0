#!/usr/bin/env python
"""R-MAT workloads of Table "tab:syn" on one B200.

For each graph: scoring time (twc_score, device-resident CSR, CUDA events, L2 flushed), score +
cluster at one threshold (the median TW; R-MAT's TW is negative everywhere), and the same end to
end from pinned host buffers through twc_pipeline_host (one synchronous call).  The paper's
16-thread CPU time for its TW framework on the same (n, m) is printed beside it as context only
(other hardware, other implementation).  One JSON line per graph; the list is also written to
profiles/rmat_<tag>.json.

    python scripts/bench_rmat.py [--tag r1] [--graphs vs-1e7,s-1e7,...] [--reps 10]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--graphs", default=",".join(gg.RMAT_CONFIGS))
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    twc.load_library()
    dev = torch.device("cuda")
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev)
    out = []
    for name in args.graphs.split(","):
        t0 = time.time()
        g = gg.rmat_graph(name)
        gen_s = time.time() - t0
        n, m = g.n, g.m
        rp, ci = harness.to_device(g, dev)
        rb = rp.element_size()
        ws_s = torch.empty(twc.twc_score_workspace_bytes(n, m, rb), dtype=torch.uint8, device=dev)
        ws_c = torch.empty(twc.twc_cluster_workspace_bytes(n, m, rb), dtype=torch.uint8, device=dev)
        t, w, tw = (torch.empty(m, dtype=torch.int32, device=dev) for _ in range(3))
        labels = torch.empty(n, dtype=torch.int32, device=dev)
        stats = torch.empty(2, dtype=torch.int64, device=dev)
        twc.twc_score(rp, ci, out=(t, w, tw), workspace=ws_s)
        torch.cuda.synchronize()
        delta = harness.nearest_rank(tw.cpu().numpy(), 50)
        sc, cl = [], []
        for i in range(args.reps + 3):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            twc.twc_score(rp, ci, out=(t, w, tw), workspace=ws_s)
            e[1].record()
            twc.twc_cluster(rp, ci, tw, delta, labels=labels, stats=stats, workspace=ws_c)
            e[2].record()
            torch.cuda.synchronize()
            if i >= 3:
                sc.append(e[0].elapsed_time(e[1]))
                cl.append(e[0].elapsed_time(e[2]))
        rp_h = torch.from_numpy(np.ascontiguousarray(g.rowptr)).pin_memory()
        ci_h = torch.from_numpy(np.ascontiguousarray(g.colidx)).pin_memory()
        ws_p = torch.empty(twc.twc_pipeline_workspace_bytes(n, m, rb, 1), dtype=torch.uint8,
                           device=dev)
        res = {"tw": torch.empty(m, dtype=torch.int32, pin_memory=True),
               "labels": torch.empty((1, n), dtype=torch.int32, pin_memory=True),
               "stats": torch.empty((1, 2), dtype=torch.int64, pin_memory=True)}
        e2e = []
        for i in range(max(3, args.reps // 2) + 1):
            t1 = time.perf_counter()
            twc.twc_pipeline_host(rp_h, ci_h, [delta], out=res, workspace=ws_p, device=dev)
            if i:
                e2e.append(time.perf_counter() - t1)
        assert torch.equal(res["labels"][0], labels.cpu())
        deg = np.diff(g.rowptr.astype(np.int64))
        paper = gg.RMAT_CONFIGS[name]["paper_tw_s"]
        cl_ms = statistics.median(cl)
        line = {"graph": "rmat-" + name, "n": n, "m_requested": gg.RMAT_CONFIGS[name]["m"],
                "m": m, "max_degree": int(deg.max()), "triangles": int(t.sum(dtype=torch.int64).item()) // 3,
                "delta_p50": delta, "kept": int(stats[0].item()), "components": int(stats[1].item()),
                "score_ms": statistics.median(sc), "score_edges_per_s": m / (statistics.median(sc) / 1e3),
                "score_cluster_ms": cl_ms, "score_cluster_edges_per_s": m / (cl_ms / 1e3),
                "e2e_pipeline_host_ms": 1e3 * statistics.median(e2e),
                "e2e_edges_per_s": m / statistics.median(e2e),
                "paper_tw_16threads_s": paper,
                "context_ratio_vs_paper_cpu": paper / (cl_ms / 1e3),
                "generation_s": gen_s}
        print(json.dumps(line), flush=True)
        out.append(line)
        del rp, ci, ws_s, ws_c, t, w, tw, ws_p
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"rmat_{args.tag}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
