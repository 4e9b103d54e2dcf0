#!/usr/bin/env python
"""SURVEY 8(d) "Oracle timing": the CPU oracle (oracle/, test infrastructure) as it stands, timed
on this host -- O2 (per-edge scoring), O3 (threshold filter) and O4 (BFS labelling) separately
with the oracle's own steady clock, excluding graph generation/load.  Two runs: 1 thread and all
cores (OpenMP; only O2 is parallel).  Best of 3 for configs 1-4; config 5 once.  Every config's
thresholds are its harness thresholds (reading C17); CC runs on the FULL graph.

    python scripts/oracle_baseline.py [--configs 1 2 3 4 5] [--out profiles/oracle_baseline_TAG]
Writes OUT.json and OUT.md.  A reported baseline, not an optimisation target.
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import graphgen as gg  # noqa: E402
import harness  # noqa: E402
import oracle  # noqa: E402


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        info = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                info[k.strip()] = v.strip()
        return {"model": info.get("Model name"), "sockets": info.get("Socket(s)"),
                "cores_per_socket": info.get("Core(s) per socket"),
                "threads_per_core": info.get("Thread(s) per core"), "cpus": info.get("CPU(s)"),
                "max_mhz": info.get("CPU max MHz")}
    except Exception:
        return {"model": platform.processor()}


def run_config(k, threads, reps):
    g = gg.config_graph(k)
    oracle.set_threads(threads)
    best = None
    for _ in range(reps):
        _, _, tw = oracle.score(g)
        o2 = oracle.last_times()["O2"]
        deltas = harness.thresholds(k, tw)
        o3 = o4 = 0.0
        for d in deltas:
            oracle.cluster(g, tw, d)
            tt = oracle.last_times()
            o3 += tt["O3"]
            o4 += tt["O4"]
        rec = {"O2_s": o2, "O3_s": o3, "O4_s": o4, "total_s": o2 + o3 + o4}
        if best is None or rec["total_s"] < best["total_s"]:
            best = rec
    best.update(config=k, n=g.n, m=g.m, thresholds=len(deltas), threads=threads, reps=reps,
                edges_per_s=g.m / best["total_s"], score_edges_per_s=g.m / best["O2_s"])
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "oracle_baseline"))
    a = ap.parse_args()
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    res = {"host": cpu_model(), "cores_available": cores, "runs": [],
           "note": "oracle/twc_oracle.c as it stands (gcc -O2 -fopenmp): O2 = per-edge full-list "
                   "merge (OpenMP over rows), O3 = threshold filter (materialises the kept graph), "
                   "O4 = BFS labelling in ascending id order; CC on the full graph; "
                   "steady clock inside the oracle, graph generation excluded"}
    for k in a.configs:
        for th in (1, cores):
            reps = 1 if k == 5 else 3
            t0 = time.time()
            r = run_config(k, th, reps)
            r["wall_s"] = time.time() - t0
            res["runs"].append(r)
            print(json.dumps(r), flush=True)
    with open(a.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = [f"# CPU oracle baseline ({os.path.basename(a.out)})", "",
             f"Host: {res['host'].get('model')}, {cores} cores available "
             f"(lscpu: {res['host']}).  {res['note']}.", "",
             "| config | n | m | thresholds | threads | O2 score s | O3 filter s | O4 BFS s | "
             "total s | edges/s (whole path) |", "|---|---|---|---|---|---|---|---|---|---|"]
    for r in res["runs"]:
        lines.append(f"| {r['config']} | {r['n']:,} | {r['m']:,} | {r['thresholds']} | "
                     f"{r['threads']} | {r['O2_s']:.4f} | {r['O3_s']:.4f} | {r['O4_s']:.4f} | "
                     f"{r['total_s']:.4f} | {r['edges_per_s']:.3e} |")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
