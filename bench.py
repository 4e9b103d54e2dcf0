#!/usr/bin/env python
"""bench.py -- TW scoring + threshold sweep (arXiv 2412.12382, Alg. 1 with Eq. 2) on B200.

One step = the whole hot path on BASELINE config 5 (DC-SBM,
n = 4,000,000, m ~ 35M, int64 rowptr): twc_score (orientation, intersection, fused score
epilogue) followed by twc_sweep over the 16 thresholds -30, -28, ..., 0 reusing the
scores (filter + connected components per threshold).  Inputs are resident in HBM when the
timed region starts; `e2e` times the same step through twc_pipeline_host_async from pinned
host buffers (H2D of the whole CSR and D2H of TW + labels + stats of every step inside the
timed region, three steps in flight so one step's copies back overlap the next steps' copy in;
the single synchronous call's latency is reported beside it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

N > 1 runs under torchrun: every rank scores its own replica of the workload (independent
problems, no data-path collective, "scaling": "weak").  --impl reference
times the CPU oracle (oracle/, test infrastructure) on bounded samples of the same workload.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen as gg  # noqa: E402
import harness  # noqa: E402

METRIC = "edges scored/sec (TW) and end-to-end cluster time; achieved HBM GB/s vs peak"
UNIT = "edges/s"
E2E_INFLIGHT = 3  # twc_pipeline_host_async calls in flight in the e2e measurement
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # N > 1: NCCL on a B200 node.  gloo + --same-device runs every rank on cuda:0 with host-side
    # exchanges (a functional check of this code path on a one-GPU box, not a measurement)
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--same-device", action="store_true")
    return ap.parse_args()


def config_dict(cfg, g, deltas, world):
    """The `config` object of the JSON line; identical for both arms (--impl b200|reference)."""
    return {"workload": workload_desc(cfg, g, len(deltas)), "n": g.n, "m": g.m,
            "thresholds": list(deltas), "rowptr": str(g.rowptr.dtype),
            "graph_sha256": g.sha256(),
            "parallelism": (f"one graph split over {world} GPUs (SURVEY 8(e) row ranges, NCCL "
                            "exchanges)") if world > 1 else "single GPU",
            "l2": "explicit 512 MiB L2 flush between timed steps; inputs (CSR 312 MB) and "
                  "outputs exceed the 126 MB L2"}


def workload_desc(cfg, g, k):
    c = gg.CONFIGS[cfg]
    kind = "planted-partition SBM" if c["kind"] == "pp" else "degree-corrected SBM"
    return (f"config{cfg}: {kind} n={g.n} m={g.m} (BASELINE.json configs[{cfg - 1}], seed "
            f"{c['seed']}); step = twc_score_sweep: score + {k}-threshold filter + CC sweep, fused")


# ----------------------------------------------------------------------------- host stats
def orientation_stats(g):
    """Sum_v d-(v) d+(v) for the degree orientation (the pivot-staged intersection volume)."""
    rp = g.rowptr.astype(np.int64)
    deg = np.diff(rp)
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    dst = g.colidx.astype(np.int64)
    out = (deg[src] < deg[dst]) | ((deg[src] == deg[dst]) & (src < dst))
    dplus = np.bincount(src[out], minlength=g.n).astype(np.int64)
    dminus = deg - dplus
    return int((dminus * dplus).sum()), int(dplus.max()) if g.n else 0


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(graph_sha):
    """DRAM bytes per K2 launch from the committed `ncu --set full` capture
    (profiles/k2_ncu_summary.json, written by scripts/summarize_ncu.py), used only when that
    capture profiled THIS graph (same sha256); else (None, None)."""
    p = os.path.join(ROOT, "profiles", "k2_ncu_summary.json")
    try:
        d = json.load(open(p))
    except Exception:
        return None, None
    if d.get("graph_sha256") != graph_sha:
        return None, None
    return d.get("dram_bytes_per_launch"), d


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        if getattr(self, "_summary", None) is not None:
            return self._summary
        self._summary = self._summarize()
        return self._summary

    def _summarize(self):
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


# ----------------------------------------------------------------------------- CPU oracle arm
# The oracle (oracle/, test infrastructure) as it stands, timed with its own steady clock
# (oracle.last_times: O2 scoring, O3 filter, O4 BFS labelling).  Scoring uses all
# host cores (OpenMP over rows); the filter and the BFS are single-threaded and run on the FULL
# graph, like the GPU sweep.
def row_windows(g, n_windows=64):
    """Row windows [r0, r1) with their canonical edge ranges [a, b) (harness bookkeeping)."""
    s, _ = g.canonical_pairs()
    bounds = np.linspace(0, g.n, n_windows + 1).astype(np.int64)
    lo = np.searchsorted(s, bounds[:-1], side="left")
    hi = np.searchsorted(s, bounds[1:], side="left")
    return [(int(bounds[w]), int(bounds[w + 1]), int(lo[w]), int(hi[w])) for w in range(n_windows)]


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_cpu_baseline(g, deltas, cc_thresholds=2):
    """The whole path on the whole workload where affordable: O2 over ALL canonical edges (all
    cores), then O3 + O4 on the full graph for `cc_thresholds` of the k thresholds (the two
    extremes), extrapolated to k.  ~15-30 s on config 5."""
    import oracle
    oracle.build()
    cores = cpu_cores()
    oracle.set_threads(cores)
    _, _, tw = oracle.score(g)
    o2 = oracle.last_times()["O2"]
    k = len(deltas)
    pick = sorted(set([0, k - 1][:cc_thresholds])) if k > cc_thresholds else list(range(k))
    o3 = o4 = 0.0
    for i in pick:
        oracle.cluster(g, tw, deltas[i])
        tt = oracle.last_times()
        o3 += tt["O3"]
        o4 += tt["O4"]
    scale = k / len(pick)
    total = o2 + scale * (o3 + o4)
    return {"value": g.m / total, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "phases_s": {"O2_score": o2, "O3_filter": o3 * scale, "O4_bfs": o4 * scale},
            "sample": (f"all {g.m} canonical edges scored (O2, {cores} OpenMP threads, "
                       f"{o2:.1f} s); filter (O3) + BFS labelling (O4) on the full graph, "
                       f"single thread, timed at {len(pick)} of the {k} thresholds "
                       f"({', '.join(str(deltas[i]) for i in pick)}) and scaled x{scale:g}")}


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    g = gg.config_graph(cfg)
    import oracle
    oracle.build()
    cores = cpu_cores()
    oracle.set_threads(cores)
    _, _, tw = oracle.score(g)            # setup: the full TW the CC steps filter (untimed)
    deltas = harness.thresholds(cfg, tw)
    k = len(deltas)
    # a step scores 1/8 of the rows of config 5 (~2 s; the oracle's per-call canonical-offset
    # pass then costs a few %), all rows of the smaller configs
    wins = row_windows(g, 8 if g.m > 10_000_000 else 1)

    def step(i):
        r0, r1, a, b = wins[i % len(wins)]
        oracle.score(g, rows=(r0, r1))
        o2 = oracle.last_times()["O2"]
        oracle.cluster(g, tw, deltas[i % k])
        tt = oracle.last_times()
        return b - a, o2, tt["O3"] + tt["O4"]

    for i in range(args.warmup):
        step(i)
    edges = 0
    o2s = 0.0
    ccs = []
    for i in range(args.steps):
        e, o2, cc = step(args.warmup + i)
        edges += e
        o2s += o2
        ccs.append(cc)
    # each step = one row window scored + the full-graph CC at one threshold; the metric
    # is edges/s of the whole path: the measured scoring rate over all m edges plus k CC passes
    full_s = g.m / (edges / o2s) + k * statistics.mean(ccs)
    value = g.m / full_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * full_s, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config_dict(cfg, g, deltas, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": (f"each step = one of {len(wins)} row windows of config "
                                        f"{cfg} scored (O2, {cores} threads) + filter and BFS "
                                        f"labelling of the FULL graph at one of the {k} "
                                        "thresholds (cycling); ms_per_step = the extrapolated "
                                        "whole step: m / (measured scoring rate) + k x mean "
                                        "CC pass")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- B200 arm
def main_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2412_12382_b200 as twc
    from paper_2412_12382_b200 import build as twc_build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        twc_build.build()
    if world > 1:
        dist.barrier()
    twc.load_library()

    cfg = args.config
    g = gg.config_graph(cfg)
    n, m = g.n, g.m
    rp, ci = harness.to_device(g, dev)
    rb = rp.element_size()
    stream = torch.cuda.current_stream()
    ws_s = torch.empty(twc.twc_score_workspace_bytes(n, m, rb), dtype=torch.uint8, device=dev)
    ws_c = torch.empty(twc.twc_cluster_workspace_bytes(n, m, rb), dtype=torch.uint8, device=dev)
    ws_f = torch.empty(twc.twc_score_sweep_workspace_bytes(n, m, rb), dtype=torch.uint8,
                       device=dev)
    t, w, tw = (torch.empty(m, dtype=torch.int32, device=dev) for _ in range(3))
    twc.twc_score(rp, ci, out=(t, w, tw), workspace=ws_s)
    torch.cuda.synchronize()
    deltas = harness.thresholds(cfg, tw.cpu().numpy())
    k = len(deltas)
    labels = torch.empty((k, n), dtype=torch.int32, device=dev)
    stats = torch.empty((k, 2), dtype=torch.int64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def mk(nev):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
        for e in evs:
            e.record(stream)
        return evs

    def step(ev=None):
        # the whole hot path, fused: score (orient, intersect, epilogue + band binning) + sweep
        twc.twc_score_sweep(rp, ci, deltas, out=(t, w, tw), labels=labels, stats=stats,
                            workspace=ws_f, events=ev)

    def step_separate(se=None, we=None):
        # the same path through the two separate ABI calls
        twc.twc_score(rp, ci, out=(t, w, tw), workspace=ws_s, events=se)
        twc.twc_sweep(rp, ci, tw, deltas, labels=labels, stats=stats, workspace=ws_c, events=we)

    for _ in range(args.warmup):
        step()
        step_separate()
    torch.cuda.synchronize()

    K = args.steps
    fev = [mk(6) for _ in range(K)]
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    torch.cuda.synchronize()
    l0 = twc.twc_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        wall0 = time.perf_counter()
        for i in range(K):
            flush.zero_()                      # L2 flush between timed steps (not timed)
            starts[i].record(stream)
            step(fev[i])
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    launches = (twc.twc_kernel_launches() - l0) / K
    step_ms = [starts[i].elapsed_time(ends[i]) for i in range(K)]

    def ph(a, b):
        return statistics.mean(fev[i][a].elapsed_time(fev[i][b]) for i in range(K))

    k2_ms = [fev[i][1].elapsed_time(fev[i][2]) for i in range(K)]
    phases = {"orient": ph(0, 1), "intersect_k2": ph(1, 2), "epilogue_k3_bin": ph(2, 3),
              "band_place": ph(3, 4), "sweep16_loop": ph(4, 5), "score": ph(0, 3)}
    total_s = harness.max_over_ranks(sum(step_ms) / 1000.0, dev)
    value = harness.weak_scaling_value(m * K, world, total_s)
    ms_per_step = 1000.0 * total_s / K

    # ---- the same step through the separate twc_score + twc_sweep calls (context)
    Ks = min(K, 10)
    sev = [mk(4) for _ in range(Ks)]
    wev = [mk(3) for _ in range(Ks)]
    torch.cuda.synchronize()
    for i in range(Ks):
        flush.zero_()
        step_separate(sev[i], wev[i])
    torch.cuda.synchronize()
    separate = {"score_ms": statistics.mean(sev[i][0].elapsed_time(sev[i][3]) for i in range(Ks)),
                "sweep16_ms": statistics.mean(wev[i][0].elapsed_time(wev[i][2]) for i in range(Ks))}
    separate["step_ms"] = separate["score_ms"] + separate["sweep16_ms"]

    # ---- the same fused step captured once in a CUDA graph and replayed (the library makes no
    # host synchronisation and no host->device copy inside the call, so it is capturable)
    graph = None
    try:
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            step()                              # warm on the capture stream
            torch.cuda.synchronize()
            with torch.cuda.graph(cg, stream=gs):
                step()
        torch.cuda.synchronize()
        Kg = min(K, 20)
        gse = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(Kg)]
        for i in range(Kg):
            flush.zero_()
            gse[i][0].record(stream)
            cg.replay()
            gse[i][1].record(stream)
        torch.cuda.synchronize()
        g_ms = statistics.mean(a.elapsed_time(b) for a, b in gse)
        graph = {"ms_per_step": g_ms, "value": m / (g_ms / 1000.0), "steps": Kg,
                 "note": "twc_score_sweep captured in one CUDA graph, replayed; L2 flushed between"}
        del cg
    except Exception as exc:  # capture is reported, never required
        graph = {"error": repr(exc)[:200]}

    # ---- NEXT(2): statistics of the k partitions + the selection rules (reported, not in value)
    ws_ps = torch.empty(max(1, twc.twc_partition_stats_workspace_bytes(n, m, rb)),
                        dtype=torch.uint8, device=dev)
    counts = torch.empty((k, 4), dtype=torch.int64, device=dev)
    qv = torch.empty(k, dtype=torch.float64, device=dev)
    twc.twc_partition_stats(rp, ci, labels, counts=counts, modularity=qv, workspace=ws_ps)
    st_ms = []
    for _ in range(3):
        flush.zero_()
        e0, e1 = mk(2)
        e0.record(stream)
        twc.twc_partition_stats(rp, ci, labels, counts=counts, modularity=qv, workspace=ws_ps)
        e1.record(stream)
        torch.cuda.synchronize()
        st_ms.append(e0.elapsed_time(e1))
    cl, ql, sl = counts.cpu().tolist(), qv.cpu().tolist(), stats.cpu().tolist()
    idx, rule = twc.twc_select_threshold(deltas, [c[1] for c in cl], ql, n)
    selection = {"partition_stats_ms": statistics.mean(st_ms), "k": k,
                 "selected_delta": deltas[idx], "rule": rule, "modularity": ql[idx],
                 "norm_cc": cl[idx][0] / n, "norm_edges": sl[idx][0] / m,
                 "norm_largest_cc": cl[idx][1] / n}

    # ---- roofline of the dominant kernel (K2, oriented intersection), DESIGN.md Sec. 6
    # algorithmic bytes of the pivot-staged intersection = 4 (m + S), S = sum_v
    # d-(v) d+(v) (N+(u) read once per pivot, N+(v) once per in-edge), exact from this graph.
    S, dplus_max = orientation_stats(g)
    T = int(t.sum(dtype=torch.int64).item()) // 3
    k2_bytes = 4 * (m + S)
    k2_bytes_ext = 4 * (n + 1 + 4 * m + S + T)
    k2_avg_s = statistics.mean(k2_ms) / 1000.0
    peak, peak_src = measured_peak()
    achieved = k2_bytes / k2_avg_s / 1e9
    graph_sha = g.sha256()
    traffic, k2prof = ncu_traffic(graph_sha)
    roofline = {"bound": "hbm", "kernel": "k2_intersect", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": k2_bytes,
                "algorithmic_model": "SURVEY 8(d) pivot-staged: 4*(m + S), S = sum_v d-(v)*d+(v)",
                "peak_source": peak_src, "k2_ms_avg": 1000 * k2_avg_s,
                "frac_of_8000": achieved / 8000.0,
                "extended_model": {
                    "bytes": k2_bytes_ext, "achieved": k2_bytes_ext / k2_avg_s / 1e9,
                    "frac": k2_bytes_ext / k2_avg_s / 1e9 / peak,
                    "model": "4*(n+1 + 4m + S + T): + rp_or per pivot and per out-neighbour, "
                             "one count flush per slot, one RED per triangle"}}
    if traffic:
        # SURVEY 8(d) figure 1: measured DRAM bytes per launch (ncu capture of this graph, tag
        # below) over the live K2 time, against the measured copy peak and north_star's ~8 TB/s
        dram_gbs = traffic / k2_avg_s / 1e9
        roofline["traffic_source"] = {"tag": k2prof.get("tag"), "file": k2prof.get("source"),
                                      "ncu_k2_duration": k2prof.get("duration")}
        roofline["dram"] = {"achieved": dram_gbs, "unit": "GB/s", "frac": dram_gbs / peak,
                            "frac_of_8000": dram_gbs / 8000.0,
                            "traffic_over_algorithmic": traffic / k2_bytes}
    if k2prof and k2prof.get("l2_sectors_per_launch"):
        # SURVEY 8(d) figure 3: L2 traffic (32-byte sectors of the same capture) over the live time
        roofline["l2"] = {"achieved": 32.0 * k2prof["l2_sectors_per_launch"] / k2_avg_s / 1e9,
                          "unit": "GB/s", "hit_pct": k2prof.get("l2_hit_pct"),
                          "lsu_pipe_pct": k2prof.get("lsu_pipe_pct"),
                          "warp_execution_efficiency": (k2prof.get("threads_per_inst") or 0) / 32.0}
    if k2prof and k2prof.get("warp_inst_per_launch"):
        # K2 is co-limited by instruction issue and the L1/shared pipe: its
        # warp instructions per launch (same capture) over the live K2 time, against 4
        # schedulers x SMs x max SM clock (one warp instruction per cycle each)
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        smax = clk.summary().get("sm_max_mhz") or 1965.0  # B200 max SM clock if unsampled
        peak_ginst = 4 * sms * smax / 1000.0
        ach_ginst = k2prof["warp_inst_per_launch"] / k2_avg_s / 1e9
        roofline["issue"] = {"warp_inst_per_launch": k2prof["warp_inst_per_launch"],
                             "achieved": ach_ginst, "peak": peak_ginst, "unit": "G warp-inst/s",
                             "frac": ach_ginst / peak_ginst,
                             "ncu_issue_active_pct": k2prof.get("issue_active_pct")}

    # ---- end to end through the public host API
    e2e = None
    if not args.no_e2e:
        rp_h = torch.from_numpy(np.ascontiguousarray(g.rowptr)).pin_memory()
        ci_h = torch.from_numpy(np.ascontiguousarray(g.colidx)).pin_memory()
        out_h = {"tw": torch.empty(m, dtype=torch.int32, pin_memory=True),
                 "labels": torch.empty((k, n), dtype=torch.int32, pin_memory=True),
                 "stats": torch.empty((k, 2), dtype=torch.int64, pin_memory=True)}
        ws_p = torch.empty(twc.twc_pipeline_workspace_bytes(n, m, rb, k), dtype=torch.uint8,
                           device=dev)
        for _ in range(2):
            twc.twc_pipeline_host(rp_h, ci_h, deltas, out=out_h, workspace=ws_p, device=dev)
        if world > 1:
            dist.barrier()
        # latency: one synchronous call per step
        lat = []
        for _ in range(3):
            t0 = time.perf_counter()
            twc.twc_pipeline_host(rp_h, ci_h, deltas, out=out_h, workspace=ws_p, device=dev)
            lat.append(time.perf_counter() - t0)
        assert torch.equal(out_h["tw"], tw.cpu()) and torch.equal(out_h["labels"], labels.cpu())
        # throughput: INFLIGHT calls in flight (own stream, workspace and host output set each),
        # so one step's copies back overlap the next steps' copy in and compute; every step
        # still copies its whole CSR in and its results out
        lanes = [(torch.cuda.Stream(dev), ws_p, out_h)]
        for _ in range(E2E_INFLIGHT - 1):
            lanes.append((torch.cuda.Stream(dev), torch.empty_like(ws_p),
                          {key: torch.empty_like(v).pin_memory() for key, v in out_h.items()}))
        for st_, w_, o_ in lanes:
            twc.twc_pipeline_host(rp_h, ci_h, deltas, out=o_, workspace=w_, device=dev,
                                  stream=st_, asynchronous=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        E = max(4, min(K, 20))
        t0 = time.perf_counter()
        for i in range(E):
            st_, w_, o_ = lanes[i % len(lanes)]
            twc.twc_pipeline_host(rp_h, ci_h, deltas, out=o_, workspace=w_, device=dev,
                                  stream=st_, asynchronous=True)
        torch.cuda.synchronize()
        e_s = harness.max_over_ranks((time.perf_counter() - t0) / E, dev)
        for _, _, o_ in lanes:
            assert torch.equal(o_["tw"], tw.cpu()) and torch.equal(o_["labels"], labels.cpu())
        e2e = {"value": harness.weak_scaling_value(m, world, e_s), "unit": UNIT,
               "h2d_bytes_per_step": rp_h.numel() * rp_h.element_size() + ci_h.numel() * 4,
               "d2h_bytes_per_step": 4 * m + 4 * k * n + 16 * k, "ms_per_step": 1000 * e_s,
               "steps": E, "in_flight": len(lanes), "api": "twc_pipeline_host_async",
               "latency_ms_single_call": 1000 * statistics.median(lat)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(g, deltas)

    csum = clk.summary()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config_dict(cfg, g, deltas, world),
            "phases_ms": phases, "separate_calls_ms": separate, "selection": selection,
            "score_edges_per_s": world * m / (phases["score"] / 1000.0),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": csum, "wall_s_timed": wall, "cuda_graph": graph,
            "graph": {"triangles": T, "sum_dminus_dplus": S, "max_dplus": dplus_max,
                      "max_degree": int(np.diff(g.rowptr.astype(np.int64)).max())}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main_b200_dist(args):
    """N > 1 (torchrun, one process per GPU): ONE graph split over the N GPUs (
    paper_2412_12382_b200/dist.py): every rank runs the six twc_dist_* phases on its row range
    with the three NCCL exchanges between them.  Strong scaling: value = m * K / (max over ranks
    of the device time of K steps).  DESIGN.md Sec. 7."""
    import torch
    import torch.distributed as dist

    import paper_2412_12382_b200 as twc
    from paper_2412_12382_b200 import build as twc_build
    from paper_2412_12382_b200 import dist as tdist

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    if rank == 0:
        twc_build.build()
    dist.barrier()
    twc.load_library()
    cfg = args.config
    g = gg.config_graph(cfg)
    n, m = g.n, g.m
    rp, ci = harness.to_device(g, dev)
    stream = torch.cuda.current_stream()
    deltas = harness.SWEEP_GRID if cfg == 5 else None
    if deltas is None:  # the thresholds of the smaller configs come from the scores
        _, _, tw0 = twc.twc_score(rp, ci)
        deltas = harness.thresholds(cfg, tw0.cpu().numpy())
    k = len(deltas)
    comm = tdist.TorchComm()
    st = tdist.DistRank(rp, ci, deltas, rank, world)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step():
        return tdist.run_phases([st], comm)[0]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    l0 = twc.twc_kernel_launches()
    dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        wall0 = time.perf_counter()
        for i in range(K):
            flush.zero_()
            starts[i].record(stream)
            info = step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    dist.barrier()
    launches = (twc.twc_kernel_launches() - l0) / K
    total_s = harness.max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / 1000.0,
                                     dev if args.backend == "nccl" else None)
    value = m * K / total_s
    # end to end: every rank copies the CSR in from pinned host memory, runs the step and copies
    # its slice of TW back; rank 0 also copies the labels and stats of all k thresholds back
    rows, cb = tdist.slice_bounds(rp, ci, world)
    c0, c1 = cb[rank], cb[rank + 1]
    rp_h = torch.from_numpy(np.ascontiguousarray(g.rowptr)).pin_memory()
    ci_h = torch.from_numpy(np.ascontiguousarray(g.colidx)).pin_memory()
    tw_h = torch.empty(max(1, c1 - c0), dtype=torch.int32, pin_memory=True)
    lab_h = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
    st_h = torch.empty((k, 2), dtype=torch.int64, pin_memory=True)
    E = max(4, min(K, 10))
    dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(E):
        rp.copy_(rp_h, non_blocking=True)
        ci.copy_(ci_h, non_blocking=True)
        step()
        tw_h[:c1 - c0].copy_(st.tw[c0:c1], non_blocking=True)
        if rank == 0:
            lab_h.copy_(st.labels, non_blocking=True)
            st_h.copy_(st.stats, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e_s = harness.max_over_ranks(e0.elapsed_time(e1) / 1000.0 / E,
                                 dev if args.backend == "nccl" else None)
    csr_bytes = rp_h.numel() * rp_h.element_size() + ci_h.numel() * 4
    e2e = {"value": m / e_s, "unit": UNIT, "h2d_bytes_per_step": world * csr_bytes,
           "d2h_bytes_per_step": 4 * m + 4 * k * n + 16 * k, "ms_per_step": 1000 * e_s,
           "steps": E, "api": "paper_2412_12382_b200.dist.score_sweep path (DistRank.run)",
           "note": "every rank copies the whole CSR in; the TW slices (all ranks) and the "
                   "labels (rank 0) come back"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": 1000.0 * total_s / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic", "config": config_dict(cfg, g, deltas, world),
            "exchange": {"backend": args.backend, "records_last_step_rank0": info,
                         "slice_rows_rank0": [rows[0], rows[1]]},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "wall_s_timed": wall,
            "roofline": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return main_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return main_b200_dist(args)
    return main_b200(args)


if __name__ == "__main__":
    sys.exit(main())
