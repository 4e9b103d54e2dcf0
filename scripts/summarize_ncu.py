#!/usr/bin/env python
"""Summarise an ncu capture and a launch list into profiles/ (run here, no GPU needed).

    python scripts/summarize_ncu.py TAG gpurun_out/prof_TAG.ncu-rep gpurun_out/launches_TAG.csv

Writes profiles/TAG_ncu_full.md (per-kernel metrics of the --set full capture),
profiles/TAG_launches.md (per-kernel device time and share of one bench step from the
--metrics gpu__time_duration.sum launch list; ncu serialises and cold-starts each launch, so
compare SHARES, not absolute times) and profiles/k2_ncu_summary.json (DRAM bytes per K2
launch, read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sectors.sum", "L2 sectors (x 32 B = L2 bytes)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data pipe (LSU wavefronts) % peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smem atomic bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst (of 32)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "global RED requests"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "global atomic requests"),
]


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def bench_identity(tag):
    """config / graph identity of the bench line captured in the same gpurun (gpurun_out/
    bench_TAG.json), so bench.py only uses this capture's DRAM bytes for the same graph."""
    # the full bench line, else the plain run that preceded the ncu passes (same graph)
    for name in (f"bench_{tag}.json", f"plain_{tag}.log"):
        p = os.path.join(ROOT, "gpurun_out", name)
        try:
            d = json.loads(open(p).read().strip().splitlines()[-1])
            c = d["config"]
            return {"graph_sha256": c.get("graph_sha256"), "n": c.get("n"), "m": c.get("m"),
                    "workload": c.get("workload"), "bench_line": f"profiles/{tag}_bench.json"}
        except Exception:
            continue
    return {}


def full_summary(tag, rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary ({tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(scripts/gpu_iter.sh); config 5 workload (DC-SBM n=4M, m=35M), one bench step.", ""]
    k2 = None
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            ck = key if key in col else next((h for h in col if h.endswith("." + key)), None)
            if ck is not None:
                lines.append(f"| {label} (`{key}`) | {r[col[ck]]} {units[col[ck]]} |")
        try:  # derived: sectors per global load request
            sec = float(r[col["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]].replace(",", ""))
            req = float(r[col["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]].replace(",", ""))
            lines.append(f"| sectors per global load request | {sec / req:.2f} |")
        except (KeyError, ValueError, ZeroDivisionError):
            pass
        lines.append("")
        if "k2_intersect" in name and k2 is None:
            rd = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
            wr = to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
            k2 = {"tag": tag, "dram_bytes_read": rd, "dram_bytes_write": wr,
                  "dram_bytes_per_launch": rd + wr,
                  "warp_inst_per_launch": float(r[col["smsp__inst_executed.sum"]].replace(",", "")),
                  "issue_active_pct": float(r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]]),
                  "duration": r[col["gpu__time_duration.sum"]] + " " + units[col["gpu__time_duration.sum"]],
                  "source": f"profiles/{tag}_ncu_full.md", **bench_identity(tag)}
            for key, name2 in (("lts__t_sectors.sum", "l2_sectors_per_launch"),
                               ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
                               ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                                "lsu_pipe_pct"),
                               ("smsp__thread_inst_executed_per_inst_executed.ratio",
                                "threads_per_inst")):
                try:  # third bandwidth figure (L2) and the evidence counters
                    k2[name2] = float(r[col[key]].replace(",", ""))
                except (KeyError, ValueError):
                    pass
    with open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if k2:
        with open(os.path.join(PROF, "k2_ncu_summary.json"), "w") as f:
            json.dump(k2, f, indent=1)


def launch_summary(tag, path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    seq = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")))
           for r in data if len(r) > vi]
    idx = [k for k, (nm, _) in enumerate(seq) if "k0_degrees" in nm] + [len(seq)]
    # the last complete fused step (twc_score_sweep: contains k_band_place)
    steps = [seq[a:b] for a, b in zip(idx[:-1], idx[1:])]
    fused = [st for st in steps if any("k_band_place" in nm for nm, _ in st)]
    # complete = as many sweep steps as any fused step (the capture limit can cut the last one)
    nfin = [sum("k_finalize" in nm for nm, _ in st) for st in fused]
    full = [st for st, c in zip(fused, nfin) if nfin and c == max(nfin)]
    chosen = full[-1] if full else steps[-1]
    # a fused step ends at its last k_finalize (the separate calls may follow in the same chunk)
    last_fin = max((k for k, (nm, _) in enumerate(chosen) if "k_finalize" in nm), default=len(chosen) - 1)
    last = [x for x in chosen[:last_fin + 1] if not x[0].startswith("at::")]
    tot = sum(v for _, v in last)
    agg, cnt = OrderedDict(), OrderedDict()
    for nm, v in last:
        agg[nm] = agg.get(nm, 0.0) + v
        cnt[nm] = cnt.get(nm, 0) + 1
    lines = [f"# Launch list of one bench step ({tag})", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline` (config 5); the "
             "last complete fused step (`twc_score_sweep`).  ncu serialises launches and starts each cold, so the SHARES "
             "are what compare with bench.py's live phase timings, not the absolute times.", "",
             "| kernel | launches | device time (us) | share |", "|---|---|---|---|"]
    for nm, v in agg.items():
        lines.append(f"| `{nm}` | {cnt[nm]} | {v / 1000:.1f} | {100 * v / tot:.1f}% |")
    lines.append(f"| **total** | {sum(cnt.values())} | {tot / 1000:.1f} | 100% |")
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    tag, rep, launches = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs(PROF, exist_ok=True)
    full_summary(tag, rep)
    launch_summary(tag, launches)
    print("wrote profiles/ for", tag)
