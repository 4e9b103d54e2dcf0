#!/usr/bin/env python
"""Per-instruction executed counts and stall samples from an ncu source page (SASS view).

    ncu -i REP --page source --csv --print-source sass > x.csv
    python scripts/sass_hot.py x.csv [min_share]
Prints the instructions in address order with their share of executed warp instructions and of
the stall samples, and marks backward branches (loop ends).
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ismp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":  # next kernel of a multi-kernel page: keep the first only
        break
    if len(r) <= iex or r[ia] == "Address":
        continue
    data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ismp] or 0)))
base = data[0][0]
tot = sum(d[2] for d in data)
tsm = sum(d[3] for d in data)
mins = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
print(f"total warp instructions {tot:,}  samples {tsm:,}")
for a, s, e, m in data:
    if e / tot >= mins or m / max(tsm, 1) >= 0.01:
        print(f"{a - base:6x} {e:12,d} {100 * e / tot:5.2f}% {100 * m / max(tsm, 1):5.2f}%  {s}")

if len(sys.argv) > 3:  # region summary: comma-separated hex boundaries (offsets from the base)
    cuts = [0] + [int(x, 16) for x in sys.argv[3].split(",")] + [1 << 40]
    for lo, hi in zip(cuts, cuts[1:]):
        e = sum(d[2] for d in data if lo <= d[0] - base < hi)
        m = sum(d[3] for d in data if lo <= d[0] - base < hi)
        print(f"[{lo:6x}, {hi:6x})  inst {100 * e / tot:5.1f}%  samples {100 * m / max(tsm, 1):5.1f}%")
