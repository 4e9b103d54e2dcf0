#!/usr/bin/env python
"""PCIe bound of the e2e step: pinned H2D of the config-5 CSR bytes and D2H of the result bytes,
each alone and both at once on two streams (CUDA events).  python scripts/pcie_bound.py"""
import json
import torch

H2D, D2H = 311_919_504, 395_960_004
dev = torch.device("cuda")
hi = torch.empty(H2D, dtype=torch.uint8, pin_memory=True)
ho = torch.empty(D2H, dtype=torch.uint8, pin_memory=True)
di = torch.empty(H2D, dtype=torch.uint8, device=dev)
do = torch.empty(D2H, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_event(a)
        s2.wait_event(a)
        if h2d:
            with torch.cuda.stream(s1):
                di.copy_(hi, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


r = {"h2d_ms": run(True, False), "d2h_ms": run(False, True), "both_ms": run(True, True)}
r["h2d_gbs"] = H2D / r["h2d_ms"] / 1e6
r["d2h_gbs"] = D2H / r["d2h_ms"] / 1e6
print(json.dumps(r))
