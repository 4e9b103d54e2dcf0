#!/usr/bin/env python
"""Score one R-MAT graph a few times (for an ncu launch list of its kernels).

    python scripts/prof_rmat_one.py rmat-d-1e7 [reps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
import harness  # noqa: E402
import paper_2412_12382_b200 as twc  # noqa: E402

g = gg.rmat_graph(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rp, ci = harness.to_device(g, "cuda")
for _ in range(reps):
    twc.twc_score(rp, ci)
torch.cuda.synchronize()
print("ok", g.n, g.m)
