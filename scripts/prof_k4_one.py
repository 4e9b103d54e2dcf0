#!/usr/bin/env python
"""Run twc_score_k4 on one graph (config number or R-MAT name) for an ncu launch list."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
import harness  # noqa: E402
import paper_2412_12382_b200 as twc  # noqa: E402

name = sys.argv[1]
g = gg.config_graph(int(name)) if name.isdigit() else gg.rmat_graph(name)
rp, ci = harness.to_device(g, "cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    twc.twc_score_k4(rp, ci)
torch.cuda.synchronize()
print("ok")
