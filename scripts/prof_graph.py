"""Score one named graph a few times (for ncu launch lists): python scripts/prof_graph.py rmat-d-1e7"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = gg.rmat_graph(name[5:]) if name.startswith("rmat-") else gg.config_graph(int(name))
twc.load_library()
rp, ci = harness.to_device(g)
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    twc.twc_score(rp, ci)
    e1.record()
    torch.cuda.synchronize()
    print("score ms", e0.elapsed_time(e1))
