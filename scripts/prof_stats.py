"""Run twc_partition_stats once on config 5's 16 sweep partitions (for an ncu launch list)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import graphgen as gg
import harness
import paper_2412_12382_b200 as twc

twc.load_library()
g = gg.config_graph(5)
rp, ci = harness.to_device(g)
deltas = [float(x) for x in range(-30, 1, 2)]
_, _, tw, labels, stats = twc.twc_score_sweep(rp, ci, deltas)
torch.cuda.synchronize()
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    counts, q = twc.twc_partition_stats(rp, ci, labels)
    e1.record()
    torch.cuda.synchronize()
    print("partition_stats ms", e0.elapsed_time(e1))
print(counts.cpu().tolist())
