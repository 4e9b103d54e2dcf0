#!/usr/bin/env python
"""One small end-to-end pass of the CUDA path for compute-sanitizer (scripts/gpu_sanitize.sh):
twc_score_sweep, twc_score_k4, twc_similarity + twc_sweep_f64, twc_partition_stats and the
separate score / sweep calls on BASELINE configs 1 and 2, each checked against the CPU oracle
(test infrastructure).  Exit code 0 = all results identical."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import graphgen as gg  # noqa: E402
import harness  # noqa: E402
import oracle  # noqa: E402
import paper_2412_12382_b200 as twc  # noqa: E402


def main():
    twc.load_library()
    for k in (1, 2):
        g = gg.config_graph(k)
        rp, ci = harness.to_device(g)
        ot, ow, otw = oracle.score(g)
        deltas = harness.thresholds(k, otw)
        t, w, tw, lab, st = twc.twc_score_sweep(rp, ci, deltas)
        torch.cuda.synchronize()
        assert np.array_equal(t.cpu().numpy(), ot) and np.array_equal(tw.cpu().numpy(), otw)
        for i, d in enumerate(deltas):
            ol, kept, ncomp = oracle.cluster(g, otw, d)
            assert np.array_equal(lab[i].cpu().numpy(), ol)
        t2, w2, tw2, k4 = twc.twc_score_k4(rp, ci)
        assert np.array_equal(k4.cpu().numpy(), oracle.k4(g))
        sim = twc.twc_similarity(rp, ci, t, "jaccard")
        assert np.array_equal(sim.cpu().numpy(), oracle.similarity(g, ot, "jaccard"))
        twc.twc_sweep_f64(rp, ci, sim, [0.1, 0.3])
        twc.twc_partition_stats(rp, ci, lab)
        ts, ws_, tws = twc.twc_score(rp, ci)
        lab2, _ = twc.twc_sweep(rp, ci, tws, deltas)
        torch.cuda.synchronize()
        assert torch.equal(lab2, lab)
        print(f"config {k}: ok (n={g.n}, m={g.m})", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
