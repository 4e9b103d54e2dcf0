#!/usr/bin/env python
"""Write tests/golden/graph_manifest.json: the realised statistics of the five BASELINE.json
workloads (SURVEY 8(d) "Conventions": n, m, d_max, sum d, sum d^2, W, T, S, sum over oriented
edges of d+(u) + d+(v), realised intra-block fraction, number of blocks, numpy version, seed,
sha256 of the CSR bytes).

The triangle count T comes from the CPU ORACLE (sum of its per-edge t / 3), never from the
CUDA path; every other figure is degree bookkeeping of the generated CSR.  Run here (no GPU):
    python scripts/make_manifest.py [configs...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "graph_manifest.json")
TARGET_DMAX = {3: 550, 4: 28_000, 5: 15_000}  # BASELINE.json configs[2..4] "max degree ~"


def stats(k):
    g = gg.config_graph(k)
    c = gg.CONFIGS[k]
    rp = g.rowptr.astype(np.int64)
    deg = np.diff(rp)
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    dst = g.colidx.astype(np.int64)
    # degree orientation with the strict (deg, id) key (reading C9)
    out = (deg[src] < deg[dst]) | ((deg[src] == deg[dst]) & (src < dst))
    dplus = np.bincount(src[out], minlength=g.n).astype(np.int64)
    dminus = deg - dplus
    up = dst > src
    if c["kind"] == "pp":
        blk = np.arange(g.n, dtype=np.int64) // c["s"]
        nblocks = c["n_blocks"]
    else:
        blk = g.meta["block_of"]
        nblocks = int(g.meta["blocks"])
    intra = float(np.mean(blk[src[up]] == blk[dst[up]])) if g.m else 0.0
    oracle.set_threads(oracle.max_threads())
    t, _, _ = oracle.score(g)
    T = int(t.astype(np.int64).sum()) // 3
    rec = {"config": k, "kind": c["kind"], "seed": c["seed"], "n": g.n, "m": g.m,
           "rowptr": str(g.rowptr.dtype), "d_max": int(deg.max()), "sum_d": int(deg.sum()),
           "sum_d2": int((deg * deg).sum()), "W": int((deg * (deg - 1) // 2).sum()),
           "T_oracle": T, "S_sum_dminus_dplus": int((dminus * dplus).sum()),
           "sum_oriented_dplus_u_plus_dplus_v": int((dplus[src[out]] + dplus[dst[out]]).sum()),
           "max_dplus": int(dplus.max()), "blocks": nblocks, "intra_block_fraction": intra,
           "numpy": np.__version__, "sha256": g.sha256()}
    if c["kind"] == "dcsbm":
        rec.update(m_target=c["m_target"], d_max_target=TARGET_DMAX[k], mu_target=c["mu"],
                   gamma=c["gamma"], eps=c["eps"], theta_max=c["theta_max"])
    else:
        n = g.n
        s = c["s"]
        pairs_in = c["n_blocks"] * s * (s - 1) // 2
        pairs_out = n * (n - 1) // 2 - pairs_in
        rec.update(p_in=c["p_in"], p_out=c["p_out"],
                   m_expected=pairs_in * c["p_in"] + pairs_out * c["p_out"],
                   m_sd=float(np.sqrt(pairs_in * c["p_in"] * (1 - c["p_in"]) +
                                      pairs_out * c["p_out"] * (1 - c["p_out"]))))
    return rec


if __name__ == "__main__":
    ks = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    man = json.load(open(OUT)) if os.path.exists(OUT) else {}
    man["_about"] = ("Realised statistics of the BASELINE.json workloads (graphgen.config_graph); "
                     "T from the CPU oracle; written by scripts/make_manifest.py")
    for k in ks:
        man[str(k)] = stats(k)
        print(json.dumps(man[str(k)]), flush=True)
    with open(OUT, "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)
