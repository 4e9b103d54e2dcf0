"""Calibrate the DC-SBM configs (3-5) so the realised graph hits BASELINE.json's targets.

Targets: realised m within +-2% of m_target, realised max degree within +-10%
of the stated max degree.  Two knobs per config: eps (edge over-sampling, compensating
self-loops and duplicate collapse) and theta_max (hubs' intra draws saturate at block size,
so theta_max must exceed the target degree).  Prints the constants to paste into
graphgen.CONFIGS.  Run:  python -m graphgen.calibrate [3 4 5]
"""
import sys

import numpy as np

import graphgen as gg

TARGET_DMAX = {3: 550, 4: 28_000, 5: 15_000}


def realised(k, eps, tmax):
    c = dict(gg.CONFIGS[k])
    g = gg.dc_sbm(c["n"], c["m_target"], c["gamma"], tmax, c["smin"], c["smax"], c["mu"],
                  c["seed"], eps=eps, rowptr_dtype=np.int64)
    d = np.diff(g.rowptr)
    return g.m, int(d.max())


def calibrate(k, iters=12):
    c = gg.CONFIGS[k]
    eps, tmax = c["eps"], c["theta_max"]
    mt, dt = c["m_target"], TARGET_DMAX[k]
    for it in range(iters):
        m, dmax = realised(k, eps, tmax)
        print(f"cfg{k} it{it} eps={eps:.5f} tmax={tmax:.1f} -> m={m} ({m / mt - 1:+.3%}) "
              f"dmax={dmax} ({dmax / dt - 1:+.3%})", flush=True)
        if abs(m / mt - 1) < 0.01 and abs(dmax / dt - 1) < 0.05:
            break
        eps = (1 + eps) * (mt / m) ** 1.2 - 1
        tmax = tmax * (dt / dmax) ** 1.1
    return eps, tmax


if __name__ == "__main__":
    ks = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
    for k in ks:
        e, t = calibrate(k)
        print(f"CONFIG {k}: eps={e:.6f} theta_max={t:.3f}")
