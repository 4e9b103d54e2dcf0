"""Harness helpers shared by tests/ and bench.py: threshold recipes and tensor plumbing.

Threshold recipes follow DESIGN.md reading C17 (BASELINE.json's configs state them loosely):
  config 1  delta = (min TW + max TW) / 2 (fp64, "mid-range"), plus floor() of it (a tie case)
  config 2  the 10th / 30th / 50th percentiles of TW, nearest rank: sorted(TW)[ceil(p*m/100)-1]
  config 3-4  the 50th percentile
  config 5  the paper's TW grid with the end point included: -30, -28, ..., 0 (16 values)
Nothing here computes scores or labels.
"""
from __future__ import annotations

import math

import numpy as np

SWEEP_GRID = [float(d) for d in range(-30, 1, 2)]  # 16 thresholds (P:718 TW row, end included)


def nearest_rank(tw: np.ndarray, p: float) -> float:
    s = np.sort(np.asarray(tw))
    k = max(1, math.ceil(p * s.size / 100.0))
    return float(s[k - 1])


def thresholds(config: int, tw: np.ndarray):
    tw = np.asarray(tw)
    if config == 1:
        mid = (float(tw.min()) + float(tw.max())) / 2.0
        return [mid, float(math.floor(mid))]
    if config == 2:
        return [nearest_rank(tw, p) for p in (10, 30, 50)]
    if config in (3, 4):
        return [nearest_rank(tw, 50)]
    return list(SWEEP_GRID)


def to_device(g, device="cuda"):
    import torch
    rowptr = torch.from_numpy(np.ascontiguousarray(g.rowptr)).to(device)
    colidx = torch.from_numpy(np.ascontiguousarray(g.colidx)).to(device)
    return rowptr, colidx


# ------------------------------------------------------------------ multi-rank (bench.py, N > 1)
def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over all ranks (device timings are max-over-ranks, never wall
    clock); identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_scaling_value(units_per_rank: float, world: int, seconds_max: float) -> float:
    """Whole-job throughput: every rank processes its own replica of the workload
    (independent problems, no data-path collective), so units = world x units_per_rank."""
    return world * units_per_rank / seconds_max

