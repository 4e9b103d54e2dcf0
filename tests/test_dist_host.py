"""Host-side checks of the distributed step's bookkeeping (paper_2412_12382_b200/dist.py, CPU):
the row split partitions the vertices and the canonical edges, balances the degree-oriented slots
(SURVEY 8(e)), and the in-process exchange routing (Emulated) is a permutation of the records."""
import numpy as np
import pytest
import torch

import graphgen as gg
from paper_2412_12382_b200 import dist as tdist


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_slice_bounds_partition_and_balance(world):
    for seed, g in enumerate([gg.config_graph(1), gg.erdos_renyi(700, 0.03, seed=4),
                              gg.star(300, 5), gg.complete(60)]):
        rp = torch.from_numpy(np.ascontiguousarray(g.rowptr))
        ci = torch.from_numpy(np.ascontiguousarray(g.colidx))
        rows, cb = tdist.slice_bounds(rp, ci, world)
        assert rows[0] == 0 and rows[-1] == g.n and all(a <= b for a, b in zip(rows, rows[1:]))
        assert cb[0] == 0 and cb[-1] == g.m and all(a <= b for a, b in zip(cb, cb[1:]))
        # canonical slice r = the canonical edges whose smaller endpoint lies in rows r
        s, _ = g.canonical_pairs()
        for r in range(world):
            inside = (s >= rows[r]) & (s < rows[r + 1])
            assert int(inside.sum()) == cb[r + 1] - cb[r]
        # oriented slots per slice within one row's worth of m / P (the split is by rows)
        deg = np.diff(g.rowptr.astype(np.int64))
        src = np.repeat(np.arange(g.n), deg)
        dst = g.colidx.astype(np.int64)
        out = (deg[src] < deg[dst]) | ((deg[src] == deg[dst]) & (src < dst))
        dplus = np.bincount(src[out], minlength=g.n)
        for r in range(world):
            slots = int(dplus[rows[r]:rows[r + 1]].sum())
            assert abs(slots - g.m / world) <= int(dplus.max()) + 1


def test_emulated_all_to_all_is_a_permutation():
    rng = np.random.default_rng(2)
    for world in (1, 2, 4, 7):
        sends, sizes = [], []
        for r in range(world):
            sz = [int(x) for x in rng.integers(0, 6, size=world)]
            recs = np.stack([np.full(sum(sz), r), np.arange(sum(sz))], axis=1).astype(np.int32)
            sends.append(torch.from_numpy(recs.reshape(-1).copy()))
            sizes.append(sz)
        outs, rsz = tdist.Emulated(world).all_to_all(sends, sizes, 2)
        for q in range(world):
            got = outs[q].numpy().reshape(-1, 2)
            assert rsz[q] == [sizes[r][q] for r in range(world)]
            # records from rank r to q, in r's order, sources ascending
            exp = []
            for r in range(world):
                start = sum(sizes[r][:q])
                exp += [(r, start + i) for i in range(sizes[r][q])]
            assert [tuple(x) for x in got] == exp
