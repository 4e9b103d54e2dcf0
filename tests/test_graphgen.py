"""Host-side checks of the seeded input generators (graphgen/): shape, CSR invariants and the
R-MAT recursion's quadrant law.  Generators are harness code, not the method."""
import numpy as np

import graphgen as gg


def _csr_ok(g):
    rp = g.rowptr.astype(np.int64)
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == 2 * g.m
    src = np.repeat(np.arange(g.n), np.diff(rp))
    assert np.all(g.colidx != src)                                  # no loops
    for u in range(0, g.n, max(1, g.n // 50)):                      # sorted unique rows
        row = g.colidx[rp[u]:rp[u + 1]]
        assert np.all(np.diff(row) > 0)
    a = np.sort(src * g.n + g.colidx)
    b = np.sort(g.colidx.astype(np.int64) * g.n + src)
    assert np.array_equal(a, b)                                     # symmetric


def test_rmat_quadrant_law_and_exact_n():
    # top-level quadrant of each draw: P(u high) = a21 + a22 = 0.40, P(v high) = a12 + a22 = 0.40,
    # P(both high) = a22 = 0.25 (before dedup; tested on a large sparse draw where dedup is rare)
    g = gg.rmat(16, 200_000, seed=3)
    s, d = g.canonical_pairs()
    _csr_ok(g)
    half = 1 << 15
    # canonical pairs are (min, max): the joint law of (min high, max high) is symmetric-free
    both = np.mean((s >= half) & (d >= half))
    none = np.mean((s < half) & (d < half))
    assert abs(both - 0.25) < 0.01 and abs(none - 0.45) < 0.01
    g = gg.rmat(10, 20_000, seed=1, n=700)
    _csr_ok(g)
    assert g.n == 700 and g.colidx.max() < 700 and g.m <= 20_000


def test_rmat_configs_shapes():
    assert set(gg.RMAT_CONFIGS) == {"vs-1e7", "vs-1e8", "s-1e7", "s-1e8", "d-1e7", "d-1e8"}
    for name, c in gg.RMAT_CONFIGS.items():
        dens = name.split("-")[0]
        if dens == "vs":
            assert c["m"] == 5 * c["n"]
        elif dens == "s":
            assert c["m"] == 50 * c["n"]
        else:
            assert abs(c["m"] - c["n"] ** 1.5) / c["m"] < 1e-3
