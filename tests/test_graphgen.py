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


# ------------------------------------------------------------------ manifest + calibration pins
# the realised graphs are pinned by their manifest (tests/golden/graph_manifest.json,
# written by scripts/make_manifest.py; T there comes from the CPU oracle) and the DC-SBM
# calibration must land m within +-2% of its target and d_max within +-10% (the shapes of the
# paper's Amazon / Youtube / LiveJournal rows, P:661/663/664, stood in for by these graphs).

def _degree_stats(g):
    rp = g.rowptr.astype(np.int64)
    deg = np.diff(rp)
    return {"n": g.n, "m": g.m, "d_max": int(deg.max()), "sum_d": int(deg.sum()),
            "sum_d2": int((deg * deg).sum()), "W": int((deg * (deg - 1) // 2).sum()),
            "rowptr": str(g.rowptr.dtype), "sha256": g.sha256()}


import pytest  # noqa: E402


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_config_matches_manifest(k):
    man = gg.manifest()[str(k)]
    g = gg.config_graph(k)
    _csr_ok(g)
    got = _degree_stats(g)
    for key, val in got.items():
        assert man[key] == val, (k, key, man[key], val)


def test_manifest_calibration_tolerances():
    man = gg.manifest()
    for k in (3, 4, 5):
        r = man[str(k)]
        assert abs(r["m"] / r["m_target"] - 1) <= 0.02, (k, r["m"], r["m_target"])
        assert abs(r["d_max"] / r["d_max_target"] - 1) <= 0.10, (k, r["d_max"])
        assert r["rowptr"] == ("int64" if k == 5 else "int32")
        # the generator's edge mass split: intra draws saturate at block size for hubs and
        # collapse as duplicates, so the realised intra fraction sits below mu, never above
        assert 0.5 <= r["intra_block_fraction"] <= r["mu_target"]
    for k in (1, 2):
        r = man[str(k)]
        assert abs(r["m"] - r["m_expected"]) <= 4 * r["m_sd"], (k, r["m"], r["m_expected"])
    # invariants between the recorded sums: sum d = 2m, W = (sum d^2 - sum d) / 2
    for k in range(1, 6):
        r = man[str(k)]
        assert r["sum_d"] == 2 * r["m"] and 2 * r["W"] == r["sum_d2"] - r["sum_d"]
        assert r["S_sum_dminus_dplus"] <= r["sum_oriented_dplus_u_plus_dplus_v"]


def test_graph_cache_roundtrip(tmp_path, monkeypatch):
    monkeypatch.setenv("TWC_GRAPH_CACHE", str(tmp_path))
    a = gg.config_graph(3)
    assert (tmp_path / "config3.npz").exists()
    b = gg.config_graph(3)                    # served from the cache, same bytes
    assert b.sha256() == a.sha256() == gg.manifest()["3"]["sha256"]
    assert np.array_equal(a.meta["block_of"], b.meta["block_of"])
