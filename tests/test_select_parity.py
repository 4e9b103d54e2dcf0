"""Host-logic parity (no GPU needed): the library's twc_select_threshold against oracle.select
on seeded random sweep reports, including ties, NaN modularity, duplicate deltas and reports
with and without a qualifying jump (reading C22)."""
import numpy as np
import pytest

import paper_2412_12382_b200 as twc
from paper_2412_12382_b200 import build as twc_build


@pytest.fixture(scope="module", autouse=True)
def _lib():
    twc_build.build()
    twc.load_library()


@pytest.mark.parametrize("seed", range(200))
def test_select_matches_oracle(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 20))
    n = int(rng.integers(1, 1000))
    deltas = rng.choice(np.arange(-30, 1, 2), size=k, replace=bool(k > 16 or rng.integers(0, 2))).astype(float)
    largest = rng.integers(1, n + 1, size=k)
    if rng.random() < 0.5:   # a monotone curve as a real sweep produces
        largest = np.sort(largest)[np.argsort(np.argsort(-deltas, kind="stable"), kind="stable")]
    q = np.round(rng.uniform(-0.5, 1.0, size=k), 1)     # coarse values -> ties
    if rng.random() < 0.2:
        q[rng.integers(0, k)] = np.nan
    jump = float(rng.choice([0.0, 0.05, 0.1, 0.3, 1.0]))
    i, rule = twc.twc_select_threshold(deltas, largest, q, n, jump)
    oi, orule = oracle_mod.select(deltas, largest, n, q, jump)
    assert (i, rule) == (oi, {0: "largest_cc_jump", 1: "max_modularity"}[orule])
