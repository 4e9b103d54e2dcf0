"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every function that
include/twc.h declares, and rejects bad arguments before touching the device."""
import ctypes

import numpy as np
import pytest

import paper_2412_12382_b200 as twc
from paper_2412_12382_b200 import build as twc_build


@pytest.fixture(scope="module")
def lib():
    twc_build.build()
    return twc.load_library()


def test_exports_every_header_function(lib):
    names = twc.header_functions()
    assert len(names) >= 11
    for name in names:
        assert hasattr(lib, name), name
    assert lib.twc_version() == 100


def test_status_strings(lib):
    for s in range(5):
        assert lib.twc_status_string(s)
    assert lib.twc_status_string(99) == b"unknown twc_status"


def test_workspace_queries_are_host_only(lib):
    for n, m in [(0, 0), (10, 20), (4_000_000, 35_000_000)]:
        a = lib.twc_score_workspace_bytes(n, m, 8)
        b = lib.twc_cluster_workspace_bytes(n, m, 8)
        c = lib.twc_pipeline_workspace_bytes(n, m, 8, 16)
        assert a > 0 and b > 0 and c >= a
    # score workspace ~ 5 n + 4.25 m int32 + small
    n, m = 4_000_000, 35_000_000
    a = lib.twc_score_workspace_bytes(n, m, 8)
    assert 4 * (2 * m + 3 * n) <= a <= 4 * (5 * m + 14 * n)
    assert lib.twc_pipeline_workspace_bytes(10, 10, 3, 1) == 0


def _csr(n, m, rb=4, rowptr=256, colidx=512):  # fake, suitably aligned device pointers
    return twc._Csr(n, m, ctypes.c_void_p(rowptr), rb, ctypes.c_void_p(colidx))


def test_argument_errors_before_device(lib):
    P = ctypes.c_void_p
    g = _csr(10, 5, rb=3)
    assert lib.twc_score(ctypes.byref(g), None, 0, P(1), P(1), P(1), None) == twc.TWC_EINVAL
    assert b"rowptr_bytes" in lib.twc_last_error()
    g = _csr(-1, 5)
    assert lib.twc_score(ctypes.byref(g), None, 0, P(1), P(1), P(1), None) == twc.TWC_EINVAL
    g = _csr(10, 1 << 31, rb=8)
    assert lib.twc_score(ctypes.byref(g), None, 0, P(1), P(1), P(1), None) == twc.TWC_EINVAL
    g = _csr(10, 1 << 30, rb=4)          # 2m does not fit int32 rowptr
    assert lib.twc_score(ctypes.byref(g), None, 0, P(1), P(1), P(1), None) == twc.TWC_EINVAL
    g = _csr(10, 5)
    assert lib.twc_score(ctypes.byref(g), None, 0, None, P(1), P(1), None) == twc.TWC_EINVAL
    assert lib.twc_score(ctypes.byref(g), None, 0, P(1), P(1), P(1), None) == twc.TWC_EWORKSPACE
    assert lib.twc_score(ctypes.byref(g), P(256), 16, P(1), P(1), P(1), None) == twc.TWC_EWORKSPACE
    assert lib.twc_score(ctypes.byref(g), P(100), 1 << 30, P(1), P(1), P(1), None) == twc.TWC_EWORKSPACE
    assert b"aligned" in lib.twc_last_error()
    assert lib.twc_cluster(ctypes.byref(g), P(1), float("nan"), None, 0, P(1), None, None) == twc.TWC_EINVAL
    d = (ctypes.c_double * 1)(0.0)
    assert lib.twc_sweep(ctypes.byref(g), P(1), ctypes.cast(d, P), 0, None, 0, P(1), None, None) == twc.TWC_EINVAL
    assert lib.twc_sweep(ctypes.byref(g), P(1), None, 1, None, 0, P(1), None, None) == twc.TWC_EINVAL
    assert lib.twc_validate_csr(ctypes.byref(g), None, None) == twc.TWC_EINVAL
    assert lib.twc_score(None, None, 0, P(1), P(1), P(1), None) == twc.TWC_EINVAL
    # partition statistics (NEXT(2))
    assert lib.twc_partition_stats(ctypes.byref(g), P(1), 0, None, 0, P(1), None, None) == twc.TWC_EINVAL
    assert lib.twc_partition_stats(ctypes.byref(g), None, 1, None, 0, P(1), None, None) == twc.TWC_EINVAL
    assert lib.twc_partition_stats(ctypes.byref(g), P(1), 1, None, 0, None, None, None) == twc.TWC_EINVAL
    assert lib.twc_partition_stats(ctypes.byref(g), P(1), 1, None, 0, P(1), None, None) == twc.TWC_EWORKSPACE
    big = _csr(1 << 30, 1_600_000_000, rb=8)
    assert lib.twc_partition_stats(ctypes.byref(big), P(1), 1, None, 0, P(1), None, None) == twc.TWC_EINVAL
    assert b"4m^2" in lib.twc_last_error()
    assert lib.twc_partition_stats_workspace_bytes(4_000_000, 35_000_000, 8) >= 12 * 4_000_000
    # alignment: device colidx 16-byte, rowptr rowptr_bytes-aligned, else EINVAL
    for rp, ci, rb in [(256, 516, 4), (256, 520, 8), (258, 512, 4), (260, 512, 8)]:
        g = _csr(10, 5, rb=rb, rowptr=rp, colidx=ci)
        assert lib.twc_score(ctypes.byref(g), P(256), 1 << 30, P(1), P(1), P(1), None) == twc.TWC_EINVAL
        assert b"aligned" in lib.twc_last_error()
    # host pipeline: host pointers need no alignment (copied into the aligned workspace)
    g = _csr(10, 5, rb=4, rowptr=258, colidx=516)
    assert lib.twc_pipeline_host_async(ctypes.byref(g), ctypes.cast(d, P), 1, None, 0, None, None,
                                       None, None, None, None) == twc.TWC_EWORKSPACE


def test_sweep_norm_stats_host(lib):
    import torch
    counts = torch.tensor([[4, 7, 30, 900], [10, 1, 0, 100]], dtype=torch.int64)
    kept = torch.tensor([[40, 4], [0, 10]], dtype=torch.int64)
    norm = twc.twc_sweep_norm_stats(10, 50, counts, kept)
    assert norm.tolist() == [[4 / 10, 40 / 50, 7 / 10], [10 / 10, 0 / 50, 1 / 10]]
    norm = twc.twc_sweep_norm_stats(0, 0, counts, None)
    assert torch.isnan(norm).all()
    P = ctypes.c_void_p
    assert lib.twc_sweep_norm_stats(10, 5, 0, P(1), None, P(1)) == twc.TWC_EINVAL
    assert lib.twc_sweep_norm_stats(10, 5, 1, None, None, P(1)) == twc.TWC_EINVAL


def _select(lib, deltas, largest, q, n, jump=0.1):
    k = len(deltas)
    d = (ctypes.c_double * k)(*deltas)
    lg = (ctypes.c_int64 * k)(*largest)
    qq = (ctypes.c_double * k)(*q)
    i, r = ctypes.c_int32(-1), ctypes.c_int32(-1)
    st = lib.twc_select_threshold(ctypes.cast(d, ctypes.c_void_p), ctypes.cast(lg, ctypes.c_void_p),
                                  ctypes.cast(qq, ctypes.c_void_p), k, n, jump, ctypes.byref(i),
                                  ctypes.byref(r))
    return st, i.value, r.value


def test_select_threshold_is_host_logic(lib):
    # host-only entry point: runs without a GPU.  S:372: single 0 -> 0.9 jump between 4 and 2.
    st, i, r = _select(lib, [0, 2, 4, 6, 8], [9, 9, 0, 0, 0], [0.1, 0.2, 0.3, 0.2, 0.1], 10)
    assert (st, i, r) == (twc.TWC_OK, 2, 0)
    # constant largest -> max modularity, ties to the larger delta
    st, i, r = _select(lib, [0, 2, 4, 6], [5, 5, 5, 5], [0.1, 0.4, 0.4, float("nan")], 10)
    assert (st, i, r) == (twc.TWC_OK, 2, 1)
    assert _select(lib, [0.0], [1], [0.0], 0)[0] == twc.TWC_EINVAL
    assert _select(lib, [float("nan"), 1.0], [1, 1], [0.0, 0.0], 5)[0] == twc.TWC_EINVAL
    assert lib.twc_select_threshold(None, None, None, 0, 1, 0.1, None, None) == twc.TWC_EINVAL


def test_empty_graph_score_is_ok_without_device(lib):
    g = _csr(5, 0)
    assert lib.twc_score(ctypes.byref(g), None, 0, None, None, None, None) == twc.TWC_OK


def test_product_package_never_imports_oracle():
    import pathlib
    root = pathlib.Path(twc.__file__).parent
    for p in list(root.rglob("*.py")) + list(root.rglob("*.cu")) + list(root.rglob("*.cuh")) + list(root.rglob("*.h")):
        txt = p.read_text()
        assert "import oracle" not in txt and "from oracle" not in txt and "twc_oracle" not in txt, p
