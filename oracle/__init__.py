"""CPU oracle for the TW clustering hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package.  The product path (paper_2412_12382_b200/) never imports it.

The arithmetic lives in twc_oracle.c (plain C, see its header for the PAPER.md citations);
this file only builds/loads it with ctypes and marshals numpy arrays.

    score(g, rows=None)          -> (t, wedge, tw)   int32[m] each, canonical (u<v lex) order
    cluster(g, tw, delta)        -> (labels int32[n], kept_edges, n_components)
    sweep(g, tw, deltas)         -> list of cluster() results
    similarity(g, t, kind)       -> float64[m] Table-1 score (tw, tectonic, jaccard, k3, effres)
    cluster_f64(g, score, delta) -> cluster() on real-valued scores
    partition_stats(g, labels)   -> (n_communities, largest, intra_edges, sum_D2, modularity)
    sweep_report(g, tw, deltas)  -> per-delta points (kept, #CC, largest, E_in, sum_D2, Q)
    select(deltas, largest, n, modularity, jump_factor=0.1) -> (index, rule)
    k4(g)                        -> int64[m] 4-cliques containing each canonical edge

Every function is pinned in tests/test_oracle_pins.py against brute force, closed forms,
invariants and library routines (scipy / networkx); see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "twc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile twc_oracle.c with gcc (-O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-shared", "-fPIC",
                               "-Wall", "-Wextra", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_score.argtypes = [I64, P, P, I64, I64, P, P, P]
        lib.oracle_score.restype = ctypes.c_int
        lib.oracle_cluster.argtypes = [I64, P, P, P, ctypes.c_double, P, P]
        lib.oracle_cluster.restype = ctypes.c_int
        lib.oracle_similarity.argtypes = [I64, P, P, P, ctypes.c_int32, P]
        lib.oracle_similarity.restype = ctypes.c_int
        lib.oracle_cluster_f64.argtypes = [I64, P, P, P, ctypes.c_double, P, P]
        lib.oracle_cluster_f64.restype = ctypes.c_int
        lib.oracle_partition_stats.argtypes = [I64, P, P, P, P, P]
        lib.oracle_partition_stats.restype = ctypes.c_int
        lib.oracle_select.argtypes = [ctypes.c_int32, P, P, I64, P, ctypes.c_double, P]
        lib.oracle_select.restype = ctypes.c_int32
        lib.oracle_k4.argtypes = [I64, P, P, P]
        lib.oracle_k4.restype = ctypes.c_int
        lib.oracle_times.argtypes = [P]
        lib.oracle_times.restype = None
        lib.oracle_max_threads.restype = ctypes.c_int
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else None


def _csr(g):
    rowptr = np.ascontiguousarray(g.rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(g.colidx, dtype=np.int32)
    return rowptr, colidx


def set_threads(k: int) -> None:
    _load().oracle_set_threads(int(k))


def last_times():
    """Steady-clock seconds of the last score() (O2) and of the filter (O3) and BFS (O4) parts of
    the last cluster() -- SURVEY 8(d) oracle timing; measurement only."""
    out = np.zeros(3, dtype=np.float64)
    _load().oracle_times(_ptr(out))
    return {"O2": float(out[0]), "O3": float(out[1]), "O4": float(out[2])}


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def score(g, rows=None):
    """Per-edge (t, wedge, TW) for every canonical edge, or only for the edges whose smaller
    endpoint lies in rows=(u_begin, u_end) (other entries stay 0)."""
    lib = _load()
    rowptr, colidx = _csr(g)
    m = int(rowptr[-1]) // 2 if g.n > 0 else 0
    t = np.zeros(m, dtype=np.int32)
    wedge = np.zeros(m, dtype=np.int32)
    tw = np.zeros(m, dtype=np.int32)
    u0, u1 = (0, g.n) if rows is None else rows
    if m:
        rc = lib.oracle_score(g.n, _ptr(rowptr), _ptr(colidx), int(u0), int(u1),
                              _ptr(t), _ptr(wedge), _ptr(tw))
        if rc:
            raise MemoryError("oracle_score allocation failed")
    return t, wedge, tw


def cluster(g, tw, delta: float):
    lib = _load()
    rowptr, colidx = _csr(g)
    tw = np.ascontiguousarray(tw, dtype=np.int32)
    labels = np.empty(g.n, dtype=np.int32)
    stats = np.zeros(2, dtype=np.int64)
    rc = lib.oracle_cluster(g.n, _ptr(rowptr), _ptr(colidx), _ptr(tw), float(delta),
                            _ptr(labels), _ptr(stats))
    if rc:
        raise MemoryError("oracle_cluster allocation failed")
    return labels, int(stats[0]), int(stats[1])


def sweep(g, tw, deltas):
    return [cluster(g, tw, d) for d in deltas]


KINDS = {"tw": 0, "tectonic": 1, "jaccard": 2, "k3": 3, "effres": 4}


def similarity(g, t, kind):
    """Table 1 scores (fp64) from the triangle counts t; kind in KINDS."""
    lib = _load()
    rowptr, colidx = _csr(g)
    t = np.ascontiguousarray(t, dtype=np.int32)
    out = np.zeros(t.size, dtype=np.float64)
    if t.size:
        rc = lib.oracle_similarity(g.n, _ptr(rowptr), _ptr(colidx), _ptr(t), KINDS[kind], _ptr(out))
        if rc:
            raise ValueError("bad kind")
    return out


def cluster_f64(g, score, delta: float):
    lib = _load()
    rowptr, colidx = _csr(g)
    score = np.ascontiguousarray(score, dtype=np.float64)
    labels = np.empty(g.n, dtype=np.int32)
    stats = np.zeros(2, dtype=np.int64)
    rc = lib.oracle_cluster_f64(g.n, _ptr(rowptr), _ptr(colidx), _ptr(score), float(delta),
                                _ptr(labels), _ptr(stats))
    if rc:
        raise MemoryError("oracle_cluster_f64 allocation failed")
    return labels, int(stats[0]), int(stats[1])


def partition_stats(g, labels):
    """(n_communities, largest, intra_edges, sum_c D_c^2, modularity) of labels[n]."""
    lib = _load()
    rowptr, colidx = _csr(g)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    out = np.zeros(4, dtype=np.int64)
    q = np.zeros(1, dtype=np.float64)
    rc = lib.oracle_partition_stats(g.n, _ptr(rowptr), _ptr(colidx), _ptr(labels), _ptr(out),
                                    _ptr(q))
    if rc == 1:
        raise MemoryError("oracle_partition_stats allocation failed")
    if rc == 2:
        raise ValueError("label out of range")
    return int(out[0]), int(out[1]), int(out[2]), int(out[3]), float(q[0])


def select(deltas, largest, n, modularity, jump_factor=0.1):
    """Selection rules of P:898-900 -> (index into deltas, rule 0 = jump / 1 = modularity)."""
    lib = _load()
    d = np.ascontiguousarray(deltas, dtype=np.float64)
    lg = np.ascontiguousarray(largest, dtype=np.int64)
    q = np.ascontiguousarray(modularity, dtype=np.float64)
    rule = np.zeros(1, dtype=np.int32)
    idx = lib.oracle_select(int(d.size), _ptr(d), _ptr(lg), int(n), _ptr(q), float(jump_factor),
                            _ptr(rule))
    return int(idx), int(rule[0])


def sweep_report(g, tw, deltas):
    """One dict per delta (input order): kept, n_cc, largest, intra, sum_d2, modularity."""
    pts = []
    for d in deltas:
        labels, kept, ncc = cluster(g, tw, d)
        nc, largest, intra, sd2, q = partition_stats(g, labels)
        assert nc == ncc
        pts.append({"delta": float(d), "kept": kept, "n_cc": nc, "largest": largest,
                    "intra": intra, "sum_d2": sd2, "modularity": q})
    return pts


def k4(g):
    """K4 participation per canonical edge (Table 1), int64[m]."""
    lib = _load()
    rowptr, colidx = _csr(g)
    m = int(rowptr[-1]) // 2 if g.n > 0 else 0
    out = np.zeros(m, dtype=np.int64)
    if m:
        if lib.oracle_k4(g.n, _ptr(rowptr), _ptr(colidx), _ptr(out)):
            raise MemoryError("oracle_k4 allocation failed")
    return out
