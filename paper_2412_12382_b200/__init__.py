"""paper_2412_12382_b200 -- B200 (sm_100a) triangle/wedge (TW) edge scoring and motif-based
clustering (arXiv 2412.12382, Alg. 1 with the TW score of Eq. 2).

Thin ctypes binding over libtwc.so (include/twc.h): argument marshalling only; every step of
the path runs in the library's CUDA kernels.  PyTorch supplies device memory and streams.
There is no CPU fallback: if libtwc.so is missing or no CUDA device is present, calls raise.

    t, wedge, tw      = twc_score(rowptr, colidx)                  # device int32[m] each
    labels, stats     = twc_cluster(rowptr, colidx, tw, delta)     # int32[n], int64[2]
    labels, stats     = twc_sweep(rowptr, colidx, tw, deltas)      # int32[k, n], int64[k, 2]
    out               = twc_pipeline_host(rowptr_h, colidx_h, deltas)   # host in, host out
    t, wedge, tw, labels, stats = twc_score_sweep(rowptr, colidx, deltas)   # fused device path
    twc_validate_csr(rowptr, colidx)                                # raises TwcError if invalid
    counts, q         = twc_partition_stats(rowptr, colidx, labels)  # int64[k, 4], float64[k]
    index, rule       = twc_select_threshold(deltas, largest, q, n)  # host, rules of thumb
    report            = sweep_report(rowptr, colidx, deltas)         # the selection workflow
    t, wedge, tw, k4  = twc_score_k4(rowptr, colidx)                 # + 4-clique participation

rowptr: int32 or int64 tensor [n+1]; colidx: int32 tensor [2m] (CUDA tensors, except for
twc_pipeline_host which takes CPU tensors, ideally pinned).  Outputs are in canonical edge
order: the edges (u, v), u < v, lexicographically.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtwc.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "twc.h")

TWC_OK, TWC_EINVAL, TWC_EWORKSPACE, TWC_ECUDA, TWC_EGRAPH = range(5)


class TwcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class _Csr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("rowptr", ctypes.c_void_p),
                ("rowptr_bytes", ctypes.c_int32), ("colidx", ctypes.c_void_p)]


_lib = None


def load_library(path: str | None = None):
    """Load libtwc.so (raises OSError loudly when it was not built).  TWC_LIB=checked selects the
    checked build libtwc_checked.so (device-side asserts, build.py); TWC_LIB=<name> an A/B variant
    libtwc_<name>.so built with `build.py --variant <name> -D...`."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None:
        path = LIB_PATH
        if os.environ.get("TWC_LIB"):  # "checked", or an A/B variant built by build.py --variant
            path = os.path.join(_HERE, f"libtwc_{os.environ['TWC_LIB']}.so")
    if not os.path.exists(path):
        raise OSError(f"{path} not found: build it with `python -m paper_2412_12382_b200.build` "
                      "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    CP = ctypes.POINTER(_Csr)
    sig = {
        "twc_score_workspace_bytes": (SZ, [I64, I64, I32]),
        "twc_score": (ctypes.c_int, [CP, P, SZ, P, P, P, P]),
        "twc_cluster_workspace_bytes": (SZ, [I64, I64, I32]),
        "twc_cluster": (ctypes.c_int, [CP, P, ctypes.c_double, P, SZ, P, P, P]),
        "twc_sweep": (ctypes.c_int, [CP, P, P, I32, P, SZ, P, P, P]),
        "twc_pipeline_workspace_bytes": (SZ, [I64, I64, I32, I32]),
        "twc_pipeline_host": (ctypes.c_int, [CP, P, I32, P, SZ, P, P, P, P, P, P]),
        "twc_pipeline_host_async": (ctypes.c_int, [CP, P, I32, P, SZ, P, P, P, P, P, P]),
        "twc_validate_csr": (ctypes.c_int, [CP, P, P]),
        "twc_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "twc_last_error": (ctypes.c_char_p, []),
        "twc_version": (I32, []),
        "twc_score_ex": (ctypes.c_int, [CP, P, SZ, P, P, P, P, P]),
        "twc_sweep_ex": (ctypes.c_int, [CP, P, P, I32, P, SZ, P, P, P, P]),
        "twc_kernel_launches": (I64, []),
        "twc_score_sweep_workspace_bytes": (SZ, [I64, I64, I32]),
        "twc_score_sweep": (ctypes.c_int, [CP, P, I32, P, SZ, P, P, P, P, P, P, P]),
        "twc_similarity": (ctypes.c_int, [CP, P, I32, P, SZ, P, P]),
        "twc_sweep_f64": (ctypes.c_int, [CP, P, P, I32, P, SZ, P, P, P]),
        "twc_score_k4_workspace_bytes": (SZ, [I64, I64, I32]),
        "twc_score_k4": (ctypes.c_int, [CP, P, SZ, P, P, P, P, P]),
        "twc_partition_stats_workspace_bytes": (SZ, [I64, I64, I32]),
        "twc_partition_stats": (ctypes.c_int, [CP, P, I32, P, SZ, P, P, P]),
        "twc_select_threshold": (ctypes.c_int, [P, P, P, I32, I64, ctypes.c_double, P, P]),
        "twc_sweep_norm_stats": (ctypes.c_int, [I64, I64, I32, P, P, P]),
        "twc_dist_workspace_bytes": (SZ, [I64, I64, I32, I32]),
        "twc_dist_count": (ctypes.c_int, [CP, I32, I32, P, SZ, P, P, P]),
        "twc_dist_apply": (ctypes.c_int, [CP, I32, P, SZ, P, I64, P]),
        "twc_dist_epilogue": (ctypes.c_int, [CP, I32, I32, P, I32, P, SZ, P, P, P, P, P, P]),
        "twc_dist_serve": (ctypes.c_int, [CP, I32, P, SZ, P, I64, P, P]),
        "twc_dist_forest": (ctypes.c_int, [CP, I32, P, I32, P, SZ, P, P, P, P, P, P, P, P, P]),
        "twc_dist_sweep": (ctypes.c_int, [CP, I32, P, I32, P, SZ, P, I64, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def header_functions(path: str = HEADER_PATH):
    """Names of every function include/twc.h declares (for the ABI export test)."""
    txt = open(path).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(twc_[a-z_]+)\s*\(", txt)))


def _check(status: int):
    if status != TWC_OK:
        lib = load_library()
        raise TwcError(status, f"{lib.twc_status_string(status).decode()}: "
                               f"{lib.twc_last_error().decode()}")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


def _graph(rowptr, colidx, need_cuda=True):
    if rowptr.dtype not in (torch.int32, torch.int64) or colidx.dtype != torch.int32:
        raise TypeError("rowptr must be int32/int64 and colidx int32")
    if need_cuda and (not rowptr.is_cuda or not colidx.is_cuda):
        raise ValueError("rowptr/colidx must be CUDA tensors")
    if not rowptr.is_contiguous() or not colidx.is_contiguous():
        raise ValueError("rowptr/colidx must be contiguous")
    n = rowptr.numel() - 1
    m = colidx.numel() // 2
    g = _Csr(n, m, _ptr(rowptr) if n >= 0 else None, rowptr.element_size(), _ptr(colidx))
    return g, n, m


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _workspace(nbytes, device, workspace=None, stream=None):
    """The caller's workspace if it is large enough, else a temporary one.  A temporary is
    allocated on torch's current stream; when the library runs on another `stream`, the
    temporary is tied to that stream (record_stream) so that the caching allocator does not hand
    its memory out again before the enqueued kernels are done with it."""
    if workspace is not None and workspace.numel() >= nbytes:
        return workspace
    ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
    if stream is not None and stream != torch.cuda.current_stream(ws.device):
        ws.record_stream(stream)
    return ws


def twc_score_workspace_bytes(n, m, rowptr_bytes=4):
    return int(load_library().twc_score_workspace_bytes(n, m, rowptr_bytes))


def twc_cluster_workspace_bytes(n, m, rowptr_bytes=4):
    return int(load_library().twc_cluster_workspace_bytes(n, m, rowptr_bytes))


def twc_pipeline_workspace_bytes(n, m, rowptr_bytes=4, k=1):
    return int(load_library().twc_pipeline_workspace_bytes(n, m, rowptr_bytes, k))


def _events(events):
    """torch.cuda.Event list -> C array of cudaEvent_t (events must already exist: record once)."""
    if events is None:
        return None
    arr = (ctypes.c_void_p * len(events))(*[ctypes.c_void_p(e.cuda_event) for e in events])
    return ctypes.cast(arr, ctypes.c_void_p), arr


def twc_kernel_launches():
    return int(load_library().twc_kernel_launches())


def twc_score(rowptr, colidx, out=None, workspace=None, stream=None, events=None):
    """Per-edge (t, wedge, TW) -- P:337 and Eq. 2 -- for every canonical edge.

    events: optional list of 4 torch.cuda.Event recorded at the phase boundaries
    (TWC_SCORE_NEVENTS, include/twc.h)."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    if out is None:
        out = tuple(torch.empty(m, dtype=torch.int32, device=dev) for _ in range(3))
    t, wedge, tw = out
    ws = _workspace(lib.twc_score_workspace_bytes(n, m, rowptr.element_size()),
                    dev, workspace, stream)
    ev = _events(events)
    _check(lib.twc_score_ex(ctypes.byref(g), _ptr(ws), ws.numel(), _ptr(t), _ptr(wedge), _ptr(tw),
                            _stream(stream), ev[0] if ev else None))
    return t, wedge, tw


def twc_cluster(rowptr, colidx, tw, delta, labels=None, stats=None, workspace=None, stream=None):
    """Alg. 1 at one threshold: labels[u] = min vertex id of u's component."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=dev)
    if stats is None:
        stats = torch.empty(2, dtype=torch.int64, device=dev)
    ws = _workspace(lib.twc_cluster_workspace_bytes(n, m, rowptr.element_size()),
                    dev, workspace, stream)
    _check(lib.twc_cluster(ctypes.byref(g), _ptr(tw), float(delta), _ptr(ws), ws.numel(),
                           _ptr(labels), _ptr(stats), _stream(stream)))
    return labels, stats


def twc_sweep(rowptr, colidx, tw, deltas, labels=None, stats=None, workspace=None, stream=None,
              events=None):
    """Alg. 1 for k thresholds reusing the scores: labels[i] for deltas[i].

    events: optional list of 3 torch.cuda.Event (TWC_SWEEP_NEVENTS, include/twc.h)."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    deltas = [float(d) for d in deltas]
    k = len(deltas)
    if labels is None:
        labels = torch.empty((k, n), dtype=torch.int32, device=dev)
    if stats is None:
        stats = torch.empty((k, 2), dtype=torch.int64, device=dev)
    arr = (ctypes.c_double * k)(*deltas)
    ws = _workspace(lib.twc_cluster_workspace_bytes(n, m, rowptr.element_size()),
                    dev, workspace, stream)
    ev = _events(events)
    _check(lib.twc_sweep_ex(ctypes.byref(g), _ptr(tw), ctypes.cast(arr, ctypes.c_void_p), k,
                            _ptr(ws), ws.numel(), _ptr(labels), _ptr(stats), _stream(stream),
                            ev[0] if ev else None))
    return labels, stats


def twc_score_sweep_workspace_bytes(n, m, rowptr_bytes=4):
    return int(load_library().twc_score_sweep_workspace_bytes(n, m, rowptr_bytes))


def twc_score_sweep(rowptr, colidx, deltas, out=None, labels=None, stats=None, workspace=None,
                    stream=None, events=None):
    """twc_score + twc_sweep in one fused call: returns (t, wedge, tw, labels[k, n], stats[k, 2]).

    events: optional list of 6 torch.cuda.Event (see include/twc.h)."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    deltas = [float(d) for d in deltas]
    k = len(deltas)
    if out is None:
        out = tuple(torch.empty(m, dtype=torch.int32, device=dev) for _ in range(3))
    if labels is None:
        labels = torch.empty((k, n), dtype=torch.int32, device=dev)
    if stats is None:
        stats = torch.empty((k, 2), dtype=torch.int64, device=dev)
    t, wedge, tw = out
    arr = (ctypes.c_double * k)(*deltas)
    ws = _workspace(lib.twc_score_sweep_workspace_bytes(n, m, rowptr.element_size()), dev,
                    workspace, stream)
    ev = _events(events)
    _check(lib.twc_score_sweep(ctypes.byref(g), ctypes.cast(arr, ctypes.c_void_p), k, _ptr(ws),
                               ws.numel(), _ptr(t), _ptr(wedge), _ptr(tw), _ptr(labels),
                               _ptr(stats), _stream(stream), ev[0] if ev else None))
    return t, wedge, tw, labels, stats


SIM_KINDS = {"tw": 0, "tectonic": 1, "jaccard": 2, "k3": 3, "effres": 4}


def twc_similarity(rowptr, colidx, t, kind, out=None, workspace=None, stream=None):
    """Table-1 edge similarity (fp64, canonical order) from the triangle counts t:
    kind in 'tw', 'tectonic', 'jaccard', 'k3', 'effres'."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    if out is None:
        out = torch.empty(m, dtype=torch.float64, device=dev)
    ws = _workspace(lib.twc_cluster_workspace_bytes(n, m, rowptr.element_size()),
                    dev, workspace, stream)
    _check(lib.twc_similarity(ctypes.byref(g), _ptr(t), SIM_KINDS[kind], _ptr(ws), ws.numel(),
                              _ptr(out), _stream(stream)))
    return out


def twc_sweep_f64(rowptr, colidx, score, deltas, labels=None, stats=None, workspace=None,
                  stream=None):
    """Alg. 1 for k thresholds on real-valued scores: keep e iff NOT (score[e] < delta)."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    deltas = [float(d) for d in deltas]
    k = len(deltas)
    if labels is None:
        labels = torch.empty((k, n), dtype=torch.int32, device=dev)
    if stats is None:
        stats = torch.empty((k, 2), dtype=torch.int64, device=dev)
    arr = (ctypes.c_double * k)(*deltas)
    ws = _workspace(lib.twc_cluster_workspace_bytes(n, m, rowptr.element_size()),
                    dev, workspace, stream)
    _check(lib.twc_sweep_f64(ctypes.byref(g), _ptr(score), ctypes.cast(arr, ctypes.c_void_p), k,
                             _ptr(ws), ws.numel(), _ptr(labels), _ptr(stats), _stream(stream)))
    return labels, stats


def twc_pipeline_host(rowptr, colidx, deltas, want_scores=True, out=None, workspace=None,
                      stream=None, device=None, asynchronous=False):
    """Host CSR in, host results out: H2D copy, score, sweep, D2H copy (one C call).

    rowptr/colidx: CPU tensors (pinned for full PCIe speed).  Returns dict with host tensors
    t, wedge, tw (if want_scores), labels [k, n] and stats [k, 2].  asynchronous=True calls
    twc_pipeline_host_async: the results are valid once `stream` completes."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx, need_cuda=False)
    deltas = [float(d) for d in deltas]
    k = len(deltas)
    dev = torch.device("cuda") if device is None else torch.device(device)
    if out is None:
        pin = torch.cuda.is_available()
        out = {"labels": torch.empty((k, n), dtype=torch.int32, pin_memory=pin),
               "stats": torch.empty((k, 2), dtype=torch.int64, pin_memory=pin)}
        if want_scores:
            for key in ("t", "wedge", "tw"):
                out[key] = torch.empty(m, dtype=torch.int32, pin_memory=pin)
    arr = (ctypes.c_double * k)(*deltas)
    ws = _workspace(lib.twc_pipeline_workspace_bytes(n, m, rowptr.element_size(), k), dev,
                    workspace, stream)
    fn = lib.twc_pipeline_host_async if asynchronous else lib.twc_pipeline_host
    _check(fn(ctypes.byref(g), ctypes.cast(arr, ctypes.c_void_p), k, _ptr(ws), ws.numel(),
              _ptr(out.get("t")), _ptr(out.get("wedge")), _ptr(out.get("tw")),
              _ptr(out["labels"]), _ptr(out["stats"]), _stream(stream)))
    if asynchronous:
        # the device keeps using the workspace and the host buffers after this returns: the
        # workspace is tied to `stream` (_workspace); keep the inputs referenced from out
        out["_inflight"] = (rowptr, colidx, ws)
    return out


def twc_validate_csr(rowptr, colidx, stream=None):
    """Raise TwcError(TWC_EGRAPH) unless the CSR is symmetric, sorted, loop-free (row a0)."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    verdict = torch.zeros(1, dtype=torch.int32, device=colidx.device)
    _check(lib.twc_validate_csr(ctypes.byref(g), _ptr(verdict), _stream(stream)))
    return 0


RULES = {0: "largest_cc_jump", 1: "max_modularity"}


def twc_partition_stats_workspace_bytes(n, m, rowptr_bytes=4):
    return int(load_library().twc_partition_stats_workspace_bytes(n, m, rowptr_bytes))


def twc_partition_stats(rowptr, colidx, labels, counts=None, modularity=None, workspace=None,
                        stream=None):
    """Per-partition statistics of labels [k, n] (or [n]) on the input
    graph: counts [k, 4] = (n_communities, largest, intra_edges, sum_deg_sq) and the
    modularity [k] (float64).  Synchronises the stream."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    lab = labels.reshape(-1, n) if n > 0 else labels.reshape(-1, 0)
    if labels.dtype != torch.int32 or not labels.is_contiguous() or not labels.is_cuda:
        raise ValueError("labels must be a contiguous int32 CUDA tensor")
    k = lab.shape[0] if n > 0 else max(1, labels.numel())
    if counts is None:
        counts = torch.empty((k, 4), dtype=torch.int64, device=dev)
    if modularity is None:
        modularity = torch.empty(k, dtype=torch.float64, device=dev)
    ws = _workspace(lib.twc_partition_stats_workspace_bytes(n, m, rowptr.element_size()), dev,
                    workspace, stream)
    _check(lib.twc_partition_stats(ctypes.byref(g), _ptr(labels), k, _ptr(ws), ws.numel(),
                                   _ptr(counts), _ptr(modularity), _stream(stream)))
    return counts, modularity


def twc_select_threshold(deltas, largest, modularity, n, jump_factor=0.1):
    """The rules of thumb of P:895-900 (reading C22) over k sweep points (host values):
    returns (index into deltas, rule name)."""
    lib = load_library()
    k = len(deltas)
    d = (ctypes.c_double * k)(*[float(x) for x in deltas])
    lg = (ctypes.c_int64 * k)(*[int(x) for x in largest])
    q = (ctypes.c_double * k)(*[float(x) for x in modularity])
    idx, rule = ctypes.c_int32(-1), ctypes.c_int32(-1)
    _check(lib.twc_select_threshold(ctypes.cast(d, ctypes.c_void_p), ctypes.cast(lg, ctypes.c_void_p),
                                    ctypes.cast(q, ctypes.c_void_p), k, int(n), float(jump_factor),
                                    ctypes.byref(idx), ctypes.byref(rule)))
    return int(idx.value), RULES[rule.value]


def twc_sweep_norm_stats(n, m, counts, kept_stats=None):
    """P:887-889's normalised sweep statistics from host int64 counts [k, 4] and kept_stats
    [k, 2]: float64 [k, 3] = (n_communities / n, kept / m, largest / n) (computed in C)."""
    lib = load_library()
    counts = counts.to(torch.int64).contiguous().reshape(-1, 4)
    k = counts.shape[0]
    kept = None if kept_stats is None else kept_stats.to(torch.int64).contiguous().reshape(-1, 2)
    norm = torch.empty((k, 3), dtype=torch.float64)
    _check(lib.twc_sweep_norm_stats(int(n), int(m), k, _ptr(counts), _ptr(kept), _ptr(norm)))
    return norm


def sweep_report(rowptr, colidx, deltas, tw=None, jump_factor=0.1, stream=None):
    """The threshold-selection workflow: score once (unless tw is
    given), filter + label at every delta, the statistics of each partition and the selected
    delta.  Returns {"points": [{delta, norm_cc, norm_edges, norm_largest_cc, modularity,
    n_cc, kept, largest, intra_edges, sum_deg_sq}, ...] in input order, "selected_delta",
    "selected_index", "rule", "labels" (device [k, n])}."""
    n = rowptr.numel() - 1
    m = colidx.numel() // 2
    if tw is None:
        _, _, tw, labels, stats = twc_score_sweep(rowptr, colidx, deltas, stream=stream)
    else:
        labels, stats = twc_sweep(rowptr, colidx, tw, deltas, stream=stream)
    counts, q = twc_partition_stats(rowptr, colidx, labels, stream=stream)
    norm = twc_sweep_norm_stats(n, m, counts.cpu(), stats.cpu())
    counts, q, stats = counts.cpu().tolist(), q.cpu().tolist(), stats.cpu().tolist()
    pts = []
    for d, c, qq, st, nm in zip(deltas, counts, q, stats, norm.tolist()):
        pts.append({"delta": float(d), "n_cc": c[0], "largest": c[1], "intra_edges": c[2],
                    "sum_deg_sq": c[3], "kept": st[0], "modularity": qq,
                    "norm_cc": nm[0], "norm_edges": nm[1], "norm_largest_cc": nm[2]})
    out = {"points": pts, "labels": labels}
    if n > 0:
        i, rule = twc_select_threshold(deltas, [p["largest"] for p in pts], q, n, jump_factor)
        out.update(selected_index=i, selected_delta=float(deltas[i]), rule=rule)
    return out


def twc_score_k4_workspace_bytes(n, m, rowptr_bytes=4):
    return int(load_library().twc_score_k4_workspace_bytes(n, m, rowptr_bytes))


def twc_score_k4(rowptr, colidx, out=None, workspace=None, stream=None):
    """twc_score plus K4 participation (Table 1): returns (t, wedge, tw, k4), k4 an
    int64 tensor of 4-clique counts per canonical edge."""
    lib = load_library()
    g, n, m = _graph(rowptr, colidx)
    dev = colidx.device
    if out is None:
        out = tuple(torch.empty(m, dtype=torch.int32, device=dev) for _ in range(3)) + (
            torch.empty(m, dtype=torch.int64, device=dev),)
    t, wedge, tw, k4 = out
    ws = _workspace(lib.twc_score_k4_workspace_bytes(n, m, rowptr.element_size()),
                    dev, workspace, stream)
    _check(lib.twc_score_k4(ctypes.byref(g), _ptr(ws), ws.numel(), _ptr(t), _ptr(wedge), _ptr(tw),
                            _ptr(k4), _stream(stream)))
    return t, wedge, tw, k4
