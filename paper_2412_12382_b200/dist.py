"""One graph over P GPUs (include/twc.h `twc_dist_*`).

The six phases run in libtwc.so; this module only marshals arguments and runs the three
exchanges between them over a communicator:

    t, wedge, tw, labels, stats, (c0, c1) = score_sweep_distributed(rowptr, colidx, deltas)

on every rank (one process per GPU, torch.distributed initialised; NCCL on a B200 node, where
the exchanges are NCCL all-to-alls / all-gathers over NVLink).  t / wedge / tw are full-length
device arrays of which this rank wrote its canonical slice [c0, c1); labels [k, n] and stats
[k, 2] are complete on every rank.  `Emulated(world)` drives all ranks of one graph inside one
process (ranks run one after the other; the exchanges are buffer routing) -- the parity and
timing harness for a single GPU.
"""
from __future__ import annotations

import ctypes

import torch

from . import _check, _graph, _ptr, _stream, load_library


class TorchComm:
    """The exchanges over a torch.distributed process group.  With the gloo backend (CPU tests)
    device buffers are staged through host memory; with NCCL they stay on the device."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host = dist.get_backend(group) == "gloo"

    def _io(self, x):
        return x.cpu() if self.host else x

    def all_to_all(self, sends, sizes, width):
        """sends[0]: int32 buffer holding, in destination order, sizes[0][q] records of `width`
        ints for rank q.  Returns ([received buffer], [records received from each rank])."""
        send, ssz = sends[0], [int(x) for x in sizes[0]]
        dev = send.device
        ss = torch.tensor(ssz, dtype=torch.int64, device="cpu" if self.host else dev)
        rs = torch.empty_like(ss)
        self.dist.all_to_all_single(rs, ss, group=self.group)
        rsz = [int(x) for x in rs.tolist()]
        out = torch.empty(max(1, width * sum(rsz)), dtype=send.dtype,
                          device="cpu" if self.host else dev)
        src = self._io(send[:width * sum(ssz)]) if sum(ssz) else \
            torch.empty(0, dtype=send.dtype, device=out.device)
        self.dist.all_to_all_single(out[:width * sum(rsz)], src,
                                    [width * x for x in rsz], [width * x for x in ssz],
                                    group=self.group)
        return [out.to(dev)], [rsz]

    def all_gather(self, xs):
        """xs[0]: equal-shaped tensor on every rank -> [stacked [world, ...] tensor]."""
        x = xs[0]
        parts = [torch.empty_like(self._io(x)) for _ in range(self.world)]
        self.dist.all_gather(parts, self._io(x).contiguous(), group=self.group)
        return [torch.stack(parts).to(x.device)]

    def max_int(self, vals):
        v = torch.tensor([int(vals[0])], dtype=torch.int64,
                         device="cpu" if self.host else torch.device("cuda"))
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(v.item())


class Emulated:
    """All `world` ranks of one graph in this process: the exchanges route buffers."""

    def __init__(self, world):
        self.world = world

    def all_to_all(self, sends, sizes, width):
        P = self.world
        sizes = [[int(x) for x in s] for s in sizes]
        starts = []
        for r in range(P):
            acc, st = 0, []
            for q in range(P):
                st.append(acc)
                acc += sizes[r][q]
            starts.append(st)
        outs, rsz = [], []
        for q in range(P):
            segs = [sends[r][width * starts[r][q]: width * (starts[r][q] + sizes[r][q])]
                    for r in range(P)]
            outs.append(torch.cat(segs) if segs else torch.empty(0, dtype=torch.int32))
            rsz.append([sizes[r][q] for r in range(P)])
        return outs, rsz

    def all_gather(self, xs):
        st = torch.stack(list(xs))
        return [st for _ in range(self.world)]

    def max_int(self, vals):
        return max(int(v) for v in vals)


class DistRank:
    """One rank's buffers and workspace (they carry the oriented CSR and counts between the
    phases, include/twc.h)."""

    def __init__(self, rowptr, colidx, deltas, rank, world, stream=None):
        self.lib = load_library()
        self.rowptr, self.colidx = rowptr, colidx
        self.g, self.n, self.m = _graph(rowptr, colidx)
        self.rank, self.world = int(rank), int(world)
        self.deltas = [float(d) for d in deltas]
        self.k = len(self.deltas)
        self._d = (ctypes.c_double * self.k)(*self.deltas)
        self.stream = stream
        dev = colidx.device
        n, m = self.n, self.m
        rb = rowptr.element_size()
        self.ws = torch.empty(max(1, self.lib.twc_dist_workspace_bytes(n, m, rb, world)),
                              dtype=torch.uint8, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        self.send = torch.empty(max(2, 2 * m), **i32)
        self.send_sizes = torch.zeros(world, **i64)
        self.req = torch.empty(max(1, m), **i32)
        self.req_sizes = torch.zeros(world, **i64)
        self.t, self.wedge, self.tw = (torch.zeros(m, **i32) for _ in range(3))
        self.forest = torch.empty(max(2, 2 * (n - 1)), **i32)
        self.forest_cum = torch.zeros(self.k, **i64)
        self.kept_sizes = torch.zeros(self.k, **i64)
        self.nforest = torch.zeros(1, **i64)
        self.labels = torch.empty((self.k, n), **i32)
        self.stats = torch.empty((self.k, 2), **i64)

    def _s(self):
        return _stream(self.stream)

    def count(self):
        _check(self.lib.twc_dist_count(ctypes.byref(self.g), self.rank, self.world,
                                       _ptr(self.ws), self.ws.numel(), _ptr(self.send),
                                       _ptr(self.send_sizes), self._s()))
        return self.send, self.send_sizes.tolist()

    def apply(self, recv, nrecv):
        _check(self.lib.twc_dist_apply(ctypes.byref(self.g), self.world, _ptr(self.ws),
                                       self.ws.numel(), _ptr(recv), int(nrecv), self._s()))

    def epilogue(self):
        _check(self.lib.twc_dist_epilogue(ctypes.byref(self.g), self.rank, self.world,
                                          ctypes.cast(self._d, ctypes.c_void_p), self.k,
                                          _ptr(self.ws), self.ws.numel(), _ptr(self.t),
                                          _ptr(self.wedge), _ptr(self.tw), _ptr(self.req),
                                          _ptr(self.req_sizes), self._s()))
        return self.req, self.req_sizes.tolist()

    def serve(self, req_in, nreq):
        reply = torch.empty(max(1, int(nreq)), dtype=torch.int32, device=self.colidx.device)
        _check(self.lib.twc_dist_serve(ctypes.byref(self.g), self.world, _ptr(self.ws),
                                       self.ws.numel(), _ptr(req_in), int(nreq), _ptr(reply),
                                       self._s()))
        return reply

    def forest_phase(self, reply):
        _check(self.lib.twc_dist_forest(ctypes.byref(self.g), self.world,
                                        ctypes.cast(self._d, ctypes.c_void_p), self.k,
                                        _ptr(self.ws), self.ws.numel(), _ptr(reply),
                                        _ptr(self.t), _ptr(self.wedge), _ptr(self.tw),
                                        _ptr(self.forest), _ptr(self.forest_cum),
                                        _ptr(self.kept_sizes), _ptr(self.nforest), self._s()))
        return int(self.nforest.item())

    def sweep(self, forests, cap, fcum_all, kept_all):
        _check(self.lib.twc_dist_sweep(ctypes.byref(self.g), self.world,
                                       ctypes.cast(self._d, ctypes.c_void_p), self.k,
                                       _ptr(self.ws), self.ws.numel(), _ptr(forests), int(cap),
                                       _ptr(fcum_all), _ptr(kept_all), _ptr(self.labels),
                                       _ptr(self.stats), self._s()))


def run_phases(ranks, comm):
    """The distributed step for the ranks this process drives (1 with TorchComm, all of them
    with Emulated).  Returns per rank the number of records each exchange moved."""
    P = ranks[0].world
    # 1: counts owed to other ranks -> all-to-all -> applied
    sends, sizes = zip(*[r.count() for r in ranks])
    recvs, rsz = comm.all_to_all(list(sends), list(sizes), 2)
    for r, buf, s in zip(ranks, recvs, rsz):
        r.apply(buf, sum(s))
    # 2: epilogue of the slice; counts of foreign slots requested from their owners
    reqs, qsz = zip(*[r.epilogue() for r in ranks])
    req_in, req_in_sz = comm.all_to_all(list(reqs), list(qsz), 1)
    replies_out = [r.serve(buf, sum(s)) for r, buf, s in zip(ranks, req_in, req_in_sz)]
    replies, _ = comm.all_to_all(replies_out, req_in_sz, 1)
    # 3: local forests -> all-gather -> global sweep
    nf = [r.forest_phase(rep) for r, rep in zip(ranks, replies)]
    cap = max(1, comm.max_int(nf))
    forests = comm.all_gather([r.forest[:2 * cap] if r.forest.numel() >= 2 * cap else
                               torch.nn.functional.pad(r.forest, (0, 2 * cap - r.forest.numel()))
                               for r in ranks])
    fcum = comm.all_gather([r.forest_cum for r in ranks])
    kept = comm.all_gather([r.kept_sizes for r in ranks])
    for r, f, c, k in zip(ranks, forests, fcum, kept):
        r.sweep(f.contiguous(), cap, c.contiguous(), k.contiguous())
    return [{"counts_pairs_in": sum(s), "requests_in": sum(q), "forest_pairs": f,
             "forest_cap": cap} for s, q, f in zip(rsz, req_in_sz, nf)]


def slice_bounds(rowptr, colidx, world):
    """Host restatement of the row split (k_dist_bounds) for tests and reporting: rows[r] = first u
    with rp_or[u] >= r m / P over the degree orientation, and the canonical slices eoff[rows]."""
    import numpy as np
    rp = rowptr.cpu().numpy().astype(np.int64)
    ci = colidx.cpu().numpy().astype(np.int64)
    n = rp.size - 1
    m = int(rp[-1]) // 2 if n > 0 else 0
    deg = np.diff(rp)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    out = (deg[src] < deg[ci]) | ((deg[src] == deg[ci]) & (src < ci))
    rp_or = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src[out], minlength=n), out=rp_or[1:])
    eoff = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src[ci > src], minlength=n), out=eoff[1:])
    rows = [0] + [int(np.searchsorted(rp_or, m * r // world, side="left"))
                  for r in range(1, world)] + [n]
    return rows, [int(eoff[u]) for u in rows]


def score_sweep_distributed(rowptr, colidx, deltas, group=None, stream=None):
    """The step on this process's GPU as rank dist.get_rank(group) of the group."""
    comm = TorchComm(group)
    r = DistRank(rowptr, colidx, deltas, comm.rank, comm.world, stream)
    info = run_phases([r], comm)[0]
    return r.t, r.wedge, r.tw, r.labels, r.stats, info


def score_sweep_emulated(rowptr, colidx, deltas, world):
    """All `world` ranks on this GPU, one after the other (parity / per-rank timing harness)."""
    ranks = [DistRank(rowptr, colidx, deltas, r, world) for r in range(world)]
    info = run_phases(ranks, Emulated(world))
    return ranks, info
