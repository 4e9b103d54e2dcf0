// twc_dist.cu -- the hot path of ONE graph split over P GPUs.
//
// One process per GPU; every rank holds the whole (read-only) CSR.  The vertices are split into
// P contiguous row ranges R_r of equal oriented-slot counts (k_dist_bounds, twc_score.cu); rank r
// owns the oriented slots O_r of its rows and the canonical edges C_r of its rows.  Between the
// phases below the caller runs the exchange steps with its collective library (torch.distributed
// over NCCL on a B200 node; the binding does it, paper_2412_12382_b200/dist.py):
//
//   A  twc_dist_count     K0 + K1 (replicated) and K2 over the pivots of R_r: every triangle is
//                         found once, from its lowest-key vertex (P:337 counts, orientation prior
//                         art P:380).  Its (u,v), (u,w) increments land in O_r; the (v,w) ones may
//                         land in any slice.  The nonzero counts of foreign slots are compacted
//                         into (slot, count) pairs, grouped by owner (slot order = owner order).
//      -- exchange 1: all-to-all of those pairs (sparse: ~T/P pairs per rank, not m) --
//   B  twc_dist_apply     adds the received counts: t on O_r is now final.
//   C  twc_dist_epilogue  K3 over C_r: wedge = d_u + d_v - 2t - 2, TW = 3t - d_u - d_v + 2
//                         (Eq. 2) for the edges whose oriented slot is in O_r (aligned
//                         edges always are); a reversed edge whose slot belongs to rank q is
//                         recorded and its slot requested from q (requests grouped by owner).
//      -- exchange 2: all-to-all of requested slots, owners answer (twc_dist_serve), all-to-all
//         of the answers back --
//   E  twc_dist_forest    completes the requested edges; bins every kept edge of C_r by sweep
//                         step (Alg. 1 line 1), then runs union-find over the rank's kept
//                         edges, band by band in descending threshold order, and records every
//                         successful hook (ra -> rb): per band, the rank's spanning-forest edges.
//                         They connect exactly what the rank's kept edges connect.
//      -- exchange 3: all-gather of the P forests (<= n - 1 pairs each) --
//   F  twc_dist_sweep     union-find over the P forests band by band (min-id roots, so the
//                         labels are canonical whatever the order, reading C19) and one label
//                         snapshot per threshold (Alg. 1 line 2): every rank ends with
//                         the same labels[k][n] and stats, and t / wedge / TW for its C_r.
#include <algorithm>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

constexpr int kDistThreads = 256;
constexpr int kDistTile = 2048;  // slots per block pass in the compaction

// ---- workspace ------------------------------------------------------------------------------
struct DistWs {
    void* score;          // the score workspace (oriented CSR, counts) -- kept between phases
    size_t score_bytes;
    int* bounds;          // [3 (world + 1)]: rows, oriented slice bounds, canonical slice bounds
    int* ctr;             // [0] remote records, [1] kept edges
    int4* rec;            // remote reversed edges {c, u, v, slot}, as found
    int4* rec_g;          // the same grouped by owner (the order of the requests)
    int* tcnt;            // per-tile counts of the compaction, then their exclusive scan
    int* toff;
    int* scan_tmp;
    int *ohist, *ocur;    // [world + 1] per-owner counts / cursors
    long long* thr;       // thresholds, sorted descending
    int *order, *cnt, *off, *cursor;
    int2 *kept, *pairs;
    unsigned short* kband;
    int* parent;
    int* fcnt;            // forest pairs recorded in each band
    int2* gpairs;         // F: the P forests, band-segmented
    int* goff;            // F: band offsets into gpairs
    unsigned long long* stats;
};

static DistWs carve_dist(Carver& cv, int64_t n, int64_t m, int world) {
    DistWs w;
    w.score_bytes = score_ws_bytes(n, m);
    w.score = cv.take<char>(w.score_bytes);
    w.bounds = cv.take<int>(3 * (world + 1));
    w.ctr = cv.take<int>(4);
    w.rec = cv.take<int4>(m);
    w.rec_g = cv.take<int4>(m);
    const int64_t nt = (m + kDistTile - 1) / kDistTile;
    w.tcnt = cv.take<int>(nt + 1);
    w.toff = cv.take<int>(nt + 1);
    w.scan_tmp = cv.take<int>(scan_temp_bytes(nt + 1) / sizeof(int) + 1);
    w.ohist = cv.take<int>(world + 1);
    w.ocur = cv.take<int>(world + 1);
    w.thr = cv.take<long long>(kMaxK);
    w.order = cv.take<int>(kMaxK);
    w.cnt = cv.take<int>(kMaxK + 1);
    w.off = cv.take<int>(kMaxK + 1);
    w.cursor = cv.take<int>(kMaxK + 1);
    w.kept = cv.take<int2>(m);
    w.pairs = cv.take<int2>(m);
    w.kband = cv.take<unsigned short>(m);
    w.parent = cv.take<int>(n);
    w.fcnt = cv.take<int>(kMaxK);
    w.gpairs = cv.take<int2>((size_t)world * (size_t)std::max<int64_t>(n - 1, 1));
    w.goff = cv.take<int>(kMaxK + 1);
    w.stats = cv.take<unsigned long long>(2 * kMaxK);
    return w;
}

size_t dist_ws_bytes(int64_t n, int64_t m, int world) {
    Carver cv(nullptr, 0);
    carve_dist(cv, n, m, world);
    return cv.used;
}

__device__ __forceinline__ int owner_of(const int* __restrict__ ob, int world, int slot) {
    int lo = 0, hi = world;  // ob[0] = 0 <= slot < ob[world] = m: last r with ob[r] <= slot
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ob[mid] <= slot) lo = mid; else hi = mid;
    }
    return lo;
}

// ---- A: compaction of the foreign nonzero counts ----------------------------------------------
__device__ __forceinline__ bool foreign_nz(const int* t_or, int s, int lo, int hi, int64_t m) {
    return s < m && (s < lo || s >= hi) && t_or[s] != 0;
}

__global__ void __launch_bounds__(kDistThreads) k_foreign_count(int64_t m, const int* __restrict__ t_or,
                                                                 const int* __restrict__ ob,
                                                                 int rank, int* __restrict__ tcnt) {
    __shared__ int s_sum[kDistThreads / 32];
    const int lo = ob[rank], hi = ob[rank + 1];
    const int64_t nt = (m + kDistTile - 1) / kDistTile;
    for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x) {
        const int64_t base = tile * kDistTile;
        int c = 0;
        for (int j = threadIdx.x; j < kDistTile; j += kDistThreads)
            c += foreign_nz(t_or, (int)(base + j), lo, hi, m);
        c = __reduce_add_sync(FULL, c);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int i = 0; i < kDistThreads / 32; ++i) t += s_sum[i];
            tcnt[tile] = t;
        }
    }
}

// pairs (slot, count) in slot order; per-owner pair counts into send_sizes (int64, zeroed)
__global__ void __launch_bounds__(kDistThreads) k_foreign_write(
    int64_t m, const int* __restrict__ t_or, const int* __restrict__ ob, int rank, int world,
    const int* __restrict__ toff, int* __restrict__ send, unsigned long long* __restrict__ sizes) {
    __shared__ int s_wsum[kDistThreads / 32];
    __shared__ int s_hist[64];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int lo = ob[rank], hi = ob[rank + 1];
    const int64_t nt = (m + kDistTile - 1) / kDistTile;
    for (int i = threadIdx.x; i < 64; i += kDistThreads) s_hist[i] = 0;
    for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x) {
        const int64_t base = tile * kDistTile;
        int run = toff[tile];
        for (int j0 = 0; j0 < kDistTile; j0 += kDistThreads) {
            const int s = (int)(base + j0 + threadIdx.x);
            const bool nz = foreign_nz(t_or, s, lo, hi, m);
            const unsigned b = __ballot_sync(FULL, nz);
            __syncthreads();
            if (lane == 0) s_wsum[wid] = __popc(b);
            __syncthreads();
            int pre = 0, tot = 0;
#pragma unroll
            for (int i = 0; i < kDistThreads / 32; ++i) {
                pre += (i < wid) ? s_wsum[i] : 0;
                tot += s_wsum[i];
            }
            const int q = nz ? owner_of(ob, world, s) : -1 - lane;  // unique dummy if none
            const unsigned grp = __match_any_sync(FULL, q);
            if (nz) {
                const int pos = run + pre + __popc(b & ((1u << lane) - 1u));
                TWC_ASSERT(pos >= 0 && pos < m);
                send[2 * pos] = s;
                send[2 * pos + 1] = t_or[s];
                if (lane == __ffs(grp) - 1) atomicAdd(&s_hist[q], __popc(grp));
            }
            run += tot;
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < world; q += kDistThreads)
        if (s_hist[q]) atomicAdd(&sizes[q], (unsigned long long)s_hist[q]);
}

// ---- B: apply received counts -----------------------------------------------------------------
__global__ void k_apply(int64_t nrecv, const int* __restrict__ recv, int* __restrict__ t_or) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrecv;
         i += (int64_t)gridDim.x * blockDim.x)
    {
        TWC_ASSERT(recv[2 * i] >= 0 && recv[2 * i + 1] > 0);
        atomicAdd(&t_or[recv[2 * i]], recv[2 * i + 1]);
    }
}

// ---- C: group the remote records by owner ------------------------------------------------------
__global__ void k_req_hist(const int4* __restrict__ rec, const int* __restrict__ nrec,
                           const int* __restrict__ ob, int world, int* __restrict__ hist) {
    __shared__ int s_hist[64];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const int n = *nrec;
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        const int i = base + threadIdx.x;
        const int q = i < n ? owner_of(ob, world, rec[i].w) : -1 - lane;
        const unsigned grp = __match_any_sync(FULL, q);
        if (i < n && lane == __ffs(grp) - 1) atomicAdd(&s_hist[q], __popc(grp));
    }
    __syncthreads();
    for (int q = threadIdx.x; q < world; q += blockDim.x)
        if (s_hist[q]) atomicAdd(&hist[q], s_hist[q]);
}

__global__ void k_req_offsets(int world, const int* __restrict__ hist, int* __restrict__ cur,
                              unsigned long long* __restrict__ sizes) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int run = 0;
    for (int q = 0; q < world; ++q) {
        cur[q] = run;
        sizes[q] = (unsigned long long)hist[q];
        run += hist[q];
    }
}

// Requests grouped by owner: per chunk of blockDim records, one reservation per owner and block
// (a handful of owners: per-record global atomics on them would serialise).
__global__ void __launch_bounds__(kDistThreads) k_req_scatter(
    const int4* __restrict__ rec, const int* __restrict__ nrec, const int* __restrict__ ob,
    int world, int* __restrict__ cur, int4* __restrict__ rec_g, int* __restrict__ req) {
    __shared__ int s_cnt[64], s_base[64];
    const int lane = threadIdx.x & 31;
    const int n = *nrec;
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        for (int q = threadIdx.x; q < world; q += blockDim.x) s_cnt[q] = 0;
        __syncthreads();
        const int i = base + threadIdx.x;
        int4 r = make_int4(0, 0, 0, 0);
        int q = -1 - lane;
        if (i < n) {
            r = rec[i];
            q = owner_of(ob, world, r.w);
        }
        const unsigned grp = __match_any_sync(FULL, q);
        const int leader = __ffs(grp) - 1;
        int wb = 0;
        if (i < n && lane == leader) wb = atomicAdd(&s_cnt[q], __popc(grp));
        wb = __shfl_sync(FULL, wb, leader);
        const int rk = wb + __popc(grp & ((1u << lane) - 1u));
        __syncthreads();
        for (int qq = threadIdx.x; qq < world; qq += blockDim.x)
            if (s_cnt[qq]) s_base[qq] = atomicAdd(&cur[qq], s_cnt[qq]);
        __syncthreads();
        if (i < n) {
            const int pos = s_base[q] + rk;
            TWC_ASSERT(pos >= 0 && pos < n);
            rec_g[pos] = r;
            req[pos] = r.w;
        }
        __syncthreads();
    }
}

// ---- D: serve -----------------------------------------------------------------------------------
__global__ void k_serve(int64_t nreq, const int* __restrict__ req, const int* __restrict__ t_or,
                        int* __restrict__ reply) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nreq;
         i += (int64_t)gridDim.x * blockDim.x)
    {
        TWC_ASSERT(req[i] >= 0);
        reply[i] = t_or[req[i]];
    }
}

// ---- E: complete the remote edges (+ binning), local forest -------------------------------------
__global__ void __launch_bounds__(kDistThreads) k_finish_remote(
    const int4* __restrict__ rec_g, const int* __restrict__ nrec, const int* __restrict__ reply,
    const int* __restrict__ deg, int* __restrict__ t, int* __restrict__ wedge,
    int* __restrict__ tw, BinSpec bin) {
    extern __shared__ __align__(8) unsigned char fin_dyn[];  // thr[k] (i64), hist[k]
    long long* s_thr = reinterpret_cast<long long*>(fin_dyn);
    int* s_hist = reinterpret_cast<int*>(fin_dyn + 8 * (size_t)bin.k);
    for (int i = threadIdx.x; i < bin.k; i += blockDim.x) {
        s_thr[i] = bin.thr[i];
        s_hist[i] = 0;
    }
    __syncthreads();
    const int n = *nrec;
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        const int i = base + threadIdx.x;
        int b = -1 - lane;  // unique dummy for lanes without a kept edge
        int4 r = make_int4(0, 0, 0, 0);
        if (i < n) {
            r = rec_g[i];
            const int tt = reply[i];
            TWC_ASSERT(tt >= 0 && r.y >= 0 && r.z > r.y);
            const int dsum = deg[r.y] + deg[r.z];
            const int score = 3 * tt - dsum + 2;           // Eq. 2 with the P:337 closed form
            t[r.x] = tt;
            wedge[r.x] = dsum - 2 * tt - 2;
            tw[r.x] = score;
            if ((long long)score >= s_thr[bin.k - 1])     // kept at the smallest threshold
                b = band_of(score, s_thr, bin.k);
        }
        const unsigned kb = __ballot_sync(FULL, b >= 0);
        if (kb) {  // one reservation per warp, one smem atomic per distinct band
            int wpos = 0;
            if (lane == __ffs(kb) - 1) wpos = atomicAdd(bin.nkept, __popc(kb));
            wpos = __shfl_sync(FULL, wpos, __ffs(kb) - 1);
            const unsigned grp = __match_any_sync(FULL, b);
            if (b >= 0) {
                const int pos = wpos + __popc(kb & ((1u << lane) - 1u));
                bin.kept[pos] = make_int2(r.y, r.z);
                bin.kband[pos] = (unsigned short)b;
                if (lane == __ffs(grp) - 1) atomicAdd(&s_hist[b], __popc(grp));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bin.k; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&bin.cnt[i], s_hist[i]);
}

// hooks of band b; every successful hook (a -> b) is recorded: the band's forest edges, placed
// after those of the earlier bands (their counts fcnt[0..b) are final: stream order)
__global__ void __launch_bounds__(256) k_hook_record(const int2* __restrict__ pairs,
                                                     const int* __restrict__ off, int b,
                                                     int* __restrict__ parent,
                                                     int* __restrict__ forest,
                                                     int* __restrict__ fcnt, int64_t cap) {
    __shared__ int s_base[32];
    int part = 0;
    for (int j = threadIdx.x; j < b; j += blockDim.x) part += fcnt[j];
    part = __reduce_add_sync(FULL, part);
    if ((threadIdx.x & 31) == 0) s_base[threadIdx.x >> 5] = part;
    __syncthreads();
    int band_base = 0;
    for (int wv = 0; wv < (int)(blockDim.x >> 5); ++wv) band_base += s_base[wv];
    int* fpos = fcnt + b;
    const int beg = off[b], end = off[b + 1];
    const unsigned size = (unsigned)(end - beg);
    unsigned p2 = 1;  // scrambled visiting order as k_hook_list (twc_cluster.cu)
    while (p2 < size) p2 <<= 1;
    const int lane = threadIdx.x & 31;
    for (unsigned i0 = blockIdx.x * blockDim.x; i0 < p2; i0 += gridDim.x * blockDim.x) {
        const unsigned j = ((i0 + threadIdx.x) * 2654435761u) & (p2 - 1u);
        int ra = 0, rb = 0;
        bool hooked = false;
        if (i0 + threadIdx.x < p2 && j < size) {
            const int2 e = pairs[beg + j];
            hooked = uf_unite(parent, e.x, e.y, &ra, &rb);
        }
        const unsigned hb = __ballot_sync(FULL, hooked);
        if (hb) {  // one reservation per warp
            int wpos = 0;
            if (lane == __ffs(hb) - 1) wpos = atomicAdd(fpos, __popc(hb));
            wpos = __shfl_sync(FULL, wpos, __ffs(hb) - 1);
            if (hooked) {
                const int pos = band_base + wpos + __popc(hb & ((1u << lane) - 1u));
                TWC_ASSERT(ra > rb && rb >= 0 && pos < cap);
                forest[2 * pos] = ra;
                forest[2 * pos + 1] = rb;
            }
        }
    }
}

// outputs of E as int64 (the caller's collective buffers)
__global__ void k_forest_sizes(int k, const int* __restrict__ fcnt, const int* __restrict__ cnt,
                               unsigned long long* __restrict__ forest_cum,
                               unsigned long long* __restrict__ kept_sizes,
                               unsigned long long* __restrict__ nforest) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) kept_sizes[i] = (unsigned long long)cnt[i];
    if (threadIdx.x == 0) {  // k <= 1024: one serial prefix
        unsigned long long run = 0;
        for (int i = 0; i < k; ++i) {
            run += (unsigned long long)fcnt[i];
            forest_cum[i] = run;
        }
        *nforest = run;
    }
}

// ---- F: the global sweep over the P forests ------------------------------------------------------
// goff[i] = first pair of band i; kept stats of every threshold (caller index order[i])
__global__ void k_gsweep_offsets(int world, int k, const long long* __restrict__ fcum_all,
                                 const long long* __restrict__ kept_all,
                                 const int* __restrict__ order, int* __restrict__ goff,
                                 unsigned long long* __restrict__ stats) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    long long run = 0, kept = 0;
    for (int i = 0; i < k; ++i) {
        goff[i] = (int)run;
        for (int r = 0; r < world; ++r) {
            const long long lo = i ? fcum_all[r * k + i - 1] : 0;
            run += fcum_all[r * k + i] - lo;
            kept += kept_all[r * k + i];
        }
        stats[2 * order[i]] = (unsigned long long)kept;
    }
    goff[k] = (int)run;
}

// block (i, r): copy rank r's band-i forest pairs into band i's segment
__global__ void k_gsweep_copy(int world, int k, const int* __restrict__ forests, int64_t cap,
                              const long long* __restrict__ fcum_all,
                              const int* __restrict__ goff, int2* __restrict__ gpairs) {
    const int i = blockIdx.x, r = blockIdx.y;
    int64_t dst = goff[i];
    for (int q = 0; q < r; ++q)
        dst += fcum_all[q * k + i] - (i ? fcum_all[q * k + i - 1] : 0);
    const int64_t lo = i ? fcum_all[r * k + i - 1] : 0, hi = fcum_all[r * k + i];
    const int2* src = reinterpret_cast<const int2*>(forests + 2 * cap * (int64_t)r);
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) gpairs[dst + j - lo] = src[j];
}

// ---- host --------------------------------------------------------------------------------------
static int dgrid(int64_t items, int threads) {
    const int64_t b = (items + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 8));
}

template <typename RP>
cudaError_t dist_count_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, int rank,
                            int world, void* ws, size_t ws_bytes, int* send,
                            long long* send_sizes, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    DistWs w = carve_dist(cv, n, m, world);
    cudaMemsetAsync(send_sizes, 0, sizeof(long long) * (size_t)world, s);
    cudaError_t e = dist_stage_a<RP>(n, m, rowptr, colidx, w.score, w.score_bytes, rank, world,
                                     w.bounds, s);
    if (e != cudaSuccess) return e;
    Carver sc(w.score, w.score_bytes);
    const ScoreWs sw = carve_score(sc, n, m);
    const int* ob = w.bounds + (world + 1);
    const int64_t nt = (m + kDistTile - 1) / kDistTile;
    const int grid = (int)std::min<int64_t>(nt, (int64_t)num_sms() * 8);
    k_foreign_count<<<grid, kDistThreads, 0, s>>>(m, sw.t_or, ob, rank, w.tcnt);
    exclusive_scan(w.tcnt, w.toff, nt, w.scan_tmp, s);
    k_foreign_write<<<grid, kDistThreads, 0, s>>>(m, sw.t_or, ob, rank, world, w.toff, send,
                                                  reinterpret_cast<unsigned long long*>(send_sizes));
    count_launches(2);
    return cudaGetLastError();
}

cudaError_t dist_apply_impl(int64_t n, int64_t m, int world, void* ws, size_t ws_bytes,
                            const int* recv, int64_t nrecv, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    DistWs w = carve_dist(cv, n, m, world);
    Carver sc(w.score, w.score_bytes);
    const ScoreWs sw = carve_score(sc, n, m);
    if (nrecv > 0) {
        k_apply<<<dgrid(nrecv, 256), 256, 0, s>>>(nrecv, recv, sw.t_or);
        count_launches(1);
    }
    return cudaGetLastError();
}

template <typename RP>
cudaError_t dist_epilogue_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                               int rank, int world, const long long* thr, int k, void* ws,
                               size_t ws_bytes, int* t, int* wedge, int* tw, int* req,
                               long long* req_sizes, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    DistWs w = carve_dist(cv, n, m, world);
    SweepPlan P;
    sweep_plan(thr, k, &P);
    sweep_upload(P, w.thr, w.order, s);
    cudaMemsetAsync(w.cnt, 0, sizeof(int) * (k + 1), s);
    cudaMemsetAsync(w.ctr, 0, 4 * sizeof(int), s);
    cudaMemsetAsync(w.ohist, 0, sizeof(int) * (world + 1), s);
    const BinSpec bin{w.thr, k, w.cnt, w.ctr + 1, w.kept, w.kband};
    DistK3 d;
    d.cb = w.bounds + 2 * (world + 1);
    d.ob = w.bounds + (world + 1);
    d.rank = rank;
    d.rec = w.rec;
    d.nrec = w.ctr;
    cudaError_t e = dist_epilogue<RP>(n, m, rowptr, colidx, w.score, w.score_bytes, t, wedge, tw,
                                      bin, d, s);
    if (e != cudaSuccess) return e;
    const int g = num_sms() * 4;
    k_req_hist<<<g, 256, 0, s>>>(w.rec, w.ctr, d.ob, world, w.ohist);
    k_req_offsets<<<1, 32, 0, s>>>(world, w.ohist, w.ocur,
                                   reinterpret_cast<unsigned long long*>(req_sizes));
    k_req_scatter<<<g, kDistThreads, 0, s>>>(w.rec, w.ctr, d.ob, world, w.ocur, w.rec_g, req);
    count_launches(3);
    return cudaGetLastError();
}

cudaError_t dist_serve_impl(int64_t n, int64_t m, int world, void* ws, size_t ws_bytes,
                            const int* req, int64_t nreq, int* reply, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    DistWs w = carve_dist(cv, n, m, world);
    Carver sc(w.score, w.score_bytes);
    const ScoreWs sw = carve_score(sc, n, m);
    if (nreq > 0) {
        k_serve<<<dgrid(nreq, 256), 256, 0, s>>>(nreq, req, sw.t_or, reply);
        count_launches(1);
    }
    return cudaGetLastError();
}

cudaError_t dist_forest_impl(int64_t n, int64_t m, int world, const long long* thr, int k,
                             void* ws, size_t ws_bytes, const int* reply, int* t, int* wedge,
                             int* tw, int* forest, long long* forest_cum, long long* kept_sizes,
                             long long* nforest, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    DistWs w = carve_dist(cv, n, m, world);
    Carver sc(w.score, w.score_bytes);
    const ScoreWs sw = carve_score(sc, n, m);
    SweepPlan P;
    sweep_plan(thr, k, &P);
    const BinSpec bin{w.thr, k, w.cnt, w.ctr + 1, w.kept, w.kband};
    k_finish_remote<<<num_sms() * 4, kDistThreads, (size_t)k * 12, s>>>(w.rec_g, w.ctr, reply,
                                                                       sw.deg, t, wedge, tw, bin);
    count_launches(1);
    // local kept edges -> band segments (the fused path's machinery), then the local forest
    band_offsets(w.cnt, k, w.order, w.off, w.cursor, w.stats, s);
    band_place(w.kept, w.kband, w.ctr + 1, m, k, w.cursor, w.pairs, s);
    init_parent(n, w.parent, s);
    cudaMemsetAsync(w.fcnt, 0, sizeof(int) * (size_t)k, s);
    const int hook_grid = num_sms() * 8;
    for (int i = 0; i < k; ++i) {
        if (m > 0 && P.fresh[i]) {
            k_hook_record<<<hook_grid, 256, 0, s>>>(w.pairs, w.off, i, w.parent, forest, w.fcnt,
                                                    std::max<int64_t>(n - 1, 1));
            count_launches(1);
        }
    }
    k_forest_sizes<<<1, 256, 0, s>>>(k, w.fcnt, w.cnt,
                                     reinterpret_cast<unsigned long long*>(forest_cum),
                                     reinterpret_cast<unsigned long long*>(kept_sizes),
                                     reinterpret_cast<unsigned long long*>(nforest));
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t dist_sweep_impl(int64_t n, int64_t m, int world, const long long* thr, int k,
                            void* ws, size_t ws_bytes, const int* forests, int64_t cap,
                            const long long* fcum_all, const long long* kept_all, int* labels,
                            long long* stats, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    DistWs w = carve_dist(cv, n, m, world);
    SweepPlan P;
    sweep_plan(thr, k, &P);
    unsigned long long* st = stats ? reinterpret_cast<unsigned long long*>(stats) : w.stats;
    cudaMemsetAsync(st, 0, sizeof(long long) * 2 * (size_t)k, s);
    if (n == 0) return cudaGetLastError();
    k_gsweep_offsets<<<1, 32, 0, s>>>(world, k, fcum_all, kept_all, w.order, w.goff, st);
    k_gsweep_copy<<<dim3(k, world), 256, 0, s>>>(world, k, forests, cap, fcum_all, w.goff,
                                                  w.gpairs);
    count_launches(2);
    init_parent(n, w.parent, s);
    sweep_loop(n, m, P, w.gpairs, w.goff, w.parent, labels, st, s);
    return cudaGetLastError();
}

#define TWC_INST(RP)                                                                            \
    template cudaError_t dist_count_impl<RP>(int64_t, int64_t, const RP*, const int*, int, int,  \
                                             void*, size_t, int*, long long*, cudaStream_t);     \
    template cudaError_t dist_epilogue_impl<RP>(int64_t, int64_t, const RP*, const int*, int,    \
                                                int, const long long*, int, void*, size_t, int*, \
                                                int*, int*, int*, long long*, cudaStream_t);
TWC_INST(int)
TWC_INST(long long)
#undef TWC_INST

}  // namespace twc
