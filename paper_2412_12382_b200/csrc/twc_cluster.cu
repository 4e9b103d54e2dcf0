// twc_cluster.cu -- Alg. 1: threshold edge filter + connected components, and the
// multi-threshold sweep; CSR validation (row a0).
//
// Filter: edge e is kept iff NOT (TW(e) < delta) (reading C4).  TW is an integer, so
// this is exactly TW(e) >= ceil(delta); the host converts delta to that integer threshold
// (twc_api.cu) and the kernels compare integers.
//
// Connected components: lock-free union-find.  A hook always links the LARGER root under the
// SMALLER one with atomicCAS, so parent[x] <= x at all times and the surviving root of every
// tree is its minimum vertex id; compression then yields labels[u] = min id of u's component,
// the canonical labelling of S:208-210 / S:228 (reading C6), independent of the order in which
// racing hooks win (reading C19).
//
// Sweep: for thresholds taken in DESCENDING order the kept sets are nested, so one
// union-find is grown incrementally.  One pass buckets every kept edge by the first step that
// keeps it (its "band": thr_i <= TW < thr_{i-1}); step i then hooks only band i's edges and
// snapshots the compressed labels.
#include <algorithm>
#include <cstring>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

__global__ void k_init_parent(int64_t n, int* __restrict__ parent) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) parent[u] = (int)u;
}

constexpr int kSweepThreads = 256;
constexpr int kItemsPerThread = kTile / kSweepThreads;  // 4
constexpr int kMaxTileRows = 2048;

// Pass 1: histogram of bands (edges kept at no threshold are not counted).
template <typename S, typename TH>
__global__ void __launch_bounds__(kSweepThreads) k_band_count(int64_t m, const S* __restrict__ tw,
                                                              const TH* __restrict__ thr_g,
                                                              int k, int* __restrict__ cnt) {
    __shared__ TH s_thr[kMaxK];
    __shared__ int s_hist[kMaxK];
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        s_thr[i] = thr_g[i];
        s_hist[i] = 0;
    }
    __syncthreads();
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int b = band_of_t(tw[c], s_thr, k);
        if (b < k) atomicAdd(&s_hist[b], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&cnt[i], s_hist[i]);
}

// Band offsets (exclusive scan, k <= 1024), cursors, and the kept-edge statistics of every
// threshold (kept(i) = edges in bands 0..i), written at the caller's index order[i].
__global__ void k_band_offsets(const int* __restrict__ cnt, int k, const int* __restrict__ order,
                               int* __restrict__ off, int* __restrict__ cursor,
                               unsigned long long* __restrict__ stats) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int run = 0;
    for (int i = 0; i < k; ++i) {
        off[i] = run;
        cursor[i] = run;
        run += cnt[i];
        if (stats) stats[2 * order[i]] = (unsigned long long)run;
    }
    off[k] = run;
}

// Pass 2: scatter each kept edge (u, v) into its band's segment.  Each CTA reserves, per band,
// one contiguous range per tile (one global atomic per band and tile).  A thread handles
// kItemsPerThread consecutive canonical ids: one row search, then a walk along the rows.
template <typename RP, typename S, typename TH>
__global__ void __launch_bounds__(kSweepThreads) k_band_scatter(
    int64_t m, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ eoff, const int* __restrict__ trow, const S* __restrict__ tw,
    const TH* __restrict__ thr_g, int k, int* __restrict__ cursor,
    int2* __restrict__ pairs) {
    __shared__ TH s_thr[kMaxK];
    __shared__ int s_cnt[kMaxK];
    __shared__ int s_off[kMaxTileRows + 1];
    for (int i = threadIdx.x; i < k; i += blockDim.x) s_thr[i] = thr_g[i];
    const int64_t ntiles = num_tiles(m);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c0 = (int)(tile * kTile);
        const int c1 = (int)min((int64_t)c0 + kTile, m);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;
        const bool cached = nr <= kMaxTileRows;
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x) s_cnt[i] = 0;
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_off[i] = eoff[r0 + i];
        __syncthreads();
        const int cs = c0 + threadIdx.x * kItemsPerThread;
        int band[kItemsPerThread];
        int rank[kItemsPerThread];
        bool any = false;
#pragma unroll
        for (int it = 0; it < kItemsPerThread; ++it) {
            const int c = cs + it;
            band[it] = k;
            rank[it] = 0;
            if (c < c1) {
                band[it] = band_of_t(tw[c], s_thr, k);
                if (band[it] < k) {
                    rank[it] = atomicAdd(&s_cnt[band[it]], 1);
                    any = true;
                }
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x)
            if (s_cnt[i]) s_cnt[i] = atomicAdd(&cursor[i], s_cnt[i]);
        __syncthreads();
        if (!any) continue;
        int ri = cached ? last_le(s_off, nr + 1, cs) : last_le(eoff + r0, nr + 1, cs);
        int eu = cached ? s_off[ri] : eoff[r0 + ri];
        int ee = cached ? s_off[ri + 1] : eoff[r0 + ri + 1];
        int u = r0 + ri;
        RP rb = rowptr[u];
        int du = (int)(rowptr[u + 1] - rb);
#pragma unroll
        for (int it = 0; it < kItemsPerThread; ++it) {
            const int c = cs + it;
            if (band[it] >= k) continue;
            if (c >= ee) {
                do {
                    ++ri;
                    eu = ee;
                    ee = cached ? s_off[ri + 1] : eoff[r0 + ri + 1];
                } while (c >= ee);
                u = r0 + ri;
                rb = rowptr[u];
                du = (int)(rowptr[u + 1] - rb);
            }
            const int v = colidx[rb + (RP)(du - (ee - eu)) + (RP)(c - eu)];
            pairs[s_cnt[band[it]] + rank[it]] = make_int2(u, v);
        }
    }
}

// Hook the edges of band b (one step of the sweep).
__global__ void __launch_bounds__(256) k_hook_list(const int2* __restrict__ pairs,
                                                   const int* __restrict__ off, int b,
                                                   int* __restrict__ parent, int64_t n) {
    const int beg = off[b], end = off[b + 1];
    const unsigned size = (unsigned)(end - beg);
    // A large first band unites singletons: with every thread of the GPU hooking at once, half of
    // the CAS attempts fail (the root found is no longer a root) and the walks get long, so the
    // band is taken by max(n / 8, size / 64, 32 Ki) threads only -- fewer concurrent hooks per
    // vertex, still enough threads for the band's bulk (measured on configs 2-4 and the R-MAT
    // graphs; config 3's sweep 0.24 -> 0.13 ms).
    unsigned nblk = gridDim.x;
    if (b == 0 && (int64_t)size * 16 >= n) {
        const int64_t thr = max(max(n / 8, (int64_t)size / 64), (int64_t)32768);
        nblk = (unsigned)min((int64_t)gridDim.x, (thr + blockDim.x - 1) / blockDim.x);
    }
    if (blockIdx.x >= nblk) return;
    // visit the band in a scrambled order so that edges sharing a vertex (neighbours in the
    // band, which keeps canonical row order) are not handled by neighbouring threads at the
    // same time: j = (i * odd) mod 2^p is a bijection of [0, 2^p) (2^p >= size); the j >= size
    // are skipped, so every edge of the band is visited exactly once
    unsigned p2 = 1;
    while (p2 < size) p2 <<= 1;
    const unsigned mask = p2 - 1u;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < p2; i += nblk * blockDim.x) {
        const unsigned j = (i * 2654435761u) & mask;
        if (j >= size) continue;
        const int2 e = pairs[beg + j];
        TWC_ASSERT(e.x >= 0 && e.y >= 0 && e.x != e.y);
        // equal parents: already in one tree (the previous step's finalize left every vertex
        // pointing at its root, so this settles most edges inside an existing component with
        // two reads instead of two root walks)
        if (parent[e.x] == parent[e.y]) continue;
        uf_unite(parent, e.x, e.y);
    }
}

// labels[u] = root(u) (= min id of its component); compress; count roots.
__global__ void __launch_bounds__(256) k_finalize(int64_t n, int* __restrict__ parent,
                                                  int* __restrict__ labels,
                                                  unsigned long long* __restrict__ ncomp) {
    __shared__ long long s_tmp[32];
    long long roots = 0;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int p = parent[u];
        const int r = (p == (int)u) ? p : uf_find(parent, (int)u);
        __stcs(&labels[u], r);            // streaming store: labels are not re-read
        if (r != p) parent[u] = r;        // full compression, only when it changes
        roots += (r == (int)u);
    }
    const long long tot = block_sum_ll(roots, s_tmp);
    if (threadIdx.x == 0 && tot && ncomp) atomicAdd(ncomp, (unsigned long long)tot);
}

// Thresholds (sorted descending) and their caller indices into the workspace, 64 per launch
// through kernel parameters (no host->device memcpy, so the sweep is graph-capturable).
struct ThrChunk {
    long long thr[64];
    int order[64];
};

__global__ void k_set_thresholds(ThrChunk c, int base, int cnt, long long* __restrict__ thr,
                                 int* __restrict__ order) {
    const int i = threadIdx.x;
    if (i < cnt) {
        thr[base + i] = c.thr[i];
        order[base + i] = c.order[i];
    }
}

struct ClusterWs {
    int *up, *eoff, *scan_tmp, *trow, *parent, *cnt, *off, *cursor, *order;
    long long* thr;
    int2* pairs;
    unsigned long long* stats;  // 2 per threshold (used when caller passes NULL)
};

static ClusterWs carve_cluster(Carver& cv, int64_t n, int64_t m) {
    ClusterWs w;
    w.up = cv.take<int>(n);
    w.eoff = cv.take<int>(n + 1);
    w.scan_tmp = cv.take<int>(scan_temp_bytes(n) / sizeof(int));
    w.trow = cv.take<int>(num_tiles(m) + 1);
    w.parent = cv.take<int>(n);
    w.cnt = cv.take<int>(kMaxK + 1);
    w.off = cv.take<int>(kMaxK + 1);
    w.cursor = cv.take<int>(kMaxK + 1);
    w.order = cv.take<int>(kMaxK);
    w.thr = cv.take<long long>(kMaxK);
    w.pairs = cv.take<int2>(m);
    w.stats = cv.take<unsigned long long>(2 * kMaxK);
    return w;
}

size_t cluster_ws_bytes(int64_t n, int64_t m) {
    Carver cv(nullptr, 0);
    carve_cluster(cv, n, m);
    return cv.used;
}

// ------------------------------------------------------------------ sweep building blocks
void sweep_plan(const long long* thr, int k, SweepPlan* P) {
    P->k = k;
    for (int i = 0; i < k; ++i) P->order[i] = i;
    for (int i = 1; i < k; ++i)  // insertion sort (stable), k is small
        for (int j = i; j > 0 && thr[P->order[j]] > thr[P->order[j - 1]]; --j) {
            int tmp = P->order[j]; P->order[j] = P->order[j - 1]; P->order[j - 1] = tmp;
        }
    for (int i = 0; i < k; ++i) P->thr[i] = thr[P->order[i]];
    for (int i = 0; i < k; ++i) P->fresh[i] = (i == 0) || (P->thr[i] < P->thr[i - 1]);
}

void sweep_plan_f64(const double* thr, int k, SweepPlan* P) {
    P->k = k;
    for (int i = 0; i < k; ++i) P->order[i] = i;
    for (int i = 1; i < k; ++i)
        for (int j = i; j > 0 && thr[P->order[j]] > thr[P->order[j - 1]]; --j) {
            int tmp = P->order[j]; P->order[j] = P->order[j - 1]; P->order[j - 1] = tmp;
        }
    for (int i = 0; i < k; ++i) {
        const double d = thr[P->order[i]];
        memcpy(&P->thr[i], &d, sizeof(double));  // bit pattern, uploaded as is
        P->fresh[i] = (i == 0) || (d < thr[P->order[i - 1]]);
    }
}

void sweep_upload(const SweepPlan& P, long long* thr_dev, int* order_dev, cudaStream_t s) {
    for (int b = 0; b < P.k; b += 64) {
        ThrChunk c;
        const int cnt = std::min(64, P.k - b);
        for (int i = 0; i < cnt; ++i) {
            c.thr[i] = P.thr[b + i];
            c.order[i] = P.order[b + i];
        }
        k_set_thresholds<<<1, 64, 0, s>>>(c, b, cnt, thr_dev, order_dev);
        count_launches(1);
    }
}

void band_offsets(const int* cnt, int k, const int* order_dev, int* off, int* cursor,
                  unsigned long long* stats, cudaStream_t s) {
    k_band_offsets<<<1, 32, 0, s>>>(cnt, k, order_dev, off, cursor, stats);
    count_launches(1);
}

// Place a compact list of kept edges into their band segments: per block, one reservation
// per band (smem histogram), then smem ranks.
__global__ void __launch_bounds__(kSweepThreads) k_band_place(
    const int2* __restrict__ kept, const unsigned short* __restrict__ kband,
    const int* __restrict__ nkept, int k, int* __restrict__ cursor, int2* __restrict__ pairs) {
    __shared__ int s_cnt[kMaxK];
    const int total = *nkept;
    constexpr int kChunk = kSweepThreads * 4;
    for (int base = blockIdx.x * kChunk; base < total; base += gridDim.x * kChunk) {
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        int b[4], r[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int i = base + it * kSweepThreads + threadIdx.x;
            b[it] = -1;
            if (i < total) {
                b[it] = kband[i];
                TWC_ASSERT(b[it] >= 0 && b[it] < k);
                r[it] = atomicAdd(&s_cnt[b[it]], 1);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x)
            if (s_cnt[i]) s_cnt[i] = atomicAdd(&cursor[i], s_cnt[i]);
        __syncthreads();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int i = base + it * kSweepThreads + threadIdx.x;
            if (b[it] >= 0) pairs[s_cnt[b[it]] + r[it]] = kept[i];
        }
    }
}

void band_place(const int2* kept, const unsigned short* kband, const int* nkept, int64_t cap,
                int k, int* cursor, int2* pairs, cudaStream_t s) {
    const int64_t chunks = (cap + kSweepThreads * 4 - 1) / (kSweepThreads * 4);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)num_sms() * 8));
    k_band_place<<<grid, kSweepThreads, 0, s>>>(kept, kband, nkept, k, cursor, pairs);
    count_launches(1);
}

void init_parent(int64_t n, int* parent, cudaStream_t s) {
    k_init_parent<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, parent);
    count_launches(1);
}

// Steps in descending threshold order: hook band i, snapshot labels for threshold order[i].
void sweep_loop(int64_t n, int64_t m, const SweepPlan& P, const int2* pairs, const int* off,
                int* parent, int* labels, unsigned long long* st, cudaStream_t s,
                cudaEvent_t* step_ev) {
    const int sms = num_sms();
    const int hook_grid = sms * 8;
    const int fin_grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
    for (int i = 0; i < P.k; ++i) {
        const int idx = P.order[i];
        if (m > 0 && P.fresh[i]) {
            k_hook_list<<<hook_grid, 256, 0, s>>>(pairs, off, i, parent, n);
            count_launches(1);
        }
        k_finalize<<<fin_grid, 256, 0, s>>>(n, parent, labels + (size_t)idx * n, st + 2 * idx + 1);
        count_launches(1);
        if (step_ev) cudaEventRecord(step_ev[i], s);  // labels of threshold order[i] final
    }
}

template <typename RP>
cudaError_t sweep_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, const int* tw,
                       const long long* thr, int k, void* ws, size_t ws_bytes, int* labels,
                       long long* stats, cudaStream_t s, cudaEvent_t* ev) {
    Carver cv(ws, ws_bytes);
    ClusterWs w = carve_cluster(cv, n, m);
    record(ev, 0, s);
    unsigned long long* st = stats ? reinterpret_cast<unsigned long long*>(stats) : w.stats;
    cudaMemsetAsync(st, 0, sizeof(long long) * 2 * (size_t)k, s);
    if (n == 0) {
        record(ev, 1, s);
        record(ev, 2, s);
        return cudaGetLastError();
    }
    const int sms = num_sms();
    SweepPlan P;
    sweep_plan(thr, k, &P);
    sweep_upload(P, w.thr, w.order, s);
    cudaMemsetAsync(w.cnt, 0, sizeof(int) * (k + 1), s);
    init_parent(n, w.parent, s);
    if (m > 0) {
        upper_counts<RP>(n, rowptr, colidx, w.up, s);
        exclusive_scan(w.up, w.eoff, n, w.scan_tmp, s);
        tile_first_rows(w.eoff, (int)n, m, w.trow, s);
        const int cgrid = (int)std::min<int64_t>((m + kSweepThreads - 1) / kSweepThreads,
                                                 (int64_t)sms * 8);
        k_band_count<int, long long><<<cgrid, kSweepThreads, 0, s>>>(m, tw, w.thr, k, w.cnt);
        count_launches(1);
        band_offsets(w.cnt, k, w.order, w.off, w.cursor, st, s);
        const int64_t nt = num_tiles(m);
        const int sgrid = (int)std::min<int64_t>(nt, (int64_t)sms * 8);
        k_band_scatter<RP, int, long long><<<sgrid, kSweepThreads, 0, s>>>(
            m, rowptr, colidx, w.eoff, w.trow, tw, w.thr, k, w.cursor, w.pairs);
        count_launches(1);
    }
    record(ev, 1, s);
    sweep_loop(n, m, P, w.pairs, w.off, w.parent, labels, st, s);
    record(ev, 2, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ fused score + sweep
struct FusedWs {
    void* score;
    size_t score_bytes;
    int *parent, *cnt, *off, *cursor, *order, *nkept;
    long long* thr;
    int2 *kept, *pairs;
    unsigned short* kband;
    unsigned long long* stats;
};

static FusedWs carve_fused(Carver& cv, int64_t n, int64_t m) {
    FusedWs w;
    w.score_bytes = std::max(score_ws_bytes(n, m), cluster_ws_bytes(n, m));
    w.score = cv.take<char>(w.score_bytes);
    w.parent = cv.take<int>(n);
    w.cnt = cv.take<int>(kMaxK + 1);
    w.off = cv.take<int>(kMaxK + 1);
    w.cursor = cv.take<int>(kMaxK + 1);
    w.order = cv.take<int>(kMaxK);
    w.nkept = cv.take<int>(1);
    w.thr = cv.take<long long>(kMaxK);
    w.kept = cv.take<int2>(m);
    w.pairs = cv.take<int2>(m);
    w.kband = cv.take<unsigned short>(m);
    w.stats = cv.take<unsigned long long>(2 * kMaxK);
    return w;
}

size_t score_sweep_ws_bytes(int64_t n, int64_t m) {
    Carver cv(nullptr, 0);
    carve_fused(cv, n, m);
    return cv.used;
}

// events: [0] start, [1] orientation done, [2] intersection done, [3] epilogue + binning
// done, [4] bands placed, [5] all thresholds labelled.
template <typename RP>
cudaError_t score_sweep_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                             const long long* thr, int k, void* ws, size_t ws_bytes, int* t,
                             int* wedge, int* tw, int* labels, long long* stats, cudaStream_t s,
                             cudaEvent_t* ev, cudaEvent_t* step_ev) {
    Carver cv(ws, ws_bytes);
    FusedWs w = carve_fused(cv, n, m);
    unsigned long long* st = stats ? reinterpret_cast<unsigned long long*>(stats) : w.stats;
    if (m == 0 || n == 0) {  // nothing to score: every vertex is its own component
        for (int i = 0; i < 6; ++i) record(ev, i, s);
        cudaError_t e = sweep_impl<RP>(n, m, rowptr, colidx, tw, thr, k, w.score, w.score_bytes,
                                       labels, stats, s, nullptr);
        if (step_ev)
            for (int i = 0; i < k; ++i) cudaEventRecord(step_ev[i], s);
        return e;
    }
    SweepPlan P;
    sweep_plan(thr, k, &P);
    cudaMemsetAsync(st, 0, sizeof(long long) * 2 * (size_t)k, s);
    sweep_upload(P, w.thr, w.order, s);
    cudaMemsetAsync(w.cnt, 0, sizeof(int) * (k + 1), s);
    cudaMemsetAsync(w.nkept, 0, sizeof(int), s);
    BinSpec bin{w.thr, k, w.cnt, w.nkept, w.kept, w.kband, w.parent};  // K0 initialises parent
    cudaError_t e = score_impl<RP>(n, m, rowptr, colidx, w.score, w.score_bytes, t, wedge, tw, s,
                                   ev, &bin);
    if (e != cudaSuccess) return e;
    band_offsets(w.cnt, k, w.order, w.off, w.cursor, st, s);
    band_place(w.kept, w.kband, w.nkept, m, k, w.cursor, w.pairs, s);
    record(ev, 4, s);
    sweep_loop(n, m, P, w.pairs, w.off, w.parent, labels, st, s, step_ev);
    record(ev, 5, s);
    return cudaGetLastError();
}

template cudaError_t score_sweep_impl<int>(int64_t, int64_t, const int*, const int*,
                                           const long long*, int, void*, size_t, int*, int*,
                                           int*, int*, long long*, cudaStream_t, cudaEvent_t*,
                                           cudaEvent_t*);
template cudaError_t score_sweep_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                                 const long long*, int, void*, size_t, int*,
                                                 int*, int*, int*, long long*, cudaStream_t,
                                                 cudaEvent_t*, cudaEvent_t*);

template cudaError_t sweep_impl<int>(int64_t, int64_t, const int*, const int*, const int*,
                                     const long long*, int, void*, size_t, int*, long long*,
                                     cudaStream_t, cudaEvent_t*);
template cudaError_t sweep_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                           const int*, const long long*, int, void*, size_t,
                                           int*, long long*, cudaStream_t, cudaEvent_t*);

// ------------------------------------------------------------------ sweep on fp64 scores
// Alg. 1 for any Table-1 score: keep e iff NOT (score(e) < delta) in IEEE double;
// identical band / union-find machinery with double thresholds.
template <typename RP>
cudaError_t sweep_f64_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                           const double* score, const double* deltas, int k, void* ws,
                           size_t ws_bytes, int* labels, long long* stats, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    ClusterWs w = carve_cluster(cv, n, m);
    unsigned long long* st = stats ? reinterpret_cast<unsigned long long*>(stats) : w.stats;
    cudaMemsetAsync(st, 0, sizeof(long long) * 2 * (size_t)k, s);
    if (n == 0) return cudaGetLastError();
    const int sms = num_sms();
    SweepPlan P;
    sweep_plan_f64(deltas, k, &P);
    sweep_upload(P, w.thr, w.order, s);  // bit patterns of the doubles
    const double* thr_d = reinterpret_cast<const double*>(w.thr);
    cudaMemsetAsync(w.cnt, 0, sizeof(int) * (k + 1), s);
    init_parent(n, w.parent, s);
    if (m > 0) {
        upper_counts<RP>(n, rowptr, colidx, w.up, s);
        exclusive_scan(w.up, w.eoff, n, w.scan_tmp, s);
        tile_first_rows(w.eoff, (int)n, m, w.trow, s);
        const int cgrid = (int)std::min<int64_t>((m + kSweepThreads - 1) / kSweepThreads,
                                                 (int64_t)sms * 8);
        k_band_count<double, double><<<cgrid, kSweepThreads, 0, s>>>(m, score, thr_d, k, w.cnt);
        count_launches(1);
        band_offsets(w.cnt, k, w.order, w.off, w.cursor, st, s);
        const int64_t nt = num_tiles(m);
        const int sgrid = (int)std::min<int64_t>(nt, (int64_t)sms * 8);
        k_band_scatter<RP, double, double><<<sgrid, kSweepThreads, 0, s>>>(
            m, rowptr, colidx, w.eoff, w.trow, score, thr_d, k, w.cursor, w.pairs);
        count_launches(1);
    }
    sweep_loop(n, m, P, w.pairs, w.off, w.parent, labels, st, s);
    return cudaGetLastError();
}

template cudaError_t sweep_f64_impl<int>(int64_t, int64_t, const int*, const int*, const double*,
                                         const double*, int, void*, size_t, int*, long long*,
                                         cudaStream_t);
template cudaError_t sweep_f64_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                               const double*, const double*, int, void*, size_t,
                                               int*, long long*, cudaStream_t);

// ------------------------------------------------------------------------ validation
template <typename RP>
__global__ void k_validate_rowptr(int64_t n, int64_t m, const RP* __restrict__ rowptr,
                                  int* __restrict__ verdict) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u > n) return;
    bool bad = false;
    if (u == 0) bad |= rowptr[0] != 0;
    if (u == n) bad |= (long long)rowptr[n] != 2 * (long long)m;
    if (u < n) bad |= rowptr[u] > rowptr[u + 1];
    if (bad) atomicOr(verdict, 1);
}

template <typename RP>
__global__ void k_validate_rows(int64_t n, const RP* __restrict__ rowptr,
                                const int* __restrict__ colidx, int* __restrict__ verdict) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int bits = 0;
    for (int64_t u = warp; u < n; u += nwarps) {
        const RP beg = rowptr[u], end = rowptr[u + 1];
        for (RP p = beg + lane; p < end; p += 32) {
            const int v = colidx[p];
            if (v < 0 || v >= n) { bits |= 2; continue; }
            if (p > beg && colidx[p - 1] >= v) bits |= 4;
            if (v == (int)u) bits |= 8;
            const RP vb = rowptr[v];
            const int dv = (int)(rowptr[v + 1] - vb);
            const int q = lower_bound(colidx + vb, dv, (int)u);
            if (q >= dv || colidx[vb + q] != (int)u) bits |= 16;
        }
    }
    if (bits) atomicOr(verdict, bits);
}

template <typename RP>
cudaError_t validate_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                          int* verdict, cudaStream_t s) {
    cudaMemsetAsync(verdict, 0, sizeof(int), s);
    k_validate_rowptr<RP><<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(n, m, rowptr, verdict);
    count_launches(1);
    int h = 0;
    cudaMemcpyAsync(&h, verdict, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess || h != 0 || n == 0) return e;
    const int grid = (int)std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 16);
    k_validate_rows<RP><<<grid, 256, 0, s>>>(n, rowptr, colidx, verdict);
    count_launches(1);
    return cudaStreamSynchronize(s);
}

template cudaError_t validate_impl<int>(int64_t, int64_t, const int*, const int*, int*,
                                        cudaStream_t);
template cudaError_t validate_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                              int*, cudaStream_t);

}  // namespace twc
