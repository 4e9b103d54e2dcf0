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

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

__device__ __forceinline__ int uf_find(int* parent, int x) {
    int cur = parent[x];
    if (cur != x) {
        int prev = x, next;
        while (cur > (next = parent[cur])) {
            parent[prev] = next;  // path halving; benign race, keeps parent[y] <= y
            prev = cur;
            cur = next;
        }
    }
    return cur;
}

__device__ __forceinline__ void uf_unite(int* parent, int u, int v) {
    int ru = uf_find(parent, u), rv = uf_find(parent, v);
    while (ru != rv) {
        if (ru < rv) { int tmp = ru; ru = rv; rv = tmp; }  // hook the larger root ru under rv
        const int old = atomicCAS(&parent[ru], ru, rv);
        if (old == ru) break;
        ru = uf_find(parent, old);
        rv = uf_find(parent, rv);
    }
}

__global__ void k_init_parent(int64_t n, int* __restrict__ parent) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) parent[u] = (int)u;
}

constexpr int kSweepThreads = 256;
constexpr int kItemsPerThread = kTile / kSweepThreads;  // 4
constexpr int kMaxTileRows = 2048;
constexpr int kMaxK = 1024;

// Band of an edge: the first step (thresholds sorted descending) at which it is kept,
// b = #{i : thr_sorted[i] > TW}; b == k means kept at no threshold.
__device__ __forceinline__ int band_of(long long val, const long long* thr, int k) {
    int lo = 0, hi = k;  // thr descending: predicate thr[i] > val is true on a prefix
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (thr[mid] > val) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Pass 1: histogram of bands (edges kept at no threshold are not counted).
__global__ void __launch_bounds__(kSweepThreads) k_band_count(int64_t m, const int* __restrict__ tw,
                                                              const long long* __restrict__ thr_g,
                                                              int k, int* __restrict__ cnt) {
    __shared__ long long s_thr[kMaxK];
    __shared__ int s_hist[kMaxK];
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        s_thr[i] = thr_g[i];
        s_hist[i] = 0;
    }
    __syncthreads();
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int b = band_of(tw[c], s_thr, k);
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
template <typename RP>
__global__ void __launch_bounds__(kSweepThreads) k_band_scatter(
    int64_t m, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ eoff, const int* __restrict__ trow, const int* __restrict__ tw,
    const long long* __restrict__ thr_g, int k, int* __restrict__ cursor,
    int2* __restrict__ pairs) {
    __shared__ long long s_thr[kMaxK];
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
                band[it] = band_of(tw[c], s_thr, k);
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
                                                   int* __restrict__ parent) {
    const int beg = off[b], end = off[b + 1];
    for (int i = beg + blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += gridDim.x * blockDim.x) {
        const int2 e = pairs[i];
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
        const int r = uf_find(parent, (int)u);
        labels[u] = r;
        parent[u] = r;
        roots += (r == (int)u);
    }
    const long long tot = block_sum_ll(roots, s_tmp);
    if (threadIdx.x == 0 && tot && ncomp) atomicAdd(ncomp, (unsigned long long)tot);
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
    // thresholds in descending order (fewest kept edges first): kept sets nest
    int order[kMaxK];
    long long thr_sorted[kMaxK];
    for (int i = 0; i < k; ++i) order[i] = i;
    for (int i = 1; i < k; ++i)  // insertion sort, k is small
        for (int j = i; j > 0 && thr[order[j]] > thr[order[j - 1]]; --j) {
            int tmp = order[j]; order[j] = order[j - 1]; order[j - 1] = tmp;
        }
    for (int i = 0; i < k; ++i) thr_sorted[i] = thr[order[i]];
    // pageable host -> device copies: staged by the driver before the call returns
    cudaMemcpyAsync(w.thr, thr_sorted, sizeof(long long) * k, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(w.order, order, sizeof(int) * k, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(w.cnt, 0, sizeof(int) * (k + 1), s);
    const unsigned nb = (unsigned)((n + 255) / 256);
    k_init_parent<<<nb, 256, 0, s>>>(n, w.parent);
    count_launches(1);
    if (m > 0) {
        upper_counts<RP>(n, rowptr, colidx, w.up, s);
        exclusive_scan(w.up, w.eoff, n, w.scan_tmp, s);
        tile_first_rows(w.eoff, (int)n, m, w.trow, s);
        const int cgrid = (int)std::min<int64_t>((m + kSweepThreads - 1) / kSweepThreads,
                                                 (int64_t)sms * 8);
        k_band_count<<<cgrid, kSweepThreads, 0, s>>>(m, tw, w.thr, k, w.cnt);
        k_band_offsets<<<1, 32, 0, s>>>(w.cnt, k, w.order, w.off, w.cursor, st);
        const int64_t nt = num_tiles(m);
        const int sgrid = (int)std::min<int64_t>(nt, (int64_t)sms * 8);
        k_band_scatter<RP><<<sgrid, kSweepThreads, 0, s>>>(m, rowptr, colidx, w.eoff, w.trow, tw,
                                                           w.thr, k, w.cursor, w.pairs);
        count_launches(3);
    }
    record(ev, 1, s);
    const int hook_grid = sms * 8;
    const int fin_grid = (int)std::min<int64_t>((int64_t)nb, (int64_t)sms * 8);
    for (int i = 0; i < k; ++i) {
        const int idx = order[i];
        if (m > 0 && (i == 0 || thr_sorted[i] < thr_sorted[i - 1])) {
            k_hook_list<<<hook_grid, 256, 0, s>>>(w.pairs, w.off, i, w.parent);
            count_launches(1);
        }
        k_finalize<<<fin_grid, 256, 0, s>>>(n, w.parent, labels + (size_t)idx * n,
                                            st + 2 * idx + 1);
        count_launches(1);
    }
    record(ev, 2, s);
    return cudaGetLastError();
}

template cudaError_t sweep_impl<int>(int64_t, int64_t, const int*, const int*, const int*,
                                     const long long*, int, void*, size_t, int*, long long*,
                                     cudaStream_t, cudaEvent_t*);
template cudaError_t sweep_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                           const int*, const long long*, int, void*, size_t,
                                           int*, long long*, cudaStream_t, cudaEvent_t*);

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
