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
// union-find is grown incrementally: step i hooks only the edges with thr_i <= TW < thr_{i-1}
// and snapshots the compressed labels.
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

constexpr int kHookThreads = 256;
constexpr int kMaxTileRows = 2048;

// Hook every canonical edge with lo <= TW < hi; count edges with TW >= lo into *kept.
template <typename RP>
__global__ void __launch_bounds__(kHookThreads) k_hook_band(
    int64_t n, int64_t m, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ eoff, const int* __restrict__ trow, const int* __restrict__ tw,
    long long lo, long long hi, int* __restrict__ parent, unsigned long long* __restrict__ kept) {
    __shared__ int s_off[kMaxTileRows + 1];
    __shared__ long long s_tmp[32];
    const int64_t ntiles = num_tiles(m);
    long long nkept = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c0 = (int)(tile * kTile);
        const int c1 = (int)min((int64_t)c0 + kTile, m);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;
        const bool cached = nr <= kMaxTileRows;
        __syncthreads();
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_off[i] = eoff[r0 + i];
        __syncthreads();
        for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
            const long long val = tw[c];
            nkept += (val >= lo);
            if (val >= lo && val < hi) {
                const int ri = cached ? last_le(s_off, nr + 1, c) : last_le(eoff + r0, nr + 1, c);
                const int u = r0 + ri;
                const int eu = cached ? s_off[ri] : eoff[u];
                const int upu = (cached ? s_off[ri + 1] : eoff[u + 1]) - eu;
                const RP rb = rowptr[u];
                const int du = (int)(rowptr[u + 1] - rb);
                const int v = colidx[rb + (RP)(du - upu) + (RP)(c - eu)];
                uf_unite(parent, u, v);
            }
        }
    }
    const long long tot = block_sum_ll(nkept, s_tmp);
    if (threadIdx.x == 0 && tot) atomicAdd(kept, (unsigned long long)tot);
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
        roots += (r == (int)u);
    }
    const long long tot = block_sum_ll(roots, s_tmp);
    if (threadIdx.x == 0 && tot && ncomp) atomicAdd(ncomp, (unsigned long long)tot);
}

struct ClusterWs {
    int *up, *eoff, *scan_tmp, *trow, *parent;
    unsigned long long* stats;  // 2 per threshold (used when caller passes NULL)
};

static ClusterWs carve_cluster(Carver& cv, int64_t n, int64_t m) {
    ClusterWs w;
    w.up = cv.take<int>(n);
    w.eoff = cv.take<int>(n + 1);
    w.scan_tmp = cv.take<int>(scan_temp_bytes(n) / sizeof(int));
    w.trow = cv.take<int>(num_tiles(m) + 1);
    w.parent = cv.take<int>(n);
    w.stats = cv.take<unsigned long long>(2);
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
    const int sms = num_sms();
    if (stats) cudaMemsetAsync(stats, 0, sizeof(long long) * 2 * (size_t)k, s);
    if (n == 0) {
        record(ev, 1, s);
        record(ev, 2, s);
        return cudaGetLastError();
    }
    // thresholds in descending order (fewest kept edges first)
    int order[1024];
    for (int i = 0; i < k; ++i) order[i] = i;
    for (int i = 1; i < k; ++i)  // insertion sort, k is small
        for (int j = i; j > 0 && thr[order[j]] > thr[order[j - 1]]; --j) {
            int tmp = order[j]; order[j] = order[j - 1]; order[j - 1] = tmp;
        }
    const unsigned nb = (unsigned)((n + 255) / 256);
    k_init_parent<<<nb, 256, 0, s>>>(n, w.parent);
    count_launches(1);
    if (m > 0) {
        upper_counts<RP>(n, rowptr, colidx, w.up, s);
        exclusive_scan(w.up, w.eoff, n, w.scan_tmp, s);
        tile_first_rows(w.eoff, (int)n, m, w.trow, s);
    }
    record(ev, 1, s);
    const long long kInf = (long long)1 << 62;
    long long hi = kInf;
    const int64_t nt = num_tiles(m);
    const int hook_grid = (int)std::min<int64_t>(std::max<int64_t>(nt, 1), (int64_t)sms * 8);
    const int fin_grid = (int)std::min<int64_t>((int64_t)nb, (int64_t)sms * 8);
    for (int i = 0; i < k; ++i) {
        const int idx = order[i];
        const long long lo = thr[idx];
        unsigned long long* st = stats ? reinterpret_cast<unsigned long long*>(stats) + 2 * idx
                                       : w.stats;
        if (!stats) cudaMemsetAsync(w.stats, 0, 2 * sizeof(unsigned long long), s);
        if (m > 0 && lo < hi) {
            k_hook_band<RP><<<hook_grid, kHookThreads, 0, s>>>(n, m, rowptr, colidx, w.eoff,
                                                               w.trow, tw, lo, hi, w.parent, st);
            count_launches(1);
        } else if (m > 0 && stats && i > 0) {
            // duplicate threshold: same kept count as the previous (equal) threshold
            k_hook_band<RP><<<hook_grid, kHookThreads, 0, s>>>(n, m, rowptr, colidx, w.eoff,
                                                               w.trow, tw, lo, lo, w.parent, st);
            count_launches(1);
        }
        k_finalize<<<fin_grid, 256, 0, s>>>(n, w.parent, labels + (size_t)idx * n, st + 1);
        count_launches(1);
        if (lo < hi) hi = lo;
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
