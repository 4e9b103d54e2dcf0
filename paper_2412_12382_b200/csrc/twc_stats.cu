// twc_stats.cu -- statistics of the sweep's partitions for the threshold-selection workflow
// ("norm # CC, norm edges, norm |largest CC|" and modularity).
//
// For each of k partitions labels[j*n .. j*n+n) (label values in [0, n), e.g. the min-id
// labels of twc_sweep) the library computes four exact integers
//     n_communities  #distinct labels
//     largest        size of the largest community
//     intra_edges    E_in = #edges {u, v} of the INPUT graph with labels[u] == labels[v]
//     sum_deg_sq     sum over communities c of D_c^2, D_c = sum of deg(u) over u in c
// and the modularity of P:350-352 as one IEEE division of exact integers (reading C21):
//     Q = (4 m E_in - sum_c D_c^2) / (4 m^2).
//
// Kernels (all HBM/L2 streaming; none is a contraction):
//   k_part_vertex  one pass over the labels and degrees: per-label size and D_c by atomics into
//                  two n-long arrays.  Each lane run-length-encodes its strided labels (a giant
//                  component costs one atomic per run, not per vertex) and a warp merges the
//                  runs that end on the same label with __match_any_sync.
//   k_part_roots   one pass over the label-indexed arrays: count / max / sum of squares of the
//                  non-empty entries, and resets them to zero for the next partition.
//   k_part_edges   one pass over the CSR for a GROUP of G partitions whose label arrays fit the
//                  L2 together (G * 4n bytes <= ~48 MB): per slot (u, v), v > u, compares
//                  labels[u] and labels[v] of each partition of the group -- the gathers hit L2.
//   k_modularity   one thread per partition.
#include <algorithm>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

constexpr int kStatThreads = 256;
constexpr int kVertItems = 8;       // vertices per lane in k_part_vertex
constexpr int kEdgeRows = 2048;     // rowptr entries cached per edge tile
constexpr int kMaxGroup = 8;        // partitions per k_part_edges pass
static_assert(kTile % kStatThreads == 0, "k_part_edges: whole slots per thread");

template <typename RP>
__global__ void __launch_bounds__(kStatThreads) k_part_vertex(
    int64_t n, const RP* __restrict__ rowptr, const int* __restrict__ lab,
    int* __restrict__ size, unsigned long long* __restrict__ dsum, int* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 32 * kVertItems; base < n; base += nwarps * 32 * kVertItems) {
        int cur = -1, cnt = 0;
        unsigned long long ds = 0;
#pragma unroll
        for (int i = 0; i < kVertItems; ++i) {
            const int64_t u = base + i * 32 + lane;
            if (u >= n) break;
            const int l = __ldcs(lab + u);
            const unsigned long long d = (unsigned long long)(rowptr[u + 1] - rowptr[u]);
            if (l < 0 || (int64_t)l >= n) {
                atomicOr(bad, 1);
                continue;
            }
            if (l != cur) {
                if (cnt) {
                    atomicAdd(size + cur, cnt);
                    atomicAdd(dsum + cur, ds);
                }
                cur = l;
                cnt = 0;
                ds = 0;
            }
            ++cnt;
            ds += d;
        }
        // merge the open runs of the warp that end on the same label (typical: one giant label)
        const unsigned grp = __match_any_sync(0xffffffffu, cur);
        const int leader = __ffs(grp) - 1;
        int csum = __reduce_add_sync(grp, (unsigned)cnt);
        unsigned long long dtot = 0;
        for (int src = 0; src < 32; ++src) {
            const unsigned long long v = __shfl_sync(0xffffffffu, ds, src);
            if ((grp >> src) & 1u) dtot += v;
        }
        if (lane == leader && cur >= 0 && csum) {
            atomicAdd(size + cur, csum);
            atomicAdd(dsum + cur, dtot);
        }
    }
}

// acc[4j + 0] communities, [4j + 1] largest, [4j + 3] sum of D_c^2 (as unsigned long long)
__global__ void __launch_bounds__(kStatThreads) k_part_roots(
    int64_t n, int* __restrict__ size, unsigned long long* __restrict__ dsum,
    unsigned long long* __restrict__ acc) {
    __shared__ unsigned long long s_cnt, s_sq;
    __shared__ int s_max;
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_sq = 0;
        s_max = 0;
    }
    __syncthreads();
    unsigned long long cnt = 0, sq = 0;
    int mx = 0;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n;
         l += (int64_t)gridDim.x * blockDim.x) {
        const int sz = size[l];
        if (sz) {
            const unsigned long long d = dsum[l];
            ++cnt;
            sq += d * d;
            mx = max(mx, sz);
            size[l] = 0;
            dsum[l] = 0;
        }
    }
    cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
    mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0 && (cnt || mx)) {
        atomicAdd(&s_cnt, cnt);
        atomicAdd(&s_sq, sq);
        atomicMax(&s_max, mx);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) {
        atomicAdd(acc + 0, s_cnt);
        atomicMax(acc + 1, (unsigned long long)s_max);
        atomicAdd(acc + 3, s_sq);
    }
}

// E_in for partitions j0 .. j0+G-1: acc[4j + 2]
template <typename RP>
__global__ void __launch_bounds__(kStatThreads) k_part_edges(
    int64_t n, int64_t slots, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ trow, const int* __restrict__ lab, int G,
    unsigned long long* __restrict__ acc) {
    __shared__ RP s_off[kEdgeRows + 1];
    __shared__ unsigned long long s_in[kMaxGroup];
    if (threadIdx.x < kMaxGroup) s_in[threadIdx.x] = 0;
    const int64_t ntiles = num_tiles(slots);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p0 = tile * kTile;
        const int64_t p1 = min(p0 + kTile, slots);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;
        const bool cached = nr <= kEdgeRows;
        __syncthreads();
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_off[i] = rowptr[r0 + i];
        __syncthreads();
        int c[kMaxGroup];
#pragma unroll
        for (int g = 0; g < kMaxGroup; ++g) c[g] = 0;
        const int64_t p = p0 + threadIdx.x;
        #pragma unroll
        for (int it = 0; it < kTile / kStatThreads; ++it) {
            const int64_t q = p + it * kStatThreads;
            if (q >= p1) break;
            const RP qq = (RP)q;
            const int ri = cached ? last_le(s_off, nr + 1, qq) : last_le(rowptr + r0, nr + 1, qq);
            const int u = r0 + ri;
            const int v = __ldcs(colidx + q);
            if (v > u) {
#pragma unroll
                for (int g = 0; g < kMaxGroup; ++g)
                    if (g < G) c[g] += (lab[(int64_t)g * n + u] == lab[(int64_t)g * n + v]);
            }
        }
#pragma unroll
        for (int g = 0; g < kMaxGroup; ++g) {
            if (g >= G) break;
            const unsigned w = __reduce_add_sync(0xffffffffu, (unsigned)c[g]);
            if ((threadIdx.x & 31) == 0 && w) atomicAdd(&s_in[g], (unsigned long long)w);
        }
    }
    __syncthreads();
    if (threadIdx.x < G && s_in[threadIdx.x]) atomicAdd(acc + 4 * threadIdx.x + 2, s_in[threadIdx.x]);
}

__global__ void k_modularity(int k, long long m, const long long* __restrict__ acc,
                             double* __restrict__ q) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    if (m == 0) {
        q[j] = __longlong_as_double(0x7ff8000000000000ll);  // NaN: undefined
        return;
    }
    const long long num = 4 * m * acc[4 * j + 2] - acc[4 * j + 3];
    q[j] = (double)num / (double)(4 * m * m);
}

size_t partition_stats_ws_bytes(int64_t n, int64_t m) {
    Carver cv(nullptr, 0);
    cv.take<int>(n);                       // size
    cv.take<unsigned long long>(n);        // dsum
    cv.take<int>(num_tiles(2 * m) + 1);    // tile rows of the full CSR
    cv.take<int>(1);                       // bad-label flag
    return cv.used;
}

template <typename RP>
cudaError_t partition_stats_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                                 const int* labels, int k, void* ws, size_t ws_bytes,
                                 long long* counts, double* q, int* bad_host, cudaStream_t s) {
    *bad_host = 0;
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(counts);
    cudaError_t e = cudaMemsetAsync(acc, 0, sizeof(long long) * 4 * (size_t)k, s);
    if (e != cudaSuccess) return e;
    if (n > 0) {
        Carver cv(ws, ws_bytes);
        int* size = cv.take<int>(n);
        unsigned long long* dsum = cv.take<unsigned long long>(n);
        int* trow = cv.take<int>(num_tiles(2 * m) + 1);
        int* bad = cv.take<int>(1);
        cudaMemsetAsync(size, 0, sizeof(int) * n, s);
        cudaMemsetAsync(dsum, 0, sizeof(unsigned long long) * n, s);
        cudaMemsetAsync(bad, 0, sizeof(int), s);
        const int sms = num_sms();
        const int64_t vwarps = (n + 32 * kVertItems - 1) / (32 * kVertItems);
        const int vgrid = (int)std::min<int64_t>((vwarps + kStatThreads / 32 - 1) / (kStatThreads / 32),
                                                 (int64_t)sms * 8);
        const int rgrid = (int)std::max<int64_t>(
            1, std::min<int64_t>((n + kStatThreads - 1) / kStatThreads, (int64_t)sms * 8));
        for (int j = 0; j < k; ++j) {
            k_part_vertex<RP><<<vgrid, kStatThreads, 0, s>>>(n, rowptr, labels + (int64_t)j * n,
                                                             size, dsum, bad);
            k_part_roots<<<rgrid, kStatThreads, 0, s>>>(n, size, dsum, acc + 4 * j);
        }
        count_launches(2 * k);
        if (m > 0) {
            const int64_t slots = 2 * m;
            tile_rows<RP>(rowptr, (int)n, slots, kTile, trow, s);
            // partitions per pass: their label arrays should sit in L2 together
            const int64_t l2_budget = (int64_t)48 << 20;
            const int G = (int)std::max<int64_t>(1, std::min<int64_t>(kMaxGroup, l2_budget / (4 * n)));
            const int egrid = (int)std::min<int64_t>(num_tiles(slots), (int64_t)sms * 8);
            for (int j0 = 0; j0 < k; j0 += G) {
                const int g = std::min(G, k - j0);
                k_part_edges<RP><<<egrid, kStatThreads, 0, s>>>(
                    n, slots, rowptr, colidx, trow, labels + (int64_t)j0 * n, g, acc + 4 * j0);
                count_launches(1);
            }
        }
        e = cudaMemcpyAsync(bad_host, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return e;
    }
    if (q) {
        k_modularity<<<(k + 127) / 128, 128, 0, s>>>(k, (long long)m, counts, q);
        count_launches(1);
    }
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template cudaError_t partition_stats_impl<int>(int64_t, int64_t, const int*, const int*,
                                               const int*, int, void*, size_t, long long*, double*,
                                               int*, cudaStream_t);
template cudaError_t partition_stats_impl<long long>(int64_t, int64_t, const long long*,
                                                     const int*, const int*, int, void*, size_t,
                                                     long long*, double*, int*, cudaStream_t);

}  // namespace twc
