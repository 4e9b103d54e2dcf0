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
// Kernels (HBM streaming plus one random 32-byte gather per edge; none is a contraction):
//   k_part_degrees  deg[u] once.
//   k_part_vertex   per partition: one coalesced pass over its labels; per label one packed
//                   64-bit counter (size << 32 | D_c; D_c <= 2m < 2^32) updated with one atomic
//                   per distinct label per warp (__match_any_sync).  A warp keeps a "hot" label
//                   (the last label held by >= 4 lanes of one warp load) in lane-local registers, so a giant
//                   component costs no atomics at all (same-address atomics serialise).
//   k_part_roots    per partition: count / max / sum of squares over the non-zero counters.
//   k_part_pack     per chunk of 8 partitions: labels [8][n] -> [n][8] (32 bytes per vertex).
//   k_part_edges    per chunk: one pass over the CSR slots (8 consecutive slots per thread, one
//                   row search, then a walk); for every slot (u, v) with v > u one 32-byte gather
//                   of v's 8 labels compared with u's -> E_in of all 8 partitions at once.
//   k_modularity    one thread per partition.
#include <algorithm>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

constexpr int kStatThreads = 256;
constexpr int kChunk = 8;                               // partitions per packed edge pass
constexpr int kEdgeItems = 8;                           // slots per thread in k_part_edges
constexpr int kEdgeTile = kStatThreads * kEdgeItems;    // 2048 slots
constexpr int kEdgeRows = 1024;                         // rowptr entries cached per tile

template <typename RP>
__global__ void k_part_degrees(int64_t n, const RP* __restrict__ rowptr, int* __restrict__ deg) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) deg[u] = (int)(rowptr[u + 1] - rowptr[u]);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

__global__ void __launch_bounds__(kStatThreads) k_part_vertex(
    int64_t n, const int* __restrict__ deg, const int* __restrict__ lab,
    unsigned long long* __restrict__ packed, int* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int hot = -1;                   // warp-uniform
    unsigned long long hacc = 0;    // lane-local (count << 32 | degree sum) of the hot label
    for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
        const int64_t u = base + lane;
        int l = -1;
        unsigned d = 0;
        if (u < n) {
            l = __ldcs(lab + u);
            d = (unsigned)deg[u];
            if (l < 0 || (int64_t)l >= n) {
                atomicOr(bad, 1);
                l = -1;
            }
        }
        if (l >= 0 && l == hot) hacc += (1ull << 32) | d;
        const unsigned grp = __match_any_sync(FULL, l);
        // degrees of distinct vertices: the group sum is <= 2m < 2^32
        const unsigned dg = __reduce_add_sync(grp, d);
        const int gsz = __popc(grp);
        if (l >= 0 && l != hot && lane == __ffs(grp) - 1)
            atomicAdd(packed + l, ((unsigned long long)gsz << 32) + dg);
        const unsigned big = __ballot_sync(FULL, gsz >= 4 && l >= 0 && l != hot);
        if (big) {  // a new frequent label: flush the old hot one, adopt the new
            const unsigned long long tot = warp_sum_u64(hacc);
            if (lane == 0 && hot >= 0 && tot) atomicAdd(packed + hot, tot);
            hacc = 0;
            hot = __shfl_sync(FULL, l, __ffs(big) - 1);
        }
    }
    const unsigned long long tot = warp_sum_u64(hacc);
    if (lane == 0 && hot >= 0 && tot) atomicAdd(packed + hot, tot);
}

// acc[0] communities, [1] largest, [3] sum of D_c^2 (as unsigned long long)
__global__ void __launch_bounds__(kStatThreads) k_part_roots(
    int64_t n, const unsigned long long* __restrict__ packed, unsigned long long* __restrict__ acc) {
    __shared__ unsigned long long s_cnt, s_sq;
    __shared__ unsigned s_max;
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_sq = 0;
        s_max = 0;
    }
    __syncthreads();
    unsigned cnt = 0, mx = 0;
    unsigned long long sq = 0;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n;
         l += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = __ldcs(packed + l);
        if (x) {
            const unsigned long long dc = x & 0xffffffffull;
            ++cnt;
            sq += dc * dc;
            mx = max(mx, (unsigned)(x >> 32));
        }
    }
    cnt = __reduce_add_sync(FULL, cnt);
    mx = __reduce_max_sync(FULL, mx);
    sq = warp_sum_u64(sq);
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicAdd(&s_cnt, (unsigned long long)cnt);
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

// labT[u * 8 + i] = lab[i * n + u] for i < g (unused lanes -1)
__global__ void k_part_pack(int64_t n, const int* __restrict__ lab, int g, int4* __restrict__ labT) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    int x[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) x[i] = (i < g) ? __ldcs(lab + (int64_t)i * n + u) : -1;
    labT[2 * u] = make_int4(x[0], x[1], x[2], x[3]);
    labT[2 * u + 1] = make_int4(x[4], x[5], x[6], x[7]);
}

__device__ __forceinline__ void count_equal(const int4& a, const int4& b, const int4& ua,
                                            const int4& ub, int* c) {
    c[0] += a.x == ua.x; c[1] += a.y == ua.y; c[2] += a.z == ua.z; c[3] += a.w == ua.w;
    c[4] += b.x == ub.x; c[5] += b.y == ub.y; c[6] += b.z == ub.z; c[7] += b.w == ub.w;
}

// E_in of the (up to 8) partitions packed in labT: acc[4i + 2]
template <typename RP>
__global__ void __launch_bounds__(kStatThreads) k_part_edges(
    int64_t slots, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ trow, const int4* __restrict__ labT, int g,
    unsigned long long* __restrict__ acc) {
    __shared__ RP s_rp[kEdgeRows + 1];
    __shared__ unsigned long long s_in[kChunk];
    if (threadIdx.x < kChunk) s_in[threadIdx.x] = 0;
    const int64_t ntiles = (slots + kEdgeTile - 1) / kEdgeTile;
    int c[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) c[i] = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p0 = tile * kEdgeTile;
        const int64_t p1 = min(p0 + kEdgeTile, slots);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;
        const bool cached = nr <= kEdgeRows;
        __syncthreads();
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_rp[i] = rowptr[r0 + i];
        __syncthreads();
        const int64_t q0 = p0 + (int64_t)threadIdx.x * kEdgeItems;
        if (q0 >= p1) continue;
        int v[kEdgeItems];
        if (q0 + kEdgeItems <= p1) {
            const int4* src = reinterpret_cast<const int4*>(colidx + q0);
            const int4 a = __ldcs(src), b = __ldcs(src + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < kEdgeItems; ++j) v[j] = (q0 + j < p1) ? colidx[q0 + j] : -1;
        }
        // rows of the 8 slots: one search, then a walk
        int uj[kEdgeItems];
        {
            const RP q = (RP)q0;
            int ri = cached ? last_le(s_rp, nr + 1, q) : last_le(rowptr + r0, nr + 1, q);
            RP re = cached ? s_rp[ri + 1] : rowptr[r0 + ri + 1];
#pragma unroll
            for (int j = 0; j < kEdgeItems; ++j) {
                while ((RP)(q0 + j) >= re && q0 + j < p1) {
                    ++ri;
                    re = cached ? s_rp[ri + 1] : rowptr[r0 + ri + 1];
                }
                uj[j] = r0 + ri;
            }
        }
        int ucur = -1;
        int4 ua = make_int4(0, 0, 0, 0), ub = ua;
#pragma unroll
        for (int j = 0; j < kEdgeItems; ++j) {
            if (v[j] > uj[j]) {
                if (uj[j] != ucur) {
                    ucur = uj[j];
                    ua = labT[2 * (int64_t)ucur];
                    ub = labT[2 * (int64_t)ucur + 1];
                }
                const int4 a = labT[2 * (int64_t)v[j]], b = labT[2 * (int64_t)v[j] + 1];
                count_equal(a, b, ua, ub, c);
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
        if (i >= g) break;
        const unsigned w = __reduce_add_sync(FULL, (unsigned)c[i]);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(&s_in[i], (unsigned long long)w);
    }
    __syncthreads();
    if (threadIdx.x < g && s_in[threadIdx.x]) atomicAdd(acc + 4 * threadIdx.x + 2, s_in[threadIdx.x]);
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
    cv.take<int>(n);                                            // deg
    cv.take<unsigned long long>(n);                             // packed counters
    cv.take<int4>(2 * n);                                       // labels of 8 partitions, [n][8]
    cv.take<int>((2 * m + kEdgeTile - 1) / kEdgeTile + 1);      // tile rows of the full CSR
    cv.take<int>(1);                                            // bad-label flag
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
        int* deg = cv.take<int>(n);
        unsigned long long* packed = cv.take<unsigned long long>(n);
        int4* labT = cv.take<int4>(2 * n);
        int* trow = cv.take<int>((2 * m + kEdgeTile - 1) / kEdgeTile + 1);
        int* bad = cv.take<int>(1);
        cudaMemsetAsync(bad, 0, sizeof(int), s);
        const int sms = num_sms();
        const unsigned vb = (unsigned)((n + kStatThreads - 1) / kStatThreads);
        k_part_degrees<RP><<<vb, kStatThreads, 0, s>>>(n, rowptr, deg);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(vb, (int64_t)sms * 8));
        for (int j = 0; j < k; ++j) {
            cudaMemsetAsync(packed, 0, sizeof(unsigned long long) * n, s);
            k_part_vertex<<<grid, kStatThreads, 0, s>>>(n, deg, labels + (int64_t)j * n, packed,
                                                        bad);
            k_part_roots<<<grid, kStatThreads, 0, s>>>(n, packed, acc + 4 * j);
        }
        count_launches(1 + 2 * k);
        if (m > 0) {
            const int64_t slots = 2 * m;
            const int64_t et = (slots + kEdgeTile - 1) / kEdgeTile;
            tile_rows<RP>(rowptr, (int)n, slots, kEdgeTile, trow, s);
            const int egrid = (int)std::min<int64_t>(et, (int64_t)sms * 8);
            for (int j0 = 0; j0 < k; j0 += kChunk) {
                const int g = std::min(kChunk, k - j0);
                k_part_pack<<<vb, kStatThreads, 0, s>>>(n, labels + (int64_t)j0 * n, g, labT);
                k_part_edges<RP><<<egrid, kStatThreads, 0, s>>>(slots, rowptr, colidx, trow, labT,
                                                                g, acc + 4 * j0);
                count_launches(2);
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
