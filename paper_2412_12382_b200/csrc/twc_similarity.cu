// twc_similarity.cu -- the other edge similarities of Table 1 from the triangle
// counts, in fp64, canonical edge order.
//
//   kind 0  TW        t - wedge = 3t - d_u - d_v + 2          (Eq. 2)
//   kind 1  Tectonic  t / (d_u + d_v)
//   kind 2  Jaccard   t / (d_u + d_v - t)
//   kind 3  K3        t
//   kind 4  -R_eff proxy  -2 / (2 + t)                         (P:450 upper bound 2/(2+t),
//                                                               negated as Table 1's -R_eff)
// Each score is one IEEE double operation on exact integers, so it is correctly rounded and
// bit-identical to any other correctly rounded evaluation (reading C18).
#include <algorithm>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

constexpr int kSimThreads = 256;
constexpr int kSimTileRows = 2048;

// #upper(u) = #{v in N(u): v > u} and, for the degree kinds, deg[u] (one pass over rowptr)
template <typename RP>
__global__ void k_sim_rows(int64_t n, const RP* __restrict__ rowptr,
                           const int* __restrict__ colidx, int* __restrict__ up,
                           int* __restrict__ deg) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const RP beg = rowptr[u];
    const int d = (int)(rowptr[u + 1] - beg);
    up[u] = d - lower_bound(colidx + beg, d, (int)u);  // rows are strictly increasing
    deg[u] = d;
}

__device__ __forceinline__ double sim_value(int kind, long long tt, long long dsum) {
    switch (kind) {
        case 0: return (double)(3 * tt - dsum + 2);
        case 1: return (double)tt / (double)dsum;
        case 2: return (double)tt / (double)(dsum - tt);
        case 3: return (double)tt;
        default: return -2.0 / (2.0 + (double)tt);
    }
}

// kinds K3 and -R_eff depend on t alone: a streaming pass (12 bytes per edge), no CSR
__global__ void __launch_bounds__(kSimThreads) k_similarity_t(int64_t m, const int* __restrict__ t,
                                                              int kind, double* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += stride)
        __stcs(out + c, sim_value(kind, (long long)__ldcs(t + c), 0));
}

// The degree kinds (TW, Tectonic, Jaccard), one canonical edge per thread and tile pass.  (A
// variant with four consecutive edges per thread -- one row search and a walk, 16-byte reads
// of t and 32-byte writes -- was measured slower: 0.55-0.60 ms against 0.42-0.47 ms on config
// 5, 48 registers and four scalar colidx reads per thread into the same sectors.)
// The far endpoint's degree comes from a 4-byte deg[] (16 MB for config 5, L2-resident) rather
// than from two 8-byte rowptr reads of a 32 MB array: one random L2 sector per edge.
template <typename RP>
__global__ void __launch_bounds__(kSimThreads) k_similarity(
    int64_t m, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ eoff, const int* __restrict__ trow, const int* __restrict__ deg,
    const int* __restrict__ t, int kind, double* __restrict__ out) {
    __shared__ int s_off[kSimTileRows + 1];
    const int64_t ntiles = num_tiles(m);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c0 = (int)(tile * kTile);
        const int c1 = (int)min((int64_t)c0 + kTile, m);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;
        const bool cached = nr <= kSimTileRows;
        __syncthreads();
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_off[i] = eoff[r0 + i];
        __syncthreads();
        for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
            const int ri = cached ? last_le(s_off, nr + 1, c) : last_le(eoff + r0, nr + 1, c);
            const int u = r0 + ri;
            const int eu = cached ? s_off[ri] : eoff[u];
            const int upu = (cached ? s_off[ri + 1] : eoff[u + 1]) - eu;
            const RP rb = rowptr[u];
            const long long du = (long long)(rowptr[u + 1] - rb);
            const int v = colidx[rb + (RP)(du - upu) + (RP)(c - eu)];
            const long long dv = (long long)deg[v];
            const long long tt = t[c];
            out[c] = sim_value(kind, tt, du + dv);
        }
    }
}

template <typename RP>
cudaError_t similarity_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                            const int* t, int kind, void* ws, size_t ws_bytes, double* out,
                            cudaStream_t s) {
    if (m == 0 || n == 0) return cudaGetLastError();
    if (kind == 3 || kind == 4) {
        const int grid = (int)std::min<int64_t>((m + kSimThreads - 1) / kSimThreads,
                                                (int64_t)num_sms() * 16);
        k_similarity_t<<<grid, kSimThreads, 0, s>>>(m, t, kind, out);
        count_launches(1);
        return cudaGetLastError();
    }
    // reuse the cluster workspace layout for the canonical offsets: up, eoff, scan, tile rows
    Carver cv(ws, ws_bytes);
    int* up = cv.take<int>(n);
    int* eoff = cv.take<int>(n + 1);
    int* scan_tmp = cv.take<int>(scan_temp_bytes(n) / sizeof(int));
    int* trow = cv.take<int>(num_tiles(m) + 1);
    int* deg = cv.take<int>(n);
    k_sim_rows<RP><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rowptr, colidx, up, deg);
    exclusive_scan(up, eoff, n, scan_tmp, s);
    tile_first_rows(eoff, (int)n, m, trow, s);
    const int grid = (int)std::min<int64_t>(num_tiles(m), (int64_t)num_sms() * 8);
    k_similarity<RP><<<grid, kSimThreads, 0, s>>>(m, rowptr, colidx, eoff, trow, deg, t, kind,
                                                  out);
    count_launches(2);
    return cudaGetLastError();
}

template cudaError_t similarity_impl<int>(int64_t, int64_t, const int*, const int*, const int*,
                                          int, void*, size_t, double*, cudaStream_t);
template cudaError_t similarity_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                                const int*, int, void*, size_t, double*,
                                                cudaStream_t);

}  // namespace twc
