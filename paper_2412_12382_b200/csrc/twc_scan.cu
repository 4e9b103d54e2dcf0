// twc_scan.cu -- device-wide exclusive scan, row tiling and canonical edge offsets.
//
// Canonical edge order (reading C5): the edges (u,v), u<v, in
// lexicographic order = the upper triangle of the CSR in row order.  With up[u] = #{v in N(u):
// v > u} and eoff = exclusive scan of up, the canonical id of the upper slot p of row u is
// eoff[u] + (p - rowptr[u] - lo[u]), lo[u] = deg(u) - up[u].
#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

constexpr int SB = 512;   // scan block
constexpr int SIPT = 8;   // items per thread
constexpr int SCHUNK = SB * SIPT;

__global__ void __launch_bounds__(SB) k_scan_reduce(const int* __restrict__ in, int64_t len,
                                                     int* __restrict__ bsum) {
    __shared__ long long s_tmp[32];
    int64_t base = (int64_t)blockIdx.x * SCHUNK;
    long long acc = 0;
#pragma unroll
    for (int k = 0; k < SIPT; ++k) {
        int64_t i = base + (int64_t)k * SB + threadIdx.x;
        if (i < len) acc += in[i];
    }
    long long tot = block_sum_ll(acc, s_tmp);
    if (threadIdx.x == 0) bsum[blockIdx.x] = (int)tot;
}

// Exclusive scan of bsum[0..nb) in place (one block), bsum[nb] = total.
__global__ void __launch_bounds__(1024) k_scan_spine(int* __restrict__ bsum, int nb) {
    __shared__ int s_w[32];
    __shared__ int s_carry;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        int i = base + threadIdx.x;
        int v = (i < nb) ? bsum[i] : 0;
        int incl = warp_incl_scan(v, lane);
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int w = s_w[lane];
            int wi = warp_incl_scan(w, lane);
            s_w[lane] = wi - w;
        }
        __syncthreads();
        int carry = s_carry;
        if (i < nb) bsum[i] = carry + s_w[wid] + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + s_w[wid] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = s_carry;
}

__global__ void __launch_bounds__(SB) k_scan_down(const int* __restrict__ in, int64_t len,
                                                   const int* __restrict__ boff,
                                                   int* __restrict__ out) {
    __shared__ int s_w[SB / 32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = (int64_t)blockIdx.x * SCHUNK + (int64_t)threadIdx.x * SIPT;
    int v[SIPT];
    int tsum = 0;
#pragma unroll
    for (int k = 0; k < SIPT; ++k) {
        int64_t i = base + k;
        v[k] = (i < len) ? in[i] : 0;
        tsum += v[k];
    }
    int incl = warp_incl_scan(tsum, lane);
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int w = (lane < SB / 32) ? s_w[lane] : 0;
        int wi = warp_incl_scan(w, lane);
        if (lane < SB / 32) s_w[lane] = wi - w;
    }
    __syncthreads();
    int run = boff[blockIdx.x] + s_w[wid] + incl - tsum;
#pragma unroll
    for (int k = 0; k < SIPT; ++k) {
        int64_t i = base + k;
        run += v[k];
        if (i < len) out[i + 1] = run;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

size_t scan_temp_bytes(int64_t len) {
    int64_t nb = (len + SCHUNK - 1) / SCHUNK;
    return align_up(sizeof(int) * (size_t)(nb + 2));
}

void exclusive_scan(const int* in, int* out, int64_t len, int* temp, cudaStream_t s) {
    if (len <= 0) {
        cudaMemsetAsync(out, 0, sizeof(int), s);
        return;
    }
    int nb = (int)((len + SCHUNK - 1) / SCHUNK);
    k_scan_reduce<<<nb, SB, 0, s>>>(in, len, temp);
    k_scan_spine<<<1, 1024, 0, s>>>(temp, nb);
    k_scan_down<<<nb, SB, 0, s>>>(in, len, temp, out);
    count_launches(3);
}

template <typename OT>
__global__ void k_tile_rows(const OT* __restrict__ off, int nrows, int64_t total, int tile,
                            int64_t ntiles, int* __restrict__ trow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > ntiles) return;
    const OT item = (OT)((i < ntiles) ? i * tile : total - 1);
    int r = last_le(off, nrows + 1, item);
    trow[i] = min(r, nrows - 1);
}

template <typename OT>
void tile_rows(const OT* off, int nrows, int64_t total, int tile, int* trow, cudaStream_t s) {
    const int64_t nt = (total + tile - 1) / tile;
    if (nt == 0) return;
    const int64_t threads = nt + 1;
    k_tile_rows<OT><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(off, nrows, total, tile, nt,
                                                                      trow);
    count_launches(1);
}

template void tile_rows<int>(const int*, int, int64_t, int, int*, cudaStream_t);
template void tile_rows<long long>(const long long*, int, int64_t, int, int*, cudaStream_t);

void tile_first_rows(const int* off, int nrows, int64_t total, int* trow, cudaStream_t s) {
    tile_rows<int>(off, nrows, total, kTile, trow, s);
}

template <typename RP>
__global__ void k_upper_counts(int64_t n, const RP* __restrict__ rowptr,
                               const int* __restrict__ colidx, int* __restrict__ up) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    RP beg = rowptr[u], end = rowptr[u + 1];
    int d = (int)(end - beg);
    int lo = lower_bound(colidx + beg, d, (int)u);  // #{v < u}: rows are strictly increasing
    up[u] = d - lo;
}

template <typename RP>
void upper_counts(int64_t n, const RP* rowptr, const int* colidx, int* up, cudaStream_t s) {
    if (n <= 0) return;
    k_upper_counts<RP><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rowptr, colidx, up);
    count_launches(1);
}

template void upper_counts<int>(int64_t, const int*, const int*, int*, cudaStream_t);
template void upper_counts<long long>(int64_t, const long long*, const int*, int*, cudaStream_t);

}  // namespace twc
