// twc_score.cu -- per-edge triangle / wedge / TW scoring on sm_100a.
//
//   a1  K0 degrees                      deg[u] = rowptr[u+1] - rowptr[u]
//   a2  K1 degree-ordered orientation   u -> v iff key(u) < key(v), key = (deg, id)   (P:380
//       + oriented CSR                  prior art; strict key = DESIGN.md reading C9)
//   a3  K2 oriented intersection        every triangle {u,v,w} found once, from its lowest-key
//                                       vertex u (the pivot): +1 to t of (u,v), (u,w), (v,w)
//   a4  K3 fused score epilogue         t  = |N(u) & N(v)|  gathered to canonical order
//                                       wedge = d_u + d_v - 2t - 2  (P:337 under a0)
//                                       TW = t - wedge = 3t - d_u - d_v + 2  (Eq. 2)
// The paper's own method (a full-list merge per edge, O(sum d^2) work) is replaced by
// the oriented count (O(m * arboricity) work); the paper rejected it only for its per-worker
// count arrays, which one int32 array plus atomics avoids on a GPU.  DESIGN.md Sec. 4.
#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

// ------------------------------------------------------------------------------ K0 degrees
template <typename RP>
__global__ void k0_degrees(int64_t n, const RP* __restrict__ rowptr, int* __restrict__ deg) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) deg[u] = (int)(rowptr[u + 1] - rowptr[u]);
}

// ------------------------------------------------------- K1a count: up[u], d+[u] per row
// VW lanes cooperate on one row (VW chosen from the average degree); rows of a warp are
// consecutive, so the colidx reads of a warp are one contiguous range.
template <typename RP, int VW>
__global__ void __launch_bounds__(256) k1_count(int64_t n, const RP* __restrict__ rowptr,
                                                const int* __restrict__ colidx,
                                                const int* __restrict__ deg,
                                                int* __restrict__ up, int* __restrict__ dplus) {
    constexpr int RPW = 32 / VW;
    const int lane = threadIdx.x & 31, g = lane / VW, gl = lane % VW;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u0 = warp * RPW; u0 < n; u0 += nwarps * RPW) {
        const int64_t u = u0 + g;
        const bool valid = u < n;
        const RP beg = valid ? rowptr[u] : 0;
        const int d = valid ? (int)(rowptr[u + 1] - beg) : 0;
        const int dmax = warp_max(d);
        int lower = 0, out = 0;
        for (int k = gl; k < dmax; k += VW) {
            if (k < d) {
                const int v = colidx[beg + k];
                lower += (v < (int)u);
                out += key_less(d, (int)u, deg[v], v);
            }
        }
        lower = group_sum<VW>(lower);
        out = group_sum<VW>(out);
        if (valid && gl == 0) {
            up[u] = d - lower;
            dplus[u] = out;
        }
    }
}

// ------------------------------------------- K1b scatter: oriented CSR, rows stay sorted
template <typename RP, int VW>
__global__ void __launch_bounds__(256) k1_scatter(int64_t n, const RP* __restrict__ rowptr,
                                                  const int* __restrict__ colidx,
                                                  const int* __restrict__ deg,
                                                  const int* __restrict__ rp_or,
                                                  int* __restrict__ col_or) {
    constexpr int RPW = 32 / VW;
    const int lane = threadIdx.x & 31, g = lane / VW, gl = lane % VW;
    const unsigned below = (1u << gl) - 1u;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u0 = warp * RPW; u0 < n; u0 += nwarps * RPW) {
        const int64_t u = u0 + g;
        const bool valid = u < n;
        const RP beg = valid ? rowptr[u] : 0;
        const int d = valid ? (int)(rowptr[u + 1] - beg) : 0;
        const int base = valid ? rp_or[u] : 0;
        const int dmax = warp_max(d);
        int run = 0;
        for (int k0 = 0; k0 < dmax; k0 += VW) {
            const int k = k0 + gl;
            bool pred = false;
            int v = 0;
            if (k < d) {
                v = colidx[beg + k];
                pred = key_less(d, (int)u, deg[v], v);
            }
            const unsigned bal = __ballot_sync(FULL, pred);
            const unsigned gm = (VW == 32) ? bal : ((bal >> (g * VW)) & ((1u << VW) - 1u));
            if (pred) col_or[base + run + __popc(gm & below)] = v;
            run += __popc(gm);
        }
    }
}

// ---------------------------------------------------------- K2 oriented intersection
// One warp per pivot u (dynamic, chunked work queue).  N+(u) is staged in shared memory (up
// to kCap entries; longer lists are probed in place in global memory).  The warp flattens
// the work items {(v, w): v in N+(u), w in N+(v)} so consecutive lanes read consecutive
// entries of N+(v) (coalesced), and tests w in N+(u) by binary search.  A hit at
// N+(u)[q] is the triangle {u, v, w}:  t(u,w) and t(u,v) are accumulated in per-warp smem
// counters (flushed once per pivot), t(v,w) takes one global reduction.
constexpr int kK2Warps = 8;
constexpr int kCap = 512;
constexpr int kPivotChunk = 32;

__global__ void __launch_bounds__(kK2Warps * 32) k2_intersect(int64_t n,
                                                              const int* __restrict__ rp_or,
                                                              const int* __restrict__ col_or,
                                                              int* __restrict__ t_or,
                                                              int* __restrict__ work) {
    __shared__ int s_list[kK2Warps][kCap];
    __shared__ int s_cnt[kK2Warps][kCap];
    __shared__ int s_pre[kK2Warps][33];
    __shared__ int s_vst[kK2Warps][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* list_s = s_list[wid];
    int* cnt_s = s_cnt[wid];
    int* pre = s_pre[wid];
    int* vst = s_vst[wid];
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(work, kPivotChunk);
        base = __shfl_sync(FULL, base, 0);
        if (base >= n) break;
        const int uend = (int)min((int64_t)base + kPivotChunk, n);
        for (int u = base; u < uend; ++u) {
            const int a = rp_or[u];
            const int du = rp_or[u + 1] - a;
            if (du < 2) continue;  // a pivot needs two out-neighbours
            const bool in_smem = du <= kCap;
            if (in_smem) {
                for (int j = lane; j < du; j += 32) {
                    list_s[j] = col_or[a + j];
                    cnt_s[j] = 0;
                }
            }
            __syncwarp();
            const int* list = in_smem ? list_s : col_or + a;
            const int lmin = list[0], lmax = list[du - 1];
            for (int j0 = 0; j0 < du; j0 += 32) {
                const int j = j0 + lane;
                int vs = 0, vd = 0;
                if (j < du) {
                    const int v = list[j];
                    vs = rp_or[v];
                    vd = rp_or[v + 1] - vs;
                }
                const int incl = warp_incl_scan(vd, lane);
                const int total = __shfl_sync(FULL, incl, 31);
                pre[lane] = incl - vd;
                vst[lane] = vs;
                __syncwarp();
                for (int k0 = 0; k0 < total; k0 += 32) {
                    const int k = k0 + lane;
                    if (k < total) {
                        const int jj = last_le(pre, 32, k);
                        const int sv = vst[jj] + (k - pre[jj]);  // oriented slot of v -> w
                        const int w = col_or[sv];
                        if (w >= lmin && w <= lmax) {
                            const int q = lower_bound_bl(list, du, w);
                            if (list[q] == w) {
                                if (in_smem) {
                                    atomicAdd(&cnt_s[q], 1);
                                    atomicAdd(&cnt_s[j0 + jj], 1);
                                } else {
                                    atomicAdd(&t_or[a + q], 1);
                                    atomicAdd(&t_or[a + j0 + jj], 1);
                                }
                                atomicAdd(&t_or[sv], 1);
                            }
                        }
                    }
                }
                __syncwarp();
            }
            if (in_smem) {
                for (int j = lane; j < du; j += 32) {
                    const int c = cnt_s[j];
                    if (c) atomicAdd(&t_or[a + j], c);
                }
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------- K3 fused score epilogue
// Edge-parallel over canonical ids; each CTA takes tiles of kTile ids, caches the tile's
// canonical row offsets in smem and maps id -> row by binary search.  The oriented slot of
// (u,v) is found by binary search in the (short) oriented list of its lower-key endpoint.
constexpr int kK3Threads = 256;
constexpr int kMaxTileRows = 2048;

template <typename RP>
__global__ void __launch_bounds__(kK3Threads) k3_score(
    int64_t n, int64_t m, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ deg, const int* __restrict__ eoff, const int* __restrict__ trow,
    const int* __restrict__ rp_or, const int* __restrict__ col_or,
    const int* __restrict__ t_or, int* __restrict__ t, int* __restrict__ wedge,
    int* __restrict__ tw) {
    __shared__ int s_off[kMaxTileRows + 1];
    const int64_t ntiles = num_tiles(m);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c0 = (int)(tile * kTile);
        const int c1 = (int)min((int64_t)c0 + kTile, m);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;  // rows touched by this tile
        const bool cached = nr + 1 <= kMaxTileRows + 1;
        __syncthreads();
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_off[i] = eoff[r0 + i];
        __syncthreads();
        for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
            const int ri = cached ? last_le(s_off, nr + 1, c) : last_le(eoff + r0, nr + 1, c);
            const int u = r0 + ri;
            const int eu = cached ? s_off[ri] : eoff[u];
            const int upu = (cached ? s_off[ri + 1] : eoff[u + 1]) - eu;
            const int du = deg[u];
            const RP p = rowptr[u] + (RP)(du - upu) + (RP)(c - eu);  // upper slot of (u,v)
            const int v = colidx[p];
            const int dv = deg[v];
            int x = u, y = v;
            if (!key_less(du, u, dv, v)) { x = v; y = u; }
            const int ob = rp_or[x];
            const int s = ob + lower_bound(col_or + ob, rp_or[x + 1] - ob, y);
            const int tt = t_or[s];
            t[c] = tt;
            wedge[c] = du + dv - 2 * tt - 2;
            tw[c] = 3 * tt - du - dv + 2;
        }
    }
}

// ------------------------------------------------------------------------ host side
struct ScoreWs {
    int *deg, *up, *eoff, *dplus, *rp_or, *scan_tmp, *trow, *col_or, *t_or, *work;
};

static ScoreWs carve_score(Carver& cv, int64_t n, int64_t m) {
    ScoreWs w;
    w.deg = cv.take<int>(n);
    w.up = cv.take<int>(n);
    w.eoff = cv.take<int>(n + 1);
    w.dplus = cv.take<int>(n);
    w.rp_or = cv.take<int>(n + 1);
    w.scan_tmp = cv.take<int>(scan_temp_bytes(n) / sizeof(int));
    w.trow = cv.take<int>(num_tiles(m) + 1);
    w.col_or = cv.take<int>(m);
    w.t_or = cv.take<int>(m);
    w.work = cv.take<int>(1);
    return w;
}

size_t score_ws_bytes(int64_t n, int64_t m) {
    Carver cv(nullptr, 0);
    carve_score(cv, n, m);
    return cv.used;
}

static int grid_for(int64_t items, int per_block, int max_blocks) {
    int64_t b = (items + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

template <typename RP, int VW>
static void launch_k1(int64_t n, const RP* rowptr, const int* colidx, const ScoreWs& w,
                      cudaStream_t s) {
    const int sms = num_sms();
    const int rows_per_block = 256 / VW;
    const int grid = grid_for(n, rows_per_block, sms * 8 * 4);
    k1_count<RP, VW><<<grid, 256, 0, s>>>(n, rowptr, colidx, w.deg, w.up, w.dplus);
    count_launches(1);
}

template <typename RP, int VW>
static void launch_k1b(int64_t n, const RP* rowptr, const int* colidx, const ScoreWs& w,
                       cudaStream_t s) {
    const int sms = num_sms();
    const int rows_per_block = 256 / VW;
    const int grid = grid_for(n, rows_per_block, sms * 8 * 4);
    k1_scatter<RP, VW><<<grid, 256, 0, s>>>(n, rowptr, colidx, w.deg, w.rp_or, w.col_or);
    count_launches(1);
}

static int pick_vw(int64_t n, int64_t m) {
    const double avg = n > 0 ? 2.0 * (double)m / (double)n : 0.0;
    if (avg <= 6) return 4;
    if (avg <= 12) return 8;
    if (avg <= 24) return 16;
    return 32;
}

template <typename RP>
cudaError_t score_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                       size_t ws_bytes, int* t, int* wedge, int* tw, cudaStream_t s,
                       cudaEvent_t* ev) {
    if (m == 0 || n == 0) return cudaGetLastError();
    Carver cv(ws, ws_bytes);
    ScoreWs w = carve_score(cv, n, m);
    const int sms = num_sms();
    record(ev, 0, s);
    k0_degrees<RP><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rowptr, w.deg);
    count_launches(1);
    switch (pick_vw(n, m)) {
        case 4: launch_k1<RP, 4>(n, rowptr, colidx, w, s); break;
        case 8: launch_k1<RP, 8>(n, rowptr, colidx, w, s); break;
        case 16: launch_k1<RP, 16>(n, rowptr, colidx, w, s); break;
        default: launch_k1<RP, 32>(n, rowptr, colidx, w, s); break;
    }
    exclusive_scan(w.up, w.eoff, n, w.scan_tmp, s);
    exclusive_scan(w.dplus, w.rp_or, n, w.scan_tmp, s);
    switch (pick_vw(n, m)) {
        case 4: launch_k1b<RP, 4>(n, rowptr, colidx, w, s); break;
        case 8: launch_k1b<RP, 8>(n, rowptr, colidx, w, s); break;
        case 16: launch_k1b<RP, 16>(n, rowptr, colidx, w, s); break;
        default: launch_k1b<RP, 32>(n, rowptr, colidx, w, s); break;
    }
    tile_first_rows(w.eoff, (int)n, m, w.trow, s);
    cudaMemsetAsync(w.t_or, 0, sizeof(int) * (size_t)m, s);
    cudaMemsetAsync(w.work, 0, sizeof(int), s);
    {
        static int occ = 0;
        if (occ == 0) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k2_intersect, kK2Warps * 32, 0);
            if (occ < 1) occ = 1;
        }
        record(ev, 1, s);
        k2_intersect<<<sms * occ, kK2Warps * 32, 0, s>>>(n, w.rp_or, w.col_or, w.t_or, w.work);
        count_launches(1);
        record(ev, 2, s);
    }
    {
        const int64_t nt = num_tiles(m);
        const int grid = grid_for(nt, 1, sms * 8);
        k3_score<RP><<<grid, kK3Threads, 0, s>>>(n, m, rowptr, colidx, w.deg, w.eoff, w.trow,
                                                  w.rp_or, w.col_or, w.t_or, t, wedge, tw);
        count_launches(1);
        record(ev, 3, s);
    }
    return cudaGetLastError();
}

template cudaError_t score_impl<int>(int64_t, int64_t, const int*, const int*, void*, size_t,
                                     int*, int*, int*, cudaStream_t, cudaEvent_t*);
template cudaError_t score_impl<long long>(int64_t, int64_t, const long long*, const int*,
                                           void*, size_t, int*, int*, int*, cudaStream_t,
                                           cudaEvent_t*);

}  // namespace twc
