// twc_k4.cu -- per-edge K4 participation (kappa-clique participation with kappa = 4, Table 1
// P:417; "we only consider K_4").
//
// On the degree-oriented graph of K1 every 4-clique {a, b, c, d} has one key order
// a < b < c < d, so it is found exactly once from its lowest vertex a (the pivot):
//   for every slot a -> b:  C = N+(a) & N+(b)            (c with a -> c and b -> c)
//   for every c in C:       D = N+(c) & C                (d with c -> d as well)
// and each (c, d) adds one to the K4 count of all six edges ab, ac, ad, bc, bd, cd, each at its
// oriented slot (ab, ac, ad in N+(a); bc, bd in N+(b); cd in N+(c)).  Work per pivot is
// sum over b of |N+(b)| membership tests against N+(a) plus, per triangle, |N+(c)| tests
// against C: O(m * alpha^2) as Table 1 states.
//
// k4_masks<W>: pivots with |N+(a)| <= 64 W (W = 1, 2, 4): the 4-cliques of pivot a are the
//   triangles of the graph G_a induced on N+(a); its edges are found by K2's flattened item
//   scan (filter + search in the staged N+(a)) and kept as W-word neighbour masks, so the
//   count of every edge is a popcount of two masks (see the kernel).
// k4_pivot<true> / k4_big: the few pivots with longer lists, N+(a) read from global memory and
//   C = N+(a) & N+(b) kept in a per-warp global scratch (|C| <= |N+(b)| <= sqrt(2m) under the
//   degree orientation), each c in C probed against N+(c).
// The counts are accumulated in oriented-slot order (64-bit) and gathered to canonical order by
// the score epilogue (K3) together with t, wedge and TW.
#include <algorithm>
#include <climits>
#include <cmath>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

constexpr int kK4Warps = 8;
constexpr int kK4Cap = 256;

struct K4WarpSmem {
    int list[kK4Cap];  // N+(a)
    int cnt[kK4Cap];   // K4 increments of the edges (a, x), x in N+(a)
    int cid[kK4Cap];   // C = N+(a) & N+(b): ids (ascending)
    int cpa[kK4Cap];   //   slot of c in N+(a), relative to its start
    int cpb[kK4Cap];   //   absolute oriented slot of c in N+(b)
};

// position of x in the sorted list L[0, len), or -1
__device__ __forceinline__ int find_sorted(const int* L, int len, int x) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (L[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return (lo < len && L[lo] == x) ? lo : -1;
}

template <bool BIG>
__device__ __forceinline__ void k4_pivot(int a, int lane, const int* __restrict__ rp_or,
                                         const int* __restrict__ col_or,
                                         unsigned long long* __restrict__ k4_or, int* s_list,
                                         int* s_cnt, int* cid, int* cpa, int* cpb) {
    const unsigned lt = (1u << lane) - 1u;
    const int A = rp_or[a], da = rp_or[a + 1] - A;
    const int* L = BIG ? col_or + A : s_list;
    if (!BIG) {
        for (int i = lane; i < da; i += 32) {
            s_list[i] = col_or[A + i];
            s_cnt[i] = 0;
        }
        __syncwarp();
    }
    for (int i = 0; i < da; ++i) {  // slot a -> b
        const int b = L[i];
        const int B0 = rp_or[b], db = rp_or[b + 1] - B0;
        if (db < 2) continue;  // c and d both come from N+(b)
        int nC = 0;
        for (int j0 = 0; j0 < db; j0 += 32) {
            const int j = j0 + lane;
            const int c = j < db ? col_or[B0 + j] : -1;
            const int pa = c >= 0 ? find_sorted(L, da, c) : -1;
            const unsigned bal = __ballot_sync(FULL, pa >= 0);
            if (pa >= 0) {
                const int pos = nC + __popc(bal & lt);
                cid[pos] = c;
                cpa[pos] = pa;
                cpb[pos] = B0 + j;
            }
            nC += __popc(bal);
        }
        __syncwarp();
        if (nC >= 2) {
            for (int jc = 0; jc < nC; ++jc) {  // c in C; d in N+(c) & C
                const int c = cid[jc];
                const int C0 = rp_or[c], dc = rp_or[c + 1] - C0;
                int hits = 0;
                for (int k0 = 0; k0 < dc; k0 += 32) {
                    const int k = k0 + lane;
                    const int d = k < dc ? col_or[C0 + k] : -1;
                    const int q = d >= 0 ? find_sorted(cid, nC, d) : -1;
                    if (q >= 0) {  // the 4-clique {a, b, c, d}
                        if (BIG) atomicAdd(&k4_or[A + cpa[q]], 1ull);  // ad
                        else atomicAdd(&s_cnt[cpa[q]], 1);
                        atomicAdd(&k4_or[cpb[q]], 1ull);                 // bd
                        atomicAdd(&k4_or[C0 + k], 1ull);                 // cd
                    }
                    hits += __popc(__ballot_sync(FULL, q >= 0));
                }
                if (hits && lane == 0) {
                    if (BIG) {
                        atomicAdd(&k4_or[A + i], (unsigned long long)hits);       // ab
                        atomicAdd(&k4_or[A + cpa[jc]], (unsigned long long)hits); // ac
                    } else {
                        atomicAdd(&s_cnt[i], hits);
                        atomicAdd(&s_cnt[cpa[jc]], hits);
                    }
                    atomicAdd(&k4_or[cpb[jc]], (unsigned long long)hits);         // bc
                }
            }
        }
        __syncwarp();  // C is rebuilt for the next slot
    }
    if (!BIG) {
        __syncwarp();
        for (int i = lane; i < da; i += 32) {
            const int c = s_cnt[i];
            if (c) atomicAdd(&k4_or[A + i], (unsigned long long)c);
        }
        __syncwarp();
    }
}

// ---- pivots with 3 <= |N+(a)| <= 64: the 4-cliques whose lowest vertex is a are the triangles
// of the graph G_a induced on N+(a).  One warp per pivot, N+(a) staged in shared memory with a
// 2,048-bit filter; the items (x in N+(a), y in N+(x)) are flattened across the lanes (segment
// owner lookup) and y is searched in N+(a) only when the filter hits.  Pass 1 finds every edge
// {x, y} of G_a and records it in 64-bit neighbour masks nbr[]; pass 2 finds the same edges
// again and, for each, k = popc(nbr[x] & nbr[y]) = the triangles of G_a on it = the 4-cliques
// {a, x, y, z} on edge (x, y) counted from pivot a, added to (x, y)'s oriented slot; the pivot
// edges (a, x) get half the sum of k over the edges of G_a at x.  (Each 4-clique is counted from
// its lowest vertex only, as in k4_pivot.)
// W = 1 with pivots GROUPED like K2: consecutive pivots whose lists total <= 64 slots share one
// staged list, filter and mask array (bits are only ever set between two entries of the same
// pivot, so a mask popcount still counts within one G_a), which amortises the per-pivot setup
// over ~7 pivots on config 5.  prp[] holds the group's pivot offsets; a slot's pivot is found by
// a short search in it.
constexpr int kK4Edges = 128;

// W 64-bit words per neighbour mask: up to 64 W slots staged, a 2,048 W-bit filter
template <int W>
struct K4GroupSmem {
    int list[64 * W];
    unsigned filt[64 * W];
    unsigned long long nbr[64 * W * W];  // nbr[i * W + w]
    int acc[64 * W];
    int prp[33];
    int4 seg[32];
    int owner[32];
    int2 edge[kK4Edges];  // edges of the G_a found by pass 1: {slot of x -> y, ix | iy << 10}
    int nedge;
};

template <int W>
__device__ __forceinline__ unsigned k4_filt_word(unsigned h) {
    return h >> (W == 1 ? 26 : W == 2 ? 25 : 24);  // 64 W words
}

template <int W, int PASS>
__device__ __forceinline__ void k4_group_pass(K4GroupSmem<W>& S, int lane, int len, int np,
                                              const int* __restrict__ rp_or,
                                              const int* __restrict__ col_or,
                                              unsigned long long* __restrict__ k4_or) {
    for (int r0 = 0; r0 < len; r0 += 32) {  // rounds of 32 slots of the group
        const int ix = r0 + lane;
        int wt = 0, xs = 0, xe = 0, plo = 0, phi = 0;
        if (ix < len) {
            const int pi = last_le(S.prp, np + 1, ix);
            plo = S.prp[pi];
            phi = S.prp[pi + 1];
            if (phi - plo >= 3) {  // a pivot with < 3 oriented neighbours has no 4-clique
                const int x = S.list[ix];
                xs = rp_or[x];
                xe = rp_or[x + 1];
                wt = (xe - (xs & ~7) + 7) >> 3;  // aligned 8-entry sectors covering [xs, xe)
            }
        }
        const int incl = warp_incl_scan(wt, lane);
        const int total = __shfl_sync(FULL, incl, 31);
        const int pre = incl - wt;
        // {first sector - 8 * first item, end, start, the pivot's slots [plo, phi) in the group}
        S.seg[lane] = make_int4((xs & ~7) - 8 * pre, xe, xs, plo | (phi << 10));
        const unsigned nz = __ballot_sync(FULL, wt > 0);
        int cur = nz ? __ffs(nz) - 1 : 0;
        __syncwarp();
        for (int k0 = 0; k0 < total; k0 += 32) {
            const bool starts = wt > 0 && pre >= k0 && pre < k0 + 32;
            if (starts) S.owner[pre - k0] = lane;
            const unsigned bits = __reduce_or_sync(FULL, starts ? (1u << (pre - k0)) : 0u);
            __syncwarp();
            const unsigned mine = bits & ((2u << lane) - 1u);
            const int own = S.owner[msb_pos(mine | 1u)];
            const int jj = mine ? own : cur;
            const int4 sg = S.seg[jj];
            const int sv0 = sg.x + 8 * (k0 + lane);  // 32-byte aligned
            int y[8];
            ldg_sector(col_or + min(sv0, (sg.y - 1) & ~7), y);  // one LDG.E.256
            unsigned cm = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const unsigned h = (unsigned)y[e] * 2654435761u;
                const unsigned word = S.filt[k4_filt_word<W>(h)];
                cm |= __funnelshift_r(word, word, h - (unsigned)e) & (1u << e);
            }
            cm &= ((1u << min(max(sg.y - sv0, 0), 8)) - 1u) &
                  (0xffu << min(max(sg.z - sv0, 0), 8));
            const int lo = sg.w & 1023, hi = sg.w >> 10, ixx = r0 + jj;
            while (cm) {  // filter hits (rare): search the pivot's staged list
                const int e = __ffs(cm) - 1;
                cm &= cm - 1u;
                const int q = find_sorted(S.list + lo, hi - lo, y[e]);
                if (q >= 0) {  // edge {x, y} of G_a
                    const int iy = lo + q;
                    if (PASS == 1) {
                        atomicOr(&S.nbr[ixx * W + (iy >> 6)], 1ull << (iy & 63));
                        atomicOr(&S.nbr[iy * W + (ixx >> 6)], 1ull << (ixx & 63));
                        const int pos = atomicAdd(&S.nedge, 1);  // kept for the counting step
                        if (pos < kK4Edges) S.edge[pos] = make_int2(sv0 + e, ixx | (iy << 10));
                    } else {
                        int k = 0;
#pragma unroll
                        for (int q = 0; q < W; ++q) k += __popcll(S.nbr[ixx * W + q] & S.nbr[iy * W + q]);
                        if (k) {
                            atomicAdd(&k4_or[sv0 + e], (unsigned long long)k);  // (x, y)
                            atomicAdd(&S.acc[ixx], k);
                            atomicAdd(&S.acc[iy], k);
                        }
                    }
                }
            }
            cur = __shfl_sync(FULL, jj, 31);
            __syncwarp();
        }
        __syncwarp();
    }
}

// W = 1: groups of consecutive pivots with |N+(a)| <= 64 (<= 64 slots per group); W = 2, 4: one
// pivot with 32 W < |N+(a)| <= 64 W per group.
template <int W>
__global__ void __launch_bounds__(kK4Warps * 32) k4_groups(int64_t n, int chunk,
                                                           const int* __restrict__ rp_or,
                                                           const int* __restrict__ col_or,
                                                           unsigned long long* __restrict__ k4_or,
                                                           int* __restrict__ work) {
    extern __shared__ __align__(16) unsigned char k4g_smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    K4GroupSmem<W>& S = reinterpret_cast<K4GroupSmem<W>*>(k4g_smem_raw)[wid];
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(work, chunk);
        base = __shfl_sync(FULL, base, 0);
        if (base >= n) break;
        const int gend = (int)min((int64_t)base + chunk, n);
        int u = base;
        while (u < gend) {
            const int np_max = W == 1 ? min(32, gend - u) : 1;
            const int A = rp_or[u];
            const int e_l = (lane < np_max) ? rp_or[u + lane + 1] : INT_MAX;
            const unsigned fit = __ballot_sync(
                FULL, lane < np_max && e_l - A <= 64 * W && (W == 1 || e_l - A > 32 * W));
            if (fit == 0u) {  // another size class (or k4_big)
                ++u;
                continue;
            }
            const int np = __popc(fit);
            const int B = __shfl_sync(FULL, e_l, np - 1), len = B - A;
            if (lane == 0) S.prp[0] = 0;
            if (lane < np) S.prp[lane + 1] = e_l - A;
            for (int i = lane; i < 64 * W; i += 32) {
                S.filt[i] = 0u;
                S.acc[i] = 0;
            }
            for (int i = lane; i < len * W; i += 32) S.nbr[i] = 0ull;
            __syncwarp();
            for (int i = lane; i < len; i += 32) {
                const int x = col_or[A + i];
                S.list[i] = x;
                const unsigned h = (unsigned)x * 2654435761u;
                atomicOr(&S.filt[k4_filt_word<W>(h)], 1u << (h & 31));
            }
            __syncwarp();
            if (lane == 0) S.nedge = 0;
            __syncwarp();
            k4_group_pass<W, 1>(S, lane, len, np, rp_or, col_or, k4_or);
            __syncwarp();
            const int ne = S.nedge;
            if (ne <= kK4Edges) {  // count from the kept edge list
                for (int i = lane; i < ne; i += 32) {
                    const int2 ed = S.edge[i];
                    const int ixx = ed.y & 1023, iy = ed.y >> 10;
                    int k = 0;
#pragma unroll
                    for (int q = 0; q < W; ++q) k += __popcll(S.nbr[ixx * W + q] & S.nbr[iy * W + q]);
                    if (k) {
                        atomicAdd(&k4_or[ed.x], (unsigned long long)k);  // (x, y)
                        atomicAdd(&S.acc[ixx], k);
                        atomicAdd(&S.acc[iy], k);
                    }
                }
            } else {  // too many edges to keep: find them again
                k4_group_pass<W, 2>(S, lane, len, np, rp_or, col_or, k4_or);
            }
            __syncwarp();
            for (int i = lane; i < len; i += 32) {
                const int c = S.acc[i];
                if (c) atomicAdd(&k4_or[A + i], (unsigned long long)(c / 2));  // (a, x)
            }
            __syncwarp();
            u += np;
        }
    }
}

template <int W>
static void launch_k4_groups(int64_t n, const int* rp_or, const int* col_or,
                             unsigned long long* k4_or, int* work, cudaStream_t s) {
    const size_t smem = kK4Warps * sizeof(K4GroupSmem<W>);
    const int occ = kernel_setup((const void*)k4_groups<W>, kK4Warps * 32, smem);
    const int sms = num_sms();
    const int64_t warps = (int64_t)sms * occ * kK4Warps;
    const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(32, n / (8 * warps)));
    k4_groups<W><<<sms * occ, kK4Warps * 32, smem, s>>>(n, chunk, rp_or, col_or, k4_or, work);
}

// big[] = pivots with more than kK4Cap oriented neighbours
__global__ void k4_find_big(int64_t n, const int* __restrict__ rp_or, int* __restrict__ big,
                            int* __restrict__ nbig) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool is = u < n && rp_or[u + 1] - rp_or[u] > kK4Cap;
    const unsigned b = __ballot_sync(FULL, is);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(b) - 1) base = atomicAdd(nbig, __popc(b));
    base = __shfl_sync(FULL, base, __ffs(b) - 1);
    if (is) big[base + __popc(b & ((1u << lane) - 1u))] = (int)u;
}

// Big pivots: one warp each; C in a per-warp global scratch of 3 * cmax ints.
__global__ void __launch_bounds__(128) k4_big(const int* __restrict__ big,
                                              const int* __restrict__ nbig,
                                              const int* __restrict__ rp_or,
                                              const int* __restrict__ col_or,
                                              unsigned long long* __restrict__ k4_or,
                                              int* __restrict__ scratch, int cmax,
                                              int* __restrict__ work) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int* cid = scratch + gw * 3 * (int64_t)cmax;
    int* cpa = cid + cmax;
    int* cpb = cpa + cmax;
    const int nb = *nbig;
    for (;;) {
        int h = 0;
        if (lane == 0) h = atomicAdd(work, 1);
        h = __shfl_sync(FULL, h, 0);
        if (h >= nb) break;
        k4_pivot<true>(big[h], lane, rp_or, col_or, k4_or, nullptr, nullptr, cid, cpa, cpb);
    }
}

size_t k4_ws_bytes(int64_t n, int64_t m) {
    Carver cv(nullptr, 0);
    cv.take<unsigned long long>(m);  // k4_or
    cv.take<int>(n);                 // big pivots
    cv.take<int>(5);                 // counters
    const int64_t cmax = (int64_t)std::sqrt(2.0 * (double)m) + 2;
    cv.take<int>((size_t)k4_big_warps() * 3 * cmax);
    return cv.used;
}

int k4_big_warps() { return num_sms() * 4; }

cudaError_t k4_count(int64_t n, int64_t m, const int* rp_or, const int* col_or, void* ws,
                     size_t ws_bytes, unsigned long long** k4_or_out, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    unsigned long long* k4_or = cv.take<unsigned long long>(m);
    int* big = cv.take<int>(n);
    int* ctr = cv.take<int>(5);  // [0] masks W=1, [1] big count, [2] big queue, [3] W=2, [4] W=4
    const int64_t cmax = (int64_t)std::sqrt(2.0 * (double)m) + 2;
    int* scratch = cv.take<int>((size_t)k4_big_warps() * 3 * cmax);
    *k4_or_out = k4_or;
    cudaMemsetAsync(k4_or, 0, sizeof(unsigned long long) * (size_t)m, s);
    cudaMemsetAsync(ctr, 0, 5 * sizeof(int), s);
    // pivots with |N+(a)| <= 256 by size class (mask words W = 1, 2, 4); longer lists below
    launch_k4_groups<1>(n, rp_or, col_or, k4_or, ctr + 0, s);
    launch_k4_groups<2>(n, rp_or, col_or, k4_or, ctr + 3, s);
    launch_k4_groups<4>(n, rp_or, col_or, k4_or, ctr + 4, s);
    k4_find_big<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rp_or, big, ctr + 1);
    k4_big<<<k4_big_warps() / 4, 128, 0, s>>>(big, ctr + 1, rp_or, col_or, k4_or, scratch,
                                               (int)cmax, ctr + 2);
    count_launches(5);
    return cudaGetLastError();
}

}  // namespace twc
