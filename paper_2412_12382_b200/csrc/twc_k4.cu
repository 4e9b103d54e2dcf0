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
// k4_pivots<false>: one warp per pivot with |N+(a)| <= kK4Cap; N+(a), its per-slot counters and
//   the current C (ids, slot in N+(a), slot in N+(b)) live in the warp's shared memory; every
//   membership test is a binary search in shared memory; counters of N+(a) are flushed once.
// k4_pivots<true>:  the few pivots with longer lists, N+(a) read from global memory and C kept
//   in a per-warp global scratch (|C| <= |N+(b)| <= sqrt(2m) under the degree orientation).
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

// Small pivots (3 <= |N+(a)| <= kK4Cap): warps take chunks of consecutive pivots.
__global__ void __launch_bounds__(kK4Warps * 32) k4_small(int64_t n, int chunk,
                                                          const int* __restrict__ rp_or,
                                                          const int* __restrict__ col_or,
                                                          unsigned long long* __restrict__ k4_or,
                                                          int* __restrict__ work) {
    __shared__ K4WarpSmem smem[kK4Warps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    K4WarpSmem& S = smem[wid];
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(work, chunk);
        base = __shfl_sync(FULL, base, 0);
        if (base >= n) break;
        const int end = (int)min((int64_t)base + chunk, n);
        for (int a = base; a < end; ++a) {
            const int da = rp_or[a + 1] - rp_or[a];
            if (da < 3 || da > kK4Cap) continue;  // no 4-clique / a big pivot
            k4_pivot<false>(a, lane, rp_or, col_or, k4_or, S.list, S.cnt, S.cid, S.cpa, S.cpb);
        }
    }
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
    cv.take<int>(4);                 // counters
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
    int* ctr = cv.take<int>(4);  // [0] small queue, [1] big count, [2] big queue
    const int64_t cmax = (int64_t)std::sqrt(2.0 * (double)m) + 2;
    int* scratch = cv.take<int>((size_t)k4_big_warps() * 3 * cmax);
    *k4_or_out = k4_or;
    cudaMemsetAsync(k4_or, 0, sizeof(unsigned long long) * (size_t)m, s);
    cudaMemsetAsync(ctr, 0, 4 * sizeof(int), s);
    const int sms = num_sms();
    // one resident wave: the warps are latency-bound (a global round trip per slot and per
    // triangle), so occupancy is what hides the latency
    static int occ = 0;
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k4_small, kK4Warps * 32, 0);
        if (occ < 1) occ = 1;
    }
    const int64_t warps = (int64_t)sms * occ * kK4Warps;
    const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(16, n / (8 * warps)));
    k4_small<<<sms * occ, kK4Warps * 32, 0, s>>>(n, chunk, rp_or, col_or, k4_or, ctr);
    k4_find_big<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rp_or, big, ctr + 1);
    k4_big<<<k4_big_warps() / 4, 128, 0, s>>>(big, ctr + 1, rp_or, col_or, k4_or, scratch,
                                               (int)cmax, ctr + 2);
    count_launches(3);
    return cudaGetLastError();
}

}  // namespace twc
