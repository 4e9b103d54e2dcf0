// twc_common.cuh -- device helpers shared by the TW kernels (sm_100a).
//
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Independence").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Device-side invariant checks of the checked build (-DTWC_CHECKED, build.py): a violated
// bound or capacity stops the kernel with an assertion naming file and line (the call then
// returns TWC_ECUDA).  No code in the normal build.
#ifdef TWC_CHECKED
#include <cassert>
#define TWC_ASSERT(x) assert(x)
#else
#define TWC_ASSERT(x) ((void)0)
#endif

namespace twc {

constexpr unsigned FULL = 0xffffffffu;

// One aligned 32-byte sector of an oriented list per lane: a single 256-bit load (LDG.E.256, sm_100)
// instead of two 128-bit loads touching the same lines twice.
__device__ __forceinline__ void ldg_sector(const int* p, int (&w)[8]) {
    asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
          "=r"(w[7])
        : "l"(p));
}

// Position of the most significant set bit of x != 0 (bfind: one FLO instead of clz + 31 - clz).
__device__ __forceinline__ int msb_pos(unsigned x) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}

// Mask of the bits [lo, hi) (empty when hi <= lo; lo, hi in [0, 32]): one BMSK.
__device__ __forceinline__ unsigned bit_range(int lo, int hi) {
    unsigned r;
    asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(r) : "r"(lo), "r"(max(hi - lo, 0)));
    return r;
}

// Largest index i in [0, len) with a[i] <= x, given a sorted ascending and a[0] <= x.
template <typename T, typename U>
__device__ __forceinline__ int last_le(const T* a, int len, U x) {
    int lo = 0, hi = len;  // invariant: a[lo] <= x, answer in [lo, hi)
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// First index i in [0, len) with a[i] >= x (len if none); a sorted ascending.
template <typename T>
__device__ __forceinline__ int lower_bound(const T* a, int len, T x) {
    int lo = 0, hi = len;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Branch-light lower bound for short sorted lists (membership probes in smem).
// (integer offsets, not a moving pointer: no 64-bit address arithmetic in the loop)
template <typename T>
__device__ __forceinline__ int lower_bound_bl(const T* a, int len, T x) {
    int lo = 0, n = len;
    while (n > 1) {
        const int half = n >> 1;
        lo = (a[lo + half - 1] < x) ? lo + half : lo;
        n -= half;
    }
    return lo + ((n == 1 && a[lo] < x) ? 1 : 0);
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int y = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += y;
    }
    return v;
}

template <int W>
__device__ __forceinline__ int group_sum(int v) {
#pragma unroll
    for (int d = W >> 1; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d, W);
    return v;
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(FULL, v, d));
    return v;
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* s_tmp /*[32]*/) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    __syncthreads();
    if (lane == 0) s_tmp[wid] = v;
    __syncthreads();
    long long r = 0;
    if (wid == 0) {
        r = (lane < (int)(blockDim.x >> 5)) ? s_tmp[lane] : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) r += __shfl_xor_sync(FULL, r, d);
    }
    return r;  // valid in thread 0
}

// key(u) = (deg(u), u): u -> v iff key(u) < key(v) (strict total order, reading C9).
__device__ __forceinline__ bool key_less(int du, int u, int dv, int v) {
    return du < dv || (du == dv && u < v);
}

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

// Same for any score / threshold type (int32 TW with int64 thresholds, fp64 scores with fp64
// thresholds): b = #{i : thr[i] > val}.
template <typename V, typename T>
__device__ __forceinline__ int band_of_t(V val, const T* thr, int k) {
    int lo = 0, hi = k;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (thr[mid] > (T)val) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ---- lock-free union-find (twc_cluster.cu sweep, twc_dist.cu local forests) -------------------
// A hook always links the LARGER root under the SMALLER one with atomicCAS, so parent[x] <= x at
// all times and the surviving root of every tree is its minimum vertex id (reading C6 / C19).
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

// Root of x, then a second walk pointing every node of the path straight at it (full
// compression): keeps trees shallow while a band merges many components at once.
__device__ __forceinline__ int uf_find_compress(int* parent, int x) {
    int r = parent[x];
    if (r == x) return r;
    int next;
    while (r > (next = parent[r])) r = next;
    // Second walk, only while above r: a concurrent hook may move the path below r (r itself
    // hooked under a smaller root), and nodes at or below r must never point at r.
    int cur = x;
    while (cur > r) {
        next = parent[cur];
        if (next > r) parent[cur] = r;  // r is an ancestor of cur and r < cur: stays a tree
        cur = next;
    }
    return r;
}

// Unites the trees of u and v; returns true (and the hooked roots in *a <- *b, a > b) when this
// call performed the hook, false when u and v were already connected.
__device__ __forceinline__ bool uf_unite(int* parent, int u, int v, int* a = nullptr,
                                         int* b = nullptr) {
    int ru = uf_find_compress(parent, u), rv = uf_find_compress(parent, v);
    while (ru != rv) {
        if (ru < rv) { int tmp = ru; ru = rv; rv = tmp; }  // hook the larger root ru under rv
        const int old = atomicCAS(&parent[ru], ru, rv);
        if (old == ru) {
            if (a) { *a = ru; *b = rv; }
            return true;
        }
        ru = uf_find(parent, old);
        rv = uf_find(parent, rv);
    }
    return false;
}

}  // namespace twc
