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
#include <algorithm>
#include <climits>
#include <vector>

#include "twc_common.cuh"
#include "twc_internal.h"

namespace twc {

// ------------------------------------------------------------------------------ K0 degrees
// (+ the sweep's union-find initialisation parent[u] = u when the fused call passes `parent`)
template <typename RP>
__global__ void k0_degrees(int64_t n, const RP* __restrict__ rowptr, int* __restrict__ deg,
                           int* __restrict__ parent) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) {
        deg[u] = (int)(rowptr[u + 1] - rowptr[u]);
        if (parent) parent[u] = (int)u;
    }
}

// ------------------------------------------------ K1: orientation over full-CSR slot tiles
// Every CSR slot p (row u, neighbour v) gets two bits: out(p) = key(u) < key(v) (the oriented
// edge u -> v exists) and upper(p) = v > u (p is the canonical copy of edge {u,v}).  Because
// rows are contiguous and sorted, all oriented quantities are prefix counts over slots:
//   * the oriented slot of an out-entry p is  #out(q < p)      -> col_or[#out(q<p)] = v, and
//     filtering a sorted row keeps it sorted;
//   * the canonical id of an upper slot p is  #upper(q < p)    (S:66-69 order);
//   * rp_or[u] = #out(q < rowptr[u]),  eoff[u] = #upper(q < rowptr[u]);
//   * so the oriented slot of an aligned edge (out and upper) is #out before its upper slot.
// K1 runs over tiles of kSlotTile slots (8 consecutive slots per thread): K1a computes the bits
// and per-tile counts, one block scans the tile counts, K1b scatters col_or and stores per-32-
// slot exclusive prefixes so that K1r and K3 derive any slot's oriented / canonical index with
// one lookup and a popc.  (A single pass with a decoupled look-back was measured slower,
// DESIGN.md Sec. 4.)
constexpr int kSlotThreads = 256;
constexpr int kSlotItems = 8;
static_assert(kSlotTile == kSlotThreads * kSlotItems, "K1 tile = 2048 slots");
constexpr int kMaxSlotRows = 1024;

// K1a: out/upper bits of every slot (8 consecutive slots per thread, one row search per
// thread, then a walk along the rows), stored as 32-slot words, plus per-tile counts and the
// far endpoint's degree per slot.  The tile's row offsets are kept as 32-bit offsets relative
// to the tile (clamped to [0, kSlotTile]) with the rows' degrees beside them, so the row
// search and the walk are 32-bit smem compares and deg(u) is an smem read; they are staged
// after the colidx loads and deg gathers are issued so the round trips overlap.  Tiles
// spanning more than kMaxSlotRows rows (average degree < 2 there) read rowptr / deg from
// global memory.  (Against the RP-typed version: 0.44 -> 0.36 ms on config 5.)
template <typename RP>
__global__ void __launch_bounds__(kSlotThreads, 8) k1_bits(
    int64_t m2, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int* __restrict__ deg, const int* __restrict__ ftrow, unsigned* __restrict__ obits,
    unsigned* __restrict__ ubits, int* __restrict__ tile_out, int* __restrict__ tile_up,
    unsigned short* __restrict__ dslot) {
    __shared__ int s_rp[kMaxSlotRows + 1];  // rowptr[r0 + i] - p0, clamped to [0, kSlotTile]
    __shared__ int s_dg[kMaxSlotRows];      // deg[r0 + i]
    __shared__ unsigned s_wsum[kSlotThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ntiles = (m2 + kSlotTile - 1) / kSlotTile;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p0 = tile * kSlotTile;
        const int tlen = (int)min((int64_t)kSlotTile, m2 - p0);
        const int r0 = ftrow[tile];
        const int nr = ftrow[tile + 1] - r0 + 1;
        const bool cached = nr <= kMaxSlotRows;
        {   // L2 prefetch of this block's next tile of colidx (64 lines of 128 bytes)
            const int64_t pn = (tile + gridDim.x) * kSlotTile + 32 * (int64_t)threadIdx.x;
            if (threadIdx.x < kSlotTile / 32 && pn < m2)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(colidx + pn));
        }
        auto rend = [&](int ri) -> int {  // end of row r0 + ri relative to the tile
            if (cached) return s_rp[ri + 1];
            const int64_t o = (int64_t)rowptr[r0 + ri + 1] - p0;
            return (int)min(max(o, (int64_t)0), (int64_t)kSlotTile);
        };
        auto rdeg = [&](int ri) -> int { return cached ? s_dg[ri] : deg[r0 + ri]; };
        const int q0 = threadIdx.x * kSlotItems;
        int v[kSlotItems];
        if (q0 + kSlotItems <= tlen) {
            const int4* src = reinterpret_cast<const int4*>(colidx + p0 + q0);
            const int4 a = __ldg(src), b = __ldg(src + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < kSlotItems; ++j) v[j] = (q0 + j < tlen) ? colidx[p0 + q0 + j] : 0;
        }
        int dv[kSlotItems];
#pragma unroll
        for (int j = 0; j < kSlotItems; ++j) dv[j] = (q0 + j < tlen) ? deg[v[j]] : 0;
        // the row offsets are staged after the colidx loads and deg gathers were issued, so the
        // three memory round trips overlap
        __syncthreads();
        if (cached) {
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) {
                const int64_t o = (int64_t)rowptr[r0 + i] - p0;
                s_rp[i] = (int)min(max(o, (int64_t)0), (int64_t)kSlotTile);
                if (i < nr) s_dg[i] = deg[r0 + i];
            }
        }
        __syncthreads();
        if (q0 + kSlotItems <= tlen) {
            unsigned w4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                w4[j] = (unsigned)min(dv[2 * j], 0xffff) | ((unsigned)min(dv[2 * j + 1], 0xffff) << 16);
            __stcs(reinterpret_cast<uint4*>(dslot + p0 + q0), make_uint4(w4[0], w4[1], w4[2], w4[3]));
        } else {
#pragma unroll
            for (int j = 0; j < kSlotItems; ++j)
                if (q0 + j < tlen) dslot[p0 + q0 + j] = (unsigned short)min(dv[j], 0xffff);
        }
        unsigned ob = 0, ub = 0;
        if (q0 < tlen) {
            int ri;
            if (cached) {
                ri = last_le(s_rp, nr + 1, q0);
            } else {
                ri = last_le(rowptr + r0, nr + 1, (RP)(p0 + q0));
            }
            TWC_ASSERT(ri >= 0 && ri < nr);
            int re = rend(ri);
            int u = r0 + ri, du = rdeg(ri);
#pragma unroll
            for (int j = 0; j < kSlotItems; ++j) {
                const int q = q0 + j;
                if (q < tlen) {
                    while (q >= re) {  // next row (skipping empty rows)
                        ++ri;
                        TWC_ASSERT(ri < nr);
                        re = rend(ri);
                        ++u;
                        du = rdeg(ri);
                    }
                    ob |= (unsigned)key_less(du, u, dv[j], v[j]) << j;
                    ub |= (unsigned)(v[j] > u) << j;
                }
            }
        }
        unsigned ow = ob << (8 * (lane & 3)), uw = ub << (8 * (lane & 3));
        ow |= __shfl_xor_sync(FULL, ow, 1);
        ow |= __shfl_xor_sync(FULL, ow, 2);
        uw |= __shfl_xor_sync(FULL, uw, 1);
        uw |= __shfl_xor_sync(FULL, uw, 2);
        if ((lane & 3) == 0 && q0 < tlen) {
            obits[(p0 + q0) >> 5] = ow;
            ubits[(p0 + q0) >> 5] = uw;
        }
        unsigned cnt = (__popc(ob) << 16) | __popc(ub);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(FULL, cnt, d);
        if (lane == 0) s_wsum[wid] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned tot = 0;
#pragma unroll
            for (int i = 0; i < kSlotThreads / 32; ++i) tot += s_wsum[i];
            tile_out[tile] = (int)(tot >> 16);
            tile_up[tile] = (int)(tot & 0xffffu);
        }
    }
}

// Exclusive scans of the two per-tile count arrays (one block; ntiles ~ 2m / 2048).  Both
// counts travel packed in one 64-bit value (out << 32 | upper; each total <= m < 2^32, so the
// low half never carries).  Warp w owns one contiguous segment: a coalesced sum pass (four
// 32-tile chunks in flight), one scan of the 32 segment sums, then a warp-scan rewrite of the
// segment -- no block barrier per 1,024 tiles (config 5, 34k tiles: 39 -> 28 us in the ncu launch list).
__device__ __forceinline__ unsigned long long tile_pack(const int* a, const int* b, int64_t i) {
    return ((unsigned long long)(unsigned)a[i] << 32) | (unsigned)b[i];
}

__global__ void __launch_bounds__(1024) k1_tile_scan(int64_t ntiles, int* __restrict__ a,
                                                     int* __restrict__ b) {
    __shared__ unsigned long long s_w[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t seg = (ntiles + 31) / 32;
    const int64_t lo = min(ntiles, (int64_t)wid * seg), hi = min(ntiles, lo + seg);
    unsigned long long part = 0;
    for (int64_t base = lo; base < hi; base += 128) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = base + 32 * k + lane;
            if (i < hi) part += tile_pack(a, b, i);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(FULL, part, d);
    if (lane == 0) s_w[wid] = part;
    __syncthreads();
    if (wid == 0) {
        const unsigned long long x = s_w[lane];
        unsigned long long y = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long z = __shfl_up_sync(FULL, y, d);
            if (lane >= d) y += z;
        }
        s_w[lane] = y - x;
    }
    __syncthreads();
    unsigned long long run = s_w[wid];
    for (int64_t base = lo; base < hi; base += 128) {
        unsigned long long v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = base + 32 * k + lane;
            v[k] = i < hi ? tile_pack(a, b, i) : 0ull;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            unsigned long long incl = v[k];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long z = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl += z;
            }
            const int64_t i = base + 32 * k + lane;
            const unsigned long long ex = run + incl - v[k];
            if (i < hi) {
                a[i] = (int)(ex >> 32);
                b[i] = (int)(ex & 0xffffffffull);
            }
            run += __shfl_sync(FULL, incl, 31);
        }
    }
}

// K1b: oriented slot = #out before p, canonical id = #upper before p (tile prefix + block
// scan + popc); scatter col_or and store the per-word prefixes (K1r and K3 derive any
// slot's oriented / canonical index from them with one popc).
__global__ void __launch_bounds__(kSlotThreads) k1_write(
    int64_t m2, const int* __restrict__ colidx, const unsigned* __restrict__ obits,
    const unsigned* __restrict__ ubits, const int* __restrict__ tile_out,
    const int* __restrict__ tile_up, int* __restrict__ opre, int* __restrict__ upre,
    int* __restrict__ col_or) {
    __shared__ unsigned s_wsum[kSlotThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ntiles = (m2 + kSlotTile - 1) / kSlotTile;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p0 = tile * kSlotTile;
        const int64_t q0 = p0 + threadIdx.x * kSlotItems;
        unsigned ob = 0, ub = 0;
        if (q0 < m2) {
            const int sh = 8 * (lane & 3);
            ob = (obits[q0 >> 5] >> sh) & 0xffu;
            ub = (ubits[q0 >> 5] >> sh) & 0xffu;
        }
        const unsigned cnt = (__popc(ob) << 16) | __popc(ub);
        const unsigned incl = (unsigned)warp_incl_scan((int)cnt, lane);
        __syncthreads();
        if (lane == 31) s_wsum[wid] = incl;
        __syncthreads();
        unsigned wpre = 0;
#pragma unroll
        for (int i = 0; i < kSlotThreads / 32; ++i) wpre += (i < wid) ? s_wsum[i] : 0u;
        const unsigned ex = wpre + incl - cnt;
        const int obase = tile_out[tile] + (int)(ex >> 16);
        const int ubase = tile_up[tile] + (int)(ex & 0xffffu);
        if ((lane & 3) == 0 && q0 < m2) {
            opre[q0 >> 5] = obase;
            upre[q0 >> 5] = ubase;
        }
        if (ob) {
            int v[kSlotItems];
            if (q0 + kSlotItems <= m2) {
                const int4* src = reinterpret_cast<const int4*>(colidx + q0);
                const int4 a = __ldg(src), b = __ldg(src + 1);
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
            } else {
#pragma unroll
                for (int j = 0; j < kSlotItems; ++j) v[j] = (q0 + j < m2) ? colidx[q0 + j] : 0;
            }
#pragma unroll
            for (int j = 0; j < kSlotItems; ++j) {
                if ((ob >> j) & 1u) {
                    const unsigned below = (1u << j) - 1u;
                    const int sl = obase + __popc(ob & below);
                    TWC_ASSERT(sl >= 0 && (int64_t)sl < m2 / 2);
                    col_or[sl] = v[j];
                }
            }
        }
    }
}

// K1r: rp_or[u] = #out(q < rowptr[u]), eoff[u] = #upper(q < rowptr[u]); rp_or[n] = eoff[n] = m;
// vinfo[u] = {rp_or[u], rp_or[u+1]}: the oriented list of the far endpoint of a reversed edge
// in one 8-byte record (one sector per random lookup instead of two).
template <typename RP>
__device__ __forceinline__ int out_before(int64_t m, RP p, const unsigned* __restrict__ obits,
                                          const int* __restrict__ opre) {
    if ((int64_t)p >= 2 * m) return (int)m;
    const int64_t wi = (int64_t)(p >> 5);
    return opre[wi] + __popc(obits[wi] & ((1u << (p & 31)) - 1u));
}

template <typename RP>
__global__ void k1_rows(int64_t n, int64_t m, const RP* __restrict__ rowptr,
                        const unsigned* __restrict__ obits, const unsigned* __restrict__ ubits,
                        const int* __restrict__ opre, const int* __restrict__ upre,
                        int* __restrict__ rp_or, int* __restrict__ eoff, int2* __restrict__ vinfo) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u > n) return;
    const RP p = rowptr[u];
    const int ob = out_before(m, p, obits, opre);
    rp_or[u] = ob;
    if ((int64_t)p >= 2 * m) {
        eoff[u] = (int)m;
    } else {
        const int64_t wi = (int64_t)(p >> 5);
        eoff[u] = upre[wi] + __popc(ubits[wi] & ((1u << (p & 31)) - 1u));
    }
    if (u < n) {
        const RP pe = rowptr[u + 1];
        vinfo[u] = make_int2(ob, out_before(m, pe, obits, opre));
    }
}

// ---------------------------------------------------------- K2 oriented intersection
// Every triangle {u, v, w} is found exactly once, from its lowest-key vertex u (the pivot):
// v in N+(u), w in N+(v) and w in N+(u).  Work items are the pairs (slot u->v, w in N+(v));
// there are S = sum_v d-(v) d+(v) of them, and only T (the triangle count) of them hit.
//
// Warp-level scheme (persistent grid, chunked atomic pivot queue):
//  * a warp groups consecutive pivots whose oriented lists total <= kGroupSlots slots and
//    stages those lists (one contiguous range [A, B) of col_or) in shared memory, together
//    with a kFilterBits-bit hash filter of their entries (pivots with longer lists are hubs,
//    left to K2h);
//  * the group's slots are taken 32 at a time (one per lane, a "round"); slot u->v owns the
//    items w in N+(v) if d+(u) >= 2, cut into groups of Q = kOct entries aligned to one 32-byte
//    sector of col_or (covering [start & ~7, end)).  The groups of the 32 slots are flattened
//    across the lanes (exclusive scan of the group counts; the segment records are stored
//    compacted in slot order, so the segment owning a sector is the number of segments started
//    at or before it: one __reduce_or_sync bit mask and a popc), so each lane reads one aligned
//    sector (one 256-bit LDG.E.256) of one N+(v) and a warp reads a contiguous run.  The per-lane
//    segment record {start & ~7 - 8 * first group, end, tag, start} gives a group's slots with
//    one 16-byte smem load; loads are clamped into the list, so loads and hashes run
//    unpredicated and one validity mask (start <= slot < end) is applied per group;
//  * filter position of w: word = top bits of x = w * K, bit = x & 31 (K odd, so x & 31 is a
//    bijection of w & 31); one funnel rotate by (x - e) puts item e's bit at position e;
//  * an item whose w misses the filter cannot be in N+(u) (the common case).  A lane with
//    candidates pushes ONE record (slot of the sector, 8-bit mask, tag = slot u->v and pivot)
//    with one ballot; records are expanded into a candidate ring 32 at a time and candidates
//    verified 32 at a time by binary search in the staged sorted N+(u), so the prefix work and
//    the search run on full warps.  Record and candidate entries are self-contained, so the
//    rings carry over between the rounds of a group and drain only when full or at its end;
//  * a verified hit adds 1 to t(u,w), t(u,v) and t(v,w) with three global reductions (the
//    first two land in the group's own slot range [A, B), a few sectors per verify batch).
//    Per-warp shared byte counters were used before; K2 is bound by the L1/shared data pipe,
//    and their atomics cost bank-conflict replays plus a flush per group;
//  * the round setup prefetches each lane's N+(v) into L2, so the sector loop's loads find it.
// DESIGN.md Sec. 4.1 lists the variants measured on the way (ncu evidence per step).
constexpr int kK2Warps = 8;
constexpr int kGroupSlots = 256;
constexpr int kPivotChunk = 32;
constexpr int kOct = 8;   // K2: items per lane (one aligned 32-byte sector, one 256-bit load)
constexpr int kRing = 128;  // candidate ring, default (an expansion stops before it would overflow)
constexpr int kRec = 64;    // record ring, >= 31 + 32 pending records
constexpr unsigned kFiltK = 2654435761u;

// 4,240 bytes per warp at FLOG = 13: 5 CTAs of 8 warps fit the 196 KB smem carveout and leave
// 60 KB of L1 (DESIGN.md Sec. 4.1 for the carveout / occupancy measurements).
template <int FLOG, int RING = kRing, int SPL = 1>
struct K2WarpSmem {
    static constexpr int kFilterWords = (1 << FLOG) / 32;
    static constexpr int kRingN = RING;
    int list[kGroupSlots];          // staged col_or[A, B)
    unsigned filt[kFilterWords];
    int prp[33];                    // ends of the group's non-empty lists (list j = [prp[j], prp[j+1]))
    int4 seg[32 * SPL];             // per slot of the round: {start of N+(v) - 8 * first sector, end, tag, start}
    int2 ring[RING];                // candidates: {slot of v -> w, tag}
    int2 rec[kRec];                 // candidate sectors: {slot of the sector, mask | tag << 8}
};

template <int FLOG>
__device__ __forceinline__ unsigned filter_word(unsigned x) { return x >> (32 - FLOG + 5); }


__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));  // (.L1 instead: no difference, 1.762 / 1.760 ms)
}

// Verify ring entries [head, head + cnt) (cnt <= 32; lane i takes entry head + i).
// tag = (slot of u -> v) - A | pivot index << 8.
template <typename SM>
__device__ __forceinline__ void k2_verify(SM& S, int lane, int head, int cnt, int A,
                                          const int* __restrict__ col_or,
                                          int* __restrict__ t_or) {
    if (lane < cnt) {
        const int2 c = S.ring[(head + lane) & (SM::kRingN - 1)];
        const int sv = c.x;  // slot of v -> w
        TWC_ASSERT(sv >= 0);
        const int w = col_or[sv];
        const int pi = c.y >> 8, so = c.y & 255;
        TWC_ASSERT(pi >= 0 && pi < 32 && so >= 0 && so < kGroupSlots);
        const int plo = S.prp[pi] - A, len = S.prp[pi + 1] - S.prp[pi];
        const int* L = S.list + plo;
        const int q = lower_bound_bl(L, len, w);
        if (q < len && L[q] == w) {
            const int i = plo + q;
            TWC_ASSERT(i >= 0 && i < kGroupSlots && so < kGroupSlots);
            atomicAdd(&t_or[A + i], 1);                       // t(u, w)
            atomicAdd(&t_or[A + so], 1);                      // t(u, v)
            atomicAdd(&t_or[sv], 1);                          // t(v, w)
        }
    }
}

// Expand records [rhead, rhead + cnt) (cnt <= 32, lane i takes record rhead + i) into the
// candidate ring at tail while they fit; returns the number of records consumed (a prefix; at
// least 12 when fewer than 32 candidates are pending: a record holds at most Q = 8).
template <int Q, typename SM>
__device__ __forceinline__ int k2_expand(SM& S, int lane, int rhead, int cnt, int head,
                                         int& tail) {
    const int2 r = (lane < cnt) ? S.rec[(rhead + lane) & (kRec - 1)] : make_int2(0, 0);
    const unsigned cm = (unsigned)r.y & 0xffu;
    const int nc = __popc(cm);
    const int incl = warp_incl_scan(nc, lane);
    const bool fits = lane < cnt && incl <= SM::kRingN - (tail - head);
    const unsigned fb = __ballot_sync(FULL, fits);
    if (fits) {  // a loop over the set bits: most records hold one candidate (max ~2-3 per warp)
        int pos = tail + incl - nc;
        const int tag = r.y >> 8;
        unsigned bits = cm;
        while (bits) {
            const int e = __ffs(bits) - 1;
            bits &= bits - 1u;
            S.ring[pos & (SM::kRingN - 1)] = make_int2(r.x + e, tag);
            ++pos;
        }
    }
    const int used = __popc(fb);
    tail += __shfl_sync(FULL, incl, max(used - 1, 0)) * (used > 0);
    TWC_ASSERT(tail - head <= SM::kRingN);
    return used;
}

// Drain: expand pending records while at least `keep` remain and verify full warps of
// candidates.
template <int Q, typename SM>
__device__ __forceinline__ void k2_drain(SM& S, int lane, int keep, int A, int& rhead,
                                         int rtail, int& head, int& tail,
                                         const int* __restrict__ col_or, int* __restrict__ t_or) {
    while (rtail - rhead > keep) {
        rhead += k2_expand<Q>(S, lane, rhead, min(32, rtail - rhead), head, tail);
        __syncwarp();
        while (tail - head >= 32) {
            k2_verify(S, lane, head, 32, A, col_or, t_or);
            head += 32;
        }
        __syncwarp();
    }
}

// range: NULL (all pivots) or device {u_lo, u_hi} of a shard (the queue starts at u_lo)
// SPL: slots per lane and round (a round takes 32 * SPL slots of the group and flattens their
// sectors together).  SPL = 2 with a 64-entry candidate ring (same shared memory) was measured:
// 1.82 ms against 1.765 ms for SPL = 1 -- the second owner test per window and the smaller ring
// cost more instructions than the fuller last windows save (profiles/r2k_k2_experiments.md).
template <int Q, int FLOG, int MINB, int RING = kRing, int SPL = 1>
__global__ void __launch_bounds__(kK2Warps * 32, MINB) k2_intersect(int64_t n, int chunk,
                                                              const int* __restrict__ rp_or,
                                                              const int* __restrict__ col_or,
                                                              int* __restrict__ t_or,
                                                              int* __restrict__ work,
                                                              const int* __restrict__ range,
                                                              const int2* __restrict__ vinfo) {
    extern __shared__ __align__(16) unsigned char k2_smem_raw[];
    using SM = K2WarpSmem<FLOG, RING, SPL>;
    SM* smem = reinterpret_cast<SM*>(k2_smem_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    SM& S = smem[wid];
    const int64_t u_end = range ? (int64_t)range[1] : n;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(work, chunk);
        base = __shfl_sync(FULL, base, 0);
        if (base >= u_end) break;
        const int gend = (int)min((int64_t)base + chunk, u_end);
        int u = base;
        while (u < gend) {
            // ---- form a group of pivots [u, u+np) with <= kGroupSlots slots
            const int np_max = min(32, gend - u);
            const int A = rp_or[u];
            const int e_l = (lane < np_max) ? rp_or[u + lane + 1] : INT_MAX;
            const unsigned fit = __ballot_sync(FULL, lane < np_max && e_l - A <= kGroupSlots);
            if (fit == 0u) {  // a hub (|N+(u)| > kGroupSlots): k2_hubs takes it
                ++u;
                continue;
            }
            const int np = __popc(fit);
            const int B = __shfl_sync(FULL, e_l, np - 1);
            TWC_ASSERT(np >= 1 && np <= 32 && B - A >= 0 && B - A <= kGroupSlots);
            TWC_ASSERT(fit == (np == 32 ? FULL : (1u << np) - 1u));  // a prefix of the pivots
            // prp[] holds the ends of the group's NON-EMPTY lists only (list j = [prp[j], prp[j+1])),
            // and lane j keeps prp[j+1] in a register: the list of a slot is then found with one
            // ballot and one warp OR per round instead of a binary search in shared memory
            int b_l = __shfl_up_sync(FULL, e_l, 1);
            if (lane == 0) b_l = A;
            const unsigned nem = __ballot_sync(FULL, lane < np && e_l > b_l);
            const int npc = __popc(nem);
            if (lane == 0) S.prp[0] = A;
            if ((nem >> lane) & 1u) S.prp[__popc(nem & lt_mask) + 1] = e_l;
            for (int i = lane; i < SM::kFilterWords; i += 32) S.filt[i] = 0u;
            __syncwarp();
            const int E = (lane < npc) ? S.prp[lane + 1] : INT_MAX;
            // lists with a single entry own no items (a triangle needs two out-neighbours)
            const unsigned single = __ballot_sync(FULL, lane < npc && E - S.prp[lane] < 2);
            for (int i = lane; i < B - A; i += 32) {
                const int x = __ldcs(col_or + A + i);  // read once: staged, not kept in L1
                S.list[i] = x;
                const unsigned h = (unsigned)x * kFiltK;
                atomicOr(&S.filt[filter_word<FLOG>(h)], 1u << (h & 31));
            }
            __syncwarp();
            int head = 0, tail = 0;    // candidate ring
            int rhead = 0, rtail = 0;  // record ring
            // ---- rounds of 32 * SPL slots
            for (int r0 = A; r0 < B; r0 += 32 * SPL) {
                int swin[SPL];       // window of the slot's first sector (-1: no sectors)
                unsigned sbit[SPL];  // its position in that window, as a bit
                int total = 0, nseg = 0;
#pragma unroll
                for (int k = 0; k < SPL; ++k) {
                    const int sb = r0 + 32 * k;
                    const int s = sb + lane;
                    int w_ = 0, vs = 0, vd = 0, pi = 0;
                    if (SPL == 1 || sb < B) {
                        // list of slot s: #lists ending at or before s
                        const int pbase = __popc(__ballot_sync(FULL, E <= sb));
                        const unsigned bm = __reduce_or_sync(
                            FULL, (E > sb && E < sb + 32) ? (1u << (E - sb)) : 0u);
                        pi = pbase + __popc(bm & ((2u << lane) - 1u));
                        if (s < B) {
                            TWC_ASSERT(pi >= 0 && pi < npc && S.prp[pi] <= s && s < S.prp[pi + 1]);
                            const int v = S.list[s - A];
                            if (!((single >> pi) & 1u)) {
                                const int2 vi = vinfo[v];  // {rp_or[v], rp_or[v+1]}: one 8-byte load
                                vs = vi.x;
                                vd = vi.y - vs;
                                TWC_ASSERT(vs >= 0 && vd >= 0 && vd < 65536);
                                // items in aligned groups of Q: [vs & ~(Q-1), vs + vd)
                                w_ = (vs + vd - (vs & ~(Q - 1)) + Q - 1) / Q;
                            }
                        }
                    }
                    const int incl = warp_incl_scan(w_, lane);
                    const int pre = total + incl - w_;
                    swin[k] = w_ > 0 ? pre >> 5 : -1;
                    sbit[k] = 1u << (pre & 31);
                    // the segments with sectors are stored compacted, in slot order = order of their
                    // first sector: the j-th segment starting in a window is the (#segments
                    // started before the window + j)-th record, so no owner table is needed
                    const unsigned nz = __ballot_sync(FULL, w_ > 0);
                    if (w_ > 0) {
                        S.seg[nseg + __popc(nz & lt_mask)] =
                            make_int4((vs & ~(Q - 1)) - Q * pre, vs + vd, (s - A) | (pi << 8), vs);
                        // the sector loop below reads N+(v): L2 prefetch (3 % of K2)
                        prefetch_l2(col_or + vs);
                        if (((vs + vd - 1) >> 5) != (vs >> 5)) prefetch_l2(col_or + vs + vd - 1);
                    }
                    nseg += __popc(nz);
                    total += __shfl_sync(FULL, incl, 31);
                }
                int cb = 0;  // segments started before the current window
                __syncwarp();
                for (int k0 = 0; k0 < total; k0 += 32) {
                    unsigned sb_ = 0;
#pragma unroll
                    for (int k = 0; k < SPL; ++k) sb_ |= (swin[k] == (k0 >> 5)) ? sbit[k] : 0u;
                    const unsigned bits = __reduce_or_sync(FULL, sb_);
                    // segment of sector k0 + lane: the last one started at or before it (lanes past
                    // the last sector get the last segment and an empty validity mask)
                    const int jj = cb + __popc(bits & ((2u << lane) - 1u)) - 1;
                    cb += __popc(bits);
                    TWC_ASSERT(jj >= 0 && jj < nseg);
                    const int4 sg = S.seg[jj];
                    const int sv0 = sg.x + Q * (k0 + lane);  // 4Q-byte aligned
                    TWC_ASSERT(min(sv0, (sg.y - 1) & ~(Q - 1)) >= 0 && (sv0 & (Q - 1)) == 0);
                    // the aligned sector of this lane (clamped to the list's last group)
                    const int4* src = reinterpret_cast<const int4*>(
                        col_or + min(sv0, (sg.y - 1) & ~(Q - 1)));
                    int w[Q];
                    if (Q == 8) {  // one 256-bit load (LDG.E.256) per lane
                        ldg_sector(reinterpret_cast<const int*>(src), *reinterpret_cast<int(*)[8]>(w));
                    } else {
#pragma unroll
                        for (int h = 0; h < Q / 4; ++h) {
                            const int4 q4 = __ldg(src + h);
                            w[4 * h] = q4.x; w[4 * h + 1] = q4.y; w[4 * h + 2] = q4.z; w[4 * h + 3] = q4.w;
                        }
                    }
                    unsigned cm = 0;
#pragma unroll
                    for (int e = 0; e < Q; ++e) {
                        const unsigned x = (unsigned)w[e] * kFiltK;
                        // opaque word index: keeps ptxas from folding the shift into
                        // (x >> 22) & 0x3fc + base (3 ops) so the address is SHF + LEA
                        unsigned fw = filter_word<FLOG>(x);
                        asm("" : "+r"(fw));
                        const unsigned word = S.filt[fw];
                        cm |= __funnelshift_r(word, word, x - (unsigned)e) & (1u << e);
                    }
                    // valid entries: sg.w <= sv0 + e < sg.y
                    cm &= bit_range(max(sg.w - sv0, 0), min(sg.y - sv0, Q));
                    const unsigned hb = __ballot_sync(FULL, cm != 0u);
                    if (cm) S.rec[(rtail + __popc(hb & lt_mask)) & (kRec - 1)] =
                                make_int2(sv0, (int)cm | (sg.z << 8));
                    rtail += __popc(hb);
                    TWC_ASSERT(rtail - rhead <= kRec);
                    __syncwarp();
                    k2_drain<Q>(S, lane, 31, A, rhead, rtail, head, tail, col_or, t_or);
                }
                __syncwarp();  // seg is rewritten by the next round
            }
            k2_drain<Q>(S, lane, 0, A, rhead, rtail, head, tail, col_or, t_or);
            if (tail > head) k2_verify(S, lane, head, tail - head, A, col_or, t_or);
            __syncwarp();
            u += np;
        }
    }
}

// ------------------------------------------------------ K2h: hub pivots (|N+(u)| > 256)
// One pivot per CTA: the whole block stages N+(u) (up to kHubMax entries) and a 64K-bit filter
// of it in shared memory, and its 8 warps take the pivot's slots 32 at a time with the same
// flattened sector scan, filter and candidate ring as K2.  A list longer than kHubMax keeps only
// the filter; its candidates are verified by binary search in global memory.
constexpr int kHubMax = 2048;
constexpr int kHubQ = 8;        // items per lane: one aligned 32-byte sector (one LDG.E.256)
constexpr int kHubRing = 512;   // >= 31 + 32 * kHubQ pending candidates
constexpr int kHubFilterLog = 16;
constexpr int kHubFilterWords = (1 << kHubFilterLog) / 32;

struct K2HubWarp {
    int4 seg[32];  // per segment: {start of N+(v) & ~7 - 8 * first sector, end, start, slot's lane}
    int ring[kHubRing];
};
struct K2HubSmem {
    int list[kHubMax];
    unsigned filt[kHubFilterWords];
    K2HubWarp w[kK2Warps];
    int hub;
};

// filter position as K2's: word = top bits of x = w * K, bit = x & 31
__device__ __forceinline__ unsigned hub_word(unsigned x) { return x >> (32 - kHubFilterLog + 5); }

// hubs[] = pivots with more than kGroupSlots oriented neighbours (order irrelevant)
__global__ void k2_find_hubs(int64_t n, const int* __restrict__ rp_or, int* __restrict__ hubs,
                             int* __restrict__ nhubs, const int* __restrict__ range) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = range ? (u >= range[0] && u < range[1]) : u < n;
    const bool hub = in && rp_or[u + 1] - rp_or[u] > kGroupSlots;
    const unsigned b = __ballot_sync(FULL, hub);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(b) - 1) base = atomicAdd(nhubs, __popc(b));
    base = __shfl_sync(FULL, base, __ffs(b) - 1);
    if (hub) hubs[base + __popc(b & ((1u << lane) - 1u))] = (int)u;
}

// 6 CTAs per SM (40 registers, 36 KB of shared memory each): the hub kernel is latency-bound like
// K2, and R-MAT dense 10^8 went 121.6 -> 98.5 ms when the per-entry shared counters (32 KB) were
// replaced by global REDs (3 CTAs/SM instead of 2), -> 83.1 / 74.8 / 71.5 ms with 4,096 / 4,096 /
// 2,048 staged entries at 4 / 5 / 6 CTAs/SM (profiles/r2k_k2_experiments.md Sec. 10).
constexpr int kHubMinBlocks = 6;
__global__ void __launch_bounds__(kK2Warps * 32, kHubMinBlocks) k2_hubs(
    const int* __restrict__ rp_or, const int* __restrict__ col_or, const int* __restrict__ hubs,
    const int* __restrict__ nhubs, int* __restrict__ work, int* __restrict__ t_or) {
    extern __shared__ __align__(16) unsigned char k2h_smem_raw[];
    K2HubSmem& H = *reinterpret_cast<K2HubSmem*>(k2h_smem_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    K2HubWarp& W = H.w[wid];
    const int nh = *nhubs;
    for (;;) {
        if (threadIdx.x == 0) H.hub = atomicAdd(work, 1);
        __syncthreads();
        const int h = H.hub;
        if (h >= nh) break;
        const int u = hubs[h];
        const int A = rp_or[u], B = rp_or[u + 1], len = B - A;
        const bool staged = len <= kHubMax;
        for (int i = threadIdx.x; i < kHubFilterWords; i += blockDim.x) H.filt[i] = 0u;
        __syncthreads();
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            const int x = col_or[A + i];
            if (staged) {
                H.list[i] = x;
            }
            const unsigned hx = (unsigned)x * kFiltK;
            atomicOr(&H.filt[hub_word(hx)], 1u << (hx & 31));
        }
        __syncthreads();
        for (int r0 = A + 32 * wid; r0 < B; r0 += 32 * kK2Warps) {
            const int s = r0 + lane;
            int wt = 0, vs = 0, vd = 0;
            if (s < B) {
                const int v = staged ? H.list[s - A] : col_or[s];
                vs = rp_or[v];
                vd = rp_or[v + 1] - vs;
                wt = (vs + vd - (vs & ~7) + kHubQ - 1) / kHubQ;  // aligned 32-byte sectors
            }
            const int incl = warp_incl_scan(wt, lane);
            const int total = __shfl_sync(FULL, incl, 31);
            const int pre = incl - wt;
            // segment records compacted in slot order, as in K2: the segment of a sector is the
            // number of segments started at or before it; .w keeps the slot's lane
            const unsigned nz = __ballot_sync(FULL, wt > 0);
            if (wt > 0)
                W.seg[__popc(nz & lt_mask)] = make_int4((vs & ~7) - kHubQ * pre, vs + vd, vs, lane);
            int cb = 0;
            int head = 0, tail = 0;
            __syncwarp();
            for (int k0 = 0; k0 < total; k0 += 32) {
                const bool starts = wt > 0 && pre >= k0 && pre < k0 + 32;
                const unsigned bits = __reduce_or_sync(FULL, starts ? (1u << (pre - k0)) : 0u);
                // lanes past the end get the last segment and an empty mask
                const int jj = cb + __popc(bits & ((2u << lane) - 1u)) - 1;
                cb += __popc(bits);
                TWC_ASSERT(jj >= 0 && jj < __popc(nz));
                const int4 sg = W.seg[jj];
                const int sv0 = sg.x + kHubQ * (k0 + lane);  // 32-byte aligned
                TWC_ASSERT(min(sv0, (sg.y - 1) & ~7) >= 0);
                int wq[kHubQ];
                ldg_sector(col_or + min(sv0, (sg.y - 1) & ~7), wq);
                unsigned cm = 0;
#pragma unroll
                for (int e = 0; e < kHubQ; ++e) {
                    const unsigned x = (unsigned)wq[e] * kFiltK;
                    const unsigned word = H.filt[hub_word(x)];
                    cm |= __funnelshift_r(word, word, x - (unsigned)e) & (1u << e);
                }
                cm &= ((1u << min(max(sg.y - sv0, 0), kHubQ)) - 1u) &
                      (0xffu << min(max(sg.z - sv0, 0), kHubQ));
                const int cbase = (jj << 16) + (sv0 - sg.z);  // + e >= 0 for a valid entry
#pragma unroll
                for (int e = 0; e < kHubQ; ++e) {
                    const bool c = (cm >> e) & 1u;
                    const unsigned b = __ballot_sync(FULL, c);
                    if (c) W.ring[(tail + __popc(b & lt_mask)) & (kHubRing - 1)] = cbase + e;
                    tail += __popc(b);
                }
                TWC_ASSERT(tail - head <= kHubRing);
                __syncwarp();
                while (tail - head > 0 && (tail - head >= 32 || k0 + 32 >= total)) {
                    const int cnt = min(32, tail - head);
                    if (lane < cnt) {
                        const int e = W.ring[(head + lane) & (kHubRing - 1)];
                        const int4 cs = W.seg[e >> 16];
                        const int j = cs.w;                        // lane of the slot u -> v
                        const int sv = cs.z + (e & 0xffff);        // slot of v -> w
                        const int w = col_or[sv];
                        const int* L = staged ? H.list : col_or + A;
                        const int q = staged ? lower_bound_bl(L, len, w) : lower_bound(L, len, w);
                        if (q < len && L[q] == w) {
                            TWC_ASSERT(r0 + j - A >= 0 && r0 + j - A < len);
                            atomicAdd(&t_or[A + q], 1);              // t(u, w)
                            atomicAdd(&t_or[r0 + j], 1);             // t(u, v)
                            atomicAdd(&t_or[sv], 1);                 // t(v, w)
                        }
                    }
                    head += cnt;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        __syncthreads();
    }
}

// ---------------------------------------------------------- K3 fused score epilogue
// Edge-parallel over canonical ids; each CTA takes tiles of kTile ids, caches the tile's
// canonical row offsets in smem and maps id -> row by binary search.  The count t of edge
// (u,v) sits at its oriented slot: for an aligned edge (key(u) < key(v)) that slot is the
// number of out-slots before its upper slot (word prefix + popc); for a reversed one it is
// found by probing the (short) list N+(v) for u.
//   wedge = d_u + d_v - 2t - 2   (|N(u) | N(v)| - |N(u) & N(v)| - 2 for a simple graph)
//   TW    = t - wedge            (Eq. 2)
// Index of u in the sorted list col_or[ob, oe) (u is present).  The search works on aligned
// 32-byte sectors (8 ids): it starts at the sector where u would sit if the ids were spread
// evenly over [0, n) (interpolation) and steps one sector at a time, so a typical lookup
// touches one or two sectors instead of the log2(len) scattered sectors of a binary search.
__device__ __forceinline__ int sector_search(const int* __restrict__ col_or, int ob, int oe, int u,
                                             int64_t n) {
    const int len = oe - ob;
    int s = (ob + (int)(((long long)len * u) / n)) & ~7;
    const int s_lo = ob & ~7, s_hi = (oe - 1) & ~7;
    s = max(s_lo, min(s, s_hi));
    for (;;) {
        TWC_ASSERT(s >= s_lo && s <= s_hi && s >= 0);
        int x[8];
        ldg_sector(col_or + s, x);  // the aligned 32-byte sector, one 256-bit load
        const int first = max(ob - s, 0), last = min(oe - s, 8) - 1;  // valid entries [first, last]
        int fv = 0, lv = 0, below = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            fv = (e == first) ? x[e] : fv;
            lv = (e == last) ? x[e] : lv;
            below += (e >= first && e <= last && x[e] < u);
        }
        if (s > s_lo && fv > u) { s -= 8; continue; }
        if (s < s_hi && lv < u) { s += 8; continue; }
        return s + first + below;
    }
}

constexpr int kK3Threads = 256;
// dynamic smem of a binning K3: kept edges of a tile (int2 + u16 each), thresholds, histogram
inline size_t k3_bin_smem(int k) { return (size_t)10 * kTile + (size_t)k * 12; }
constexpr int kMaxTileRows = 2048;

// DIST: the epilogue of one rank of the distributed step (twc_dist.cu): only the
// canonical edges of the rank's slice [cb[rank], cb[rank+1]); an edge whose oriented slot lies
// outside the rank's oriented slice [ob[rank], ob[rank+1]) (a reversed edge whose far endpoint
// belongs to another rank) is not scored here but recorded as {c, u, v, slot} for the owner.
template <typename RP, bool BIN, bool K4 = false, bool DIST = false>
__global__ void __launch_bounds__(kK3Threads, 8) k3_score(
    int64_t n, int64_t m, const RP* __restrict__ rowptr, const int* __restrict__ colidx,
    const int2* __restrict__ vinfo, const unsigned short* __restrict__ dslot,
    const int* __restrict__ deg, const int* __restrict__ eoff,
    const int* __restrict__ trow,
    const int* __restrict__ col_or, const int* __restrict__ opre,
    const unsigned* __restrict__ obits, const int* __restrict__ t_or, int* __restrict__ t,
    int* __restrict__ wedge, int* __restrict__ tw, BinSpec bin,
    const unsigned long long* __restrict__ k4_or = nullptr, long long* __restrict__ k4 = nullptr,
    DistK3 dist = DistK3{}) {
    constexpr int kIt = kTile / kK3Threads;
    __shared__ int s_off[kMaxTileRows + 1];
    // BIN: the tile's kept edges wait in smem for the tile's one reservation (registers would
    // cost 12 per thread and make the 8-CTA launch spill); then thr[k] (i64), hist[k]
    extern __shared__ __align__(8) unsigned char k3_dyn[];
    int2* s_kp = reinterpret_cast<int2*>(k3_dyn);
    unsigned short* s_kb = reinterpret_cast<unsigned short*>(k3_dyn + (BIN ? 8 * kTile : 0));
    long long* s_thr = reinterpret_cast<long long*>(k3_dyn + (BIN ? 10 * kTile : 0));
    int* s_hist = reinterpret_cast<int*>(k3_dyn + (BIN ? 10 * kTile : 0) +
                                         8 * (size_t)(BIN ? bin.k : 0));
    __shared__ int s_wk[kK3Threads / 32];
    __shared__ int s_base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (BIN) {
        for (int i = threadIdx.x; i < bin.k; i += blockDim.x) {
            s_thr[i] = bin.thr[i];
            s_hist[i] = 0;
        }
    }
    int64_t tile_lo = 0, ntiles = num_tiles(m);
    int e_lo = 0, e_hi = (int)m, o_lo = 0, o_hi = (int)m;
    if (DIST) {
        e_lo = dist.cb[dist.rank];
        e_hi = dist.cb[dist.rank + 1];
        o_lo = dist.ob[dist.rank];
        o_hi = dist.ob[dist.rank + 1];
        tile_lo = e_lo / kTile;
        ntiles = num_tiles(e_hi);
    }
    for (int64_t tile = tile_lo + blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c0 = max((int)(tile * kTile), e_lo);
        const int c1 = (int)min((int64_t)tile * kTile + kTile, (int64_t)e_hi);
        const int r0 = trow[tile];
        const int nr = trow[tile + 1] - r0 + 1;  // rows touched by this tile
        const bool cached = nr <= kMaxTileRows;
        __syncthreads();
        if (cached)
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_off[i] = eoff[r0 + i];
        __syncthreads();
        unsigned kmask = 0;
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const int c = (int)(tile * kTile) + it * kK3Threads + threadIdx.x;
            int bnd = -1 - lane;  // unique dummy for lanes without a kept edge
            bool remote = false;
            int4 rrec;
            if (c >= c0 && c < c1) {
            const int ri = cached ? last_le(s_off, nr + 1, c) : last_le(eoff + r0, nr + 1, c);
            TWC_ASSERT(ri >= 0 && ri < nr);
            const int u = r0 + ri;
            const int eu = cached ? s_off[ri] : eoff[u];
            const int upu = (cached ? s_off[ri + 1] : eoff[u + 1]) - eu;
            const RP rb = rowptr[u];
            const int du = (int)(rowptr[u + 1] - rb);
            const RP p = rb + (RP)(du - upu) + (RP)(c - eu);  // upper slot of (u,v)
            const int v = __ldcs(colidx + p);
            // aligned iff the upper slot p is an out-slot; deg(v) was kept per slot by K1
            const int64_t wi = (int64_t)(p >> 5);
            const unsigned ow = obits[wi];
            int dv = __ldcs(dslot + p);
            if (dv == 0xffff) dv = deg[v];  // saturated: a vertex of degree >= 65535
            int sl;
            if ((ow >> (p & 31)) & 1u) {
                // aligned: oriented slot = #out-slots before p (word prefix + popc)
                sl = opre[wi] + __popc(ow & ((1u << (p & 31)) - 1u));
            } else {  // reversed edge: u's position in N+(v), one random 8-byte record first
                const int2 vi = vinfo[v];
                sl = sector_search(col_or, vi.x, vi.y, u, n);
            }
            TWC_ASSERT(sl >= 0 && (int64_t)sl < m);
            TWC_ASSERT(((ow >> (p & 31)) & 1u) || col_or[sl] == u);  // the reversed search found u
            if (DIST && (sl < o_lo || sl >= o_hi)) {  // counted by another rank: ask its owner
                remote = true;
                rrec = make_int4(c, u, v, sl);
            } else {
            const int tt = t_or[sl];
            if (K4) __stcs(k4 + c, (long long)k4_or[sl]);
            const int score = 3 * tt - du - dv + 2;
            __stcs(t + c, tt);
            __stcs(wedge + c, du + dv - 2 * tt - 2);
            __stcs(tw + c, score);
            if (BIN && (long long)score >= s_thr[bin.k - 1]) {  // kept at the smallest threshold
                bnd = band_of(score, s_thr, bin.k);
                s_kp[it * kK3Threads + threadIdx.x] = make_int2(u, v);
                s_kb[it * kK3Threads + threadIdx.x] = (unsigned short)bnd;
                kmask |= 1u << it;
            }
            }  // local edge
            }
            if (DIST) {  // warp-aggregated append of the remote edges
                const unsigned rb = __ballot_sync(FULL, remote);
                if (rb) {
                    int base = 0;
                    if (lane == __ffs(rb) - 1) base = atomicAdd(dist.nrec, __popc(rb));
                    base = __shfl_sync(FULL, base, __ffs(rb) - 1);
                    if (remote) dist.rec[base + __popc(rb & ((1u << lane) - 1u))] = rrec;
                }
            }
            if (BIN) {  // warp-aggregated band histogram: one smem atomic per distinct band
                const unsigned grp = __match_any_sync(FULL, bnd);
                if (bnd >= 0 && lane == __ffs(grp) - 1) atomicAdd(&s_hist[bnd], __popc(grp));
            }
        }
        if (BIN) {  // append this tile's kept edges with one reservation per tile
            const int nk = __popc(kmask);
            const int incl = warp_incl_scan(nk, lane);
            if (lane == 31) s_wk[wid] = incl;
            __syncthreads();
            int wpre = 0, tot = 0;
#pragma unroll
            for (int i = 0; i < kK3Threads / 32; ++i) {
                const int x = s_wk[i];
                wpre += (i < wid) ? x : 0;
                tot += x;
            }
            if (threadIdx.x == 0) s_base = tot ? atomicAdd(bin.nkept, tot) : 0;
            __syncthreads();
            int pos = s_base + wpre + incl - nk;
            TWC_ASSERT(pos + nk <= m);
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                if ((kmask >> it) & 1u) {
                    bin.kept[pos] = s_kp[it * kK3Threads + threadIdx.x];
                    bin.kband[pos] = s_kb[it * kK3Threads + threadIdx.x];
                    ++pos;
                }
            }
        }
    }
    if (BIN) {
        __syncthreads();
        for (int i = threadIdx.x; i < bin.k; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&bin.cnt[i], s_hist[i]);
    }
}

// ------------------------------------------------------------------------ host side
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

// A per-thread, per-device side stream with a fork and a join event (created on first use and
// kept for the life of the process); NULL if it cannot be created (then everything runs on the
// caller's stream).
struct AuxStream {
    int dev = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, begin = nullptr, zeroed = nullptr;
};

static AuxStream* aux_stream() {
    static thread_local std::vector<AuxStream> lanes;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    for (auto& x : lanes)
        if (x.dev == dev) return &x;
    AuxStream a;
    a.dev = dev;
    if (cudaStreamCreateWithFlags(&a.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.begin, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.zeroed, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    lanes.push_back(a);
    return &lanes.back();
}

// Distributed step (twc_dist.cu): the row partition of all `world` ranks, split at
// equal oriented-slot counts: rows[r] = first u with rp_or[u] >= r m / world (rows[0] = 0,
// rows[world] = n); the rank's oriented slice is [rp_or[rows[r]], rp_or[rows[r+1]]) and its
// canonical slice [eoff[rows[r]], eoff[rows[r+1]]).  bounds = {rows, ob, cb}, world + 1 each.
// Also sets this rank's K2 pivot range and points the pivot queue at it.
__global__ void k_dist_bounds(int64_t n, int64_t m, const int* __restrict__ rp_or,
                              const int* __restrict__ eoff, int rank, int world,
                              int* __restrict__ bounds, int* __restrict__ range,
                              int* __restrict__ work) {
    const int r = threadIdx.x;
    if (r > world) return;
    int u;
    if (r == 0) {
        u = 0;
    } else if (r == world) {
        u = (int)n;
    } else {
        const int64_t target = m * r / world;
        int64_t lo = 0, hi = n;  // first u in [0, n] with rp_or[u] >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)rp_or[mid] < target) lo = mid + 1; else hi = mid;
        }
        u = (int)lo;
    }
    bounds[r] = u;
    bounds[world + 1 + r] = rp_or[u];
    bounds[2 * (world + 1) + r] = eoff[u];
    if (r == rank) {
        range[0] = u;
        work[0] = u;
    }
    if (r == rank + 1) range[1] = u;
}

// K2 launch configuration: 8,192-bit filters, a 128-entry candidate ring, 5 CTAs per SM (the
// measured optimum; the filter / ring / group-cap / occupancy variants were
// A/B-tested in round 2 and lost).
constexpr int kK2FilterLog = 13;
#ifndef TWC_K2_MINB
#define TWC_K2_MINB 5
#endif
#ifndef TWC_K2_RING
#define TWC_K2_RING kRing
#endif
constexpr int kK2MinBlocks = TWC_K2_MINB;
#ifndef TWC_K2_SPL
#define TWC_K2_SPL 1
#endif
#define K2_KERNEL k2_intersect<kOct, kK2FilterLog, kK2MinBlocks, TWC_K2_RING, TWC_K2_SPL>
using K2Smem = K2WarpSmem<kK2FilterLog, TWC_K2_RING, TWC_K2_SPL>;


// Stage A: degrees, orientation + oriented CSR (K0, K1) and the intersection (K2h, K2) of all
// pivots, or of a shard's pivot range.  Events [0] start, [1] orientation done, [2] K2 done.
template <typename RP>
static bool stage_orient_intersect(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                                   const ScoreWs& w, cudaStream_t s, cudaEvent_t* ev,
                                   const ShardSpec* shard, int* parent = nullptr) {
    const int sms = num_sms();
    const int64_t m2 = 2 * m;
    const int64_t nst = (m2 + kSlotTile - 1) / kSlotTile;
    bool win = false;
    record(ev, 0, s);
    // the oriented counts and the queue counters are zeroed on the library's side stream while K1
    // runs (K1 is bound by its deg gathers, not by DRAM; the 4m-byte memset took 25 us between K1
    // and K2); K2h follows on that stream, K2 waits for `zeroed`
    AuxStream* ax = aux_stream();
    cudaStream_t sh = ax ? ax->stream : s;
    if (ax) {
        cudaEventRecord(ax->begin, s);
        cudaStreamWaitEvent(sh, ax->begin, 0);
        cudaMemsetAsync(w.t_or, 0, sizeof(int) * (size_t)m, sh);
        cudaEventRecord(ax->zeroed, sh);
    }
    // a1 + a2: degrees, orientation, oriented CSR (bits + tile counts, tile scan, scatter, rows)
    k0_degrees<RP><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rowptr, w.deg, parent);
    count_launches(1);
    tile_rows<RP>(rowptr, (int)n, m2, kSlotTile, w.ftrow, s);
    {
        const int grid = grid_for(nst, 1, sms * 8);
        k1_bits<RP><<<grid, kSlotThreads, 0, s>>>(m2, rowptr, colidx, w.deg, w.ftrow, w.obits,
                                                 w.ubits, w.tile_out, w.tile_up, w.dslot);
        k1_tile_scan<<<1, 1024, 0, s>>>(nst, w.tile_out, w.tile_up);
        k1_write<<<grid, kSlotThreads, 0, s>>>(m2, colidx, w.obits, w.ubits, w.tile_out,
                                               w.tile_up, w.opre, w.upre, w.col_or);
        // vinfo (written here, gathered by K2 and K3) stays in the persisting part of L2 until the
        // caller ends the window after K3 (twc_api.cu l2_window_begin; large graphs only)
        win = l2_window_begin(s, w.vinfo, sizeof(int2) * (size_t)n, 2 * sizeof(int) * (size_t)m);
        k1_rows<RP><<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(n, m, rowptr, w.obits, w.ubits,
                                                                   w.opre, w.upre, w.rp_or, w.eoff,
                                                                   w.vinfo);
        count_launches(4);
    }
    tile_first_rows(w.eoff, (int)n, m, w.trow, s);
    // (zeroing t_or inside K1b's scatter was measured: k1_write 0.10 -> 0.29 ms; the memset is
    // a 140 MB streaming write, ~25 us)
    if (!ax) cudaMemsetAsync(w.t_or, 0, sizeof(int) * (size_t)m, s);
    cudaMemsetAsync(w.work, 0, 2 * sizeof(int), s);
    cudaMemsetAsync(w.nhubs, 0, sizeof(int), s);
    const int* range = nullptr;  // a shard counts only the triangles of its pivot range
    if (shard) {
        k_dist_bounds<<<1, 64 * ((shard->world + 64) / 64), 0, s>>>(
            n, m, w.rp_or, w.eoff, shard->rank, shard->world, shard->bounds, w.range, w.work);
        count_launches(1);
        range = w.range;
    }
    // a3: oriented intersection
    const size_t smem = kK2Warps * sizeof(K2Smem);
    const int occ = kernel_setup((const void*)K2_KERNEL, kK2Warps * 32, smem);
    record(ev, 1, s);
    // hub pivots (|N+(u)| > kGroupSlots, one per CTA) run on a library-owned side stream,
    // forked from and joined back to s: they start first (the largest tasks) and the
    // persistent K2 grid fills the SM resources they leave, so neither kernel's tail idles
    // the GPU.  No work and an early exit when the graph has no hub.
    if (ax) {
        cudaEventRecord(ax->fork, s);
        cudaStreamWaitEvent(sh, ax->fork, 0);
        cudaStreamWaitEvent(s, ax->zeroed, 0);
    }
    k2_find_hubs<<<(unsigned)((n + 255) / 256), 256, 0, sh>>>(n, w.rp_or, w.hubs, w.nhubs, range);
    const size_t hsmem = sizeof(K2HubSmem);
    kernel_setup((const void*)k2_hubs, kK2Warps * 32, hsmem);
    k2_hubs<<<sms * kHubMinBlocks, kK2Warps * 32, hsmem, sh>>>(w.rp_or, w.col_or, w.hubs, w.nhubs,
                                                    w.work + 1, w.t_or);
    if (ax) cudaEventRecord(ax->join, sh);
    // pivots per queue grab: kPivotChunk, fewer when there are too few pivots to give every
    // warp several grabs (small dense graphs), so the queue still balances the load
    const int64_t warps = (int64_t)sms * occ * kK2Warps;
    const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(kPivotChunk, n / (8 * warps)));
    K2_KERNEL<<<sms * occ, kK2Warps * 32, smem, s>>>(n, chunk, w.rp_or, w.col_or, w.t_or, w.work,
                                                     range, w.vinfo);
    if (ax) cudaStreamWaitEvent(s, ax->join, 0);
    count_launches(3);
    record(ev, 2, s);
    return win;  // an L2 window on vinfo is open on s: the caller ends it
}

template <typename RP>
cudaError_t score_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                       size_t ws_bytes, int* t, int* wedge, int* tw, cudaStream_t s,
                       cudaEvent_t* ev, const BinSpec* bin, long long* k4) {
    if (m == 0 || n == 0) return cudaGetLastError();
    Carver cv(ws, ws_bytes);
    ScoreWs w = carve_score(cv, n, m);
    const int sms = num_sms();
    const bool win = stage_orient_intersect<RP>(n, m, rowptr, colidx, w, s, ev, nullptr,
                                                bin ? bin->parent : nullptr);
    // NEXT(4): K4 participation on the same oriented CSR (workspace after the score's)
    unsigned long long* k4_or = nullptr;
    if (k4) {
        const size_t used = score_ws_bytes(n, m);
        cudaError_t e = k4_count(n, m, w.rp_or, w.col_or, static_cast<char*>(ws) + used,
                                 ws_bytes - used, &k4_or, s);
        if (e != cudaSuccess) {
            if (win) l2_window_end(s);
            return e;
        }
    }
    // a4: canonical gather + wedge + TW
    {
        const int64_t nt = num_tiles(m);
        const int grid = grid_for(nt, 1, sms * 8);
        if (k4)
            k3_score<RP, false, true><<<grid, kK3Threads, 0, s>>>(
                n, m, rowptr, colidx, w.vinfo, w.dslot, w.deg, w.eoff, w.trow, w.col_or, w.opre,
                w.obits, w.t_or, t, wedge, tw, BinSpec{}, k4_or, k4);
        else if (bin)
            k3_score<RP, true><<<grid, kK3Threads, k3_bin_smem(bin->k), s>>>(
                n, m, rowptr, colidx, w.vinfo, w.dslot, w.deg, w.eoff, w.trow, w.col_or, w.opre, w.obits, w.t_or, t,
                wedge, tw, *bin);
        else
            k3_score<RP, false><<<grid, kK3Threads, 0, s>>>(
                n, m, rowptr, colidx, w.vinfo, w.dslot, w.deg, w.eoff, w.trow, w.col_or, w.opre, w.obits, w.t_or, t,
                wedge, tw, BinSpec{});
        count_launches(1);
        if (win) l2_window_end(s);
        record(ev, 3, s);
    }
    return cudaGetLastError();
}

template <typename RP>
cudaError_t dist_stage_a(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                         size_t ws_bytes, int rank, int world, int* bounds, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    ScoreWs w = carve_score(cv, n, m);
    const ShardSpec sh{rank, world, bounds};
    if (stage_orient_intersect<RP>(n, m, rowptr, colidx, w, s, nullptr, &sh)) l2_window_end(s);
    return cudaGetLastError();
}

template <typename RP>
cudaError_t dist_epilogue(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                          size_t ws_bytes, int* t, int* wedge, int* tw, const BinSpec& bin,
                          const DistK3& d, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    ScoreWs w = carve_score(cv, n, m);
    const int grid = grid_for(num_tiles(m), 1, num_sms() * 8);
    const bool win =
        l2_window_begin(s, w.vinfo, sizeof(int2) * (size_t)n, 2 * sizeof(int) * (size_t)m);
    k3_score<RP, true, false, true><<<grid, kK3Threads, k3_bin_smem(bin.k), s>>>(
        n, m, rowptr, colidx, w.vinfo, w.dslot, w.deg, w.eoff, w.trow, w.col_or, w.opre, w.obits,
        w.t_or, t, wedge, tw, bin, nullptr, nullptr, d);
    if (win) l2_window_end(s);
    count_launches(1);
    return cudaGetLastError();
}

#define TWC_INST(RP)                                                                            \
    template cudaError_t score_impl<RP>(int64_t, int64_t, const RP*, const int*, void*, size_t,  \
                                        int*, int*, int*, cudaStream_t, cudaEvent_t*,            \
                                        const BinSpec*, long long*);                             \
    template cudaError_t dist_stage_a<RP>(int64_t, int64_t, const RP*, const int*, void*, size_t, \
                                          int, int, int*, cudaStream_t);                        \
    template cudaError_t dist_epilogue<RP>(int64_t, int64_t, const RP*, const int*, void*,       \
                                           size_t, int*, int*, int*, const BinSpec&,             \
                                           const DistK3&, cudaStream_t);
TWC_INST(int)
TWC_INST(long long)
#undef TWC_INST

}  // namespace twc
