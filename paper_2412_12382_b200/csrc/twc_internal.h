// twc_internal.h -- host-side launchers shared between the translation units of libtwc.so.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace twc {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Bump allocator over a caller-provided workspace (the library never allocates).
struct Carver {
    char* base;
    size_t cap, used = 0;
    Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
    template <typename T>
    T* take(size_t count) {
        size_t bytes = align_up(count * sizeof(T) + 1);
        T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
        used += bytes;
        return p;
    }
    bool ok() const { return used <= cap; }
};

int num_sms();

// Launch set-up of a kernel with dynamic shared memory (K2, K2h, K4 groups; K2h needs more
// than 48 KB): sets cudaFuncAttributeMaxDynamicSharedMemorySize on the CURRENT device (the
// attribute is per device) once per (device, kernel, smem) and returns the resident blocks per
// SM (>= 1).  Thread-safe; the cache is the library's only process-wide state besides the
// launch counter and the per-thread error string.
int kernel_setup(const void* fn, int threads, size_t smem);
// persisting-L2 access-policy window on stream s for [ptr, ptr + bytes), used when the call
// streams more than the L2 holds (twc_api.cu); begin returns whether a window was set, and only
// then must end be called
bool l2_window_begin(cudaStream_t s, const void* ptr, size_t bytes, size_t streamed_bytes);
void l2_window_end(cudaStream_t s);

// Launch accounting (twc_kernel_launches) and optional phase events (twc_*_ex).
void count_launches(int k);
inline void record(cudaEvent_t* ev, int i, cudaStream_t s) {
    if (ev && ev[i]) cudaEventRecord(ev[i], s);
}

// ---- scan (twc_scan.cu): out[0] = 0, out[i+1] = in[0] + ... + in[i], for i < len ----------
size_t scan_temp_bytes(int64_t len);
void exclusive_scan(const int* in, int* out, int64_t len, int* temp, cudaStream_t s);

// ---- row tiling (twc_scan.cu): trow[i] = row holding item i*tile of offsets off[0..nrows] ---
constexpr int kTile = 1024;  // canonical edges per tile in the edge-parallel kernels
__host__ __device__ inline int64_t num_tiles(int64_t total) { return (total + kTile - 1) / kTile; }
void tile_first_rows(const int* off, int nrows, int64_t total, int* trow, cudaStream_t s);
// generic: trow[i] = row holding item i*tile of off[0..nrows] (OT = int or long long)
template <typename OT>
void tile_rows(const OT* off, int nrows, int64_t total, int tile, int* trow, cudaStream_t s);

// ---- canonical edge offsets (twc_scan.cu) ---------------------------------------------------
// up[u] = #{v in N(u): v > u};  eoff = exclusive scan of up  (S:66-69 canonical order)
template <typename RP>
void upper_counts(int64_t n, const RP* rowptr, const int* colidx, int* up, cudaStream_t s);

// ---- sweep building blocks (twc_cluster.cu) --------------------------------------------------
constexpr int kMaxK = 1024;  // thresholds per sweep
struct SweepPlan {           // thresholds sorted descending (fewest kept edges first)
    int k;
    int order[kMaxK];        // caller index of the i-th threshold
    long long thr[kMaxK];    // keep iff TW >= thr[i] (fp64 sweeps: the double's bit pattern)
    bool fresh[kMaxK];       // thr[i] differs from thr[i-1] (step i has its own band)
};
void sweep_plan(const long long* thr, int k, SweepPlan* P);
void sweep_plan_f64(const double* thr, int k, SweepPlan* P);
void sweep_upload(const SweepPlan& P, long long* thr_dev, int* order_dev, cudaStream_t s);
void band_offsets(const int* cnt, int k, const int* order_dev, int* off, int* cursor,
                  unsigned long long* stats, cudaStream_t s);
void band_place(const int2* kept, const unsigned short* kband, const int* nkept, int64_t cap,
                int k, int* cursor, int2* pairs, cudaStream_t s);
// step_ev: NULL or k events, step_ev[i] recorded once the labels of threshold order[i] are final
void sweep_loop(int64_t n, int64_t m, const SweepPlan& P, const int2* pairs, const int* off,
                int* parent, int* labels, unsigned long long* stats, cudaStream_t s,
                cudaEvent_t* step_ev = nullptr);
void init_parent(int64_t n, int* parent, cudaStream_t s);

// ---- score (twc_score.cu) ------------------------------------------------------------------
// Optional binning of kept edges by sweep step, fused into the score epilogue (K3).
struct BinSpec {
    const long long* thr;   // device, sorted descending, k entries
    int k;
    int* cnt;               // device [k] band histogram (zeroed by the caller)
    int* nkept;             // device counter (zeroed by the caller)
    int2* kept;             // device [m] (u, v) of kept edges, in no particular order
    unsigned short* kband;  // device [m] band of kept[i]
    int* parent = nullptr;  // device [n] or NULL: union-find parents, initialised by K0 (parent[u] = u)
};
size_t score_ws_bytes(int64_t n, int64_t m);

// Epilogue of one rank of the distributed step (twc_dist.cu).
struct DistK3 {
    const int* cb = nullptr;  // device [world+1] canonical slice bounds
    const int* ob = nullptr;  // device [world+1] oriented slice bounds
    int rank = 0;
    int4* rec = nullptr;      // device: remote edges {c, u, v, oriented slot}
    int* nrec = nullptr;      // device counter
};

// The score workspace layout (shared with the distributed phases, twc_dist.cu, which keep the
// oriented CSR and counts alive between their calls).
constexpr int kSlotTile = 2048;  // K1 CSR-slot tile
struct ScoreWs {
    int *deg, *eoff, *rp_or, *trow, *ftrow, *tile_out, *tile_up, *opre, *upre;
    unsigned *obits, *ubits;
    int2* vinfo;
    unsigned short* dslot;
    int *col_or, *t_or, *work, *hubs, *nhubs, *range;
};
inline ScoreWs carve_score(Carver& cv, int64_t n, int64_t m) {
    ScoreWs w;
    const int64_t nst = (2 * m + kSlotTile - 1) / kSlotTile;
    const int64_t nw = (2 * m + 31) / 32;
    w.deg = cv.take<int>(n);
    w.eoff = cv.take<int>(n + 1);
    w.rp_or = cv.take<int>(n + 1);
    w.trow = cv.take<int>(num_tiles(m) + 1);
    w.ftrow = cv.take<int>(nst + 1);
    w.tile_out = cv.take<int>(nst);
    w.tile_up = cv.take<int>(nst);
    w.obits = cv.take<unsigned>(nw);
    w.ubits = cv.take<unsigned>(nw);
    w.opre = cv.take<int>(nw);
    w.upre = cv.take<int>(nw);
    w.col_or = cv.take<int>(m);
    w.t_or = cv.take<int>(m);
    w.vinfo = cv.take<int2>(n);
    w.dslot = cv.take<unsigned short>(2 * m);
    w.work = cv.take<int>(2);  // [0] K2 pivot queue, [1] K2h hub queue
    w.hubs = cv.take<int>(n);
    w.nhubs = cv.take<int>(1);
    w.range = cv.take<int>(2);
    return w;
}
// k4: NULL, or device int64[m] that receives the K4 participation of every canonical edge
// (then ws must also hold k4_ws_bytes(n, m) after the score workspace)
// shard (the distributed step, twc_dist.cu): count only the triangles whose pivot (lowest-key
// vertex) lies in the rank's row range; bounds: device [3 (world + 1)] row /
// oriented / canonical slice bounds of every rank (k_dist_bounds)
struct ShardSpec {
    int rank, world;
    int* bounds;
};
template <typename RP>
cudaError_t score_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                       size_t ws_bytes, int* t, int* wedge, int* tw, cudaStream_t s,
                       cudaEvent_t* ev = nullptr, const BinSpec* bin = nullptr,
                       long long* k4 = nullptr);
// Distributed step (twc_dist.cu): stage A = K0, K1 and K2 over this rank's pivot rows (bounds of
// all ranks written to `bounds`); the epilogue = K3 over the rank's canonical slice (DIST mode).
template <typename RP>
cudaError_t dist_stage_a(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                         size_t ws_bytes, int rank, int world, int* bounds, cudaStream_t s);
template <typename RP>
cudaError_t dist_epilogue(int64_t n, int64_t m, const RP* rowptr, const int* colidx, void* ws,
                          size_t ws_bytes, int* t, int* wedge, int* tw, const BinSpec& bin,
                          const DistK3& d, cudaStream_t s);
// ---- distributed step (twc_dist.cu) ------------------------------------------------------------
size_t dist_ws_bytes(int64_t n, int64_t m, int world);
template <typename RP>
cudaError_t dist_count_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, int rank,
                            int world, void* ws, size_t ws_bytes, int* send,
                            long long* send_sizes, cudaStream_t s);
cudaError_t dist_apply_impl(int64_t n, int64_t m, int world, void* ws, size_t ws_bytes,
                            const int* recv, int64_t nrecv, cudaStream_t s);
template <typename RP>
cudaError_t dist_epilogue_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                               int rank, int world, const long long* thr, int k, void* ws,
                               size_t ws_bytes, int* t, int* wedge, int* tw, int* req,
                               long long* req_sizes, cudaStream_t s);
cudaError_t dist_serve_impl(int64_t n, int64_t m, int world, void* ws, size_t ws_bytes,
                            const int* req, int64_t nreq, int* reply, cudaStream_t s);
cudaError_t dist_forest_impl(int64_t n, int64_t m, int world, const long long* thr, int k,
                             void* ws, size_t ws_bytes, const int* reply, int* t, int* wedge,
                             int* tw, int* forest, long long* forest_cum, long long* kept_sizes,
                             long long* nforest, cudaStream_t s);
cudaError_t dist_sweep_impl(int64_t n, int64_t m, int world, const long long* thr, int k,
                            void* ws, size_t ws_bytes, const int* forests, int64_t cap,
                            const long long* fcum_all, const long long* kept_all, int* labels,
                            long long* stats, cudaStream_t s);

// ---- K4 participation (twc_k4.cu) -----------------------------------------------------------
int k4_big_warps();
size_t k4_ws_bytes(int64_t n, int64_t m);
// counts per oriented slot (64-bit) into a buffer carved from ws; *k4_or_out points at it
cudaError_t k4_count(int64_t n, int64_t m, const int* rp_or, const int* col_or, void* ws,
                     size_t ws_bytes, unsigned long long** k4_or_out, cudaStream_t s);

// ---- cluster (twc_cluster.cu) --------------------------------------------------------------
size_t cluster_ws_bytes(int64_t n, int64_t m);
size_t score_sweep_ws_bytes(int64_t n, int64_t m);
template <typename RP>
cudaError_t score_sweep_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                             const long long* thr, int k, void* ws, size_t ws_bytes, int* t,
                             int* wedge, int* tw, int* labels, long long* stats, cudaStream_t s,
                             cudaEvent_t* ev, cudaEvent_t* step_ev = nullptr);
// thresholds already converted to integer "keep iff tw >= thr[i]" form, any order.
template <typename RP>
cudaError_t sweep_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx, const int* tw,
                       const long long* thr, int k, void* ws, size_t ws_bytes, int* labels,
                       long long* stats, cudaStream_t s, cudaEvent_t* ev = nullptr);

// ---- real-valued scores (twc_similarity.cu / twc_cluster.cu) --------------------------------
template <typename RP>
cudaError_t similarity_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                            const int* t, int kind, void* ws, size_t ws_bytes, double* out,
                            cudaStream_t s);
template <typename RP>
cudaError_t sweep_f64_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                           const double* score, const double* deltas, int k, void* ws,
                           size_t ws_bytes, int* labels, long long* stats, cudaStream_t s);

// ---- partition statistics (twc_stats.cu) ---------------------------------------------------
size_t partition_stats_ws_bytes(int64_t n, int64_t m);
// counts: device int64[4k]; q: device double[k] or NULL; *bad_host = 1 if a label is outside
// [0, n).  Synchronises the stream.
template <typename RP>
cudaError_t partition_stats_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                                 const int* labels, int k, void* ws, size_t ws_bytes,
                                 long long* counts, double* q, int* bad_host, cudaStream_t s);

// ---- validation (twc_cluster.cu) -----------------------------------------------------------
template <typename RP>
cudaError_t validate_impl(int64_t n, int64_t m, const RP* rowptr, const int* colidx,
                          int* verdict, cudaStream_t s);

}  // namespace twc
