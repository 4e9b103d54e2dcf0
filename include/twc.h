/*
 * twc.h -- C ABI of the B200 triangle/wedge (TW) edge-scoring and motif-based clustering path
 * (arXiv 2412.12382, Chen & Tsourakakis).  Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md
 * line n, "SURVEY x" = SURVEY.md section.  Implemented by libtwc.so
 * (paper_2412_12382_b200/csrc/); sm_100a only.
 *
 * Conventions shared by every call
 * --------------------------------
 *  Graph.   twc_csr describes an undirected simple graph in CSR form with DEVICE pointers
 *           (for the *_host calls, HOST pointers): rowptr has n+1 entries of rowptr_bytes
 *           (4 = int32, 8 = int64) bytes with rowptr[0] = 0 and rowptr[n] = 2m; colidx has 2m
 *           int32 entries; every row is strictly increasing, the graph is symmetric and has
 *           no self-loops (the paper's pre-processing "sort the adjacency list by node id",
 *           P:618).  Limits: 0 <= n < 2^31, 0 <= m < 2^31.  The precondition is NOT
 *           checked by the scoring calls (the wedge closed form assumes it); twc_validate_csr
 *           checks it.
 *  Edges.   Per-edge outputs are indexed by the canonical edge id: the edges (u,v), u<v, in
 *           lexicographic order (reading C5), i.e. the upper
 *           triangle of the CSR in row order.
 *  Memory.  Every array is caller-owned.  The library never allocates device memory: all
 *           scratch comes from a caller-provided device workspace whose size is given by the
 *           matching *_workspace_bytes query (cuBLAS style).  Workspaces must be 256-byte
 *           aligned.  DEVICE colidx must be 16-byte aligned and DEVICE rowptr aligned to
 *           rowptr_bytes (the kernels read colidx with 16-byte vector loads; a view with an odd
 *           storage offset, e.g. colidx[2:], is rejected with TWC_EINVAL rather than faulting).
 *           HOST pointers of the *_host calls have no alignment requirement.
 *           Nothing is retained after a call returns; outputs must not alias inputs.
 *  Streams. `stream` is a cudaStream_t (NULL = legacy default stream).  Device calls only
 *           enqueue work on it and return without synchronising (outputs are valid once the
 *           stream reaches them), except twc_validate_csr and the *_host calls, which
 *           synchronise the stream before returning.  The scoring calls may fork part of
 *           their work (the hub-pivot intersection) onto a library-owned side stream of the
 *           calling thread and join it back to `stream` with events before they return, so
 *           stream order, event timing and CUDA-graph capture of `stream` see one call as one
 *           unit; the *_host_async calls copy results back on a library-owned copy stream the
 *           same way.
 *  Errors.  Calls return a twc_status.  TWC_EINVAL: a null pointer where data is required
 *           (n > 0 or m > 0), n or m out of range, rowptr_bytes not in {4, 8}, a misaligned
 *           device colidx / rowptr, NaN delta, k < 1.  TWC_EWORKSPACE: workspace too small or misaligned.  TWC_ECUDA: a CUDA launch
 *           or runtime error (detail in twc_last_error()).  TWC_EGRAPH: only from
 *           twc_validate_csr.  Outputs are undefined on error; nothing aborts or throws.
 *           n = 0 or m = 0 is not an error: empty score arrays; labels[u] = u.
 *  Threads. Calls are re-entrant and may target any device (the current one).  Process-wide
 *           state is limited to: the thread-local error string returned by twc_last_error(),
 *           the launch counter of twc_kernel_launches(), per-(thread, device) side/copy streams
 *           and events created on first use, and a mutex-guarded per-(device, kernel) cache of
 *           the dynamic-shared-memory attribute and occupancy (the attribute is per device).
 *  L2.      The first scoring call on a device whose graph's oriented arrays (8m bytes) exceed
 *           the L2 sets that device's persisting-L2 set-aside to 32 MiB
 *           (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize); environment TWC_L2_PERSIST_MB
 *           overrides the size, 0 = never).  Such calls put an access-policy window on `stream`
 *           around their intersection and epilogue kernels (the per-vertex record array the
 *           kernels gather from stays in L2) and clear the stream's window before they return,
 *           so a window the caller had set on `stream` is not preserved.  A later call on a small
 *           graph resets the persisting lines (cudaCtxResetPersistingL2Cache).  These are cache
 *           hints only: results never depend on them, and a device without the feature, or a
 *           first call made during stream capture, simply runs without the window.
 */
#ifndef TWC_H_
#define TWC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TWC_OK = 0,
    TWC_EINVAL = 1,
    TWC_EWORKSPACE = 2,
    TWC_ECUDA = 3,
    TWC_EGRAPH = 4
} twc_status;

typedef struct {
    int64_t n;             /* vertices, 0 <= n < 2^31                                        */
    int64_t m;             /* undirected edges; rowptr[n] == 2m, 0 <= m < 2^31              */
    const void *rowptr;    /* n+1 entries of rowptr_bytes each                               */
    int32_t rowptr_bytes;  /* 4 (int32) or 8 (int64)                                          */
    const int32_t *colidx; /* 2m entries                                                      */
} twc_csr;

/* ---------------------------------------------------------------------------------------
 * twc_score -- per-edge triangle count, wedge count and TW score.
 *
 *   t[e]     = |N(u) & N(v)|                                  ("Notations")
 *   wedge[e] = |N(u) | N(v)| - |N(u) & N(v)| - 2
 *   tw[e]    = t[e] - wedge[e]                                (Eq. 2)
 * for every canonical edge e = (u,v).  t, wedge, tw: device int32[m] each, written in full.
 * Exact integers (no rounding).  Needs a workspace of twc_score_workspace_bytes(n, m, rb).
 * ------------------------------------------------------------------------------------- */
size_t twc_score_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes);
twc_status twc_score(const twc_csr *g, void *workspace, size_t workspace_bytes,
                     int32_t *t, int32_t *wedge, int32_t *tw, void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_cluster -- Alg. 1 for one threshold on precomputed scores.
 *
 * Removes every edge e with tw[e] < delta (equality is kept, reading C4;
 * the comparison (double)tw[e] < delta is exact) and labels the connected components of the
 * remaining graph: labels[u] = the minimum vertex id of u's component (S:208-210,
 * S:228; isolated vertices are singletons).  delta may be +-infinity, not NaN.
 *   tw:     device int32[m], canonical order (e.g. from twc_score).
 *   labels: device int32[n], written in full.
 *   stats:  device int64[2] = {kept_edges, n_components}, or NULL.
 * Needs a workspace of twc_cluster_workspace_bytes(n, m, rb).
 * ------------------------------------------------------------------------------------- */
size_t twc_cluster_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes);
twc_status twc_cluster(const twc_csr *g, const int32_t *tw, double delta, void *workspace,
                       size_t workspace_bytes, int32_t *labels, int64_t *stats, void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_sweep -- twc_cluster for k thresholds reusing one score array (
 * S:384 "computed once per sweep ... T cheap CC passes").  Results equal k independent
 * twc_cluster calls.  deltas_host: HOST double[k] (any order, no NaN).  labels: device
 * int32[k*n], labels[i*n + u] for deltas_host[i].  stats: device int64[2k] or NULL.
 * Same workspace size as twc_cluster.
 * ------------------------------------------------------------------------------------- */
twc_status twc_sweep(const twc_csr *g, const int32_t *tw, const double *deltas_host, int32_t k,
                     void *workspace, size_t workspace_bytes, int32_t *labels, int64_t *stats,
                     void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_score_sweep -- twc_score followed by twc_sweep in one call (the fused device path).
 * The score epilogue also bins every edge kept at the smallest threshold by sweep step, so
 * the sweep makes no further pass over TW or the CSR.  Outputs are identical to twc_score +
 * twc_sweep (t, wedge, tw: device int32[m]; labels: device int32[k*n]; stats: device
 * int64[2k] or NULL).  deltas_host: HOST double[k], 1 <= k <= 1024, any order, no NaN.
 * `events`: NULL or 6 cudaEvent_t recorded at [0] start, [1] orientation done, [2]
 * intersection done, [3] epilogue + binning done, [4] bands placed, [5] all labelled.
 * Workspace: twc_score_sweep_workspace_bytes(n, m, rb).
 * ------------------------------------------------------------------------------------- */
size_t twc_score_sweep_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes);
twc_status twc_score_sweep(const twc_csr *g, const double *deltas_host, int32_t k,
                           void *workspace, size_t workspace_bytes, int32_t *t, int32_t *wedge,
                           int32_t *tw, int32_t *labels, int64_t *stats, void *stream,
                           void *const *events);

/* ---------------------------------------------------------------------------------------
 * twc_pipeline_host -- the whole path end to end from HOST buffers: copies the CSR to the
 * device, runs twc_score_sweep over deltas_host[k], copies the results back and
 * synchronises the stream.  g points at HOST rowptr/colidx (pinned memory gives full PCIe
 * speed; pageable works).  t, wedge, tw: HOST int32[m] each, or NULL to skip that copy-back.
 * labels: HOST int32[k*n] or NULL.  stats: HOST int64[2k] or NULL.  Needs a DEVICE workspace
 * of twc_pipeline_workspace_bytes(n, m, rb, k) (holds the device copies too).
 * The copies back run on a library-owned second stream as soon as each result is final (the
 * scores after the epilogue, each threshold's labels after its sweep step), overlapping the
 * remaining device work; `stream` is made to wait for them.
 *
 * twc_pipeline_host_async -- the same without the final synchronisation: all work, including
 * the copies back, is ordered before anything later enqueued on `stream`.  The host outputs are
 * valid, and the host inputs, host outputs and workspace may be reused, only once `stream` has
 * completed.  Two calls on two streams with two workspaces overlap one graph's copies back with
 * the next graph's copy in and compute (PCIe is full duplex).
 * ------------------------------------------------------------------------------------- */
size_t twc_pipeline_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes, int32_t k);
twc_status twc_pipeline_host(const twc_csr *g_host, const double *deltas_host, int32_t k,
                             void *workspace, size_t workspace_bytes, int32_t *t, int32_t *wedge,
                             int32_t *tw, int32_t *labels, int64_t *stats, void *stream);
twc_status twc_pipeline_host_async(const twc_csr *g_host, const double *deltas_host, int32_t k,
                                   void *workspace, size_t workspace_bytes, int32_t *t,
                                   int32_t *wedge, int32_t *tw, int32_t *labels, int64_t *stats,
                                   void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_similarity -- the other edge similarities of Table 1 from the triangle
 * counts, as IEEE doubles in canonical edge order (one correctly rounded operation each):
 *   TWC_SIM_TW        t - wedge = 3t - d_u - d_v + 2      (Eq. 2)
 *   TWC_SIM_TECTONIC  t / (d_u + d_v)
 *   TWC_SIM_JACCARD   t / (d_u + d_v - t)
 *   TWC_SIM_K3        t
 *   TWC_SIM_EFFRES    -2 / (2 + t)   (the effective-resistance upper bound 2/(2+t) of P:450,
 *                                     negated like Table 1's -R_eff)
 * t: device int32[m] (from twc_score); score: device double[m].  Workspace:
 * twc_cluster_workspace_bytes(n, m, rb).  Unknown kind: TWC_EINVAL.
 * twc_sweep_f64 -- twc_sweep on real-valued scores: keeps e iff NOT (score[e] < delta);
 * same outputs and workspace as twc_sweep.
 * ------------------------------------------------------------------------------------- */
typedef enum {
    TWC_SIM_TW = 0,
    TWC_SIM_TECTONIC = 1,
    TWC_SIM_JACCARD = 2,
    TWC_SIM_K3 = 3,
    TWC_SIM_EFFRES = 4
} twc_sim_kind;
twc_status twc_similarity(const twc_csr *g, const int32_t *t, int32_t kind, void *workspace,
                          size_t workspace_bytes, double *score, void *stream);
twc_status twc_sweep_f64(const twc_csr *g, const double *score, const double *deltas_host,
                         int32_t k, void *workspace, size_t workspace_bytes, int32_t *labels,
                         int64_t *stats, void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_score_k4 -- twc_score plus the kappa-clique participation for kappa = 4 (Table 1,
 * P:417; "we only consider K_4"): k4[e] = number of 4-cliques containing the
 * canonical edge e = number of adjacent pairs {w, x} of common neighbours of its endpoints
 * (SURVEY 8(f) NEXT(4)).  t, wedge, tw: device int32[m] as twc_score; k4: device int64[m],
 * canonical order.  Every 4-clique is counted once from its lowest (deg, id)-key vertex on the
 * same oriented CSR (O(m * alpha^2) work).  Workspace: twc_score_k4_workspace_bytes(n, m, rb)
 * (the score workspace followed by the K4 counters and scratch).
 * ------------------------------------------------------------------------------------- */
size_t twc_score_k4_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes);
twc_status twc_score_k4(const twc_csr *g, void *workspace, size_t workspace_bytes, int32_t *t,
                        int32_t *wedge, int32_t *tw, int64_t *k4, void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_dist_* -- the whole hot path (score + k-threshold sweep) of ONE graph split over P GPUs
 * ("both components of our framework are highly scalable").
 * One process per GPU, 1 <= P <= 64; every rank holds the whole CSR.  The rows are split into P
 * contiguous ranges of equal degree-oriented slot counts; rank r scores the canonical edges of
 * its rows ("its slice").  The caller runs three exchanges between the phases with its
 * collective library (the binding uses torch.distributed: NCCL on a B200 node):
 *
 *  1. twc_dist_count(g, r, P, ws, send, send_sizes): orientation (replicated) + the triangles
 *     whose lowest (deg, id)-key vertex is in rank r's rows, each found once (prior art
 *     P:380).  send: device int32[2m] capacity, (oriented slot, count) pairs owed to other
 *     ranks, grouped by destination rank in rank order; send_sizes: device int64[P], pairs per
 *     destination (own = 0).   EXCHANGE 1: all-to-all of the pairs.
 *  2. twc_dist_apply(g, P, ws, recv, nrecv): adds the nrecv received pairs (device
 *     int32[2 nrecv]).
 *  3. twc_dist_epilogue(g, r, P, deltas, k, ws, t, wedge, tw, req, req_sizes): per canonical
 *     edge of the slice, t, wedge = d_u + d_v - 2t - 2 and TW = t - wedge (Eq. 2,
 *     P:488-491) into t/wedge/tw (device int32[m]; only the slice is written), except the edges
 *     whose count lives on another rank: their oriented slots go out as requests, req (device
 *     int32[m] capacity) grouped by owner, req_sizes (device int64[P]).   EXCHANGE 2: all-to-all
 *     of the requests; each owner answers with
 *  4. twc_dist_serve(g, P, ws, req_in, nreq, reply): reply[i] = count of slot req_in[i]; the
 *     replies go back with a second all-to-all (so they arrive in the order of the requests).
 *  5. twc_dist_forest(g, P, deltas, k, ws, reply, t, wedge, tw, forest, forest_cum, kept_sizes,
 *     nforest): completes the requested edges, filters the slice (keep iff NOT TW < delta)
 *     and runs union-find over its kept edges threshold by threshold in descending order,
 *     recording every hook: forest (device int32[2(n-1)] capacity) holds (a, b) pairs, those of
 *     the i-th largest threshold before forest_cum[i] (device int64[k], cumulative); kept_sizes
 *     (device int64[k]) = the slice's edges first kept at that threshold; nforest = total pairs.
 *     EXCHANGE 3: all-gather of forest (padded to cap pairs), forest_cum and kept_sizes.
 *  6. twc_dist_sweep(g, P, deltas, k, ws, forests, cap, forest_cum_all, kept_all, labels,
 *     stats): union-find over the P forests (forests: device int32[P][2 cap]; forest_cum_all,
 *     kept_all: device int64[P][k]; cap >= every rank's nforest) and one snapshot per
 *     threshold: labels (device
 *     int32[k*n]) and stats (device int64[2k] or NULL) identical to twc_sweep's on every rank.
 * The calls of one rank must use the same g, P, deltas and workspace (it carries the oriented
 * CSR and counts between the phases): twc_dist_workspace_bytes(n, m, rb, P).  Any output can be
 * checked against the single-GPU calls: the union of the slices is twc_score's t, wedge, tw.
 * Errors as elsewhere; rank / P out of range -> TWC_EINVAL.
 * ------------------------------------------------------------------------------------- */
size_t twc_dist_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes, int32_t world);
twc_status twc_dist_count(const twc_csr *g, int32_t rank, int32_t world, void *workspace,
                          size_t workspace_bytes, int32_t *send, int64_t *send_sizes,
                          void *stream);
twc_status twc_dist_apply(const twc_csr *g, int32_t world, void *workspace,
                          size_t workspace_bytes, const int32_t *recv, int64_t nrecv,
                          void *stream);
twc_status twc_dist_epilogue(const twc_csr *g, int32_t rank, int32_t world,
                             const double *deltas_host, int32_t k, void *workspace,
                             size_t workspace_bytes, int32_t *t, int32_t *wedge, int32_t *tw,
                             int32_t *req, int64_t *req_sizes, void *stream);
twc_status twc_dist_serve(const twc_csr *g, int32_t world, void *workspace,
                          size_t workspace_bytes, const int32_t *req, int64_t nreq,
                          int32_t *reply, void *stream);
twc_status twc_dist_forest(const twc_csr *g, int32_t world, const double *deltas_host, int32_t k,
                           void *workspace, size_t workspace_bytes, const int32_t *reply,
                           int32_t *t, int32_t *wedge, int32_t *tw, int32_t *forest,
                           int64_t *forest_cum, int64_t *kept_sizes, int64_t *nforest,
                           void *stream);
twc_status twc_dist_sweep(const twc_csr *g, int32_t world, const double *deltas_host, int32_t k,
                          void *workspace, size_t workspace_bytes, const int32_t *forests,
                          int64_t cap, const int64_t *forest_cum_all, const int64_t *kept_all,
                          int32_t *labels, int64_t *stats, void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_partition_stats -- the statistics the threshold-selection study plots for each
 * partition ("norm # CC ... norm |largest CC|", modularity P:350-352; S:346;
 * SURVEY 8(f) NEXT(2)), for k partitions of the INPUT graph g at once.
 *   labels:     device int32[k*n]; labels[j*n + u] in [0, n) names u's community in
 *               partition j (the min-id labels of twc_sweep qualify; any labelling works).
 *   counts:     device int64[4k]; counts[4j + 0] = number of communities, [4j + 1] = size of the
 *               largest, [4j + 2] = E_in, the number of edges of g inside one community,
 *               [4j + 3] = sum over communities c of D_c^2, D_c = sum of deg(u), u in c.
 *   modularity: device double[k] or NULL; modularity[j] = (4 m E_in - sum D_c^2) / (4 m^2),
 *               one IEEE division of exact integers (reading C21; P:350-352's double sum over
 *               ordered pairs), NaN when m = 0.
 * The norm statistics of P:888 are counts / n and kept edges (twc_sweep stats) / m.
 * Synchronises `stream` (a device flag is read back).  TWC_EINVAL: k outside [1, 1024],
 * m > 1.5e9 (4m^2 must fit int64), NULL arrays, or a label outside [0, n) (counts are then
 * meaningless).  Workspace: twc_partition_stats_workspace_bytes(n, m, rb) (device, 256-byte
 * aligned; may be NULL when n = 0).
 * ------------------------------------------------------------------------------------- */
size_t twc_partition_stats_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes);
twc_status twc_partition_stats(const twc_csr *g, const int32_t *labels, int32_t k,
                               void *workspace, size_t workspace_bytes, int64_t *counts,
                               double *modularity, void *stream);

/* ---------------------------------------------------------------------------------------
 * twc_select_threshold -- the paper's two rules of thumb for picking delta (
 * reading C22), on HOST arrays describing k sweep points (any order):
 *   deltas[k], largest[k] (size of the largest community at deltas[i], counts[4i + 1] of
 *   twc_partition_stats), modularity[k], n = number of vertices (normalises largest).
 * Rule 1 (TWC_RULE_LARGEST_JUMP): scanning the points by DECREASING delta, find the step with
 * the largest increase (double)(largest_next - largest_prev) / (double)n (first such step on
 * ties); if it is >= jump_factor (0.1 is the documented default, not a paper value), select
 * the higher delta of that step ("a sudden increment in the size of the largest community").
 * Rule 2 (TWC_RULE_MAX_MODULARITY), otherwise: the delta with the largest modularity, the
 * larger delta on ties; NaN never wins.  Equal deltas keep input order.
 * Writes *index (into deltas) and *rule.  TWC_EINVAL: k < 1, n < 1, NULL, NaN delta.
 * Host-only; no device work.
 * ------------------------------------------------------------------------------------- */
typedef enum { TWC_RULE_LARGEST_JUMP = 0, TWC_RULE_MAX_MODULARITY = 1 } twc_rule;
twc_status twc_select_threshold(const double *deltas, const int64_t *largest,
                                const double *modularity, int32_t k, int64_t n,
                                double jump_factor, int32_t *index, int32_t *rule);

/* ---------------------------------------------------------------------------------------
 * twc_sweep_norm_stats -- the three normalised statistics the threshold-selection study plots
 * per sweep point ("norm # CC", "norm # edges", "norm |largest CC|"), from
 * HOST copies of twc_partition_stats' counts and twc_sweep's stats:
 *   counts[4k] (n_communities, largest, E_in, sum D_c^2 per partition), kept_stats[2k]
 *   ({kept_edges, n_components} per threshold; NULL -> the norm-edges column is NaN),
 *   norm[3k]:  norm[3j + 0] = counts[4j] / n        (number of communities / n)
 *              norm[3j + 1] = kept_stats[2j] / m    (edges kept at delta_j / m)
 *              norm[3j + 2] = counts[4j + 1] / n    (largest community / n)
 * each one IEEE division of exact integers; NaN when the divisor is 0.  Host-only, no device
 * work.  TWC_EINVAL: k < 1, n < 0, m < 0, NULL counts or norm.
 * ------------------------------------------------------------------------------------- */
twc_status twc_sweep_norm_stats(int64_t n, int64_t m, int32_t k, const int64_t *counts,
                                const int64_t *kept_stats, double *norm);

/* ---------------------------------------------------------------------------------------
 * twc_validate_csr -- checks the a0 precondition: rowptr[0] = 0, rowptr
 * non-decreasing, rowptr[n] = 2m, 0 <= colidx < n, rows strictly increasing, no self-loops,
 * symmetry.  Writes a bit mask to *verdict (device int32; 0 = valid; bit 0 rowptr, bit 1 id
 * range, bit 2 order/duplicates, bit 3 self-loop, bit 4 asymmetry), synchronises the stream
 * and returns TWC_OK when valid, TWC_EGRAPH otherwise.  Workspace: none needed (may be NULL).
 * ------------------------------------------------------------------------------------- */
twc_status twc_validate_csr(const twc_csr *g, int32_t *verdict, void *stream);

/* ---------------------------------------------------------------------------------------
 * Instrumented variants (bench.py): identical results to twc_score / twc_sweep.  `events` is
 * NULL or an array of caller-created cudaEvent_t handles that the call records on `stream` at
 * its phase boundaries, so the caller can time each phase with cudaEventElapsedTime:
 *   twc_score_ex: TWC_SCORE_NEVENTS = 4 events -- [0] start, [1] orientation done (K0, K1,
 *                 scans), [2] intersection done (K2), [3] epilogue done (K3).
 *   twc_sweep_ex: TWC_SWEEP_NEVENTS = 3 events -- [0] start, [1] setup done, [2] all k
 *                 thresholds filtered + labelled.
 * ------------------------------------------------------------------------------------- */
#define TWC_SCORE_NEVENTS 4
#define TWC_SWEEP_NEVENTS 3
twc_status twc_score_ex(const twc_csr *g, void *workspace, size_t workspace_bytes, int32_t *t,
                        int32_t *wedge, int32_t *tw, void *stream, void *const *events);
twc_status twc_sweep_ex(const twc_csr *g, const int32_t *tw, const double *deltas_host,
                        int32_t k, void *workspace, size_t workspace_bytes, int32_t *labels,
                        int64_t *stats, void *stream, void *const *events);

/* Number of kernels this process has launched through the library so far (monotone counter;
 * bench.py reports the per-step difference as gpu_launches). */
int64_t twc_kernel_launches(void);

/* Static description of a status code; never NULL. */
const char *twc_status_string(twc_status s);
/* Detail of this thread's last non-OK status ("" if none); valid until the next call. */
const char *twc_last_error(void);
/* ABI version: 100 * major + minor. */
int32_t twc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TWC_H_ */
