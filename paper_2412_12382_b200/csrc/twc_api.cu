// twc_api.cu -- the extern "C" boundary declared in include/twc.h: argument checks, workspace
// carving, dtype dispatch (int32 / int64 rowptr) and error reporting.  No compute here.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "twc.h"
#include "twc_internal.h"

namespace twc {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

static twc_status fail(twc_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

static twc_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return TWC_OK;
    return fail(TWC_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

int num_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

int kernel_setup(const void* fn, int threads, size_t smem) {
    struct Entry {
        int dev;
        const void* fn;
        size_t smem;
        int occ;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
        if (e.dev == dev && e.fn == fn && e.smem == smem) return e.occ;
    int occ = 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
    if (occ < 1) {
        cudaGetLastError();  // a failed query must not leak into the launch status
        occ = 1;
    }
    cache.push_back({dev, fn, smem, occ});
    return occ;
}

// Persisting-L2 window for the per-vertex record array vinfo (8n bytes), which K2 gathers once
// per oriented slot and K3 once per reversed edge.  Under the 5-6 TB/s of streaming traffic of
// those kernels a normally cached line lives ~20 us in L2, about the interval between two uses
// of a vinfo line, so a good part of those gathers went to DRAM (a 64-byte access each);
// eviction hints on the loads did not change that.  With an L2 set-aside
// (cudaLimitPersistingL2CacheSize, 32 MiB, set once per device on the first call that needs it)
// and an access-policy window on the caller's stream from k1_rows (which writes vinfo) to K3,
// the records stay in L2: config 5 K2 1.72 -> 1.68 ms, K3 0.87 -> 0.82 ms, DRAM reads -0.55 /
// -0.34 GB.  24 / 40 / 48 MiB gain less and 64 MiB costs the other data too much L2 (step 4.5
// ms).  The window is used only when the oriented arrays (col_or + t_or, 8m bytes) exceed the
// L2: on smaller graphs everything stays cached anyway and the set-aside only cost capacity
// (config 4: +3 %); such a call resets persisting lines an earlier large call left behind.
// These are cache hints: results never depend on them.  TWC_L2_PERSIST_MB overrides the
// set-aside size (0 = never use the window); a device without the feature, or a first call made
// during stream capture (the limit cannot be set then), runs without it.
#ifndef TWC_L2_PERSIST_DEFAULT_MB
#define TWC_L2_PERSIST_DEFAULT_MB 32
#endif
namespace {
struct L2Dev {
    bool done = false;    // set-aside decided for this device
    size_t cap = 0;       // set-aside bytes (0: window off)
    size_t l2 = 0;        // L2 size
    size_t max_win = 0;   // largest access-policy window
    bool dirty = false;   // persisting lines of an earlier windowed call may still be resident
};
std::mutex g_l2_mu;
L2Dev g_l2[64];
}  // namespace

static bool stream_capturing(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return cs != cudaStreamCaptureStatusNone;
}

// returns the device's record with the set-aside decided, or nullptr (feature off / not yet)
static L2Dev* l2_device(cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    L2Dev& d = g_l2[dev];
    if (!d.done) {
        if (stream_capturing(s)) return nullptr;  // decided by the first call outside a capture
        d.done = true;
        const char* e = getenv("TWC_L2_PERSIST_MB");
        const long mb = e ? atol(e) : (long)TWC_L2_PERSIST_DEFAULT_MB;
        int maxp = 0, maxw = 0, l2 = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        d.l2 = (size_t)std::max(l2, 0);
        d.max_win = (size_t)std::max(maxw, 0);
        if (mb > 0 && maxp > 0 && maxw > 0 && l2 > 0) {
            const size_t want = std::min<size_t>((size_t)mb << 20, (size_t)maxp);
            if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess)
                d.cap = want;
        }
        cudaGetLastError();
    }
    return d.cap ? &d : nullptr;
}

bool l2_window_begin(cudaStream_t s, const void* ptr, size_t bytes, size_t streamed_bytes) {
    std::lock_guard<std::mutex> lock(g_l2_mu);
    L2Dev* d = l2_device(s);
    if (!d || !bytes || !ptr) return false;
    if (streamed_bytes < d->l2) {  // everything stays cached without help
        if (d->dirty && !stream_capturing(s)) {
            cudaCtxResetPersistingL2Cache();
            cudaGetLastError();
            d->dirty = false;
        }
        return false;
    }
    cudaStreamAttrValue a;
    memset(&a, 0, sizeof(a));
    a.accessPolicyWindow.base_ptr = const_cast<void*>(ptr);
    a.accessPolicyWindow.num_bytes = std::min(bytes, d->max_win);
    a.accessPolicyWindow.hitRatio =
        std::min(1.0f, (float)((double)d->cap / (double)a.accessPolicyWindow.num_bytes));
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    d->dirty = true;
    return true;
}

void l2_window_end(cudaStream_t s) {
    cudaStreamAttrValue a;
    memset(&a, 0, sizeof(a));
    a.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
    a.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
    if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess)
        cudaGetLastError();
}

static twc_status check_csr(const twc_csr* g, bool need_ptrs = true, bool device_ptrs = true) {
    if (!g) return fail(TWC_EINVAL, "graph descriptor is NULL");
    if (g->n < 0 || g->n >= ((int64_t)1 << 31)) return fail(TWC_EINVAL, "n=%lld out of range", (long long)g->n);
    if (g->m < 0 || g->m >= ((int64_t)1 << 31)) return fail(TWC_EINVAL, "m=%lld out of range", (long long)g->m);
    if (g->rowptr_bytes != 4 && g->rowptr_bytes != 8)
        return fail(TWC_EINVAL, "rowptr_bytes=%d must be 4 or 8", g->rowptr_bytes);
    if (g->rowptr_bytes == 4 && 2 * g->m >= ((int64_t)1 << 31))
        return fail(TWC_EINVAL, "2m=%lld does not fit an int32 rowptr", (long long)(2 * g->m));
    if (g->m > 0 && g->n == 0) return fail(TWC_EINVAL, "m > 0 with n == 0");
    if (need_ptrs && g->n > 0 && !g->rowptr) return fail(TWC_EINVAL, "rowptr is NULL");
    if (need_ptrs && g->m > 0 && !g->colidx) return fail(TWC_EINVAL, "colidx is NULL");
    if (device_ptrs && g->m > 0 && reinterpret_cast<uintptr_t>(g->colidx) % 16)
        return fail(TWC_EINVAL, "device colidx must be 16-byte aligned (vector loads)");
    if (device_ptrs && g->n > 0 && reinterpret_cast<uintptr_t>(g->rowptr) % g->rowptr_bytes)
        return fail(TWC_EINVAL, "device rowptr must be %d-byte aligned", g->rowptr_bytes);
    return TWC_OK;
}

static twc_status check_ws(void* ws, size_t have, size_t need) {
    if (need == 0) return TWC_OK;
    if (!ws) return fail(TWC_EWORKSPACE, "workspace is NULL (need %zu bytes)", need);
    if (reinterpret_cast<uintptr_t>(ws) % kAlign)
        return fail(TWC_EWORKSPACE, "workspace not %zu-byte aligned", kAlign);
    if (have < need) return fail(TWC_EWORKSPACE, "workspace %zu bytes < required %zu", have, need);
    return TWC_OK;
}

// keep iff NOT(tw < delta)  <=>  tw >= ceil(delta) for integer tw (reading C4 / C18)
static twc_status delta_to_thr(double delta, long long* thr) {
    const long long kBig = (long long)1 << 62;
    if (isnan(delta)) return fail(TWC_EINVAL, "delta is NaN");
    if (delta == -INFINITY) { *thr = -kBig; return TWC_OK; }
    if (delta == INFINITY) { *thr = kBig; return TWC_OK; }
    double c = ceil(delta);
    if (c < -4.0e18) *thr = -kBig;
    else if (c > 4.0e18) *thr = kBig;
    else *thr = (long long)c;
    return TWC_OK;
}

// A per-thread, per-device copy stream plus events for twc_pipeline_host (created on first use
// and kept for the life of the process).
struct CopyLane {
    int dev = -1;
    cudaStream_t stream = nullptr;
    std::vector<cudaEvent_t> ev;  // [0] scores final, [1] copies done, [2 + i] sweep step i
};

static CopyLane* copy_lane(int k) {
    static thread_local std::vector<CopyLane> lanes;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    CopyLane* L = nullptr;
    for (auto& x : lanes)
        if (x.dev == dev) L = &x;
    if (!L) {
        lanes.emplace_back();
        L = &lanes.back();
        L->dev = dev;
        if (cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking) != cudaSuccess) {
            lanes.pop_back();
            return nullptr;
        }
    }
    while ((int)L->ev.size() < k + 2) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        L->ev.push_back(e);
    }
    return L;
}

}  // namespace twc

using namespace twc;

extern "C" {

int32_t twc_version(void) { return 100; }

const char* twc_status_string(twc_status s) {
    switch (s) {
        case TWC_OK: return "TWC_OK";
        case TWC_EINVAL: return "TWC_EINVAL: invalid argument";
        case TWC_EWORKSPACE: return "TWC_EWORKSPACE: workspace too small or misaligned";
        case TWC_ECUDA: return "TWC_ECUDA: CUDA error";
        case TWC_EGRAPH: return "TWC_EGRAPH: CSR violates the input precondition";
    }
    return "unknown twc_status";
}

const char* twc_last_error(void) { return g_err.c_str(); }

size_t twc_score_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes) {
    (void)rowptr_bytes;
    if (n < 0 || m < 0) return 0;
    return score_ws_bytes(n, m);
}

size_t twc_cluster_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes) {
    (void)rowptr_bytes;
    if (n < 0 || m < 0) return 0;
    return cluster_ws_bytes(n, m);
}

int64_t twc_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

twc_status twc_score(const twc_csr* g, void* ws, size_t ws_bytes, int32_t* t, int32_t* wedge,
                     int32_t* tw, void* stream) {
    return twc_score_ex(g, ws, ws_bytes, t, wedge, tw, stream, nullptr);
}

twc_status twc_score_ex(const twc_csr* g, void* ws, size_t ws_bytes, int32_t* t, int32_t* wedge,
                        int32_t* tw, void* stream, void* const* events) {
    cudaEvent_t* ev = reinterpret_cast<cudaEvent_t*>(const_cast<void**>(events));
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (g->m > 0 && (!t || !wedge || !tw)) return fail(TWC_EINVAL, "output array is NULL");
    if (g->m == 0) {
        if (ev) {
            cudaStream_t s0 = static_cast<cudaStream_t>(stream);
            for (int i = 0; i < 4; ++i) record(ev, i, s0);
        }
        return TWC_OK;
    }
    st = check_ws(ws, ws_bytes, score_ws_bytes(g->n, g->m));
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = score_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, ws,
                            ws_bytes, t, wedge, tw, s, ev);
    else
        e = score_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr), g->colidx,
                                  ws, ws_bytes, t, wedge, tw, s, ev);
    return cuda_status(e, "twc_score");
}

static twc_status sweep_common(const twc_csr* g, const int32_t* tw, const long long* thr, int k,
                               void* ws, size_t ws_bytes, int32_t* labels, int64_t* stats,
                               void* stream, cudaEvent_t* ev = nullptr) {
    if (g->n > 0 && !labels) return fail(TWC_EINVAL, "labels is NULL");
    if (g->m > 0 && !tw) return fail(TWC_EINVAL, "tw is NULL");
    twc_status st = check_ws(ws, ws_bytes, cluster_ws_bytes(g->n, g->m));
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = sweep_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, tw, thr, k,
                            ws, ws_bytes, labels, reinterpret_cast<long long*>(stats), s, ev);
    else
        e = sweep_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr), g->colidx,
                                  tw, thr, k, ws, ws_bytes, labels,
                                  reinterpret_cast<long long*>(stats), s, ev);
    return cuda_status(e, "twc_cluster/twc_sweep");
}

twc_status twc_cluster(const twc_csr* g, const int32_t* tw, double delta, void* ws,
                       size_t ws_bytes, int32_t* labels, int64_t* stats, void* stream) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    long long thr;
    st = delta_to_thr(delta, &thr);
    if (st) return st;
    return sweep_common(g, tw, &thr, 1, ws, ws_bytes, labels, stats, stream);
}

twc_status twc_sweep(const twc_csr* g, const int32_t* tw, const double* deltas_host, int32_t k,
                     void* ws, size_t ws_bytes, int32_t* labels, int64_t* stats, void* stream) {
    return twc_sweep_ex(g, tw, deltas_host, k, ws, ws_bytes, labels, stats, stream, nullptr);
}

twc_status twc_sweep_ex(const twc_csr* g, const int32_t* tw, const double* deltas_host,
                        int32_t k, void* ws, size_t ws_bytes, int32_t* labels, int64_t* stats,
                        void* stream, void* const* events) {
    cudaEvent_t* ev = reinterpret_cast<cudaEvent_t*>(const_cast<void**>(events));
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (k < 1 || k > 1024) return fail(TWC_EINVAL, "k=%d must be in [1, 1024]", k);
    if (!deltas_host) return fail(TWC_EINVAL, "deltas_host is NULL");
    long long thr[1024];
    for (int i = 0; i < k; ++i) {
        st = delta_to_thr(deltas_host[i], &thr[i]);
        if (st) return st;
    }
    return sweep_common(g, tw, thr, k, ws, ws_bytes, labels, stats, stream, ev);
}

size_t twc_score_sweep_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes) {
    (void)rowptr_bytes;
    if (n < 0 || m < 0) return 0;
    return score_sweep_ws_bytes(n, m);
}

twc_status twc_score_sweep(const twc_csr* g, const double* deltas_host, int32_t k, void* ws,
                           size_t ws_bytes, int32_t* t, int32_t* wedge, int32_t* tw,
                           int32_t* labels, int64_t* stats, void* stream, void* const* events) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (k < 1 || k > 1024) return fail(TWC_EINVAL, "k=%d must be in [1, 1024]", k);
    if (!deltas_host) return fail(TWC_EINVAL, "deltas_host is NULL");
    if (g->m > 0 && (!t || !wedge || !tw)) return fail(TWC_EINVAL, "output array is NULL");
    if (g->n > 0 && !labels) return fail(TWC_EINVAL, "labels is NULL");
    long long thr[1024];
    for (int i = 0; i < k; ++i) {
        st = delta_to_thr(deltas_host[i], &thr[i]);
        if (st) return st;
    }
    st = check_ws(ws, ws_bytes, score_sweep_ws_bytes(g->n, g->m));
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaEvent_t* ev = reinterpret_cast<cudaEvent_t*>(const_cast<void**>(events));
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = score_sweep_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, thr,
                                  k, ws, ws_bytes, t, wedge, tw, labels,
                                  reinterpret_cast<long long*>(stats), s, ev);
    else
        e = score_sweep_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                        g->colidx, thr, k, ws, ws_bytes, t, wedge, tw, labels,
                                        reinterpret_cast<long long*>(stats), s, ev);
    return cuda_status(e, "twc_score_sweep");
}

twc_status twc_similarity(const twc_csr* g, const int32_t* t, int32_t kind, void* ws,
                          size_t ws_bytes, double* score, void* stream) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (kind < TWC_SIM_TW || kind > TWC_SIM_EFFRES) return fail(TWC_EINVAL, "unknown kind %d", kind);
    if (g->m > 0 && (!t || !score)) return fail(TWC_EINVAL, "t or score is NULL");
    if (g->m == 0) return TWC_OK;
    st = check_ws(ws, ws_bytes, cluster_ws_bytes(g->n, g->m));
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = similarity_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, t,
                                 kind, ws, ws_bytes, score, s);
    else
        e = similarity_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                       g->colidx, t, kind, ws, ws_bytes, score, s);
    return cuda_status(e, "twc_similarity");
}

twc_status twc_sweep_f64(const twc_csr* g, const double* score, const double* deltas_host,
                         int32_t k, void* ws, size_t ws_bytes, int32_t* labels, int64_t* stats,
                         void* stream) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (k < 1 || k > 1024) return fail(TWC_EINVAL, "k=%d must be in [1, 1024]", k);
    if (!deltas_host) return fail(TWC_EINVAL, "deltas_host is NULL");
    for (int i = 0; i < k; ++i)
        if (isnan(deltas_host[i])) return fail(TWC_EINVAL, "delta is NaN");
    if (g->n > 0 && !labels) return fail(TWC_EINVAL, "labels is NULL");
    if (g->m > 0 && !score) return fail(TWC_EINVAL, "score is NULL");
    st = check_ws(ws, ws_bytes, cluster_ws_bytes(g->n, g->m));
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = sweep_f64_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, score,
                                deltas_host, k, ws, ws_bytes, labels,
                                reinterpret_cast<long long*>(stats), s);
    else
        e = sweep_f64_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                      g->colidx, score, deltas_host, k, ws, ws_bytes, labels,
                                      reinterpret_cast<long long*>(stats), s);
    return cuda_status(e, "twc_sweep_f64");
}

// ---- end-to-end from host buffers --------------------------------------------------------
struct PipeWs {
    void* rowptr;
    int *colidx, *t, *wedge, *tw, *labels;
    long long* stats;
    void* inner;
    size_t inner_bytes;
};

static PipeWs carve_pipe(Carver& cv, int64_t n, int64_t m, int rb, int k) {
    PipeWs w;
    w.rowptr = cv.take<char>((size_t)(n + 1) * rb);
    w.colidx = cv.take<int>(2 * m);
    w.t = cv.take<int>(m);
    w.wedge = cv.take<int>(m);
    w.tw = cv.take<int>(m);
    w.labels = cv.take<int>((size_t)k * n);
    w.stats = cv.take<long long>(2 * (size_t)k);
    w.inner_bytes = score_sweep_ws_bytes(n, m);
    w.inner = cv.take<char>(w.inner_bytes);
    return w;
}

size_t twc_pipeline_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes, int32_t k) {
    if (n < 0 || m < 0 || (rowptr_bytes != 4 && rowptr_bytes != 8) || k < 1) return 0;
    Carver cv(nullptr, 0);
    carve_pipe(cv, n, m, rowptr_bytes, k);
    return cv.used;
}

twc_status twc_pipeline_host(const twc_csr* gh, const double* deltas_host, int32_t k, void* ws,
                             size_t ws_bytes, int32_t* t, int32_t* wedge, int32_t* tw,
                             int32_t* labels, int64_t* stats, void* stream) {
    twc_status st = twc_pipeline_host_async(gh, deltas_host, k, ws, ws_bytes, t, wedge, tw,
                                            labels, stats, stream);
    if (st) return st;
    return cuda_status(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)),
                       "twc_pipeline_host sync");
}

twc_status twc_pipeline_host_async(const twc_csr* gh, const double* deltas_host, int32_t k,
                                   void* ws, size_t ws_bytes, int32_t* t, int32_t* wedge,
                                   int32_t* tw, int32_t* labels, int64_t* stats, void* stream) {
    g_err.clear();
    twc_status st = check_csr(gh, true, false);  // host buffers: copied to aligned device memory
    if (st) return st;
    if (k < 1 || k > 1024) return fail(TWC_EINVAL, "k=%d must be in [1, 1024]", k);
    if (!deltas_host) return fail(TWC_EINVAL, "deltas_host is NULL");
    long long thr[1024];
    for (int i = 0; i < k; ++i) {
        st = delta_to_thr(deltas_host[i], &thr[i]);
        if (st) return st;
    }
    const int64_t n = gh->n, m = gh->m;
    const int rb = gh->rowptr_bytes;
    st = check_ws(ws, ws_bytes, twc_pipeline_workspace_bytes(n, m, rb, k));
    if (st) return st;
    Carver cv(ws, ws_bytes);
    PipeWs w = carve_pipe(cv, n, m, rb, k);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CopyLane* cl = copy_lane(k);
    if (!cl) return cuda_status(cudaGetLastError(), "twc_pipeline_host copy stream");
    cudaError_t e = cudaSuccess;
    if (n > 0) e = cudaMemcpyAsync(w.rowptr, gh->rowptr, (size_t)(n + 1) * rb, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && m > 0)
        e = cudaMemcpyAsync(w.colidx, gh->colidx, sizeof(int) * 2 * (size_t)m, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "twc_pipeline_host H2D");
    // Results go back on a second stream as soon as they are final, overlapping the copies
    // with the remaining device work: the scores once the epilogue is done (event [3]), the
    // labels of each threshold once its sweep step is done.
    cudaEvent_t ev6[6] = {nullptr, nullptr, nullptr, cl->ev[0], nullptr, nullptr};
    cudaEvent_t* step_ev = cl->ev.data() + 2;
    if (rb == 4)
        e = score_sweep_impl<int>(n, m, static_cast<const int*>(w.rowptr), w.colidx, thr, k,
                                  w.inner, w.inner_bytes, w.t, w.wedge, w.tw, w.labels, w.stats,
                                  s, ev6, step_ev);
    else
        e = score_sweep_impl<long long>(n, m, static_cast<const long long*>(w.rowptr), w.colidx,
                                        thr, k, w.inner, w.inner_bytes, w.t, w.wedge, w.tw,
                                        w.labels, w.stats, s, ev6, step_ev);
    if (e != cudaSuccess) return cuda_status(e, "twc_pipeline_host score_sweep");
    if (m == 0 || n == 0) cudaEventRecord(cl->ev[0], s);
    cudaStream_t c = cl->stream;
    const size_t mb = sizeof(int) * (size_t)m;
    e = cudaStreamWaitEvent(c, cl->ev[0], 0);
    if (e == cudaSuccess && t && m) e = cudaMemcpyAsync(t, w.t, mb, cudaMemcpyDeviceToHost, c);
    if (e == cudaSuccess && wedge && m) e = cudaMemcpyAsync(wedge, w.wedge, mb, cudaMemcpyDeviceToHost, c);
    if (e == cudaSuccess && tw && m) e = cudaMemcpyAsync(tw, w.tw, mb, cudaMemcpyDeviceToHost, c);
    SweepPlan P;
    sweep_plan(thr, k, &P);
    for (int i = 0; i < k && e == cudaSuccess; ++i) {
        e = cudaStreamWaitEvent(c, step_ev[i], 0);
        if (e == cudaSuccess && labels && n)
            e = cudaMemcpyAsync(labels + (size_t)P.order[i] * n, w.labels + (size_t)P.order[i] * n,
                                sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost, c);
    }
    if (e == cudaSuccess && stats)
        e = cudaMemcpyAsync(stats, w.stats, sizeof(long long) * 2 * (size_t)k, cudaMemcpyDeviceToHost, c);
    if (e == cudaSuccess) e = cudaEventRecord(cl->ev[1], c);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, cl->ev[1], 0);  // the caller's stream sees all
    return cuda_status(e, "twc_pipeline_host D2H");
}

twc_status twc_validate_csr(const twc_csr* g, int32_t* verdict, void* stream) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (!verdict) return fail(TWC_EINVAL, "verdict is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = validate_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, verdict, s);
    else
        e = validate_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                     g->colidx, verdict, s);
    if (e != cudaSuccess) return cuda_status(e, "twc_validate_csr");
    int h = 0;
    e = cudaMemcpyAsync(&h, verdict, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "twc_validate_csr");
    if (h) return fail(TWC_EGRAPH, "CSR invalid, verdict bits 0x%x", h);
    return TWC_OK;
}

// ---- one graph over P GPUs (twc_dist.cu) ---------------------------------------
static constexpr int kDistMaxWorld = 64;

static twc_status dist_args(const twc_csr* g, int32_t rank, int32_t world) {
    twc_status st = check_csr(g);
    if (st) return st;
    if (world < 1 || world > kDistMaxWorld || rank < 0 || rank >= world)
        return fail(TWC_EINVAL, "rank %d / world %d (1 <= world <= %d)", rank, world, kDistMaxWorld);
    return TWC_OK;
}

static twc_status dist_thresholds(const double* deltas_host, int32_t k, long long* thr) {
    if (k < 1 || k > 1024) return fail(TWC_EINVAL, "k=%d must be in [1, 1024]", k);
    if (!deltas_host) return fail(TWC_EINVAL, "deltas_host is NULL");
    for (int i = 0; i < k; ++i) {
        twc_status st = delta_to_thr(deltas_host[i], &thr[i]);
        if (st) return st;
    }
    return TWC_OK;
}

size_t twc_dist_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes, int32_t world) {
    (void)rowptr_bytes;
    if (n < 0 || m < 0 || world < 1 || world > kDistMaxWorld) return 0;
    return dist_ws_bytes(n, m, world);
}

twc_status twc_dist_count(const twc_csr* g, int32_t rank, int32_t world, void* ws,
                          size_t ws_bytes, int32_t* send, int64_t* send_sizes, void* stream) {
    g_err.clear();
    twc_status st = dist_args(g, rank, world);
    if (st) return st;
    if (!send_sizes || (g->m > 0 && !send)) return fail(TWC_EINVAL, "send buffers are NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (g->m == 0 || g->n == 0)
        return cuda_status(cudaMemsetAsync(send_sizes, 0, sizeof(int64_t) * world, s),
                           "twc_dist_count");
    st = check_ws(ws, ws_bytes, dist_ws_bytes(g->n, g->m, world));
    if (st) return st;
    long long* sz = reinterpret_cast<long long*>(send_sizes);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = dist_count_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, rank,
                                 world, ws, ws_bytes, send, sz, s);
    else
        e = dist_count_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                       g->colidx, rank, world, ws, ws_bytes, send, sz, s);
    return cuda_status(e, "twc_dist_count");
}

twc_status twc_dist_apply(const twc_csr* g, int32_t world, void* ws, size_t ws_bytes,
                          const int32_t* recv, int64_t nrecv, void* stream) {
    g_err.clear();
    twc_status st = dist_args(g, 0, world);
    if (st) return st;
    if (nrecv < 0 || (nrecv > 0 && !recv)) return fail(TWC_EINVAL, "recv / nrecv");
    if (g->m == 0 || g->n == 0 || nrecv == 0) return TWC_OK;
    st = check_ws(ws, ws_bytes, dist_ws_bytes(g->n, g->m, world));
    if (st) return st;
    return cuda_status(dist_apply_impl(g->n, g->m, world, ws, ws_bytes, recv, nrecv,
                                       static_cast<cudaStream_t>(stream)),
                       "twc_dist_apply");
}

twc_status twc_dist_epilogue(const twc_csr* g, int32_t rank, int32_t world,
                             const double* deltas_host, int32_t k, void* ws, size_t ws_bytes,
                             int32_t* t, int32_t* wedge, int32_t* tw, int32_t* req,
                             int64_t* req_sizes, void* stream) {
    g_err.clear();
    twc_status st = dist_args(g, rank, world);
    if (st) return st;
    long long thr[1024];
    st = dist_thresholds(deltas_host, k, thr);
    if (st) return st;
    if (!req_sizes || (g->m > 0 && (!t || !wedge || !tw || !req)))
        return fail(TWC_EINVAL, "output array is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (g->m == 0 || g->n == 0)
        return cuda_status(cudaMemsetAsync(req_sizes, 0, sizeof(int64_t) * world, s),
                           "twc_dist_epilogue");
    st = check_ws(ws, ws_bytes, dist_ws_bytes(g->n, g->m, world));
    if (st) return st;
    long long* rs = reinterpret_cast<long long*>(req_sizes);
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = dist_epilogue_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx,
                                    rank, world, thr, k, ws, ws_bytes, t, wedge, tw, req, rs, s);
    else
        e = dist_epilogue_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                          g->colidx, rank, world, thr, k, ws, ws_bytes, t, wedge,
                                          tw, req, rs, s);
    return cuda_status(e, "twc_dist_epilogue");
}

twc_status twc_dist_serve(const twc_csr* g, int32_t world, void* ws, size_t ws_bytes,
                          const int32_t* req, int64_t nreq, int32_t* reply, void* stream) {
    g_err.clear();
    twc_status st = dist_args(g, 0, world);
    if (st) return st;
    if (nreq < 0 || (nreq > 0 && (!req || !reply))) return fail(TWC_EINVAL, "req / reply");
    if (g->m == 0 || g->n == 0 || nreq == 0) return TWC_OK;
    st = check_ws(ws, ws_bytes, dist_ws_bytes(g->n, g->m, world));
    if (st) return st;
    return cuda_status(dist_serve_impl(g->n, g->m, world, ws, ws_bytes, req, nreq, reply,
                                       static_cast<cudaStream_t>(stream)),
                       "twc_dist_serve");
}

twc_status twc_dist_forest(const twc_csr* g, int32_t world, const double* deltas_host, int32_t k,
                           void* ws, size_t ws_bytes, const int32_t* reply, int32_t* t,
                           int32_t* wedge, int32_t* tw, int32_t* forest, int64_t* forest_cum,
                           int64_t* kept_sizes, int64_t* nforest, void* stream) {
    g_err.clear();
    twc_status st = dist_args(g, 0, world);
    if (st) return st;
    long long thr[1024];
    st = dist_thresholds(deltas_host, k, thr);
    if (st) return st;
    if (!forest_cum || !kept_sizes || !nforest) return fail(TWC_EINVAL, "size outputs are NULL");
    if (g->m > 0 && g->n > 0 && (!t || !wedge || !tw || !forest))
        return fail(TWC_EINVAL, "output array is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (g->m == 0 || g->n == 0) {
        cudaError_t e = cudaMemsetAsync(forest_cum, 0, sizeof(int64_t) * k, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(kept_sizes, 0, sizeof(int64_t) * k, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(nforest, 0, sizeof(int64_t), s);
        return cuda_status(e, "twc_dist_forest");
    }
    st = check_ws(ws, ws_bytes, dist_ws_bytes(g->n, g->m, world));
    if (st) return st;
    return cuda_status(
        dist_forest_impl(g->n, g->m, world, thr, k, ws, ws_bytes, reply, t, wedge, tw, forest,
                         reinterpret_cast<long long*>(forest_cum),
                         reinterpret_cast<long long*>(kept_sizes),
                         reinterpret_cast<long long*>(nforest), s),
        "twc_dist_forest");
}

twc_status twc_dist_sweep(const twc_csr* g, int32_t world, const double* deltas_host, int32_t k,
                          void* ws, size_t ws_bytes, const int32_t* forests, int64_t cap,
                          const int64_t* forest_cum_all, const int64_t* kept_all,
                          int32_t* labels, int64_t* stats, void* stream) {
    g_err.clear();
    twc_status st = dist_args(g, 0, world);
    if (st) return st;
    long long thr[1024];
    st = dist_thresholds(deltas_host, k, thr);
    if (st) return st;
    if (cap < 0 || (g->n > 0 && (!labels || !forest_cum_all || !kept_all)) ||
        (cap > 0 && !forests))
        return fail(TWC_EINVAL, "NULL argument or cap < 0");
    st = check_ws(ws, ws_bytes, dist_ws_bytes(g->n, g->m, world));
    if (st) return st;
    return cuda_status(
        dist_sweep_impl(g->n, g->m, world, thr, k, ws, ws_bytes, forests, cap,
                        reinterpret_cast<const long long*>(forest_cum_all),
                        reinterpret_cast<const long long*>(kept_all), labels,
                        reinterpret_cast<long long*>(stats), static_cast<cudaStream_t>(stream)),
        "twc_dist_sweep");
}

// ---- K4 participation (NEXT(4)) ----------------------------------------------------------
size_t twc_score_k4_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes) {
    (void)rowptr_bytes;
    if (n < 0 || m < 0) return 0;
    return score_ws_bytes(n, m) + k4_ws_bytes(n, m);
}

twc_status twc_score_k4(const twc_csr* g, void* ws, size_t ws_bytes, int32_t* t, int32_t* wedge,
                        int32_t* tw, int64_t* k4, void* stream) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (g->m > 0 && (!t || !wedge || !tw || !k4)) return fail(TWC_EINVAL, "output array is NULL");
    if (g->m == 0) return TWC_OK;
    st = check_ws(ws, ws_bytes, score_ws_bytes(g->n, g->m) + k4_ws_bytes(g->n, g->m));
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    long long* k = reinterpret_cast<long long*>(k4);
    if (g->rowptr_bytes == 4)
        e = score_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx, ws,
                            ws_bytes, t, wedge, tw, s, nullptr, nullptr, k);
    else
        e = score_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr), g->colidx,
                                  ws, ws_bytes, t, wedge, tw, s, nullptr, nullptr, k);
    return cuda_status(e, "twc_score_k4");
}

// ---- threshold selection (NEXT(2)) -------------------------------------------------------
size_t twc_partition_stats_workspace_bytes(int64_t n, int64_t m, int32_t rowptr_bytes) {
    (void)rowptr_bytes;
    if (n < 0 || m < 0) return 0;
    return partition_stats_ws_bytes(n, m);
}

twc_status twc_partition_stats(const twc_csr* g, const int32_t* labels, int32_t k, void* ws,
                               size_t ws_bytes, int64_t* counts, double* modularity,
                               void* stream) {
    g_err.clear();
    twc_status st = check_csr(g);
    if (st) return st;
    if (k < 1 || k > 1024) return fail(TWC_EINVAL, "k=%d must be in [1, 1024]", k);
    if (g->m > 1500000000LL) return fail(TWC_EINVAL, "m=%lld: 4m^2 must fit int64", (long long)g->m);
    if (g->n > 0 && !labels) return fail(TWC_EINVAL, "labels is NULL");
    if (!counts) return fail(TWC_EINVAL, "counts is NULL");
    if (g->n > 0) {
        st = check_ws(ws, ws_bytes, partition_stats_ws_bytes(g->n, g->m));
        if (st) return st;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int bad = 0;
    cudaError_t e;
    if (g->rowptr_bytes == 4)
        e = partition_stats_impl<int>(g->n, g->m, static_cast<const int*>(g->rowptr), g->colidx,
                                      labels, k, ws, ws_bytes, reinterpret_cast<long long*>(counts),
                                      modularity, &bad, s);
    else
        e = partition_stats_impl<long long>(g->n, g->m, static_cast<const long long*>(g->rowptr),
                                            g->colidx, labels, k, ws, ws_bytes,
                                            reinterpret_cast<long long*>(counts), modularity, &bad, s);
    if (e != cudaSuccess) return cuda_status(e, "twc_partition_stats");
    if (bad) return fail(TWC_EINVAL, "a label lies outside [0, n)");
    return TWC_OK;
}

twc_status twc_sweep_norm_stats(int64_t n, int64_t m, int32_t k, const int64_t* counts,
                                const int64_t* kept_stats, double* norm) {
    g_err.clear();
    if (k < 1 || n < 0 || m < 0) return fail(TWC_EINVAL, "k=%d n=%lld m=%lld", k, (long long)n,
                                             (long long)m);
    if (!counts || !norm) return fail(TWC_EINVAL, "counts or norm is NULL");
    const double nan = NAN;
    for (int j = 0; j < k; ++j) {
        norm[3 * j + 0] = n ? (double)counts[4 * j] / (double)n : nan;
        norm[3 * j + 1] = (m && kept_stats) ? (double)kept_stats[2 * j] / (double)m : nan;
        norm[3 * j + 2] = n ? (double)counts[4 * j + 1] / (double)n : nan;
    }
    return TWC_OK;
}

twc_status twc_select_threshold(const double* deltas, const int64_t* largest,
                                const double* modularity, int32_t k, int64_t n,
                                double jump_factor, int32_t* index, int32_t* rule) {
    g_err.clear();
    if (k < 1) return fail(TWC_EINVAL, "k=%d must be >= 1", k);
    if (!deltas || !largest || !modularity || !index || !rule)
        return fail(TWC_EINVAL, "NULL argument");
    if (n < 1) return fail(TWC_EINVAL, "n=%lld must be >= 1", (long long)n);
    for (int i = 0; i < k; ++i)
        if (isnan(deltas[i])) return fail(TWC_EINVAL, "delta is NaN");
    std::vector<int> by(k);
    for (int i = 0; i < k; ++i) by[i] = i;
    // decreasing delta; equal deltas keep their input order
    std::stable_sort(by.begin(), by.end(), [&](int a, int b) { return deltas[a] > deltas[b]; });
    // rule of thumb 1: the largest increase of the largest community on that scan
    int jump_at = -1;
    double jump = 0.0;
    for (int i = 1; i < k; ++i) {
        const double inc = (double)(largest[by[i]] - largest[by[i - 1]]) / (double)n;
        if (jump_at < 0 || inc > jump) {
            jump = inc;
            jump_at = by[i - 1];
        }
    }
    if (jump_at >= 0 && jump >= jump_factor) {
        *index = jump_at;
        *rule = TWC_RULE_LARGEST_JUMP;
        return TWC_OK;
    }
    // rule of thumb 2: maximum modularity, the larger delta on ties, NaN never wins
    int best = by[0];
    for (int i = 1; i < k; ++i) {
        const double a = modularity[by[i]], b = modularity[best];
        if (!isnan(a) && (isnan(b) || a > b)) best = by[i];
    }
    *index = best;
    *rule = TWC_RULE_MAX_MODULARITY;
    return TWC_OK;
}

}  // extern "C"
