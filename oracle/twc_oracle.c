/*
 * twc_oracle.c -- plain, slow, obviously-correct CPU oracle for the TW clustering hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or execute anything under oracle/.
 * The product path (paper_2412_12382_b200/) never links, imports or calls this file and
 * shares no code, header, table or helper with it.
 *
 * What it computes (citations are PAPER.md line numbers "P:n", SPEC.md "S:n"):
 *   oracle_score   -- for every canonical edge (u,v), u<v, in lexicographic order (reading C5,
 *                     S:66-69): one two-pointer merge over the FULL sorted lists N(u), N(v)
 *                     (the paper's own per-edge method) that counts
 *                       t     = |N(u) & N(v)|
 *                       uni   = |N(u) | N(v)|  (counted directly, not via degrees)
 *                       wedge = uni - t - 2
 *                       TW    = t - wedge                          (Eq. 2)
 *   oracle_cluster -- Alg. 1: keep edge e iff NOT (TW(e) < delta) (reading
 *                     C4), then connected components by breadth-first search from every
 *                     unlabelled vertex in ascending id order, so every vertex is labelled
 *                     with the minimum id of its component (reading C6).
 *
 *   oracle_similarity -- the other scores of Table 1 from t and the degrees:
 *                     Tectonic t/(d_u+d_v), Jaccard t/(d_u+d_v-t),
 *                     K3 = t, TW = t - wedge (Eq. 2) and the effective-resistance
 *                     proxy -2/(2+t) ("upper bound 2/(2+t)", negated as Table 1's
 *                     -R_eff); one IEEE double operation per score.
 *   oracle_cluster_f64 -- Alg. 1 on real-valued scores: keep e iff NOT (sim(e) < delta).
 *
 *   oracle_partition_stats -- the statistics of one partition that the threshold-selection
 *                     study plots: number of components, size of the
 *                     largest, and the modularity
 *                       Q = (1/2m) sum_{u,v} (A_uv - d_u d_v / 2m) [c_u = c_v]
 *                     evaluated from two exact integers (reading C21): the ordered-pair sum of
 *                     A_uv over same-community pairs is 2 E_in (E_in = edges with both ends in
 *                     one community) and the sum of d_u d_v over them is sum_c D_c^2 (D_c = total
 *                     degree of community c), so Q = (4 m E_in - sum_c D_c^2) / (4 m^2), one
 *                     IEEE division of two exactly represented integers.
 *   oracle_k4      -- kappa-clique participation for kappa = 4 (Table 1; "we only
 *                     consider K_4"): for every canonical edge (u, v), the number of
 *                     4-cliques containing it = the number of pairs {w, x} of common neighbours
 *                     (w < x, both in N(u) & N(v)) that are adjacent, checked by binary search
 *                     in the sorted list N(w).  int64 per edge.
 *   oracle_select  -- the two rules of thumb of P:898-900 (reading C22): on the
 *                     decreasing-delta scan, the largest single-step increase of the normalised
 *                     largest-component size; if it is >= jump_factor return the higher delta
 *                     of that step, else the delta of maximum modularity (ties -> larger delta).
 *
 * Parallelism: the only parallelism is an OpenMP loop over rows in oracle_score (disjoint
 * writes, deterministic).  Everything is int32/int64 integer arithmetic, so there is no
 * rounding anywhere (reading C18).  The comparison (double)TW < delta is exact (|TW| < 2^53).
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Timing only (SURVEY 8(d) "Oracle timing": O2, O3 and O4 timed separately, excluding load):
 * steady-clock seconds of the last oracle_score (O2) and of the filter (O3) and BFS (O4) parts
 * of the last oracle_cluster.  No arithmetic of the method depends on these. */
static double g_times[3];
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
void oracle_times(double *out) { out[0] = g_times[0]; out[1] = g_times[1]; out[2] = g_times[2]; }

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int k) {
#ifdef _OPENMP
    if (k > 0) omp_set_num_threads(k);
#else
    (void)k;
#endif
}

/* Canonical edge offsets: eoff[u] = number of edges (a,b), a<b, with a < u.  S:66-69. */
static void canonical_offsets(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                              int64_t *eoff) {
    eoff[0] = 0;
    for (int64_t u = 0; u < n; ++u) {
        int64_t up = 0;
        for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p)
            if (colidx[p] > u) ++up;
        eoff[u + 1] = eoff[u] + up;
    }
}

/*
 * Score the canonical edges whose smaller endpoint u lies in [u_begin, u_end).
 * t/wedge/tw are full-length (m) arrays indexed by canonical edge id; entries of other rows are
 * left untouched.  Returns 0, or 1 when an allocation fails.
 */
int oracle_score(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                 int64_t u_begin, int64_t u_end,
                 int32_t *t, int32_t *wedge, int32_t *tw) {
    if (n <= 0) return 0;
    const double t0 = now_s();
    int64_t *eoff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!eoff) return 1;
    canonical_offsets(n, rowptr, colidx, eoff);
    if (u_begin < 0) u_begin = 0;
    if (u_end > n) u_end = n;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t u = u_begin; u < u_end; ++u) {
        int64_t c = eoff[u];
        for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p) {
            int64_t v = colidx[p];
            if (v <= u) continue;                      /* canonical: u < v only */
            /* one merge over N(u) and N(v): intersection and union sizes */
            int64_t i = rowptr[u], ie = rowptr[u + 1];
            int64_t j = rowptr[v], je = rowptr[v + 1];
            int64_t inter = 0, uni = 0;
            while (i < ie && j < je) {
                int32_t a = colidx[i], b = colidx[j];
                if (a == b) { ++inter; ++uni; ++i; ++j; }
                else if (a < b) { ++uni; ++i; }
                else { ++uni; ++j; }
            }
            uni += (ie - i) + (je - j);
            int64_t wdg = uni - inter - 2;
            t[c] = (int32_t)inter;
            wedge[c] = (int32_t)wdg;
            tw[c] = (int32_t)(inter - wdg);           /* Eq. 2 */
            ++c;
        }
    }
    free(eoff);
    g_times[0] = now_s() - t0;
    return 0;
}

/*
 * Alg. 1 for one threshold.  labels[n] receives the minimum vertex id of each vertex's
 * component in the kept subgraph; stats (may be NULL) receives {kept_edges, n_components}.
 * Returns 0, or 1 when an allocation fails.
 */
int oracle_cluster(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                   const int32_t *tw, double delta, int32_t *labels, int64_t *stats) {
    if (n <= 0) {
        if (stats) { stats[0] = 0; stats[1] = 0; }
        return 0;
    }
    /* line 1 of Alg. 1: remove e iff sim(e) < delta -- materialise the kept graph */
    const double t0 = now_s();
    int64_t *kdeg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!kdeg) return 1;
    int64_t c = 0, kept = 0;
    for (int64_t u = 0; u < n; ++u)
        for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p) {
            int64_t v = colidx[p];
            if (v <= u) continue;
            if (!((double)tw[c] < delta)) { kdeg[u + 1]++; kdeg[v + 1]++; ++kept; }
            ++c;
        }
    for (int64_t u = 0; u < n; ++u) kdeg[u + 1] += kdeg[u];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int32_t *kadj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * kept + 1));
    int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!fill || !kadj || !queue) { free(kdeg); free(fill); free(kadj); free(queue); return 1; }
    memcpy(fill, kdeg, sizeof(int64_t) * (size_t)n);
    c = 0;
    for (int64_t u = 0; u < n; ++u)
        for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p) {
            int64_t v = colidx[p];
            if (v <= u) continue;
            if (!((double)tw[c] < delta)) {
                kadj[fill[u]++] = (int32_t)v;
                kadj[fill[v]++] = (int32_t)u;
            }
            ++c;
        }
    /* line 2 of Alg. 1: connected components, by BFS in ascending start id */
    const double t1 = now_s();
    for (int64_t u = 0; u < n; ++u) labels[u] = -1;
    int64_t ncomp = 0;
    for (int64_t s = 0; s < n; ++s) {
        if (labels[s] >= 0) continue;
        ++ncomp;
        int64_t head = 0, tail = 0;
        labels[s] = (int32_t)s;
        queue[tail++] = (int32_t)s;
        while (head < tail) {
            int32_t x = queue[head++];
            for (int64_t p = kdeg[x]; p < kdeg[x + 1]; ++p) {
                int32_t y = kadj[p];
                if (labels[y] < 0) { labels[y] = (int32_t)s; queue[tail++] = y; }
            }
        }
    }
    if (stats) { stats[0] = kept; stats[1] = ncomp; }
    free(kdeg); free(fill); free(kadj); free(queue);
    g_times[1] = t1 - t0;
    g_times[2] = now_s() - t1;
    return 0;
}

/* Degree-based scores of Table 1 for every canonical edge, in the same order as
 * oracle_score; kind: 0 TW, 1 Tectonic, 2 Jaccard, 3 K3, 4 effective-resistance proxy. */
int oracle_similarity(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                      const int32_t *t, int32_t kind, double *out) {
    int64_t c = 0;
    for (int64_t u = 0; u < n; ++u) {
        const int64_t du = rowptr[u + 1] - rowptr[u];
        for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p) {
            const int64_t v = colidx[p];
            if (v <= u) continue;
            const int64_t dv = rowptr[v + 1] - rowptr[v];
            const double tt = (double)t[c];
            double x;
            switch (kind) {
                case 0: x = (double)(t[c] - (du + dv - 2 * (int64_t)t[c] - 2)); break;
                case 1: x = tt / (double)(du + dv); break;
                case 2: x = tt / (double)(du + dv - t[c]); break;
                case 3: x = tt; break;
                case 4: x = -2.0 / (2.0 + tt); break;
                default: return 1;
            }
            out[c++] = x;
        }
    }
    return 0;
}

/* Alg. 1 on real-valued scores (same contract as oracle_cluster). */
int oracle_cluster_f64(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                       const double *score, double delta, int32_t *labels, int64_t *stats) {
    if (n <= 0) {
        if (stats) { stats[0] = 0; stats[1] = 0; }
        return 0;
    }
    int64_t m = rowptr[n] / 2;
    /* map the real-valued keep decision onto a 0/1 integer score and reuse oracle_cluster */
    int32_t *keep = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m + 1));
    if (!keep) return 1;
    for (int64_t c = 0; c < m; ++c) keep[c] = (score[c] < delta) ? 0 : 1;
    int rc = oracle_cluster(n, rowptr, colidx, keep, 0.5, labels, stats);
    free(keep);
    return rc;
}


/*
 * Statistics of the partition labels[n] (labels[u] in [0, n) names u's community; the labels
 * of a connected-components run are its minimum vertex ids).
 * out[4] = {number of communities, size of the largest, E_in, sum_c D_c^2};
 * *q = modularity or NaN when m = 0 ("undefined marker").
 * Returns 0, 1 on allocation failure, 2 when a label is out of range.
 */
int oracle_partition_stats(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                           const int32_t *labels, int64_t *out, double *q) {
    out[0] = out[1] = out[2] = out[3] = 0;
    int64_t m = n > 0 ? rowptr[n] / 2 : 0;
    if (n <= 0) { *q = 0.0 / 0.0; return 0; }
    int64_t *size = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    int64_t *dsum = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    if (!size || !dsum) { free(size); free(dsum); return 1; }
    for (int64_t u = 0; u < n; ++u) {
        if (labels[u] < 0 || labels[u] >= n) { free(size); free(dsum); return 2; }
        size[labels[u]] += 1;
        dsum[labels[u]] += rowptr[u + 1] - rowptr[u];          /* D_c = sum of degrees */
    }
    for (int64_t c = 0; c < n; ++c) {
        if (size[c] == 0) continue;
        out[0] += 1;                                            /* communities */
        if (size[c] > out[1]) out[1] = size[c];                 /* largest */
        out[3] += dsum[c] * dsum[c];                            /* sum_c D_c^2 */
    }
    for (int64_t u = 0; u < n; ++u)                             /* E_in: each edge once (u<v) */
        for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p)
            if (colidx[p] > u && labels[colidx[p]] == labels[u]) out[2] += 1;
    if (m == 0) *q = 0.0 / 0.0;
    else *q = (double)(4 * m * out[2] - out[3]) / (double)(4 * m * m);
    free(size); free(dsum);
    return 0;
}

/*
 * The selection rules over k sweep points: deltas[k] (any order), largest[k] = size
 * of the largest community at deltas[i], modularity[k].  Returns the index of the selected
 * point and sets *rule = 0 (largest-component jump) or 1 (maximum modularity).  The
 * normalised increase of one step is (double)(largest_lower - largest_higher) / (double)n.
 */
int32_t oracle_select(int32_t k, const double *deltas, const int64_t *largest, int64_t n,
                      const double *modularity, double jump_factor, int32_t *rule) {
    /* indices by decreasing delta (insertion sort; equal deltas keep input order) */
    int32_t *ord = (int32_t *)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
    if (!ord || k <= 0) { free(ord); *rule = -1; return -1; }
    for (int32_t i = 0; i < k; ++i) {
        int32_t j = i;
        while (j > 0 && deltas[ord[j - 1]] < deltas[i]) { ord[j] = ord[j - 1]; --j; }
        ord[j] = i;
    }
    /* rule 1: "a sudden increment in the size of the largest community" on decreasing delta */
    int32_t best = -1;
    double best_inc = 0.0;
    for (int32_t i = 0; i + 1 < k; ++i) {
        double inc = (double)(largest[ord[i + 1]] - largest[ord[i]]) / (double)n;
        if (best < 0 || inc > best_inc) { best = ord[i]; best_inc = inc; }
    }
    if (best >= 0 && best_inc >= jump_factor) { *rule = 0; free(ord); return best; }
    /* rule 2: "picking a threshold that maximizes the modularity", ties -> larger delta */
    best = ord[0];
    for (int32_t i = 1; i < k; ++i) {
        double a = modularity[ord[i]], b = modularity[best];
        if (a == a && (b != b || a > b)) best = ord[i];
    }
    *rule = 1;
    free(ord);
    return best;
}

static int has_edge(const int64_t *rowptr, const int32_t *colidx, int32_t a, int32_t b) {
    int64_t lo = rowptr[a], hi = rowptr[a + 1];
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (colidx[mid] < b) lo = mid + 1; else hi = mid;
    }
    return lo < rowptr[a + 1] && colidx[lo] == b;
}

/* K4(u, v) for every canonical edge ("for each common neighbor pair w<x in
 * N(u)&N(v), count if (w,x) is an edge").  Returns 0, or 1 when an allocation fails. */
int oracle_k4(int64_t n, const int64_t *rowptr, const int32_t *colidx, int64_t *k4) {
    if (n <= 0) return 0;
    int64_t *eoff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!eoff) return 1;
    canonical_offsets(n, rowptr, colidx, eoff);
    int64_t dmax = 0;
    for (int64_t u = 0; u < n; ++u)
        if (rowptr[u + 1] - rowptr[u] > dmax) dmax = rowptr[u + 1] - rowptr[u];
    int fail = 0;
#pragma omp parallel
    {
        int32_t *common = (int32_t *)malloc(sizeof(int32_t) * (size_t)(dmax + 1));
        if (!common) {
#pragma omp atomic write
            fail = 1;
        }
#pragma omp for schedule(dynamic, 16)
        for (int64_t u = 0; u < n; ++u) {
            if (!common) continue;
            int64_t c = eoff[u];
            for (int64_t p = rowptr[u]; p < rowptr[u + 1]; ++p) {
                int32_t v = colidx[p];
                if (v <= u) continue;
                /* common neighbours by one merge of the sorted lists */
                int64_t i = rowptr[u], ie = rowptr[u + 1], j = rowptr[v], je = rowptr[v + 1];
                int64_t nc = 0;
                while (i < ie && j < je) {
                    if (colidx[i] == colidx[j]) { common[nc++] = colidx[i]; ++i; ++j; }
                    else if (colidx[i] < colidx[j]) ++i;
                    else ++j;
                }
                int64_t cnt = 0;
                for (int64_t a = 0; a < nc; ++a)
                    for (int64_t b = a + 1; b < nc; ++b)
                        cnt += has_edge(rowptr, colidx, common[a], common[b]);
                k4[c++] = cnt;
            }
        }
        free(common);
    }
    free(eoff);
    return fail;
}
