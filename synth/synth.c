/*
 * synth/synth.c -- host side of the seeded SYNTHETIC INPUT GENERATOR.
 *
 * Builds the inputs both sides consume: per-relation in-CSC (indptr over dst
 * tids, src tids), feature bytes, train ids.  Multi-threaded (OpenMP): this is
 * input data, not the method.  Recipe:
 *   in-degree  capped discrete Pareto/Lomax law, alpha = 2.5:
 *              P(D >= k) = (1 + k/x)^-(alpha-1), 1 <= k <= Dmax, x calibrated so
 *              that E[D] = |E_r| / N_dst; then a deterministic exact-count fix-up
 *              so that sum(d) == |E_r|.  (Assumption; the paper only says
 *              "most of graphs have power-law distribution in vertex degree",
 *              P:493-494.)
 *   sources    uniform over the src vertex type (sy_src_tid).
 *   features   integer bit formula (sy_feat_f32 / sy_feat_f16), no float rounding.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

#include "synth_hash.h"

static double mean_of(double x, int64_t dmax, double beta)
{
    double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
    for (int64_t k = 1; k <= dmax; ++k) s += pow(1.0 + (double)k / x, -beta);
    return s;
}

/* thresholds thr[k-1] = round((1 - P(D >= k)) * 2^32), k = 1..dmax (non-decreasing). */
int sy_degree_table(double mean, int64_t dmax, double alpha, uint64_t *thr, double *x_out)
{
    const double beta = alpha - 1.0;
    if (dmax < 1 || mean <= 0.0 || mean >= (double)dmax) return -1;
    double lo = 1e-9, hi = 1e15;
    for (int it = 0; it < 60; ++it) {          /* bisection in log space */
        double mid = sqrt(lo * hi);
        if (mean_of(mid, dmax, beta) < mean) lo = mid; else hi = mid;
    }
    double x = sqrt(lo * hi);
#pragma omp parallel for schedule(static)
    for (int64_t k = 1; k <= dmax; ++k) {
        double tail = pow(1.0 + (double)k / x, -beta);
        double t = (1.0 - tail) * 4294967296.0;
        thr[k - 1] = (uint64_t)llround(t);
    }
    for (int64_t k = 1; k < dmax; ++k)         /* guard monotonicity against rounding */
        if (thr[k] < thr[k - 1]) thr[k] = thr[k - 1];
    if (x_out) *x_out = x;
    return 0;
}

/* indptr[0..n_dst] of relation r with exactly n_edges edges. */
int sy_indptr(uint64_t G, int32_t r, int64_t n_dst, int64_t n_edges, int64_t dmax,
              double alpha, int64_t *indptr)
{
    if (n_dst <= 0) { indptr[0] = 0; return n_edges == 0 ? 0 : -1; }
    if (n_edges > n_dst * dmax) return -1;
    int64_t *deg = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_dst);
    if (!deg) return -2;
    double mean = (double)n_edges / (double)n_dst;
    if (mean >= (double)dmax) {
        for (int64_t v = 0; v < n_dst; ++v) deg[v] = dmax;
    } else if (n_edges == 0) {
        for (int64_t v = 0; v < n_dst; ++v) deg[v] = 0;
    } else {
        uint64_t *thr = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)dmax);
        if (!thr) { free(deg); return -2; }
        if (sy_degree_table(mean, dmax, alpha, thr, NULL) != 0) { free(thr); free(deg); return -1; }
#pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < n_dst; ++v) {
            uint64_t w = sy_hash(G, SY_TAG_DEG + (uint64_t)r, (uint64_t)v, 0) >> 32;
            /* d = #{k : thr[k-1] <= w} (upper bound in the sorted table) */
            int64_t lo = 0, hi = dmax;
            while (lo < hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (thr[mid] <= w) lo = mid + 1; else hi = mid;
            }
            deg[v] = lo;
        }
        free(thr);
    }
    int64_t sum = 0;
#pragma omp parallel for reduction(+ : sum) schedule(static)
    for (int64_t v = 0; v < n_dst; ++v) sum += deg[v];
    int64_t delta = n_edges - sum;             /* exact-count fix-up, cyclic in tid order */
    for (int64_t v = 0; delta != 0; v = (v + 1 == n_dst) ? 0 : v + 1) {
        if (delta > 0 && deg[v] < dmax) { deg[v]++; delta--; }
        else if (delta < 0 && deg[v] > 0) { deg[v]--; delta++; }
    }
    indptr[0] = 0;
    for (int64_t v = 0; v < n_dst; ++v) indptr[v + 1] = indptr[v] + deg[v];
    free(deg);
    return 0;
}

/* src tids of CSC positions [e_lo, e_hi) of relation r */
void sy_indices(uint64_t G, int32_t r, int64_t n_src, int64_t e_lo, int64_t e_hi, int32_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t e = e_lo; e < e_hi; ++e) out[e - e_lo] = sy_src_tid(G, r, e, n_src);
}

/* feature rows [tid_lo, tid_hi) of vertex type u, dim columns, dtype 0=f32 1=f16 */
/* planted-community src tids of CSC positions [e_lo, e_hi) of relation r; indptr is the
 * relation's global CSC row pointer (n_dst + 1) */
void sy_indices_loc(uint64_t G, int32_t r, int64_t n_src, int64_t n_dst, const int64_t *indptr, int64_t e_lo,
                    int64_t e_hi, uint32_t q_thr, int32_t n_comm, int32_t *out)
{
    if (e_hi <= e_lo) return;
#pragma omp parallel
    {
        int nt = 1, id = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        id = omp_get_thread_num();
#endif
        int64_t n = e_hi - e_lo, a = e_lo + n * id / nt, b = e_lo + n * (id + 1) / nt;
        int64_t lo = 0, hi = n_dst;                /* dst of edge a: last x with indptr[x] <= a */
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) / 2;
            if (indptr[mid] <= a) lo = mid; else hi = mid - 1;
        }
        int64_t x = lo;
        for (int64_t e = a; e < b; ++e) {
            while (x < n_dst && indptr[x + 1] <= e) ++x;
            out[e - e_lo] = sy_src_tid_loc(G, r, e, n_src, x, n_dst, q_thr, n_comm);
        }
    }
}

/* planted-community src tids of given CSC positions with their dst tids (LP positives) */
void sy_indices_at_loc(uint64_t G, int32_t r, int64_t n_src, int64_t n_dst, const int64_t *e, const int64_t *dst,
                       int64_t n, uint32_t q_thr, int32_t n_comm, int32_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = sy_src_tid_loc(G, r, e[i], n_src, dst[i], n_dst, q_thr, n_comm);
}

/* src tids of the given CSC positions of relation r (link-prediction positives) */
void sy_indices_at(uint64_t G, int32_t r, int64_t n_src, const int64_t *e, int64_t n, int32_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = sy_src_tid(G, r, e[i], n_src);
}

void sy_features(uint64_t G, int32_t u, int64_t tid_lo, int64_t tid_hi, int64_t dim,
                 int32_t dtype, void *out)
{
    if (dtype == 0) {
        uint32_t *o = (uint32_t *)out;
#pragma omp parallel for schedule(static)
        for (int64_t t = tid_lo; t < tid_hi; ++t)
            for (int64_t c = 0; c < dim; ++c) o[(t - tid_lo) * dim + c] = sy_feat_f32(G, u, t, c);
    } else {
        uint16_t *o = (uint16_t *)out;
#pragma omp parallel for schedule(static)
        for (int64_t t = tid_lo; t < tid_hi; ++t)
            for (int64_t c = 0; c < dim; ++c) o[(t - tid_lo) * dim + c] = sy_feat_f16(G, u, t, c);
    }
}

/* feature rows of an arbitrary list of tids (rows not materialised on the host) */
void sy_features_ids(uint64_t G, int32_t u, const int64_t *tids, int64_t n, int64_t dim, int32_t dtype,
                     void *out)
{
    if (dtype == 0) {
        uint32_t *o = (uint32_t *)out;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t c = 0; c < dim; ++c) o[i * dim + c] = sy_feat_f32(G, u, tids[i], c);
    } else {
        uint16_t *o = (uint16_t *)out;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t c = 0; c < dim; ++c) o[i * dim + c] = sy_feat_f16(G, u, tids[i], c);
    }
}

/* train ids: tids t in [0, n) with hash(G,'TRN_',t) < thresh (ascending);
 * returns the count (written up to cap). */
int64_t sy_select_train(uint64_t G, int32_t u, int64_t n, uint64_t thresh, int64_t *out, int64_t cap)
{
    int64_t m = 0;
    for (int64_t t = 0; t < n; ++t)
        if (sy_hash(G, SY_TAG_TRN + (uint64_t)u, (uint64_t)t, 0) < thresh) {
            if (m < cap) out[m] = t;
            ++m;
        }
    return m;
}

/* permutation keys for epoch e over a list of ids */
void sy_perm_keys(uint64_t G, int64_t epoch, const int64_t *ids, int64_t n, uint64_t *keys)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) keys[i] = sy_hash(G, SY_TAG_PERM, (uint64_t)epoch, (uint64_t)ids[i]);
}

uint64_t sy_mix(uint64_t x) { return sy_mix64(x); }
