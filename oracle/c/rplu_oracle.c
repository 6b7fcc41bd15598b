/* Plain-C restatement of the reference's dense Alg 1 (TEST INFRASTRUCTURE ONLY).
 *
 * Restates /root/reference/pkg/src/rplu/dense_pivots.py:129-209 (eliminate)
 * with _draw_rank1_pivot (:103-126) and rng.py:50-74 (sample_index) for real
 * float64 residuals -- the reference's complex128 arithmetic with a zero
 * imaginary part:
 *
 *   * row masses  einsum("ij,ij->i", R, R.conj()).real: a sequential
 *     left-to-right sum of r*r per row (the order numpy's einsum uses for this
 *     contraction), no FMA contraction;
 *   * column weights |r|^2 = r*r;
 *   * sample_index: sequential cumsum, first running sum > u*total
 *     (searchsorted side='right'), clamp to the last index, walk back over
 *     zero weights, else the first positive weight;
 *   * update  col = R[:,j] * (1/a)  (numpy's complex division by a real-valued
 *     complex, Smith's algorithm with rat = 0), R -= outer(col, row) with one
 *     rounding for the product and one for the difference;
 *   * one zero-pivot resample, then an error (:178-184); clean stop when the
 *     residual is exactly zero (:162-164); tol stop (:195-197).
 *
 * The update of step t and the row masses of step t+1 are fused into one pass
 * over R (row-parallel, OpenMP; every row's arithmetic is independent of the
 * thread split, so results do not depend on the thread count).  resid_fro is
 * sqrt(sum of the row masses) -- equal to the reference's np.linalg.norm(R) to
 * rounding (the tests compare it at rtol 1e-12).
 *
 * With `forced` != NULL the pivots are given (forced-pivot replay,
 * dense_pivots.py:185-191 with the pivots of another run), used to grade the
 * fp32 GPU factors against fp64.
 *
 * Built by oracle/Makefile into oracle/liboracle_c.so; bound by
 * oracle/c_oracle.py.  Only tests/, smoke() and bench.py's CPU legs use it.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { RULE_RPLU = 0, RULE_C2PLU = 1, RULE_CPLU = 2 };
enum { ORC_OK = 0, ORC_ZERO_PIVOT = -1, ORC_ARG = -2, ORC_UNIFORMS = -3, ORC_NOMEM = -4 };

/* rng.py:50-74 over w[0..n) with running sums in cdf; returns the index and
 * the relative distance of u*total to the nearest CDF boundary. */
static int64_t sample_index(const double *w, double *cdf, int64_t n, double u, double *margin)
{
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        s += w[k];
        cdf[k] = s;
    }
    double total = cdf[n - 1];
    double target = u * total;
    /* searchsorted(cdf, target, side='right'): first k with cdf[k] > target */
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (cdf[mid] > target) hi = mid; else lo = mid + 1;
    }
    int64_t k = lo < n - 1 ? lo : n - 1;
    if (margin) {
        double below = k > 0 ? cdf[k - 1] : 0.0;
        double a = fabs(target - below), b = fabs(cdf[k] - target);
        *margin = (a < b ? a : b) / total;
    }
    while (k > 0 && !(w[k] > 0.0)) --k;
    if (!(w[k] > 0.0)) {
        for (k = 0; k < n && !(w[k] > 0.0); ++k) {}
    }
    return k;
}

static int64_t argmax_first(const double *w, int64_t n)
{
    int64_t best = 0;
    for (int64_t k = 1; k < n; ++k)
        if (w[k] > w[best]) best = k;
    return best;
}

/* One generic dense loop per residual type T (float64: the reference's
 * arithmetic; float32: the same steps with one float rounding per product and
 * difference and 1/a rounded to float -- the C3-fp32 configuration, for which
 * no reference exists).  Masses and weights are always float64 sums of
 * (double)r * (double)r. */
#define DEFINE_DENSE(T, SUF)                                                              \
static int draw_##SUF(const T *R, int64_t n, int64_t m, int rule, const double *masses,    \
                      double *cdf, double *wrow, const double *uniforms,                  \
                      int64_t n_uniforms, int64_t *used, int64_t *pi, int64_t *pj,        \
                      double *margin)                                                     \
{                                                                                         \
    if (rule == RULE_CPLU) {                                                              \
        double best = -1.0;                                                               \
        int64_t bi = 0, bj = 0;                                                           \
        for (int64_t i = 0; i < n; ++i)                                                   \
            for (int64_t j = 0; j < m; ++j) {                                             \
                double v = fabs((double)R[i * m + j]);                                    \
                if (v > best) { best = v; bi = i; bj = j; }                               \
            }                                                                             \
        *pi = bi; *pj = bj;                                                               \
        return ORC_OK;                                                                    \
    }                                                                                     \
    if (rule == RULE_C2PLU) {                                                             \
        int64_t i = argmax_first(masses, n);                                              \
        for (int64_t j = 0; j < m; ++j) wrow[j] = fabs((double)R[i * m + j]);             \
        *pi = i;                                                                          \
        *pj = argmax_first(wrow, m);                                                      \
        return ORC_OK;                                                                    \
    }                                                                                     \
    if (*used + 2 > n_uniforms) return ORC_UNIFORMS;                                      \
    double m1 = 0.0, m2 = 0.0;                                                            \
    int64_t i = sample_index(masses, cdf, n, uniforms[(*used)++], &m1);                   \
    for (int64_t j = 0; j < m; ++j) {                                                     \
        double r = (double)R[i * m + j];                                                  \
        wrow[j] = r * r;                                                                  \
    }                                                                                     \
    int64_t j = sample_index(wrow, cdf, m, uniforms[(*used)++], &m2);                     \
    *pi = i; *pj = j;                                                                     \
    if (margin) *margin = m1 < m2 ? m1 : m2;                                              \
    return ORC_OK;                                                                        \
}                                                                                         \
                                                                                          \
int oracle_dense_##SUF(T *R, int64_t n, int64_t m, int64_t steps, int rule,               \
                       const double *uniforms, int64_t n_uniforms, const int64_t *forced, \
                       double stop_tol, int threads, int64_t *pivots, T *Lt, T *U,        \
                       double *resid_fro, double *margins, int64_t *out)                  \
{                                                                                         \
    if (threads > 0) omp_set_num_threads(threads);                                        \
    if (n <= 0 || m <= 0 || steps < 0 || steps > (n < m ? n : m) || stop_tol < 0.0)       \
        return ORC_ARG;                                                                   \
    double *masses = malloc(sizeof(double) * n);                                          \
    double *cdf = malloc(sizeof(double) * (n > m ? n : m));                               \
    double *wrow = malloc(sizeof(double) * m);                                            \
    T *row = malloc(sizeof(T) * m);                                                       \
    if (!masses || !cdf || !wrow || !row) {                                               \
        free(masses); free(cdf); free(wrow); free(row);                                   \
        return ORC_NOMEM;                                                                 \
    }                                                                                     \
    int64_t used = 0, done = 0;                                                           \
    int status = ORC_OK;                                                                  \
    out[2] = out[3] = 0;                                                                  \
    out[4] = -1;                                                                          \
    _Pragma("omp parallel for schedule(static)")                                          \
    for (int64_t i = 0; i < n; ++i) {                                                     \
        const T *r = R + i * m;                                                           \
        double s = 0.0;                                                                   \
        for (int64_t j = 0; j < m; ++j) s += (double)r[j] * (double)r[j];                 \
        masses[i] = s;                                                                    \
    }                                                                                     \
    double fro0 = fro_of(masses, n);                                                      \
    resid_fro[0] = fro0;                                                                  \
    for (int64_t t = 0; t < steps; ++t) {                                                 \
        if (resid_fro[t] == 0.0) { out[2] = 1; break; }                                   \
        int64_t i, j;                                                                     \
        double mg = INFINITY;                                                             \
        if (forced) {                                                                     \
            i = forced[2 * t];                                                            \
            j = forced[2 * t + 1];                                                        \
        } else {                                                                          \
            status = draw_##SUF(R, n, m, rule, masses, cdf, wrow, uniforms, n_uniforms,   \
                                &used, &i, &j, &mg);                                      \
            if (status) break;                                                            \
        }                                                                                 \
        T a = R[i * m + j];                                                               \
        if (a == 0 && !forced) {                                                          \
            double mg2 = INFINITY;                                                        \
            status = draw_##SUF(R, n, m, rule, masses, cdf, wrow, uniforms, n_uniforms,   \
                                &used, &i, &j, &mg2);                                     \
            if (status) break;                                                            \
            mg = mg < mg2 ? mg : mg2;                                                     \
            a = R[i * m + j];                                                             \
        }                                                                                 \
        if (a == 0) { status = ORC_ZERO_PIVOT; out[4] = t; break; }                       \
        const T inv = (T)1 / a;                                                           \
        memcpy(row, R + i * m, sizeof(T) * m);                                            \
        T *lt = Lt + t * n;                                                               \
        /* update step t fused with the masses of step t+1 */                             \
        _Pragma("omp parallel for schedule(static)")                                      \
        for (int64_t k = 0; k < n; ++k) {                                                 \
            T *r = R + k * m;                                                             \
            const T c = r[j] * inv;                                                       \
            lt[k] = c;                                                                    \
            double s = 0.0;                                                               \
            for (int64_t q = 0; q < m; ++q) {                                             \
                const T p = c * row[q];                                                   \
                const T v = r[q] - p;                                                     \
                r[q] = v;                                                                 \
                s += (double)v * (double)v;                                               \
            }                                                                             \
            masses[k] = s;                                                                \
        }                                                                                 \
        memcpy(U + t * m, row, sizeof(T) * m);                                            \
        pivots[2 * t] = i;                                                                \
        pivots[2 * t + 1] = j;                                                            \
        if (margins) margins[t] = mg;                                                     \
        done = t + 1;                                                                     \
        resid_fro[t + 1] = fro_of(masses, n);                                             \
        if (stop_tol > 0.0 && resid_fro[t + 1] <= stop_tol * fro0) { out[3] = 1; break; } \
    }                                                                                     \
    out[0] = done;                                                                        \
    out[1] = used;                                                                        \
    free(masses); free(cdf); free(wrow); free(row);                                       \
    return status;                                                                        \
}

static double fro_of(const double *masses, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += masses[i];
    return sqrt(s);
}

/* out[0] steps done, out[1] uniforms consumed, out[2] clean stop, out[3] tol
 * stop, out[4] failing step (zero pivot) or -1.  Lt is steps x n, U steps x m;
 * margins (optional) one per step (the smaller of the row and column draw). */
DEFINE_DENSE(double, f64)
DEFINE_DENSE(float, f32)
