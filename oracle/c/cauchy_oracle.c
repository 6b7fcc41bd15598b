/* Plain-C restatement of the reference's exact-norm Cauchy-like elimination
 * (TEST INFRASTRUCTURE ONLY).
 *
 * Restates /root/reference/pkg/src/rplu/cauchy.py:177-256 (structured_eliminate
 * with plan=None) with exact_row_norms (:129-137) and the generator update
 * (:140-154, :247-250):
 *
 *   u_i = sum_j |(G_i . B_:,j) / (x_i - y_j)|^2     (sequential over j)
 *   stop when max u <= 0 (degenerate) or max u <= tol^2 * u0max (:217-222)
 *   i = sample_index(u, u1) (rplu) or argmax u (c2plu)
 *   r = (G_i . B) / (x_i - y),  j = sample_index(|r|^2, u2) or argmax |r|
 *   |r_j| <= 1e-14 max |r|: one resample of j (rplu), else ZeroDivisionError
 *   c = (G . B_:,j) / (x - y_j)
 *   G -= outer(c / a, G_i),  B -= outer(B_:,j, r / a)
 *
 * Complex arithmetic is C99 `double complex`; the row masses use a different
 * association than numpy's blocked matmul + einsum, so the masses agree to
 * rounding and a draw can only change within rounding of a CDF boundary --
 * the same criterion the dense real restatement is held to.  Row-parallel
 * (OpenMP) over the n row masses and the column / G update.  x, y: complex
 * n / m; G: n x p row-major; Bt: m x p row-major (column j of B contiguous,
 * the reference's F-order B).  Built into oracle/liboracle_c.so.
 */
#include <complex.h>
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { RULE_RPLU = 0, RULE_C2PLU = 1 };
enum { C_OK = 0, C_ZERO_PIVOT = -1, C_ARG = -2, C_UNIFORMS = -3, C_NOMEM = -4 };

typedef double complex cplx;

static int64_t sample_index_c(const double *w, double *cdf, int64_t n, double u, double *margin)
{
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) { s += w[k]; cdf[k] = s; }
    const double total = cdf[n - 1], target = u * total;
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
    if (!(w[k] > 0.0))
        for (k = 0; k < n && !(w[k] > 0.0); ++k) {}
    return k;
}

static int64_t argmax_first(const double *w, int64_t n)
{
    int64_t b = 0;
    for (int64_t k = 1; k < n; ++k)
        if (w[k] > w[b]) b = k;
    return b;
}

/* out: [0] steps, [1] uniforms used, [2] tol stop, [3] degenerate stop,
 * [4] failing step (zero pivot) or -1.  rows / cols [rank]; bmax / bsum
 * [rank] (bound history, one entry per evaluated step); margins [rank];
 * Rrow (optional) rank x m kept pivot rows, Ccol (optional) rank x n kept
 * columns, apiv (optional) rank pivot values. */
int oracle_cauchy(const double *xr, const double *yr, double *Gr, double *Btr, int64_t n,
                  int64_t m, int p, int64_t rank, int rule, const double *uniforms,
                  int64_t n_uniforms, double stop_tol, int threads, int64_t *rows, int64_t *cols,
                  double *bmax, double *bsum, double *margins, double *Rrow, double *Ccol,
                  double *apiv, int64_t *out)
{
    if (threads > 0) omp_set_num_threads(threads);
    if (n <= 0 || m <= 0 || p < 1 || rank < 0 || rank > (n < m ? n : m)) return C_ARG;
    const cplx *x = (const cplx *)xr, *y = (const cplx *)yr;
    cplx *G = (cplx *)Gr, *Bt = (cplx *)Btr;
    double *u = malloc(sizeof(double) * n);
    double *cdf = malloc(sizeof(double) * (n > m ? n : m));
    double *w = malloc(sizeof(double) * m);
    cplx *r = malloc(sizeof(cplx) * m);
    cplx *c = malloc(sizeof(cplx) * n);
    cplx *gi = malloc(sizeof(cplx) * p), *bj = malloc(sizeof(cplx) * p);
    if (!u || !cdf || !w || !r || !c || !gi || !bj) {
        free(u); free(cdf); free(w); free(r); free(c); free(gi); free(bj);
        return C_NOMEM;
    }
    int64_t used = 0, done = 0;
    int status = C_OK;
    double u0max = -1.0;
    out[2] = out[3] = 0;
    out[4] = -1;
    for (int64_t t = 0; t < rank; ++t) {
        /* exact_row_norms (cauchy.py:129-137) */
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            const cplx *g = G + i * p;
            double s = 0.0;
            for (int64_t j = 0; j < m; ++j) {
                const cplx *b = Bt + j * p;
                cplx num = 0.0;
                for (int q = 0; q < p; ++q) num += g[q] * b[q];
                const cplx e = num / (x[i] - y[j]);
                s += creal(e) * creal(e) + cimag(e) * cimag(e);
            }
            u[i] = s;
        }
        double umax = u[0], usum = 0.0;
        for (int64_t i = 0; i < n; ++i) { if (u[i] > umax) umax = u[i]; usum += u[i]; }
        bmax[t] = umax;
        bsum[t] = usum;
        if (u0max < 0.0) u0max = umax;
        if (umax <= 0.0) { out[3] = 1; break; }
        if (stop_tol > 0.0 && umax <= stop_tol * stop_tol * u0max) { out[2] = 1; break; }
        int64_t i;
        double mg = INFINITY, m2 = INFINITY;
        if (rule == RULE_C2PLU) {
            i = argmax_first(u, n);
        } else {
            if (used + 2 > n_uniforms) { status = C_UNIFORMS; break; }
            i = sample_index_c(u, cdf, n, uniforms[used++], &mg);
        }
        memcpy(gi, G + i * p, sizeof(cplx) * p);
        double rmax = 0.0;
        for (int64_t j = 0; j < m; ++j) {
            cplx num = 0.0;
            for (int q = 0; q < p; ++q) num += gi[q] * Bt[j * p + q];
            r[j] = num / (x[i] - y[j]);
            const double ab = cabs(r[j]);
            w[j] = ab * ab;
            if (ab > rmax) rmax = ab;
        }
        int64_t j;
        if (rule == RULE_C2PLU) {
            j = argmax_first(w, m);
        } else {
            j = sample_index_c(w, cdf, m, uniforms[used++], &m2);
            if (m2 < mg) mg = m2;
        }
        cplx a = r[j];
        const double thr = 1e-14 * rmax;
        if (cabs(a) <= thr) {
            if (rule == RULE_C2PLU || used + 1 > n_uniforms) { status = C_ZERO_PIVOT; out[4] = t; break; }
            j = sample_index_c(w, cdf, m, uniforms[used++], NULL);
            a = r[j];
            if (cabs(a) <= thr) { status = C_ZERO_PIVOT; out[4] = t; break; }
        }
        memcpy(bj, Bt + j * p, sizeof(cplx) * p);
        #pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < n; ++k) {
            cplx num = 0.0;
            for (int q = 0; q < p; ++q) num += G[k * p + q] * bj[q];
            c[k] = num / (x[k] - y[j]);
        }
        /* G -= outer(c / a, G_i); B -= outer(B_:,j, r / a) */
        #pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < n; ++k) {
            const cplx ca = c[k] / a;
            for (int q = 0; q < p; ++q) G[k * p + q] -= ca * gi[q];
        }
        #pragma omp parallel for schedule(static)
        for (int64_t l = 0; l < m; ++l) {
            const cplx ra = r[l] / a;
            for (int q = 0; q < p; ++q) Bt[l * p + q] -= bj[q] * ra;
        }
        rows[t] = i;
        cols[t] = j;
        margins[t] = mg;
        if (Rrow) memcpy(Rrow + 2 * t * m, r, sizeof(cplx) * m);
        if (Ccol) memcpy(Ccol + 2 * t * n, c, sizeof(cplx) * n);
        if (apiv) { apiv[2 * t] = creal(a); apiv[2 * t + 1] = cimag(a); }
        done = t + 1;
    }
    out[0] = done;
    out[1] = used;
    free(u); free(cdf); free(w); free(r); free(c); free(gi); free(bj);
    return status;
}
