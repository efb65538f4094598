/*
 * oracle/rsfast.c -- multi-threaded evaluation of the oracle's kernels.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/rsref.c).  bench.py's reference arm
 * times the oracle port "with all the host threads it can use"; this file
 * gives it OpenMP versions of the reference kernels that produce the SAME
 * BITS as the sequential restatements in rsref.c (pinned by
 * tests/test_oracle_pin.py::test_fast_kernels_match_sequential):
 *
 *   matvec (sc.py:212-221): np.add.at accumulates row i's products in
 *     ascending column order from 0.0 -> a CSR row-sequential sum; rows are
 *     independent, so they are split over threads.
 *   matvec_transpose (sc.py:224-235): one reduceat segment per column,
 *     columns split over threads.
 *   sparse_lower_solve / sparse_upper_solve (sc.py:243-279): every unknown
 *     receives the column updates in the same order as the column sweep
 *     (ascending / descending columns, skipped when x_j == 0), so the row
 *     form computes identical values; unknowns of one dependency level are
 *     independent and split over threads, levels in order.
 *   sparse_lower_solve_transpose (sc.py:282-298): one gathered OpenBLAS dot
 *     per unknown (rsref.c's order), levels in order.
 *   ddot with T OpenBLAS threads: T chunk dots on T threads, summed in chunk
 *     order (the reference's blas_level1_thread order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

double rso_blas_dot(int64_t n, const double *x, const double *y);
double rso_pairwise_sum(const double *a, int64_t n);

/* CSC (m x n) -> CSR with columns ascending inside each row */
void rsf_csr(int64_t m, int64_t n, const int64_t *cp, const int64_t *ri, const double *cv, int64_t *rp,
             int64_t *ci, double *rv)
{
    memset(rp, 0, (size_t)(m + 1) * sizeof(int64_t));
    for (int64_t k = 0; k < cp[n]; k++) rp[ri[k] + 1]++;
    for (int64_t i = 0; i < m; i++) rp[i + 1] += rp[i];
    int64_t *fill = malloc((size_t)(m + 1) * sizeof(int64_t));
    memcpy(fill, rp, (size_t)(m + 1) * sizeof(int64_t));
    for (int64_t j = 0; j < n; j++)
        for (int64_t k = cp[j]; k < cp[j + 1]; k++) {
            int64_t d = fill[ri[k]]++;
            ci[d] = j;
            rv[d] = cv[k];
        }
    free(fill);
}

void rsf_matvec_csr(int64_t m, const int64_t *rp, const int64_t *ci, const double *rv, const double *x, double *y)
{
#pragma omp parallel for schedule(static, 4096)
    for (int64_t i = 0; i < m; i++) {
        double acc = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            double c = rv[k] * x[ci[k]];
            acc = acc + c;
        }
        y[i] = acc;
    }
}

void rsf_matvec_t(int64_t n, const int64_t *cp, const int64_t *ri, const double *cv, const double *y, double *z,
                  int64_t maxlen)
{
#pragma omp parallel
    {
        double *s = malloc((size_t)(maxlen > 0 ? maxlen : 1) * sizeof(double));
#pragma omp for schedule(static, 4096)
        for (int64_t j = 0; j < n; j++) {
            int64_t lo = cp[j], hi = cp[j + 1];
            if (hi == lo) {
                z[j] = 0.0;
                continue;
            }
            for (int64_t k = lo; k < hi; k++) s[k - lo] = cv[k] * y[ri[k]];
            z[j] = s[0] + rso_pairwise_sum(s + 1, hi - lo - 1);
        }
        free(s);
    }
}

/* Dependency levels.  kind 0: forward row form (CSR, deps = columns < i);
 * kind 1: backward row form (CSR, deps = columns > i); kind 2: transposed
 * lower (CSC, deps = rows > j).  Writes order[] (unknowns grouped by level,
 * ascending inside a level) and lev_ptr[0..nlev]; returns nlev. */
int64_t rsf_levels(int64_t n, const int64_t *ptr, const int64_t *idx, int kind, int64_t *order, int64_t *lev_ptr)
{
    int64_t *lev = malloc((size_t)n * sizeof(int64_t));
    int64_t nlev = 0;
    for (int64_t t = 0; t < n; t++) {
        const int64_t i = kind == 0 ? t : n - 1 - t;
        int64_t l = 0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
            const int64_t j = idx[k];
            if ((kind == 0 && j < i) || (kind != 0 && j > i))
                if (lev[j] + 1 > l) l = lev[j] + 1;
        }
        lev[i] = l;
        if (l + 1 > nlev) nlev = l + 1;
    }
    memset(lev_ptr, 0, (size_t)(nlev + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) lev_ptr[lev[i] + 1]++;
    for (int64_t l = 0; l < nlev; l++) lev_ptr[l + 1] += lev_ptr[l];
    int64_t *fill = malloc((size_t)(nlev + 1) * sizeof(int64_t));
    memcpy(fill, lev_ptr, (size_t)(nlev + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) order[fill[lev[i]]++] = i;
    free(fill);
    free(lev);
    return nlev;
}

/* sparse_lower_solve(L, b, unit_diag=True), L strictly lower, CSR */
void rsf_lower_unit(int64_t n, const int64_t *rp, const int64_t *ci, const double *rv, const double *b, double *x,
                    int64_t nlev, const int64_t *order, const int64_t *lev_ptr)
{
    for (int64_t l = 0; l < nlev; l++) {
#pragma omp parallel for schedule(static, 1024)
        for (int64_t t = lev_ptr[l]; t < lev_ptr[l + 1]; t++) {
            const int64_t i = order[t];
            double acc = b[i];
            for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
                const double xj = x[ci[k]];
                if (xj != 0.0) {
                    double c = rv[k] * xj;
                    acc = acc - c;
                }
            }
            x[i] = acc;
        }
    }
    (void)n;
}

/* sparse_upper_solve(U, b), diagonal stored in every row (CSR: last entry
 * of row i is at column >= i; the diagonal is the entry at column i) */
void rsf_upper(int64_t n, const int64_t *rp, const int64_t *ci, const double *rv, const double *b, double *x,
               int64_t nlev, const int64_t *order, const int64_t *lev_ptr)
{
    for (int64_t l = 0; l < nlev; l++) {
#pragma omp parallel for schedule(static, 1024)
        for (int64_t t = lev_ptr[l]; t < lev_ptr[l + 1]; t++) {
            const int64_t i = order[t];
            double acc = b[i];
            double d = 0.0;
            for (int64_t k = rp[i + 1] - 1; k >= rp[i]; k--) {
                const int64_t j = ci[k];
                if (j == i) {
                    d = rv[k];
                    continue;
                }
                const double xj = x[j];
                if (xj != 0.0) {
                    double c = rv[k] * xj;
                    acc = acc - c;
                }
            }
            x[i] = acc / d;
        }
    }
    (void)n;
}

/* the gathered dot of rsref.c for columns up to 256 entries */
static double gdot(const double *v, const int64_t *idx, const double *x, int64_t n)
{
    double buf[256];
    for (int64_t k = 0; k < n; k++) buf[k] = x[idx[k]];
    return rso_blas_dot(n, v, buf);
}

/* sparse_lower_solve_transpose(L, b, unit_diag=True), CSC; columns <= 256 */
void rsf_lower_t_unit(int64_t n, const int64_t *cp, const int64_t *ri, const double *cv, const double *b, double *x,
                      int64_t nlev, const int64_t *order, const int64_t *lev_ptr)
{
    for (int64_t l = 0; l < nlev; l++) {
#pragma omp parallel for schedule(static, 1024)
        for (int64_t t = lev_ptr[l]; t < lev_ptr[l + 1]; t++) {
            const int64_t j = order[t];
            double xj = b[j];
            const int64_t lo = cp[j], hi = cp[j + 1];
            if (hi > lo) xj -= gdot(cv + lo, ri + lo, x, hi - lo);
            x[j] = xj;
        }
    }
    (void)n;
}

/* a @ b with T OpenBLAS threads: chunk widths ceil(rest / threads left) */
double rsf_dot(int64_t n, const double *a, const double *b, int T)
{
    if (T <= 1 || n <= 10000) return rso_blas_dot(n, a, b);
    int64_t lo[64], w[64];
    int64_t rest = n, off = 0;
    for (int t = 0; t < T; t++) {
        w[t] = (rest + (T - t) - 1) / (T - t);
        lo[t] = off;
        off += w[t];
        rest -= w[t];
    }
    double part[64];
#pragma omp parallel for schedule(static, 1)
    for (int t = 0; t < T; t++) part[t] = rso_blas_dot(w[t], a + lo[t], b + lo[t]);
    double s = 0.0;
    for (int t = 0; t < T; t++) s = s + part[t];
    return s;
}

/* elementwise helpers the oracle loop needs at config-4 size (numpy's
 * single-threaded ops would dominate the timed iteration otherwise); each
 * is the one IEEE operation numpy performs per element */
void rsf_axpy(int64_t n, double *y, double a, const double *x, int sign) /* y += a*x | y -= a*x */
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double c = a * x[i];
        y[i] = sign > 0 ? y[i] + c : y[i] - c;
    }
}

void rsf_xpby(int64_t n, double *out, const double *h, double beta, const double *p) /* out = h + beta*p */
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double c = beta * p[i];
        out[i] = h[i] + c;
    }
}

void rsf_gather(int64_t n, double *out, const double *r, const int64_t *perm)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) out[i] = r[perm[i]];
}

void rsf_sub(int64_t n, double *out, const double *a, const double *b) /* out = a - b */
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) out[i] = a[i] - b[i];
}

void rsf_add(int64_t n, double *out, const double *a, const double *b) /* out = a + b */
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) out[i] = a[i] + b[i];
}

void rsf_copy(int64_t n, double *out, const double *a)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) out[i] = a[i];
}

void rsf_scale_div(int64_t n, double *out, const double *a, double d) /* out = a / d */
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) out[i] = a[i] / d;
}

int rsf_max_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void rsf_set_threads(int t)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(t);
#else
    (void)t;
#endif
}
