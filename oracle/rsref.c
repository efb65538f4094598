/*
 * oracle/rsref.c -- CPU restatement of the reference's sparse kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 path; nothing in paper_2603_28642_b200/ links or calls it.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load liboracle_rsref.so.
 *
 * Each function restates one kernel of the reference package `rowsplit`
 * (pkg/src/rowsplit/sparse_core.py, abbreviated sc.py below) in the exact
 * floating-point operation order numpy + OpenBLAS use there, so results
 * are bit-identical to the reference on the same inputs:
 *
 *   matvec                    sc.py:212-221  np.add.at scatter: y starts at 0.0,
 *                                            contributions added in CSC order
 *   matvec_transpose          sc.py:224-235  np.add.reduceat: z_j = p0 + pairwise(p1..)
 *                                            (numpy's pairwise summation, blocks of 8,
 *                                            PW_BLOCKSIZE 128)
 *   sparse_lower_solve        sc.py:243-263  column axpy, skip when x_j == 0
 *   sparse_upper_solve        sc.py:266-279  column axpy from the last column
 *   sparse_lower_solve_transpose sc.py:282-298  x_j -= vals @ x[rows]: OpenBLAS ddot
 *                                            (rso_blas_dot: the SkylakeX kernel's order)
 *   sparse_upper_solve_transpose sc.py:301-313  same dot recipe
 *   dense_cholesky_factorize  sc.py:585-604  right-looking, elementwise outer update
 *   dense_cholesky_solve      sc.py:607-622  forward column axpy; backward ddot
 *   rso_blas_dot              every `a @ b` / np.linalg.norm of 1-D float64 in the
 *                                            reference (sv.py, pc.py), single-threaded
 *                                            OpenBLAS; bit-exact vs numpy on the survey host
 *
 * Compiled with -ffp-contract=off so every a*b+c below is two roundings
 * unless fma() is written explicitly.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define RSO_OK 0
#define RSO_ESINGULAR 2

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * DOUBLE_pairwise_sum), restated: n < 8 sequential from -0.0; n <= 128
 * eight strided accumulators; larger n split at n/2 rounded down to a
 * multiple of 8. */
static double pairwise_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; k++) r[k] = a[k];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}


/* OpenBLAS 0.3.30 ddot as the reference host runs it (scipy-openblas,
 * DYNAMIC_ARCH SkylakeX kernel, one thread: kernel/x86_64/ddot.c with
 * ddot_microk_skylakex-2.c), restated as its association order:
 *   n1 = n & -16 elements go through the vector kernel: blocks of 32 into
 *   four 8-wide FMA accumulators, each folded 8 -> 4 (lo + hi half); a
 *   remaining block of 16 into four 4-wide FMA accumulators; then
 *   ((a0 + a1) + a2) + a3 lane-wise, (t0 + t2) + (t1 + t3);
 *   the n - n1 tail is a scalar FMA chain onto that.
 * Verified bitwise against numpy `@` on the survey host (tests/test_oracle_pin.py). */
double rso_blas_dot(int64_t n, const double *x, const double *y)
{
    int64_t n1 = n & ~(int64_t)15;
    double dot = 0.0;
    if (n1) {
        double a5[4][8];
        for (int g = 0; g < 4; g++) for (int k = 0; k < 8; k++) a5[g][k] = 0.0;
        int64_t n32 = n1 & ~(int64_t)31, i = 0;
        for (; i < n32; i += 32)
            for (int g = 0; g < 4; g++)
                for (int k = 0; k < 8; k++)
                    a5[g][k] = fma(x[i + 8 * g + k], y[i + 8 * g + k], a5[g][k]);
        double a[4][4];
        for (int g = 0; g < 4; g++) for (int k = 0; k < 4; k++) a[g][k] = a5[g][k] + a5[g][k + 4];
        for (; i < n1; i += 16)
            for (int g = 0; g < 4; g++)
                for (int k = 0; k < 4; k++)
                    a[g][k] = fma(x[i + 4 * g + k], y[i + 4 * g + k], a[g][k]);
        double t[4];
        for (int k = 0; k < 4; k++) t[k] = ((a[0][k] + a[1][k]) + a[2][k]) + a[3][k];
        dot = (t[0] + t[2]) + (t[1] + t[3]);
    }
    for (int64_t i = n1; i < n; i++) dot = fma(y[i], x[i], dot);
    return dot;
}

double rso_pairwise_sum(const double *a, int64_t n) { return pairwise_sum(a, n); }

/* y = A x, sc.py:212-221. */
void rso_matvec(int64_t nrows, int64_t ncols, const int64_t *col_ptr, const int64_t *row_idx,
                const double *vals, const double *x, double *y)
{
    for (int64_t i = 0; i < nrows; i++) y[i] = 0.0;
    for (int64_t j = 0; j < ncols; j++) {
        double xj = x[j];
        for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; k++) {
            double c = vals[k] * xj;
            y[row_idx[k]] = y[row_idx[k]] + c;
        }
    }
}

/* z = A^T y, sc.py:224-235.  scratch must hold max column length. */
void rso_matvec_transpose(int64_t nrows, int64_t ncols, const int64_t *col_ptr,
                          const int64_t *row_idx, const double *vals, const double *y,
                          double *z, double *scratch)
{
    (void)nrows;
    for (int64_t j = 0; j < ncols; j++) {
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        if (hi == lo) { z[j] = 0.0; continue; }
        for (int64_t k = lo; k < hi; k++) scratch[k - lo] = vals[k] * y[row_idx[k]];
        z[j] = scratch[0] + pairwise_sum(scratch + 1, hi - lo - 1);
    }
}

/* sc.py:243-263.  Returns the failing column + 1 as -(col+1) on a missing diagonal. */
int64_t rso_lower_solve(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                        const double *vals, const double *b, double *x, int unit_diag)
{
    memcpy(x, b, (size_t)n * sizeof(double));
    for (int64_t j = 0; j < n; j++) {
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        if (!unit_diag) {
            if (hi == lo || row_idx[lo] != j || vals[lo] == 0.0) return -(j + 1);
            x[j] /= vals[lo];
            lo += 1;
        }
        double xj = x[j];
        if (xj != 0.0 && hi > lo)
            for (int64_t k = lo; k < hi; k++) {
                double c = vals[k] * xj;
                x[row_idx[k]] = x[row_idx[k]] - c;
            }
    }
    return RSO_OK;
}

/* sc.py:266-279. */
int64_t rso_upper_solve(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                        const double *vals, const double *b, double *x)
{
    memcpy(x, b, (size_t)n * sizeof(double));
    for (int64_t j = n - 1; j >= 0; j--) {
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        if (hi == lo || row_idx[hi - 1] != j || vals[hi - 1] == 0.0) return -(j + 1);
        x[j] /= vals[hi - 1];
        double xj = x[j];
        if (xj != 0.0 && hi - 1 > lo)
            for (int64_t k = lo; k < hi - 1; k++) {
                double c = vals[k] * xj;
                x[row_idx[k]] = x[row_idx[k]] - c;
            }
    }
    return RSO_OK;
}

/* x_j -= vals @ x[rows] in the reference: numpy gathers x[rows] into a
 * contiguous temporary and calls ddot -- the recipe above. */
static double gathered_dot(const double *v, const int64_t *idx, const double *x, int64_t n)
{
    double buf[256];
    if (n <= 256) {
        for (int64_t k = 0; k < n; k++) buf[k] = x[idx[k]];
        return rso_blas_dot(n, v, buf);
    }
    /* long columns: same association, gathered on the fly */
    int64_t n1 = n & ~(int64_t)15;
    double dot = 0.0;
    if (n1) {
        double a5[4][8];
        for (int g = 0; g < 4; g++) for (int k = 0; k < 8; k++) a5[g][k] = 0.0;
        int64_t n32 = n1 & ~(int64_t)31, i = 0;
        for (; i < n32; i += 32)
            for (int g = 0; g < 4; g++)
                for (int k = 0; k < 8; k++)
                    a5[g][k] = fma(v[i + 8 * g + k], x[idx[i + 8 * g + k]], a5[g][k]);
        double a[4][4];
        for (int g = 0; g < 4; g++) for (int k = 0; k < 4; k++) a[g][k] = a5[g][k] + a5[g][k + 4];
        for (; i < n1; i += 16)
            for (int g = 0; g < 4; g++)
                for (int k = 0; k < 4; k++)
                    a[g][k] = fma(v[i + 4 * g + k], x[idx[i + 4 * g + k]], a[g][k]);
        double t[4];
        for (int k = 0; k < 4; k++) t[k] = ((a[0][k] + a[1][k]) + a[2][k]) + a[3][k];
        dot = (t[0] + t[2]) + (t[1] + t[3]);
    }
    for (int64_t i = n1; i < n; i++) dot = fma(x[idx[i]], v[i], dot);
    return dot;
}

/* sc.py:282-298. */
int64_t rso_lower_solve_transpose(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                  const double *vals, const double *b, double *x, int unit_diag)
{
    memcpy(x, b, (size_t)n * sizeof(double));
    for (int64_t j = n - 1; j >= 0; j--) {
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        if (unit_diag) {
            if (hi > lo) x[j] -= gathered_dot(vals + lo, row_idx + lo, x, hi - lo);
        } else {
            if (hi == lo || row_idx[lo] != j || vals[lo] == 0.0) return -(j + 1);
            if (hi > lo + 1) x[j] -= gathered_dot(vals + lo + 1, row_idx + lo + 1, x, hi - lo - 1);
            x[j] /= vals[lo];
        }
    }
    return RSO_OK;
}

/* sc.py:301-313. */
int64_t rso_upper_solve_transpose(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                  const double *vals, const double *b, double *x)
{
    memcpy(x, b, (size_t)n * sizeof(double));
    for (int64_t j = 0; j < n; j++) {
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        if (hi == lo || row_idx[hi - 1] != j || vals[hi - 1] == 0.0) return -(j + 1);
        if (hi - 1 > lo) x[j] -= gathered_dot(vals + lo, row_idx + lo, x, hi - 1 - lo);
        x[j] /= vals[hi - 1];
    }
    return RSO_OK;
}

/* sc.py:585-604; g is s x s column-major, overwritten by the lower factor. */
int64_t rso_cholesky_factorize(int64_t s, double *g)
{
    for (int64_t j = 0; j < s; j++) {
        double d = g[j + j * s];
        if (d <= 0.0 || !isfinite(d)) return -(j + 1);
        d = sqrt(d);
        g[j + j * s] = d;
        for (int64_t i = j + 1; i < s; i++) g[i + j * s] /= d;
        for (int64_t k = j + 1; k < s; k++)
            for (int64_t i = j + 1; i < s; i++) {
                double c = g[i + j * s] * g[k + j * s];
                g[i + k * s] = g[i + k * s] - c;
            }
    }
    for (int64_t k = 1; k < s; k++)
        for (int64_t i = 0; i < k; i++) g[i + k * s] = 0.0; /* np.tril */
    return RSO_OK;
}

/* sc.py:607-622; g column-major lower factor. */
void rso_cholesky_solve(int64_t s, const double *g, const double *b, double *x)
{
    memcpy(x, b, (size_t)s * sizeof(double));
    for (int64_t j = 0; j < s; j++) {
        x[j] /= g[j + j * s];
        for (int64_t i = j + 1; i < s; i++) {
            double c = g[i + j * s] * x[j];
            x[i] = x[i] - c;
        }
    }
    for (int64_t j = s - 1; j >= 0; j--) {
        if (j + 1 < s) {
            x[j] -= rso_blas_dot(s - j - 1, g + (j + 1) + j * s, x + j + 1);
        }
        x[j] /= g[j + j * s];
    }
}
