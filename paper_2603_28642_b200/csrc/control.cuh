// Device-side control state of pcgls and the inner CG (shared by the
// single-RHS solver, solver.cu, and the batched one, bsolver.cu), and the
// host/device restatements of the reference's scalar formulas.
#pragma once
#include <cmath>

#include "rsb_internal.h"

namespace rsb {

struct CgState {  // _cg_fixed_steps, pc.py:284-310
    double rho, pq, alpha, rho_new, beta;
    int stop;
};

enum Status { ST_RUN = 0, ST_CONVERGED = 1, ST_STOPPED = 2, ST_MAXED = 3, ST_ZERO_START = 4, ST_ERROR = 5 };

struct CglsState {  // pcgls locals, sv.py:147-241
    double norm_A, delta, b_norm;
    double rho, sigma, alpha, qq, zz, zh, zp, beta, xnorm;
    long long max_iters, iters_run, its_certified, hist_len;
    int d, ratio_raw;
    int status;
    int need_zp, skip_retry, p_copy;
};

struct PowerState {  // power_method_norm2, sc.py:428-454
    double nv, est, nt, result;
    int stop;
};


// Python 3.12 sum() of floats (Neumaier compensated), as used by
// error_estimate (sv.py:101) and the partial-window sums (sv.py:247):
// sum(a*s for ...) with an int 0 start.
__host__ __device__ inline double py_sum_products(const double *a, const double *s, long long lo,
                                                  long long hi) {
    if (hi <= lo) return 0.0;
    double f = 0.0 + a[lo] * s[lo];
    double c = 0.0;
    for (long long k = lo + 1; k < hi; ++k) {
        const double x = a[k] * s[k];
        const double t = f + x;
        if (fabs(f) >= fabs(x))
            c += (f - t) + x;
        else
            c += (x - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

// stopping_ratio, sv.py:104-117 (error flag on a non-positive denominator)
__host__ __device__ inline double py_stopping_ratio(double estim, double norm_A, double x_norm,
                                                    double b_norm, int raw, int *err) {
    const double denom = norm_A * x_norm + b_norm;
    if (denom <= 0.0) {
        *err = 1;
        return 0.0;
    }
    if (estim < 0.0) estim = 0.0;
    const double num = raw ? estim : sqrt(estim);
    return num / denom;
}


}  // namespace rsb

// Mutable state of one preconditioner application stream: vectors, the inner
// CG control block and the triangular-solve scratch.  The preconditioner
// itself is immutable (pc.py:111-113); every user of it -- its own standalone
// entry points and every solver -- owns an ApplyWs, so independent solves can
// run concurrently on different streams.
namespace rsb {
struct ApplyWs {
    rsb_ctx *ctx = nullptr;
    int64_t n = 0, s = 0;
    double *t1 = nullptr, *t2 = nullptr, *t3 = nullptr, *v = nullptr;  // n
    double *u = nullptr, *w = nullptr;                                  // s
    double *cg_r = nullptr, *cg_p = nullptr, *cg_q = nullptr;            // s
    double *cg_a = nullptr, *cg_b = nullptr, *cg_c = nullptr;            // n
    double *cg_b2 = nullptr;  // n: cg_b of the odd inner-CG steps (a solve fills its successor's output, TrsvChain)
    double *r1g = nullptr;    // n: r1 as the first solve gathered it, for the application's second solve with r1
    CgState *cg = nullptr;
    TriWs tri;
    // A solver's own workspace (only enqueue_apply touches it): t1, the first
    // solve's output, holds the sentinel between applications -- filled once
    // at allocation, then by every application's last solve.
    bool carry = false;
};

}  // namespace rsb

struct rsb_pre {
    rsb_ctx *ctx = nullptr;
    int64_t m = 0, n = 0, s = 0;
    int s_mode = 0, y_mode = 0, cg_iters = 0;
    int32_t *perm = nullptr;  // device, length m
    rsb_mat *L1 = nullptr, *L2 = nullptr, *U = nullptr, *Y = nullptr;
    rsb::TriSched *tL1 = nullptr, *tL1T = nullptr, *tU = nullptr;
    double *S = nullptr;  // s x s lower factor, column-major
    rsb::ApplyWs ws;      // for the standalone entry points (pc.py:135-186)
};

