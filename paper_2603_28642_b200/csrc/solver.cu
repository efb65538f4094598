// Preconditioner application, device-resident pcgls and the power method.
//
// The host never looks at a scalar inside an iteration: dots land in a
// device-side state block, one-thread "control" kernels evaluate the
// reference's branches there, and every vector kernel carries a Gate that
// turns it into a no-op once the control state says the reference would
// have left the loop.  One pcgls iteration is captured once as a CUDA graph
// and replayed; the host only polls the 4-byte status between batches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "control.cuh"
#include "rsb_internal.h"

namespace rsb {

// ---------------------------------------------------------------------------
// device control state
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ bool gated(const Gate &g) {
    return (g.a && *(volatile const int *)g.a) || (g.b && *(volatile const int *)g.b);
}

// ---- inner CG control (pc.py:291-309) ----
__global__ void k_cg_start(CgState *cg, Gate g) {  // rho = r@r; if rho == 0: return w (=0)
    if (gated(g)) return;
    cg->stop = (cg->rho == 0.0) ? 1 : 0;
}
__global__ void k_cg_alpha(CgState *cg, Gate g) {  // pq <= 0: break; alpha = rho/pq
    if (gated(g)) return;
    if (cg->pq <= 0.0)
        cg->stop = 1;
    else
        cg->alpha = cg->rho / cg->pq;
}
__global__ void k_cg_beta(CgState *cg, Gate g) {  // rho_new == 0: break; p = r + (rho_new/rho) p
    if (gated(g)) return;
    if (cg->rho_new == 0.0) {
        cg->stop = 1;
    } else {
        cg->beta = cg->rho_new / cg->rho;
        cg->rho = cg->rho_new;
    }
}
__global__ void k_cg_init(double *w, double *r, double *p, const double *u, int64_t s, Gate g) {
    if (gated(g)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
        w[i] = 0.0;
        r[i] = u[i];
        p[i] = u[i];
    }
}

// ---- pcgls control (sv.py:184-241) ----
__global__ void k_start_check(CglsState *st) {  // sv.py:184: z@z == 0 -> x = 0 stationary
    st->iters_run = 0;
    st->its_certified = 0;
    st->hist_len = 0;
    st->status = (st->zz == 0.0) ? ST_ZERO_START : ST_RUN;
}
__global__ void k_start_rho(CglsState *st, double *x_norms) {  // sv.py:198-199
    if (st->status) return;
    st->rho = st->zh;
    x_norms[0] = 0.0;
}
__global__ void k_it_begin(CglsState *st) {  // need z@p only when rho <= 0 (sv.py:203)
    if (st->status) return;
    st->need_zp = !(st->rho > 0.0);
}
__global__ void k_it_sigma(CglsState *st) {  // sv.py:203-208
    if (st->status) return;
    st->sigma = st->rho > 0.0 ? st->rho : st->zp;
    st->skip_retry = 1;
    if (st->sigma == 0.0) {
        st->skip_retry = 0;  // p = z.copy()
        st->sigma = st->zz;  // float(z @ z): the same z whose z@z is stored
        st->rho = st->sigma;
    }
}
__global__ void k_it_alpha(CglsState *st) {  // sv.py:210-214
    if (st->status) return;
    if (st->qq <= 0.0 || st->sigma == 0.0)
        st->status = ST_STOPPED;
    else
        st->alpha = st->sigma / st->qq;
}
__global__ void k_it_estimate(CglsState *st, double *alphas, double *sigmas, double *x_norms,
                              double *history) {  // sv.py:217-232
    if (st->status) return;
    const long long it = st->iters_run;
    alphas[it] = st->alpha;
    sigmas[it] = st->sigma;
    x_norms[it + 1] = st->xnorm;
    st->iters_run = it + 1;
    const long long i = st->iters_run - st->d;
    if (i >= 0) {
        const double estim = py_sum_products(alphas, sigmas, i, st->iters_run);
        int err = 0;
        const double ratio = py_stopping_ratio(estim, st->norm_A, x_norms[i], st->b_norm, st->ratio_raw, &err);
        if (err) {
            st->status = ST_ERROR;
            return;
        }
        history[st->hist_len++] = ratio;
        if (ratio <= st->delta) {
            st->status = ST_CONVERGED;
            st->its_certified = i;
        }
    }
}
__global__ void k_it_zz(CglsState *st) {  // sv.py:235-237
    if (st->status) return;
    if (st->zz == 0.0) st->status = ST_STOPPED;
}
__global__ void k_it_beta(CglsState *st) {  // sv.py:239-241
    if (st->status) return;
    const double rho_new = st->zh;
    if (st->rho != 0.0) {
        st->beta = rho_new / st->rho;
        st->p_copy = 0;
    } else {
        st->p_copy = 1;
    }
    st->rho = rho_new;
}
__global__ void k_it_end(CglsState *st) {  // for-loop exhausted (sv.py:202)
    if (st->status) return;
    if (st->iters_run >= st->max_iters) st->status = ST_MAXED;
}

// ---- power method control (sc.py:439-454) ----
__global__ void k_pm_start(PowerState *ps, int empty) {
    ps->stop = 0;
    ps->est = 0.0;
    if (ps->nv == 0.0 || empty) {
        ps->result = 0.0;
        ps->stop = 1;
    }
}
__global__ void k_pm_est(PowerState *ps) {
    if (ps->stop) return;
    if (ps->est == 0.0) {
        ps->result = 0.0;
        ps->stop = 1;
    }
}
__global__ void k_pm_nt(PowerState *ps) {
    if (ps->stop) return;
    if (ps->nt == 0.0) {
        ps->result = ps->est;
        ps->stop = 1;
    }
}
__global__ void k_pm_final(PowerState *ps) {
    if (ps->stop) return;
    ps->result = ps->est;
}
__global__ void k_div(double *dst, const double *src, const double *den, int64_t n, const int *stop) {
    if (stop && *(volatile const int *)stop) return;
    const double d = *den;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] / d;
}

inline int small_grid(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

inline int chk(rsb_ctx *ctx, int kernels = 1) {
    ctx->launches += kernels;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("kernel launch failed: %s", cudaGetErrorString(e));
        return RSB_ECUDA;
    }
    return RSB_OK;
}

}  // namespace

}  // namespace rsb

using namespace rsb;

// ---------------------------------------------------------------------------
// preconditioner (pc.py:106-186)
// ---------------------------------------------------------------------------
namespace {

int ws_alloc(rsb_ctx *ctx, const rsb_pre *P, ApplyWs &W, bool carry = false) {
    W.ctx = ctx;
    W.n = P->n;
    W.s = P->s;
    const size_t n8 = P->n * sizeof(double), s8 = P->s * sizeof(double);
    for (double **q : {&W.t1, &W.t2, &W.t3, &W.v, &W.cg_a, &W.cg_b, &W.cg_c, &W.cg_b2, &W.r1g})
        RSB_TRY(dev_alloc(ctx, (void **)q, n8));
    for (double **q : {&W.u, &W.w, &W.cg_r, &W.cg_p, &W.cg_q}) RSB_TRY(dev_alloc(ctx, (void **)q, s8));
    RSB_TRY(dev_alloc(ctx, (void **)&W.cg, sizeof(CgState)));
    RSB_TRY_CUDA(cudaMemsetAsync(W.cg, 0, sizeof(CgState), ctx->stream));
    int64_t cap = 0;
    for (const TriSched *T : {P->tL1, P->tL1T, P->tU})
        if (T) cap = std::max(cap, T->padded_n);
    RSB_TRY(tri_ws_alloc(ctx, W.tri, cap));
    // the implicit-Y application starts with L1: r1 -> t1 and never reads t1
    // after its first product, so its last solve can refill it
    W.carry = carry && P->s > 0 && P->y_mode != RSB_Y_EXPLICIT && trsv_wants_prefill(*P->tL1);
    if (W.carry) RSB_TRY(launch_fill(ctx, W.t1, P->n, kSentinel, Gate{}));
    return RSB_OK;
}

void ws_free(ApplyWs &W) {
    if (!W.ctx) return;
    const size_t n8 = W.n * sizeof(double), s8 = W.s * sizeof(double);
    for (double *q : {W.t1, W.t2, W.t3, W.v, W.cg_a, W.cg_b, W.cg_c, W.cg_b2, W.r1g}) dev_free(W.ctx, q, n8);
    for (double *q : {W.u, W.w, W.cg_r, W.cg_p, W.cg_q}) dev_free(W.ctx, q, s8);
    dev_free(W.ctx, W.cg, sizeof(CgState));
    tri_ws_free(W.ctx, W.tri);
    W.ctx = nullptr;
}

// The solves of one application form a chain: each fills the next one's output
// with the sentinel where that solve wants it (TrsvChain).  `ready` is the
// vector the previous solve filled.
struct SolveChain {
    rsb_ctx *ctx;
    ApplyWs &W;
    Gate g;
    double *ready;
    int run(const TriSched &T, VecIn a, const double *c, double *x, const TriSched *next, double *next_x,
            double *rhs_copy = nullptr) {
        TrsvChain ch;
        ch.rhs_copy = rhs_copy;
        ch.prefilled = ready != nullptr && ready == x;
        ch.fill_next = (next && next_x && trsv_wants_prefill(*next)) ? next_x : nullptr;
        RSB_TRY(launch_trsv(ctx, T, a, c, x, g, &W.tri, ch));
        ready = ch.fill_next;
        return RSB_OK;
    }
};

// q = S p = p + L2 L1^{-1} L1^{-T} L2^T p  (s_matvec_implicit, pc.py:149-154)
// cb: the vector between the two solves; after: the solve that follows this
// product in the chain and its output (nullptr: none)
int enqueue_s_matvec(rsb_pre *P, ApplyWs &W, const double *p, double *q, Gate g, SolveChain *chain = nullptr,
                     double *cb = nullptr, const TriSched *after = nullptr, double *after_x = nullptr) {
    rsb_ctx *ctx = W.ctx;
    SolveChain local{ctx, W, g, nullptr};
    SolveChain &C = chain ? *chain : local;
    if (!cb) cb = W.cg_b;
    const Gate outer = C.g;
    C.g = g;
    RSB_TRY(launch_spmv_t(ctx, P->L2->csc(), VecIn{p, nullptr, 0}, W.cg_a, EPI_STORE, VecIn{}, g));
    RSB_TRY(C.run(*P->tL1T, VecIn{W.cg_a, nullptr, 0}, nullptr, cb, P->tL1, W.cg_c));
    RSB_TRY(C.run(*P->tL1, VecIn{cb, nullptr, 0}, nullptr, W.cg_c, after, after_x));
    C.g = outer;
    RSB_TRY(launch_spmv(ctx, P->L2->csr(), VecIn{W.cg_c, nullptr, 0}, q, EPI_ADD, VecIn{p, nullptr, 0}, g));
    return RSB_OK;
}

// w = _cg_fixed_steps(S, u, k)  (pc.py:284-310), result in W.w
// after / after_x: the solve that follows the inner CG in the chain
int enqueue_cg(rsb_pre *P, ApplyWs &W, const double *u, Gate outer, SolveChain &C, const TriSched *after,
               double *after_x) {
    rsb_ctx *ctx = W.ctx;
    const int64_t s = P->s;
    CgState *cg = W.cg;
    k_cg_init<<<small_grid(s), 256, 0, ctx->stream>>>(W.w, W.cg_r, W.cg_p, u, s, outer);
    RSB_TRY(chk(ctx));
    RSB_TRY(launch_dot(ctx, s, VecIn{W.cg_r, nullptr, 0}, VecIn{W.cg_r, nullptr, 0}, &cg->rho, 0, outer, nullptr));
    k_cg_start<<<1, 1, 0, ctx->stream>>>(cg, outer);
    RSB_TRY(chk(ctx));
    Gate g{outer.a, &cg->stop};
    auto cb_of = [&](int it) { return (it & 1) ? W.cg_b2 : W.cg_b; };
    for (int it = 0; it < P->cg_iters; ++it) {
        const bool last = it + 1 == P->cg_iters;
        RSB_TRY(enqueue_s_matvec(P, W, W.cg_p, W.cg_q, g, &C, cb_of(it), last ? after : P->tL1T,
                                 last ? after_x : cb_of(it + 1)));
        RSB_TRY(launch_dot(ctx, s, VecIn{W.cg_p, nullptr, 0}, VecIn{W.cg_q, nullptr, 0}, &cg->pq, 0, g, nullptr));
        k_cg_alpha<<<1, 1, 0, ctx->stream>>>(cg, g);
        RSB_TRY(chk(ctx));
        RSB_TRY(launch_axpy(ctx, W.w, W.cg_p, &cg->alpha, +1, s, g));
        // the last step's r, rho_new, break test and p feed nothing: w is final
        // here and the next application starts from k_cg_init / k_cg_start
        // (which resets the stop flag), so they are not enqueued -- w, and so
        // every apply, is unchanged bit for bit
        if (last) break;
        RSB_TRY(launch_axpy(ctx, W.cg_r, W.cg_q, &cg->alpha, -1, s, g));
        RSB_TRY(launch_dot(ctx, s, VecIn{W.cg_r, nullptr, 0}, VecIn{W.cg_r, nullptr, 0}, &cg->rho_new, 0, g, nullptr));
        k_cg_beta<<<1, 1, 0, ctx->stream>>>(cg, g);
        RSB_TRY(chk(ctx));
        RSB_TRY(launch_xpby(ctx, W.cg_p, W.cg_r, &cg->beta, nullptr, s, g));
    }
    return RSB_OK;
}

// h = apply(r1, r2)  (pc.py:175-186)
int enqueue_apply(rsb_pre *P, ApplyWs &W, VecIn r1, VecIn r2, double *h, Gate g) {
    rsb_ctx *ctx = W.ctx;
    SolveChain C{ctx, W, g, W.carry ? W.t1 : nullptr};
    if (P->s > 0) {
        const bool expl = P->y_mode == RSB_Y_EXPLICIT;
        // the first solve after w = solve_S(u), and its output
        const TriSched *back = expl ? P->tL1 : P->tL1T;
        double *back_x = expl ? W.v : W.t3;
        const bool cg = P->s_mode != RSB_S_DENSE && P->s_mode != RSB_S_IDENTITY;
        VecIn r1_again = r1;
        // u = r2 - Y r1
        if (expl) {
            RSB_TRY(launch_spmv(ctx, P->Y->csr(), r1, W.u, EPI_SUB_FROM, r2, g));
        } else {
            // r1 arrives through the row permutation (a scattered gather of
            // the m-vector r): the index-order solve writes what it gathered
            // to r1g, and the application's second solve with r1 streams that
            r1_again = (r1.g && trsv_wants_prefill(*P->tL1)) ? VecIn{W.r1g, nullptr, 0} : r1;
            RSB_TRY(C.run(*P->tL1, r1, nullptr, W.t1, cg ? P->tL1T : back, cg ? W.cg_b : back_x,
                          r1_again.p == W.r1g ? W.r1g : nullptr));
            RSB_TRY(launch_spmv(ctx, P->L2->csr(), VecIn{W.t1, nullptr, 0}, W.u, EPI_SUB_FROM, r2, g));
        }
        // w = solve_S(u)
        const double *w = W.w;
        if (P->s_mode == RSB_S_DENSE) {
            RSB_TRY(launch_chol_solve(ctx, P->S, P->s, W.u, W.w, g));
        } else if (P->s_mode == RSB_S_IDENTITY) {
            w = W.u;
        } else {
            RSB_TRY(enqueue_cg(P, W, W.u, g, C, back, back_x));
        }
        // y = r1 + Y^T w ; v = L1^{-1} y
        if (expl) {
            RSB_TRY(launch_spmv_t(ctx, P->Y->csc(), VecIn{w, nullptr, 0}, W.t3, EPI_ADD, r1, g));
            RSB_TRY(C.run(*P->tL1, VecIn{W.t3, nullptr, 0}, nullptr, W.v, P->tU, h));
        } else {
            RSB_TRY(launch_spmv_t(ctx, P->L2->csc(), VecIn{w, nullptr, 0}, W.t2, EPI_STORE, VecIn{}, g));
            RSB_TRY(C.run(*P->tL1T, VecIn{W.t2, nullptr, 0}, nullptr, W.t3, P->tL1, W.v));
            RSB_TRY(C.run(*P->tL1, r1_again, W.t3, W.v, P->tU, h));
        }
    } else {
        RSB_TRY(C.run(*P->tL1, r1, nullptr, W.v, P->tU, h));
    }
    // the last solve refills the next application's first output
    return C.run(*P->tU, VecIn{W.v, nullptr, 0}, nullptr, h, W.carry ? P->tL1 : nullptr, W.carry ? W.t1 : nullptr);
}

void pre_free(rsb_pre *P) {
    rsb_ctx *ctx = P->ctx;
    dev_free(ctx, P->perm, P->m * sizeof(int32_t));
    if (P->S) dev_free(ctx, P->S, P->s * P->s * sizeof(double));
    ws_free(P->ws);
    delete P;
}

}  // namespace

// ---------------------------------------------------------------------------
// solver (sv.py:120-268)
// ---------------------------------------------------------------------------
struct rsb_solver {
    rsb_ctx *ctx = nullptr;  // the solver's stream; may differ from the matrices' (same device)
    rsb_mat *A = nullptr;
    rsb_pre *pre = nullptr;
    ApplyWs ws;              // this solver's preconditioner workspace
    int64_t m = 0, n = 0;
    double *b = nullptr, *x = nullptr, *r = nullptr, *q = nullptr, *fr = nullptr;  // m: b, r, q, fr
    double *z = nullptr, *h = nullptr, *p = nullptr, *g = nullptr;                 // n
    CglsState *st = nullptr;
    CglsState *h_st = nullptr;  // pinned mirror
    double *alphas = nullptr, *sigmas = nullptr, *x_norms = nullptr, *history = nullptr;
    int64_t cap = 0;  // capacity of the per-iteration arrays (max_iters)
    int d = 5;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t graph_kernels = 0;
    // instrumented copy of the iteration graph (bench): event-record nodes
    // around every triangular solve
    cudaGraph_t bgraph = nullptr;
    cudaGraphExec_t bexec = nullptr;
    int btrace = 0, bptrace = 0;
    bool started = false;
    rsb_cgls_cfg cfg{};
};

namespace {

int enqueue_precondition(rsb_solver *S, Gate g) {
    if (S->pre) {
        const rsb_pre *P = S->pre;
        return enqueue_apply(S->pre, S->ws, VecIn{S->r, P->perm, 0}, VecIn{S->r, P->perm, S->n}, S->h, g);
    }
    return launch_copy(S->ctx, S->h, VecIn{S->z, nullptr, 0}, S->n, g);  // h = A^T r (sv.py:166-167)
}

// one iteration of sv.py:202-241
int enqueue_iteration(rsb_solver *S) {
    rsb_ctx *ctx = S->ctx;
    CglsState *st = S->st;
    const Gate g{&st->status, nullptr};
    const int64_t m = S->m, n = S->n;
    k_it_begin<<<1, 1, 0, ctx->stream>>>(st);
    RSB_TRY(chk(ctx));
    RSB_TRY(launch_dot(ctx, n, VecIn{S->z, nullptr, 0}, VecIn{S->p, nullptr, 0}, &st->zp, 0, g, &st->need_zp));
    k_it_sigma<<<1, 1, 0, ctx->stream>>>(st);
    RSB_TRY(chk(ctx));
    RSB_TRY(launch_copy(ctx, S->p, VecIn{S->z, nullptr, 0}, n, Gate{&st->status, &st->skip_retry}));
    RSB_TRY(launch_spmv(ctx, S->A->csr(), VecIn{S->p, nullptr, 0}, S->q, EPI_STORE, VecIn{}, g));
    RSB_TRY(launch_dot(ctx, m, VecIn{S->q, nullptr, 0}, VecIn{S->q, nullptr, 0}, &st->qq, 0, g, nullptr));
    k_it_alpha<<<1, 1, 0, ctx->stream>>>(st);
    RSB_TRY(chk(ctx));
    RSB_TRY(launch_axpy(ctx, S->x, S->p, &st->alpha, +1, n, g));
    RSB_TRY(launch_axpy(ctx, S->r, S->q, &st->alpha, -1, m, g));
    // The preconditioner application reads only r (sv.py:238), so it runs on
    // the main branch while a side branch computes ||x|| with the estimator,
    // then z = A^T r and z.z (sv.py:220-237).  Everything is gated on the
    // status the estimator sets, so an application started before a stop is
    // merely wasted (z is not an output); k_it_zz runs after the join, keeping
    // the reference's order of the stopping checks.  (Not in tree-dot mode,
    // whose dots share one scratch.)
    const char *nf = getenv("RSB_NO_FORK");  // experiments: everything on the main branch
    const bool fork = !(ctx->flags & RSB_DOT_TREE) && ctx->side && !(nf && atoi(nf) != 0);
    auto on_side = [&](auto &&launches) -> int {
        cudaStream_t main = ctx->stream;
        ctx->stream = ctx->side;
        const int rc = launches();
        ctx->stream = main;
        return rc;
    };
    auto side_branch = [&]() -> int {
        RSB_TRY(launch_dot(ctx, n, VecIn{S->x, nullptr, 0}, VecIn{S->x, nullptr, 0}, &st->xnorm, 1, g, nullptr));
        k_it_estimate<<<1, 1, 0, ctx->stream>>>(st, S->alphas, S->sigmas, S->x_norms, S->history);
        RSB_TRY(chk(ctx));
        RSB_TRY(launch_spmv_t(ctx, S->A->csc(), VecIn{S->r, nullptr, 0}, S->z, EPI_STORE, VecIn{}, g));
        return launch_dot(ctx, n, VecIn{S->z, nullptr, 0}, VecIn{S->z, nullptr, 0}, &st->zz, 0, g, nullptr);
    };
    if (fork) {
        RSB_TRY_CUDA(cudaEventRecord(ctx->fork_ev[0], ctx->stream));
        RSB_TRY_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork_ev[0], 0));
        RSB_TRY(on_side(side_branch));
        RSB_TRY_CUDA(cudaEventRecord(ctx->fork_ev[2], ctx->side));
    } else {
        RSB_TRY(side_branch());
        k_it_zz<<<1, 1, 0, ctx->stream>>>(st);
        RSB_TRY(chk(ctx));
    }
    if (S->pre) RSB_TRY(enqueue_precondition(S, g));
    if (fork) {
        RSB_TRY_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->fork_ev[2], 0));
        k_it_zz<<<1, 1, 0, ctx->stream>>>(st);
        RSB_TRY(chk(ctx));
    }
    if (!S->pre) RSB_TRY(enqueue_precondition(S, g));  // plain CGLS: h = z, after the branch that computes z
    RSB_TRY(launch_dot(ctx, n, VecIn{S->z, nullptr, 0}, VecIn{S->h, nullptr, 0}, &st->zh, 0, g, nullptr));
    k_it_beta<<<1, 1, 0, ctx->stream>>>(st);
    RSB_TRY(chk(ctx));
    RSB_TRY(launch_xpby(ctx, S->p, S->h, &st->beta, &st->p_copy, n, g));
    k_it_end<<<1, 1, 0, ctx->stream>>>(st);
    return chk(ctx);
}

int ensure_capacity(rsb_solver *S, int64_t max_iters, int d) {
    if (max_iters <= S->cap && d <= S->d && S->exec) return RSB_OK;
    rsb_ctx *ctx = S->ctx;
    cudaStreamSynchronize(ctx->stream);
    if (S->exec) {
        cudaGraphExecDestroy(S->exec);
        cudaGraphDestroy(S->graph);
        S->exec = nullptr;
        S->graph = nullptr;
    }
    if (S->bexec) {
        cudaGraphExecDestroy(S->bexec);
        cudaGraphDestroy(S->bgraph);
        S->bexec = nullptr;
        S->bgraph = nullptr;
    }
    if (max_iters > S->cap || d > S->d) {
        const int64_t cap = std::max(max_iters, S->cap);
        const int dd = std::max(d, S->d);
        dev_free(ctx, S->alphas, S->cap * sizeof(double));
        dev_free(ctx, S->sigmas, S->cap * sizeof(double));
        dev_free(ctx, S->x_norms, (S->cap + 1) * sizeof(double));
        dev_free(ctx, S->history, (S->cap + S->d + 1) * sizeof(double));
        S->cap = cap;
        S->d = dd;
        RSB_TRY(dev_alloc(ctx, (void **)&S->alphas, cap * sizeof(double)));
        RSB_TRY(dev_alloc(ctx, (void **)&S->sigmas, cap * sizeof(double)));
        RSB_TRY(dev_alloc(ctx, (void **)&S->x_norms, (cap + 1) * sizeof(double)));
        RSB_TRY(dev_alloc(ctx, (void **)&S->history, (cap + dd + 1) * sizeof(double)));
    }
    // capture one iteration as a graph
    const int64_t before = ctx->launches;
    RSB_TRY_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_iteration(S);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (rc != RSB_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    RSB_TRY_CUDA(e);
    S->graph = graph;
    RSB_TRY_CUDA(cudaGraphInstantiate(&S->exec, graph, cudaGraphInstantiateFlagUseNodePriority));
    S->graph_kernels = ctx->launches - before;
    ctx->launches = before;
    return RSB_OK;
}

int read_state(rsb_solver *S) {
    rsb_ctx *ctx = S->ctx;
    RSB_TRY_CUDA(cudaMemcpyAsync(S->h_st, S->st, sizeof(CglsState), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    return RSB_OK;
}

void solver_free(rsb_solver *S) {
    rsb_ctx *ctx = S->ctx;
    cudaStreamSynchronize(ctx->stream);
    if (S->exec) cudaGraphExecDestroy(S->exec);
    if (S->graph) cudaGraphDestroy(S->graph);
    if (S->bexec) cudaGraphExecDestroy(S->bexec);
    if (S->bgraph) cudaGraphDestroy(S->bgraph);
    const size_t m8 = S->m * sizeof(double), n8 = S->n * sizeof(double);
    for (double *q : {S->b, S->r, S->q, S->fr}) dev_free(ctx, q, m8);
    for (double *q : {S->x, S->z, S->h, S->p, S->g}) dev_free(ctx, q, n8);
    dev_free(ctx, S->st, sizeof(CglsState));
    if (S->h_st) cudaFreeHost(S->h_st);
    dev_free(ctx, S->alphas, S->cap * sizeof(double));
    dev_free(ctx, S->sigmas, S->cap * sizeof(double));
    dev_free(ctx, S->x_norms, (S->cap + 1) * sizeof(double));
    dev_free(ctx, S->history, (S->cap + S->d + 1) * sizeof(double));
    ws_free(S->ws);
    delete S;
}

}  // namespace

extern "C" {

int rsb_pre_create(rsb_ctx *ctx, int64_t m, int64_t n, const int64_t *perm, rsb_mat *L1, rsb_mat *L2,
                   rsb_mat *U, rsb_mat *Y, const double *S_factor, int64_t s, int s_mode, int y_mode,
                   int cg_iters, rsb_pre **out) {
    *out = nullptr;
    if (cg_iters < 1) {
        set_error("cg_iters must be >= 1");
        return RSB_EINVAL;
    }
    if (s_mode < 0 || s_mode > 2 || y_mode < 0 || y_mode > 1) {
        set_error("unknown s_mode/y_mode");
        return RSB_EINVAL;
    }
    if (s_mode == RSB_S_DENSE && y_mode != RSB_Y_EXPLICIT) {
        set_error("dense S factorization requires the explicit Y");
        return RSB_EINVAL;
    }
    if (!L1 || !L2 || !U || L1->nrows != n || L1->ncols != n || U->nrows != n || U->ncols != n ||
        L2->ncols != n || L2->nrows != s || m != n + s) {
        set_error("inconsistent factor dimensions");
        return RSB_EINVAL;
    }
    if (y_mode == RSB_Y_EXPLICIT && (!Y || Y->nrows != s || Y->ncols != n)) {
        set_error("explicit Y mode needs Y of shape (%lld, %lld)", (long long)s, (long long)n);
        return RSB_EINVAL;
    }
    if (s_mode == RSB_S_DENSE && s > 0 && !S_factor) {
        set_error("dense S mode needs the S factor");
        return RSB_EINVAL;
    }
    for (int64_t i = 0; i < m; ++i)
        if (perm[i] < 0 || perm[i] >= m) {
            set_error("row permutation entry out of range");
            return RSB_EINVAL;
        }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    auto *P = new rsb_pre();
    P->ctx = ctx;
    P->m = m;
    P->n = n;
    P->s = s;
    P->s_mode = s_mode;
    P->y_mode = y_mode;
    P->cg_iters = cg_iters;
    P->L1 = L1;
    P->L2 = L2;
    P->U = U;
    P->Y = Y;
    int rc = RSB_OK;
    std::vector<int32_t> pm(perm, perm + m);
    const size_t n8 = n * sizeof(double), s8 = s * sizeof(double);
#define PTRY(x)                 \
    if ((rc = (x)) != RSB_OK) { \
        pre_free(P);            \
        return rc;              \
    }
    PTRY(get_tri(L1, RSB_TRI_LOWER_UNIT, &P->tL1));
    PTRY(get_tri(U, RSB_TRI_UPPER, &P->tU));
    if (s > 0) PTRY(get_tri(L1, RSB_TRI_LOWER_T_UNIT, &P->tL1T));
    PTRY(dev_upload(ctx, &P->perm, pm.data(), pm.size()));
    if (s_mode == RSB_S_DENSE && s > 0) {
        PTRY(dev_upload(ctx, &P->S, S_factor, (size_t)(s * s)));
        PTRY(prepare_chol(s));
    }
    PTRY(ws_alloc(ctx, P, P->ws));
#undef PTRY
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = P;
    return RSB_OK;
}

int rsb_pre_destroy(rsb_pre *pre) {
    if (!pre) return RSB_OK;
    cudaStreamSynchronize(pre->ctx->stream);
    pre_free(pre);
    return RSB_OK;
}

int rsb_pre_apply(rsb_pre *P, const double *r1, const double *r2, double *h, int where) {
    rsb_ctx *ctx = P->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    Staged s1, s2, sh;
    RSB_TRY(stage_in(ctx, r1, P->n, where, s1));
    RSB_TRY(stage_in(ctx, r2, P->s, where, s2));
    RSB_TRY(stage_out(ctx, h, P->n, where, sh));
    RSB_TRY(enqueue_apply(P, P->ws, VecIn{s1.d, nullptr, 0}, VecIn{s2.d, nullptr, 0}, sh.d, Gate{}));
    return finish_out(ctx, h, P->n, where, sh);
}

int rsb_pre_y_apply(rsb_pre *P, const double *r1, double *out, int where) {
    rsb_ctx *ctx = P->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    Staged s1, so;
    RSB_TRY(stage_in(ctx, r1, P->n, where, s1));
    RSB_TRY(stage_out(ctx, out, P->s, where, so));
    if (P->s > 0) {
        if (P->y_mode == RSB_Y_EXPLICIT) {
            RSB_TRY(launch_spmv(ctx, P->Y->csr(), VecIn{s1.d, nullptr, 0}, so.d, EPI_STORE, VecIn{}, Gate{}));
        } else {
            RSB_TRY(launch_trsv(ctx, *P->tL1, VecIn{s1.d, nullptr, 0}, nullptr, P->ws.t1, Gate{}, &P->ws.tri));
            RSB_TRY(launch_spmv(ctx, P->L2->csr(), VecIn{P->ws.t1, nullptr, 0}, so.d, EPI_STORE, VecIn{}, Gate{}));
        }
    }
    return finish_out(ctx, out, P->s, where, so);
}

int rsb_pre_y_apply_transpose(rsb_pre *P, const double *w, double *out, int where) {
    rsb_ctx *ctx = P->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    Staged sw, so;
    RSB_TRY(stage_in(ctx, w, P->s, where, sw));
    RSB_TRY(stage_out(ctx, out, P->n, where, so));
    if (P->y_mode == RSB_Y_EXPLICIT) {
        RSB_TRY(launch_spmv_t(ctx, P->Y->csc(), VecIn{sw.d, nullptr, 0}, so.d, EPI_STORE, VecIn{}, Gate{}));
    } else {
        RSB_TRY(launch_spmv_t(ctx, P->L2->csc(), VecIn{sw.d, nullptr, 0}, P->ws.t2, EPI_STORE, VecIn{}, Gate{}));
        RSB_TRY(launch_trsv(ctx, *P->tL1T, VecIn{P->ws.t2, nullptr, 0}, nullptr, so.d, Gate{}, &P->ws.tri));
    }
    return finish_out(ctx, out, P->n, where, so);
}

int rsb_pre_s_matvec(rsb_pre *P, const double *v, double *out, int where) {
    rsb_ctx *ctx = P->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    Staged sv, so;
    RSB_TRY(stage_in(ctx, v, P->s, where, sv));
    RSB_TRY(stage_out(ctx, out, P->s, where, so));
    if (P->s > 0) {
        RSB_TRY(enqueue_s_matvec(P, P->ws, sv.d, so.d, Gate{}));
    }
    return finish_out(ctx, out, P->s, where, so);
}

int rsb_solver_create(rsb_mat *A, rsb_pre *pre, rsb_solver **out) {
    return rsb_solver_create_on(A->ctx, A, pre, out);
}

int rsb_solver_create_on(rsb_ctx *ctx, rsb_mat *A, rsb_pre *pre, rsb_solver **out) {
    *out = nullptr;
    if (pre && (pre->m != A->nrows || pre->n != A->ncols)) {
        set_error("preconditioner does not match the matrix");
        return RSB_EINVAL;
    }
    if (A->ctx->device != ctx->device || (pre && pre->ctx->device != ctx->device)) {
        set_error("matrix, preconditioner and solver context must be on the same device");
        return RSB_EINVAL;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    // the shared matrices were uploaded on their own streams
    RSB_TRY_CUDA(cudaStreamSynchronize(A->ctx->stream));
    if (pre) RSB_TRY_CUDA(cudaStreamSynchronize(pre->ctx->stream));
    auto *S = new rsb_solver();
    S->ctx = ctx;
    S->A = A;
    S->pre = pre;
    S->m = A->nrows;
    S->n = A->ncols;
    int rc = RSB_OK;
    const size_t m8 = S->m * sizeof(double), n8 = S->n * sizeof(double);
    for (double **q : {&S->b, &S->r, &S->q, &S->fr})
        if ((rc = dev_alloc(ctx, (void **)q, m8)) != RSB_OK) break;
    for (double **q : {&S->x, &S->z, &S->h, &S->p, &S->g})
        if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)q, n8);
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->st, sizeof(CglsState));
    if (rc == RSB_OK && cudaMallocHost((void **)&S->h_st, sizeof(CglsState)) != cudaSuccess) {
        set_error("pinned allocation failed");
        rc = RSB_ENOMEM;
    }
    if (rc == RSB_OK && pre) rc = ws_alloc(ctx, pre, S->ws, /*carry=*/true);
    if (rc == RSB_OK) rc = cudaStreamSynchronize(ctx->stream) == cudaSuccess ? RSB_OK : RSB_ECUDA;
    if (rc != RSB_OK) {
        solver_free(S);
        return rc;
    }
    *out = S;
    return RSB_OK;
}

int rsb_solver_destroy(rsb_solver *S) {
    if (S) solver_free(S);
    return RSB_OK;
}

}  // extern "C"

namespace {

// sv.py:152-200 enqueued on the solver's stream, ending with an async read of
// the control block into the pinned mirror (no synchronisation)
int start_enqueue(rsb_solver *S, const double *b, int where, const rsb_cgls_cfg *cfg) {
    rsb_ctx *ctx = S->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    if (!(cfg->delta > 0.0) || cfg->estimator_delay < 1 || cfg->max_iters < 1) {
        set_error("invalid CglsConfig (delta > 0, estimator_delay >= 1, max_iters >= 1)");
        return RSB_EINVAL;
    }
    RSB_TRY(ensure_capacity(S, cfg->max_iters, cfg->estimator_delay));
    S->cfg = *cfg;
    S->started = false;
    const int64_t m = S->m, n = S->n;
    if (where != RSB_HOST) {
        RSB_TRY_CUDA(cudaMemcpyAsync(S->b, b, m * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        RSB_TRY_CUDA(cudaMemcpyAsync(S->b, b, m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    CglsState init{};
    init.norm_A = cfg->norm_A;
    init.delta = cfg->delta;
    init.max_iters = cfg->max_iters;
    init.d = cfg->estimator_delay;
    init.ratio_raw = cfg->ratio_raw;
    // the mirror may still be the source of an in-flight copy from a
    // previous start on this stream
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    *S->h_st = init;
    RSB_TRY_CUDA(cudaMemcpyAsync(S->st, S->h_st, sizeof(CglsState), cudaMemcpyHostToDevice, ctx->stream));
    CglsState *st = S->st;
    const Gate none{};
    const Gate g{&st->status, nullptr};
    // sv.py:152, 171-173
    RSB_TRY(launch_dot(ctx, m, VecIn{S->b, nullptr, 0}, VecIn{S->b, nullptr, 0}, &st->b_norm, 1, none, nullptr));
    RSB_TRY(launch_fill(ctx, S->x, n, 0ull, none));
    RSB_TRY(launch_copy(ctx, S->r, VecIn{S->b, nullptr, 0}, m, none));
    RSB_TRY(launch_spmv_t(ctx, S->A->csc(), VecIn{S->r, nullptr, 0}, S->z, EPI_STORE, VecIn{}, none));
    RSB_TRY(launch_dot(ctx, n, VecIn{S->z, nullptr, 0}, VecIn{S->z, nullptr, 0}, &st->zz, 0, none, nullptr));
    k_start_check<<<1, 1, 0, ctx->stream>>>(st);
    RSB_TRY(chk(ctx));
    // sv.py:198-200
    RSB_TRY(enqueue_precondition(S, g));
    RSB_TRY(launch_dot(ctx, n, VecIn{S->z, nullptr, 0}, VecIn{S->h, nullptr, 0}, &st->zh, 0, g, nullptr));
    k_start_rho<<<1, 1, 0, ctx->stream>>>(st, S->x_norms);
    RSB_TRY(chk(ctx));
    RSB_TRY(launch_copy(ctx, S->p, VecIn{S->h, nullptr, 0}, n, g));
    RSB_TRY_CUDA(cudaMemcpyAsync(S->h_st, S->st, sizeof(CglsState), cudaMemcpyDeviceToHost, ctx->stream));
    return RSB_OK;
}

// after start_enqueue: wait for the control block and check it
int start_complete(rsb_solver *S, int *status) {
    RSB_TRY_CUDA(cudaSetDevice(S->ctx->device));
    RSB_TRY_CUDA(cudaStreamSynchronize(S->ctx->stream));
    if (S->h_st->status == ST_ERROR) {
        set_error("zero denominator in stopping ratio");
        return RSB_EINVAL;
    }
    S->started = true;
    *status = S->h_st->status;
    return RSB_OK;
}

// enqueue up to nb iteration-graph replays and an async state read
int iterate_enqueue(rsb_solver *S, int64_t nb) {
    rsb_ctx *ctx = S->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    for (int64_t i = 0; i < nb; ++i) RSB_TRY_CUDA(cudaGraphLaunch(S->exec, ctx->stream));
    ctx->launches += nb * S->graph_kernels;
    RSB_TRY_CUDA(cudaMemcpyAsync(S->h_st, S->st, sizeof(CglsState), cudaMemcpyDeviceToHost, ctx->stream));
    return RSB_OK;
}

}  // namespace

extern "C" {

int rsb_solver_start(rsb_solver *S, const double *b, int where, const rsb_cgls_cfg *cfg, int *status) {
    RSB_TRY(start_enqueue(S, b, where, cfg));
    return start_complete(S, status);
}

int rsb_solver_iterate(rsb_solver *S, int64_t k, int64_t *iters_run, int *status) {
    rsb_ctx *ctx = S->ctx;
    if (!S->started) {
        set_error("rsb_solver_iterate before rsb_solver_start");
        return RSB_ESTATE;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    int64_t done = 0;
    int st = S->h_st->status;
    // batches of graph replays; kernels are gated on the device status, so
    // replays past a stop are no-ops
    int64_t batch = 4;
    while (st == ST_RUN && done < k) {
        const int64_t nb = std::min(batch, k - done);
        RSB_TRY(iterate_enqueue(S, nb));
        done += nb;
        RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
        st = S->h_st->status;
        batch = std::min<int64_t>(batch * 2, 64);
    }
    if (st == ST_ERROR) {
        set_error("zero denominator in stopping ratio");
        return RSB_EINVAL;
    }
    *iters_run = S->h_st->iters_run;
    *status = st;
    return RSB_OK;
}

int rsb_solver_get_x(rsb_solver *S, double *x, int where) {
    rsb_ctx *ctx = S->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    RSB_TRY_CUDA(cudaMemcpyAsync(x, S->x, S->n * sizeof(double),
                                 where != RSB_HOST ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    return RSB_OK;
}

int rsb_solver_finish(rsb_solver *S, rsb_report *rep, double *history, int64_t history_cap) {
    rsb_ctx *ctx = S->ctx;
    if (!S->started) {
        set_error("rsb_solver_finish before rsb_solver_start");
        return RSB_ESTATE;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    RSB_TRY(read_state(S));
    const CglsState st = *S->h_st;
    std::memset(rep, 0, sizeof *rep);
    if (st.status == ST_ZERO_START) {  // sv.py:184-196
        rep->its = 0;
        rep->converged = 1;
        rep->breakdown = 0;
        rep->ratio_pt_final = 0.0;
        rep->residual_norm = st.b_norm;
        rep->gradient_norm = 0.0;
        rep->history_len = 1;
        if (history_cap > 0) history[0] = 0.0;
        return RSB_OK;
    }
    const long long it_run = st.iters_run;
    std::vector<double> al(it_run), sg(it_run), xn(it_run + 1), hist(st.hist_len);
    if (it_run) {
        RSB_TRY_CUDA(cudaMemcpyAsync(al.data(), S->alphas, it_run * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        RSB_TRY_CUDA(cudaMemcpyAsync(sg.data(), S->sigmas, it_run * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    RSB_TRY_CUDA(cudaMemcpyAsync(xn.data(), S->x_norms, (it_run + 1) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (st.hist_len)
        RSB_TRY_CUDA(cudaMemcpyAsync(hist.data(), S->history, st.hist_len * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    // final residual and gradient (sv.py:256-266), enqueued before the sync
    CglsState *dst = S->st;
    RSB_TRY(launch_spmv(ctx, S->A->csr(), VecIn{S->x, nullptr, 0}, S->fr, EPI_SUB_FROM, VecIn{S->b, nullptr, 0}, Gate{}));
    RSB_TRY(launch_dot(ctx, S->m, VecIn{S->fr, nullptr, 0}, VecIn{S->fr, nullptr, 0}, &dst->qq, 1, Gate{}, nullptr));
    RSB_TRY(launch_spmv_t(ctx, S->A->csc(), VecIn{S->fr, nullptr, 0}, S->g, EPI_STORE, VecIn{}, Gate{}));
    RSB_TRY(launch_dot(ctx, S->n, VecIn{S->g, nullptr, 0}, VecIn{S->g, nullptr, 0}, &dst->zz, 1, Gate{}, nullptr));
    RSB_TRY(read_state(S));
    const double res_norm = S->h_st->qq, grad_norm = S->h_st->zz;

    bool converged = st.status == ST_CONVERGED;
    const bool stopped_early = st.status == ST_STOPPED;
    long long its_cert = st.its_certified;
    if (stopped_early && !converged) {  // sv.py:243-253
        const int d = S->cfg.estimator_delay;
        for (long long i = std::max(0LL, it_run - d + 1); i <= it_run; ++i) {
            const double estim = py_sum_products(al.data(), sg.data(), i, it_run);
            int err = 0;
            const double ratio = py_stopping_ratio(estim, S->cfg.norm_A, xn[i], st.b_norm, S->cfg.ratio_raw, &err);
            if (err) {
                set_error("zero denominator in stopping ratio");
                return RSB_EINVAL;
            }
            hist.push_back(ratio);
            if (ratio <= S->cfg.delta) {
                converged = true;
                its_cert = i;
                break;
            }
        }
    }
    rep->iters_run = it_run;
    rep->its = converged ? its_cert : it_run;
    rep->converged = converged;
    rep->breakdown = stopped_early && !converged;
    rep->ratio_pt_final = hist.empty() ? INFINITY : hist.back();
    rep->residual_norm = res_norm;
    rep->gradient_norm = grad_norm;
    rep->history_len = (int64_t)hist.size();
    for (int64_t i = 0; i < std::min<int64_t>(history_cap, (int64_t)hist.size()); ++i) history[i] = hist[i];
    return RSB_OK;
}

// Bench: k iterations, each one replay of the instrumented iteration graph
// bracketed by events, optionally preceded by an L2 flush that is outside
// the bracket.  Returns the summed device time of the iterations and of the
// triangular solves inside them.
int rsb_solver_bench(rsb_solver *S, int64_t k, int flush, double *iter_ms, double *tri_ms,
                     int64_t *tri_launches, int64_t *kernels_per_iter, int *status) {
    rsb_ctx *ctx = S->ctx;
    if (!S->started) {
        set_error("rsb_solver_bench before rsb_solver_start");
        return RSB_ESTATE;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    if (!S->bexec) {
        ctx->tracing = true;
        ctx->trace_n = 0;
        ctx->ptrace_n = 0;
        const int64_t before = ctx->launches;
        RSB_TRY_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_iteration(S);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
        ctx->tracing = false;
        ctx->launches = before;
        if (rc != RSB_OK) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        RSB_TRY_CUDA(e);
        S->bgraph = graph;
        RSB_TRY_CUDA(cudaGraphInstantiate(&S->bexec, graph, cudaGraphInstantiateFlagUseNodePriority));
        S->btrace = ctx->trace_n;
        S->bptrace = ctx->ptrace_n;
    }
    double it_total = 0.0, tri_total = 0.0, prod_total = 0.0;
    for (int64_t i = 0; i < k; ++i) {
        if (flush) RSB_TRY(launch_l2_flush(ctx));
        RSB_TRY_CUDA(cudaEventRecord(ctx->ev[14], ctx->stream));
        RSB_TRY_CUDA(cudaGraphLaunch(S->bexec, ctx->stream));
        RSB_TRY_CUDA(cudaEventRecord(ctx->ev[15], ctx->stream));
        RSB_TRY_CUDA(cudaEventSynchronize(ctx->ev[15]));
        ctx->launches += S->graph_kernels;
        float ms = 0.f;
        RSB_TRY_CUDA(cudaEventElapsedTime(&ms, ctx->ev[14], ctx->ev[15]));
        it_total += ms;
        for (int t = 0; t + 1 < S->btrace; t += 2) {
            RSB_TRY_CUDA(cudaEventElapsedTime(&ms, ctx->trace_ev[t], ctx->trace_ev[t + 1]));
            tri_total += ms;
        }
        for (int t = 0; t + 1 < S->bptrace; t += 2) {
            RSB_TRY_CUDA(cudaEventElapsedTime(&ms, ctx->ptrace_ev[t], ctx->ptrace_ev[t + 1]));
            prod_total += ms;
        }
    }
    ctx->last_prod_ms = prod_total;
    ctx->last_prod_launches = k * (S->bptrace / 2);
    RSB_TRY(read_state(S));
    *iter_ms = it_total;
    *tri_ms = tri_total;
    *tri_launches = k * (S->btrace / 2);
    *kernels_per_iter = S->graph_kernels;
    *status = S->h_st->status;
    return RSB_OK;
}

int rsb_solver_bench_products(rsb_solver *S, double *prod_ms, int64_t *prod_launches) {
    *prod_ms = S->ctx->last_prod_ms;
    *prod_launches = S->ctx->last_prod_launches;
    return RSB_OK;
}

int rsb_pcgls(rsb_solver *S, const double *b, int where, const rsb_cgls_cfg *cfg, double *x, rsb_report *rep,
              double *history, int64_t history_cap) {
    int status = 0;
    RSB_TRY(rsb_solver_start(S, b, where, cfg, &status));
    if (status == ST_RUN) {
        int64_t iters = 0;
        RSB_TRY(rsb_solver_iterate(S, cfg->max_iters, &iters, &status));
    }
    RSB_TRY(rsb_solver_finish(S, rep, history, history_cap));
    return rsb_solver_get_x(S, x, where);
}

// Independent solves on several solvers (one stream each, same device or
// not), advanced together: every solver's graph batch is enqueued before the
// host waits on any of them, so the solves overlap on the device.  Each
// solver's arithmetic is exactly rsb_pcgls's.
int rsb_pcgls_many(int count, rsb_solver *const *S, const double *const *b, int where, const rsb_cgls_cfg *cfg,
                   double *const *x, rsb_report *reps, double *history, int64_t history_cap) {
    if (count < 0) {
        set_error("count must be >= 0");
        return RSB_EINVAL;
    }
    for (int i = 0; i < count; ++i)
        for (int j = 0; j < i; ++j)
            if (S[i] == S[j] || S[i]->ctx == S[j]->ctx) {
                set_error("rsb_pcgls_many needs distinct solvers on distinct contexts");
                return RSB_EINVAL;
            }
    // How many solves iterate at once.  Single-CTA triangular solves (narrow
    // DAGs) occupy one SM each, so all run together; a grid-wide solve fills
    // most of the GPU on its own and many concurrent ones only contend (config
    // 4 at n = 8e6: 8 concurrent RHS 72 RHS-iterations/s against 84 for one
    // e2e), while two overlap each other's level tails (n = 2e6: 340 at two,
    // 290 at one, 325 at 4 or 8; profiles/batch_conc_*), so those run two at a
    // time.  RSB_BATCH_CONC overrides (experiments).
    int conc = count;
    for (int i = 0; i < count; ++i)
        if (S[i]->pre)
            for (const TriSched *T : {S[i]->pre->tL1, S[i]->pre->tL1T, S[i]->pre->tU})
                if (T && !T->single_cta) conc = std::min(conc, T->level_sync ? 1 : 2);
    if (const char *e = getenv("RSB_BATCH_CONC")) conc = std::max(1, atoi(e));
    std::vector<int> st(count, ST_RUN);
    for (int i = 0; i < count; ++i) RSB_TRY(start_enqueue(S[i], b[i], where, cfg));
    for (int i = 0; i < count; ++i) RSB_TRY(start_complete(S[i], &st[i]));
    std::vector<int64_t> done(count, 0);
    for (int g0 = 0; g0 < count; g0 += conc) {
        const int g1 = std::min(count, g0 + conc);
        int64_t batch = 4;
        for (;;) {
            bool any = false;
            for (int i = g0; i < g1; ++i) {
                if (st[i] != ST_RUN || done[i] >= cfg->max_iters) continue;
                RSB_TRY(iterate_enqueue(S[i], std::min(batch, cfg->max_iters - done[i])));
                any = true;
            }
            if (!any) break;
            for (int i = g0; i < g1; ++i) {
                if (st[i] != ST_RUN || done[i] >= cfg->max_iters) continue;
                done[i] += std::min(batch, cfg->max_iters - done[i]);
                RSB_TRY_CUDA(cudaSetDevice(S[i]->ctx->device));
                RSB_TRY_CUDA(cudaStreamSynchronize(S[i]->ctx->stream));
                st[i] = S[i]->h_st->status;
                if (st[i] == ST_ERROR) {
                    set_error("zero denominator in stopping ratio");
                    return RSB_EINVAL;
                }
            }
            batch = std::min<int64_t>(batch * 2, 64);
        }
    }
    for (int i = 0; i < count; ++i) {
        RSB_TRY(rsb_solver_finish(S[i], &reps[i], history ? history + i * history_cap : nullptr,
                                  history ? history_cap : 0));
        RSB_TRY(rsb_solver_get_x(S[i], x[i], where));
    }
    return RSB_OK;
}

// power_method_norm2 (sc.py:428-454); v0 drawn on the host
int rsb_power_norm2(rsb_mat *A, const double *v0, int iters, double *est) {
    rsb_ctx *ctx = A->ctx;
    if (iters < 1) {
        set_error("iters must be >= 1");
        return RSB_EINVAL;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    const int64_t m = A->nrows, n = A->ncols;
    double *v = nullptr, *w = nullptr;
    PowerState *ps = nullptr;
    int rc = RSB_OK;
    if ((rc = dev_alloc(ctx, (void **)&v, n * sizeof(double))) != RSB_OK) return rc;
    if ((rc = dev_alloc(ctx, (void **)&w, m * sizeof(double))) != RSB_OK) {
        dev_free(ctx, v, n * sizeof(double));
        return rc;
    }
    if ((rc = dev_alloc(ctx, (void **)&ps, sizeof(PowerState))) != RSB_OK) {
        dev_free(ctx, v, n * sizeof(double));
        dev_free(ctx, w, m * sizeof(double));
        return rc;
    }
    auto run = [&]() -> int {
        RSB_TRY_CUDA(cudaMemcpyAsync(v, v0, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        RSB_TRY(launch_dot(ctx, n, VecIn{v, nullptr, 0}, VecIn{v, nullptr, 0}, &ps->nv, 1, Gate{}, nullptr));
        k_pm_start<<<1, 1, 0, ctx->stream>>>(ps, A->nnz == 0);
        RSB_TRY(chk(ctx));
        k_div<<<small_grid(n), 256, 0, ctx->stream>>>(v, v, &ps->nv, n, &ps->stop);
        RSB_TRY(chk(ctx));
        const Gate g{&ps->stop, nullptr};
        // the `t` of sc.py:449 reuses the n-vector v once v is consumed
        for (int it = 0; it < iters; ++it) {
            RSB_TRY(launch_spmv(ctx, A->csr(), VecIn{v, nullptr, 0}, w, EPI_STORE, VecIn{}, g));
            RSB_TRY(launch_dot(ctx, m, VecIn{w, nullptr, 0}, VecIn{w, nullptr, 0}, &ps->est, 1, g, nullptr));
            k_pm_est<<<1, 1, 0, ctx->stream>>>(ps);
            RSB_TRY(chk(ctx));
            RSB_TRY(launch_spmv_t(ctx, A->csc(), VecIn{w, nullptr, 0}, v, EPI_STORE, VecIn{}, g));
            RSB_TRY(launch_dot(ctx, n, VecIn{v, nullptr, 0}, VecIn{v, nullptr, 0}, &ps->nt, 1, g, nullptr));
            k_pm_nt<<<1, 1, 0, ctx->stream>>>(ps);
            RSB_TRY(chk(ctx));
            k_div<<<small_grid(n), 256, 0, ctx->stream>>>(v, v, &ps->nt, n, &ps->stop);
            RSB_TRY(chk(ctx));
        }
        k_pm_final<<<1, 1, 0, ctx->stream>>>(ps);
        RSB_TRY(chk(ctx));
        RSB_TRY_CUDA(cudaMemcpyAsync(ctx->h_scalar, &ps->result, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
        *est = ctx->h_scalar[0];
        return RSB_OK;
    };
    rc = run();
    cudaStreamSynchronize(ctx->stream);
    dev_free(ctx, v, n * sizeof(double));
    dev_free(ctx, w, m * sizeof(double));
    dev_free(ctx, ps, sizeof(PowerState));
    return rc;
}

}  // extern "C"
