// pcgls on a batch of up to kBatch = 8 right-hand sides sharing A and the
// preconditioner (config 4's 64 RHS are sharded 8 per GPU
// with replicated factors).  The reference solves one b per call
// (sv.py:120-268); here the 8 solves advance together through one captured
// iteration graph whose kernels read every matrix and factor entry once for
// all 8 (bkernels.cu).  Each RHS keeps its own control block -- scalars,
// estimator window, stopping flags -- evaluated by one thread per RHS in
// the control kernels below, so every solve takes exactly the branches it
// would take alone and its x and SolveReport are bit-identical to
// rsb_pcgls on that b.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bsolver.cuh"

namespace rsb {
namespace {

constexpr int kB = kBatch;
constexpr int kSt = (int)sizeof(CglsState);
constexpr int kCg = (int)sizeof(CgState);

// ---- per-RHS control (one thread per RHS; the logic of solver.cu's kernels)
__global__ void kbc_cg_start(CgState *cg, const CglsState *st) {  // pc.py:293-295
    const int r = threadIdx.x;
    if (st[r].status) return;
    cg[r].stop = (cg[r].rho == 0.0) ? 1 : 0;
}
__global__ void kbc_cg_alpha(CgState *cg, const CglsState *st) {  // pc.py:298-301
    const int r = threadIdx.x;
    if (st[r].status || cg[r].stop) return;
    if (cg[r].pq <= 0.0)
        cg[r].stop = 1;
    else
        cg[r].alpha = cg[r].rho / cg[r].pq;
}
__global__ void kbc_cg_beta(CgState *cg, const CglsState *st) {  // pc.py:305-309
    const int r = threadIdx.x;
    if (st[r].status || cg[r].stop) return;
    if (cg[r].rho_new == 0.0) {
        cg[r].stop = 1;
    } else {
        cg[r].beta = cg[r].rho_new / cg[r].rho;
        cg[r].rho = cg[r].rho_new;
    }
}
__device__ void set_all_done(const CglsState *st, int *all_done) {
    __syncthreads();
    if (threadIdx.x == 0) {
        int all = 1;
        for (int q = 0; q < kB; ++q) all &= st[q].status != ST_RUN;
        *all_done = all;
    }
}
__global__ void kbc_start_check(CglsState *st, int *all_done) {  // sv.py:184
    const int r = threadIdx.x;
    st[r].iters_run = 0;
    st[r].its_certified = 0;
    st[r].hist_len = 0;
    st[r].status = (st[r].zz == 0.0) ? ST_ZERO_START : ST_RUN;
    set_all_done(st, all_done);
}
__global__ void kbc_start_rho(CglsState *st, double *x_norms, int64_t xstride) {  // sv.py:198-199
    const int r = threadIdx.x;
    if (st[r].status) return;
    st[r].rho = st[r].zh;
    x_norms[r * xstride] = 0.0;
}
__global__ void kbc_it_begin(CglsState *st) {  // sv.py:203
    const int r = threadIdx.x;
    st[r].need_zp = st[r].status ? 0 : !(st[r].rho > 0.0);
}
__global__ void kbc_it_sigma(CglsState *st) {  // sv.py:203-208
    const int r = threadIdx.x;
    if (st[r].status) return;
    CglsState &s = st[r];
    s.sigma = s.rho > 0.0 ? s.rho : s.zp;
    s.skip_retry = 1;
    if (s.sigma == 0.0) {
        s.skip_retry = 0;
        s.sigma = s.zz;
        s.rho = s.sigma;
    }
}
__global__ void kbc_it_alpha(CglsState *st) {  // sv.py:210-214
    const int r = threadIdx.x;
    if (st[r].status) return;
    if (st[r].qq <= 0.0 || st[r].sigma == 0.0)
        st[r].status = ST_STOPPED;
    else
        st[r].alpha = st[r].sigma / st[r].qq;
}
__global__ void kbc_it_estimate(CglsState *st, double *alphas, double *sigmas, double *x_norms, double *history,
                                int64_t astride, int64_t xstride, int64_t hstride) {  // sv.py:217-232
    const int r = threadIdx.x;
    CglsState &s = st[r];
    if (s.status) return;
    double *al = alphas + r * astride, *sg = sigmas + r * astride, *xn = x_norms + r * xstride;
    double *hi = history + r * hstride;
    const long long it = s.iters_run;
    al[it] = s.alpha;
    sg[it] = s.sigma;
    xn[it + 1] = s.xnorm;
    s.iters_run = it + 1;
    const long long i = s.iters_run - s.d;
    if (i >= 0) {
        const double estim = py_sum_products(al, sg, i, s.iters_run);
        int err = 0;
        const double ratio = py_stopping_ratio(estim, s.norm_A, xn[i], s.b_norm, s.ratio_raw, &err);
        if (err) {
            s.status = ST_ERROR;
            return;
        }
        hi[s.hist_len++] = ratio;
        if (ratio <= s.delta) {
            s.status = ST_CONVERGED;
            s.its_certified = i;
        }
    }
}
__global__ void kbc_it_zz(CglsState *st) {  // sv.py:235-237
    const int r = threadIdx.x;
    if (st[r].status) return;
    if (st[r].zz == 0.0) st[r].status = ST_STOPPED;
}
__global__ void kbc_it_beta(CglsState *st) {  // sv.py:239-241
    const int r = threadIdx.x;
    CglsState &s = st[r];
    if (s.status) return;
    const double rho_new = s.zh;
    if (s.rho != 0.0) {
        s.beta = rho_new / s.rho;
        s.p_copy = 0;
    } else {
        s.p_copy = 1;
    }
    s.rho = rho_new;
}
__global__ void kbc_it_end(CglsState *st, int *all_done) {  // for-loop exhausted (sv.py:202)
    const int r = threadIdx.x;
    if (!st[r].status && st[r].iters_run >= st[r].max_iters) st[r].status = ST_MAXED;
    set_all_done(st, all_done);
}

inline int cchk(rsb_ctx *ctx) { return bpost(ctx); }

}  // namespace
}  // namespace rsb

using namespace rsb;

struct rsb_bsolver {
    rsb_ctx *ctx = nullptr;
    rsb_mat *A = nullptr;
    rsb_pre *pre = nullptr;
    int64_t m = 0, n = 0, s = 0;
    int k = 0;  // right-hand sides of the current solve
    // interleaved vectors (length * 8)
    double *b = nullptr, *r = nullptr, *q = nullptr, *fr = nullptr;  // m
    double *x = nullptr, *z = nullptr, *h = nullptr, *p = nullptr, *g = nullptr;  // n
    double *t1 = nullptr, *t2 = nullptr, *t3 = nullptr, *v = nullptr, *ca = nullptr, *cb = nullptr, *cc = nullptr;  // n
    double *u = nullptr, *w = nullptr, *cr = nullptr, *cp = nullptr, *cq = nullptr;  // s
    CglsState *st = nullptr, *h_st = nullptr;
    CgState *cg = nullptr;
    int *all_done = nullptr, *h_all = nullptr;
    double *alphas = nullptr, *sigmas = nullptr, *x_norms = nullptr, *history = nullptr;
    int64_t cap = 0, d = 5;
    BDotRing ring;
    BTriWs tri;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t graph_kernels = 0;
    cudaGraph_t bgraph = nullptr;
    cudaGraphExec_t bexec = nullptr;
    int btrace = 0;
    bool started = false;
    rsb_cgls_cfg cfg{};
};

namespace {

const BGate none_g{nullptr, 0, nullptr, 0};

BGate st_gate(rsb_bsolver *S) { return BGate{&S->st[0].status, kSt, nullptr, 0}; }
BGate cg_gate(rsb_bsolver *S) { return BGate{&S->st[0].status, kSt, &S->cg[0].stop, kCg}; }

// q = S p = p + L2 L1^{-1} L1^{-T} L2^T p  (s_matvec_implicit, pc.py:149-154)
int b_s_matvec(rsb_bsolver *S, const double *p, double *q) {
    rsb_ctx *ctx = S->ctx;
    rsb_pre *P = S->pre;
    const int *ad = S->all_done;
    RSB_TRY(launch_bspmv_t(ctx, P->L2->csc(), VecIn{p, nullptr, 0}, S->ca, EPI_STORE, VecIn{}, ad));
    RSB_TRY(launch_btrsv(ctx, *P->tL1T, VecIn{S->ca, nullptr, 0}, nullptr, S->cb, S->tri, ad));
    RSB_TRY(launch_btrsv(ctx, *P->tL1, VecIn{S->cb, nullptr, 0}, nullptr, S->cc, S->tri, ad));
    return launch_bspmv(ctx, P->L2->csr(), VecIn{S->cc, nullptr, 0}, q, EPI_ADD, VecIn{p, nullptr, 0}, ad);
}

// w = _cg_fixed_steps(S, u, k)  (pc.py:284-310), per RHS
int b_cg(rsb_bsolver *S) {
    rsb_ctx *ctx = S->ctx;
    rsb_pre *P = S->pre;
    const int64_t s = P->s;
    CgState *cg = S->cg;
    const int *ad = S->all_done;
    RSB_TRY(launch_bcg_init(ctx, S->w, S->cr, S->cp, S->u, s, st_gate(S)));
    RSB_TRY(launch_bdot(ctx, S->ring, s, VecIn{S->cr, nullptr, 0}, VecIn{S->cr, nullptr, 0}, &cg[0].rho, kCg, 0, ad));
    kbc_cg_start<<<1, kB, 0, ctx->stream>>>(cg, S->st);
    RSB_TRY(cchk(ctx));
    for (int it = 0; it < P->cg_iters; ++it) {
        RSB_TRY(b_s_matvec(S, S->cp, S->cq));
        RSB_TRY(launch_bdot(ctx, S->ring, s, VecIn{S->cp, nullptr, 0}, VecIn{S->cq, nullptr, 0}, &cg[0].pq, kCg, 0, ad));
        kbc_cg_alpha<<<1, kB, 0, ctx->stream>>>(cg, S->st);
        RSB_TRY(cchk(ctx));
        RSB_TRY(launch_baxpy(ctx, S->w, S->cp, &cg[0].alpha, kCg, +1, s, cg_gate(S)));
        if (it + 1 == P->cg_iters) break;  // the last step's r, rho_new and p feed nothing (solver.cu)
        RSB_TRY(launch_baxpy(ctx, S->cr, S->cq, &cg[0].alpha, kCg, -1, s, cg_gate(S)));
        RSB_TRY(launch_bdot(ctx, S->ring, s, VecIn{S->cr, nullptr, 0}, VecIn{S->cr, nullptr, 0}, &cg[0].rho_new, kCg,
                            0, ad));
        kbc_cg_beta<<<1, kB, 0, ctx->stream>>>(cg, S->st);
        RSB_TRY(cchk(ctx));
        RSB_TRY(launch_bxpby(ctx, S->cp, S->cr, &cg[0].beta, kCg, nullptr, 0, s, cg_gate(S)));
    }
    return RSB_OK;
}

// h = apply(r[perm][:n], r[perm][n:])  (pc.py:175-186, implicit Y)
int b_apply(rsb_bsolver *S) {
    rsb_ctx *ctx = S->ctx;
    rsb_pre *P = S->pre;
    const int *ad = S->all_done;
    const VecIn r1{S->r, P->perm, 0}, r2{S->r, P->perm, S->n};
    if (P->s > 0) {
        RSB_TRY(launch_btrsv(ctx, *P->tL1, r1, nullptr, S->t1, S->tri, ad));
        RSB_TRY(launch_bspmv(ctx, P->L2->csr(), VecIn{S->t1, nullptr, 0}, S->u, EPI_SUB_FROM, r2, ad));
        const double *w = S->w;
        if (P->s_mode == RSB_S_IDENTITY)
            w = S->u;
        else
            RSB_TRY(b_cg(S));
        RSB_TRY(launch_bspmv_t(ctx, P->L2->csc(), VecIn{w, nullptr, 0}, S->t2, EPI_STORE, VecIn{}, ad));
        RSB_TRY(launch_btrsv(ctx, *P->tL1T, VecIn{S->t2, nullptr, 0}, nullptr, S->t3, S->tri, ad));
        RSB_TRY(launch_btrsv(ctx, *P->tL1, r1, S->t3, S->v, S->tri, ad));
    } else {
        RSB_TRY(launch_btrsv(ctx, *P->tL1, r1, nullptr, S->v, S->tri, ad));
    }
    return launch_btrsv(ctx, *P->tU, VecIn{S->v, nullptr, 0}, nullptr, S->h, S->tri, ad);
}

int b_precondition(rsb_bsolver *S) {
    if (S->pre) return b_apply(S);
    return launch_bcopy(S->ctx, S->h, VecIn{S->z, nullptr, 0}, S->n, st_gate(S));  // h = A^T r (sv.py:166-167)
}

// one iteration of sv.py:202-241 for every RHS of the batch
int b_iteration(rsb_bsolver *S) {
    rsb_ctx *ctx = S->ctx;
    CglsState *st = S->st;
    const int *ad = S->all_done;
    const int64_t m = S->m, n = S->n;
    kbc_it_begin<<<1, kB, 0, ctx->stream>>>(st);
    RSB_TRY(cchk(ctx));
    RSB_TRY(launch_bdot(ctx, S->ring, n, VecIn{S->z, nullptr, 0}, VecIn{S->p, nullptr, 0}, &st[0].zp, kSt, 0, ad,
                        &st[0].need_zp, kSt));
    kbc_it_sigma<<<1, kB, 0, ctx->stream>>>(st);
    RSB_TRY(cchk(ctx));
    // p = z.copy() where sigma fell back to z.z (skip_retry == 0)
    RSB_TRY(launch_bcopy(ctx, S->p, VecIn{S->z, nullptr, 0}, n, BGate{&st[0].status, kSt, &st[0].skip_retry, kSt}));
    RSB_TRY(launch_bspmv(ctx, S->A->csr(), VecIn{S->p, nullptr, 0}, S->q, EPI_STORE, VecIn{}, ad));
    RSB_TRY(launch_bdot(ctx, S->ring, m, VecIn{S->q, nullptr, 0}, VecIn{S->q, nullptr, 0}, &st[0].qq, kSt, 0, ad));
    kbc_it_alpha<<<1, kB, 0, ctx->stream>>>(st);
    RSB_TRY(cchk(ctx));
    RSB_TRY(launch_baxpy(ctx, S->x, S->p, &st[0].alpha, kSt, +1, n, st_gate(S)));
    RSB_TRY(launch_baxpy(ctx, S->r, S->q, &st[0].alpha, kSt, -1, m, st_gate(S)));
    // side branch: ||x||, the estimator, z = A^T r and z.z; the application
    // (which reads only r) on the main branch (solver.cu enqueue_iteration)
    const bool fork = ctx->side != nullptr;
    auto side = [&]() -> int {
        RSB_TRY(launch_bdot(ctx, S->ring, n, VecIn{S->x, nullptr, 0}, VecIn{S->x, nullptr, 0}, &st[0].xnorm, kSt, 1,
                            ad));
        kbc_it_estimate<<<1, kB, 0, ctx->stream>>>(st, S->alphas, S->sigmas, S->x_norms, S->history, S->cap,
                                                   S->cap + 1, S->cap + S->d + 1);
        RSB_TRY(cchk(ctx));
        RSB_TRY(launch_bspmv_t(ctx, S->A->csc(), VecIn{S->r, nullptr, 0}, S->z, EPI_STORE, VecIn{}, ad));
        return launch_bdot(ctx, S->ring, n, VecIn{S->z, nullptr, 0}, VecIn{S->z, nullptr, 0}, &st[0].zz, kSt, 0, ad);
    };
    if (fork) {
        RSB_TRY_CUDA(cudaEventRecord(ctx->fork_ev[0], ctx->stream));
        RSB_TRY_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork_ev[0], 0));
        cudaStream_t main = ctx->stream;
        ctx->stream = ctx->side;
        const int rc = side();
        ctx->stream = main;
        RSB_TRY(rc);
        RSB_TRY_CUDA(cudaEventRecord(ctx->fork_ev[2], ctx->side));
    } else {
        RSB_TRY(side());
        kbc_it_zz<<<1, kB, 0, ctx->stream>>>(st);
        RSB_TRY(cchk(ctx));
    }
    if (S->pre) RSB_TRY(b_precondition(S));
    if (fork) {
        RSB_TRY_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->fork_ev[2], 0));
        kbc_it_zz<<<1, kB, 0, ctx->stream>>>(st);
        RSB_TRY(cchk(ctx));
    }
    if (!S->pre) RSB_TRY(b_precondition(S));
    RSB_TRY(launch_bdot(ctx, S->ring, n, VecIn{S->z, nullptr, 0}, VecIn{S->h, nullptr, 0}, &st[0].zh, kSt, 0, ad));
    kbc_it_beta<<<1, kB, 0, ctx->stream>>>(st);
    RSB_TRY(cchk(ctx));
    RSB_TRY(launch_bxpby(ctx, S->p, S->h, &st[0].beta, kSt, &st[0].p_copy, kSt, n, st_gate(S)));
    kbc_it_end<<<1, kB, 0, ctx->stream>>>(st, S->all_done);
    return cchk(ctx);
}

int b_capture(rsb_bsolver *S, bool trace, cudaGraph_t *graph, cudaGraphExec_t *exec, int64_t *kernels, int *ntrace) {
    rsb_ctx *ctx = S->ctx;
    const int64_t before = ctx->launches;
    if (trace) {
        ctx->tracing = true;
        ctx->trace_n = 0;
    }
    RSB_TRY_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = b_iteration(S);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
    ctx->tracing = false;
    if (ntrace) *ntrace = ctx->trace_n;
    if (kernels) *kernels = ctx->launches - before;
    ctx->launches = before;
    if (rc != RSB_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    RSB_TRY_CUDA(e);
    *graph = g;
    RSB_TRY_CUDA(cudaGraphInstantiate(exec, g, cudaGraphInstantiateFlagUseNodePriority));
    return RSB_OK;
}

void drop_graphs(rsb_bsolver *S) {
    if (S->exec) cudaGraphExecDestroy(S->exec);
    if (S->graph) cudaGraphDestroy(S->graph);
    if (S->bexec) cudaGraphExecDestroy(S->bexec);
    if (S->bgraph) cudaGraphDestroy(S->bgraph);
    S->exec = nullptr;
    S->graph = nullptr;
    S->bexec = nullptr;
    S->bgraph = nullptr;
}

int ensure_cap(rsb_bsolver *S, int64_t max_iters, int d) {
    if (max_iters <= S->cap && d <= S->d && S->exec) return RSB_OK;
    rsb_ctx *ctx = S->ctx;
    cudaStreamSynchronize(ctx->stream);
    drop_graphs(S);
    if (max_iters > S->cap || d > S->d) {
        const int64_t cap = std::max(max_iters, S->cap), dd = std::max<int64_t>(d, S->d);
        dev_free(ctx, S->alphas, kB * S->cap * sizeof(double));
        dev_free(ctx, S->sigmas, kB * S->cap * sizeof(double));
        dev_free(ctx, S->x_norms, kB * (S->cap + 1) * sizeof(double));
        dev_free(ctx, S->history, kB * (S->cap + S->d + 1) * sizeof(double));
        S->cap = cap;
        S->d = dd;
        RSB_TRY(dev_alloc(ctx, (void **)&S->alphas, kB * cap * sizeof(double)));
        RSB_TRY(dev_alloc(ctx, (void **)&S->sigmas, kB * cap * sizeof(double)));
        RSB_TRY(dev_alloc(ctx, (void **)&S->x_norms, kB * (cap + 1) * sizeof(double)));
        RSB_TRY(dev_alloc(ctx, (void **)&S->history, kB * (cap + dd + 1) * sizeof(double)));
    }
    return b_capture(S, false, &S->graph, &S->exec, &S->graph_kernels, nullptr);
}

void bsolver_free(rsb_bsolver *S) {
    rsb_ctx *ctx = S->ctx;
    cudaStreamSynchronize(ctx->stream);
    drop_graphs(S);
    const size_t m8 = S->m * kB * sizeof(double), n8 = S->n * kB * sizeof(double), s8 = S->s * kB * sizeof(double);
    for (double *q : {S->b, S->r, S->q, S->fr}) dev_free(ctx, q, m8);
    for (double *q : {S->x, S->z, S->h, S->p, S->g, S->t1, S->t2, S->t3, S->v, S->ca, S->cb, S->cc})
        dev_free(ctx, q, n8);
    for (double *q : {S->u, S->w, S->cr, S->cp, S->cq}) dev_free(ctx, q, s8);
    dev_free(ctx, S->st, kB * sizeof(CglsState));
    dev_free(ctx, S->cg, kB * sizeof(CgState));
    dev_free(ctx, S->all_done, sizeof(int));
    if (S->h_st) cudaFreeHost(S->h_st);
    if (S->h_all) cudaFreeHost(S->h_all);
    dev_free(ctx, S->alphas, kB * S->cap * sizeof(double));
    dev_free(ctx, S->sigmas, kB * S->cap * sizeof(double));
    dev_free(ctx, S->x_norms, kB * (S->cap + 1) * sizeof(double));
    dev_free(ctx, S->history, kB * (S->cap + S->d + 1) * sizeof(double));
    dev_free(ctx, S->ring.part, (size_t)kDotSlots * kMaxBlasThreads * kB * sizeof(double));
    dev_free(ctx, S->ring.cnt, kDotSlots * sizeof(unsigned));
    dev_free(ctx, S->tri.flag, S->tri.n * sizeof(int));
    dev_free(ctx, S->tri.epoch, sizeof(unsigned));
    dev_free(ctx, S->tri.ticket, sizeof(unsigned long long));
    delete S;
}

int read_bstate(rsb_bsolver *S) {
    rsb_ctx *ctx = S->ctx;
    RSB_TRY_CUDA(cudaMemcpyAsync(S->h_st, S->st, kB * sizeof(CglsState), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaMemcpyAsync(S->h_all, S->all_done, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    return RSB_OK;
}

}  // namespace

extern "C" {

int rsb_bsolver_create(rsb_mat *A, rsb_pre *pre, rsb_bsolver **out) {
    *out = nullptr;
    rsb_ctx *ctx = A->ctx;
    if (pre && (pre->m != A->nrows || pre->n != A->ncols)) {
        set_error("preconditioner does not match the matrix");
        return RSB_EINVAL;
    }
    if (pre) {
        if (pre->s > 0 && (pre->y_mode != RSB_Y_IMPLICIT || pre->s_mode == RSB_S_DENSE)) {
            set_error("the batched solve supports the implicit Y with cg or identity coupling");
            return RSB_EINVAL;
        }
        for (const TriSched *T : {pre->tL1, pre->tL1T, pre->tU})
            if (T && !btrsv_supported(*T)) {
                set_error("the batched solve needs wide (grid) triangular schedules");
                return RSB_EINVAL;
            }
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    auto *S = new rsb_bsolver();
    S->ctx = ctx;
    S->A = A;
    S->pre = pre;
    S->m = A->nrows;
    S->n = A->ncols;
    S->s = pre ? pre->s : 0;
    int rc = RSB_OK;
    const size_t m8 = S->m * kB * sizeof(double), n8 = S->n * kB * sizeof(double), s8 = S->s * kB * sizeof(double);
    for (double **q : {&S->b, &S->r, &S->q, &S->fr})
        if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)q, m8);
    for (double **q : {&S->x, &S->z, &S->h, &S->p, &S->g})
        if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)q, n8);
    if (pre)
        for (double **q : {&S->t1, &S->t2, &S->t3, &S->v, &S->ca, &S->cb, &S->cc})
            if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)q, n8);
    if (pre && S->s > 0)
        for (double **q : {&S->u, &S->w, &S->cr, &S->cp, &S->cq})
            if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)q, s8);
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->st, kB * sizeof(CglsState));
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->cg, kB * sizeof(CgState));
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->all_done, sizeof(int));
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->ring.part, (size_t)kDotSlots * kMaxBlasThreads * kB * sizeof(double));
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->ring.cnt, kDotSlots * sizeof(unsigned));
    S->tri.n = S->n;
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->tri.flag, S->n * sizeof(int));
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->tri.epoch, sizeof(unsigned));
    if (rc == RSB_OK) rc = dev_alloc(ctx, (void **)&S->tri.ticket, sizeof(unsigned long long));
    if (rc == RSB_OK && (cudaMallocHost((void **)&S->h_st, kB * sizeof(CglsState)) != cudaSuccess ||
                         cudaMallocHost((void **)&S->h_all, sizeof(int)) != cudaSuccess)) {
        set_error("pinned allocation failed");
        rc = RSB_ENOMEM;
    }
    if (rc == RSB_OK) {
        cudaMemsetAsync(S->ring.cnt, 0, kDotSlots * sizeof(unsigned), ctx->stream);
        cudaMemsetAsync(S->tri.flag, 0, S->n * sizeof(int), ctx->stream);
        cudaMemsetAsync(S->tri.epoch, 0, sizeof(unsigned), ctx->stream);
        cudaMemsetAsync(S->cg, 0, kB * sizeof(CgState), ctx->stream);
        cudaMemsetAsync(S->all_done, 0, sizeof(int), ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
            set_error("batched solver initialisation failed");
            rc = RSB_ECUDA;
        }
    }
    if (rc != RSB_OK) {
        bsolver_free(S);
        return rc;
    }
    *out = S;
    return RSB_OK;
}

int rsb_bsolver_destroy(rsb_bsolver *S) {
    if (S) bsolver_free(S);
    return RSB_OK;
}

// sv.py:147-200 for k <= 8 right-hand sides (B: k x m row-major); status[r]
// as rsb_solver_start's
int rsb_bsolver_start(rsb_bsolver *S, int k, const double *B, int where, const rsb_cgls_cfg *cfg, int *status) {
    rsb_ctx *ctx = S->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    if (k < 1 || k > kB) {
        set_error("a batch holds 1..%d right-hand sides", kB);
        return RSB_EINVAL;
    }
    if (!(cfg->delta > 0.0) || cfg->estimator_delay < 1 || cfg->max_iters < 1) {
        set_error("invalid CglsConfig (delta > 0, estimator_delay >= 1, max_iters >= 1)");
        return RSB_EINVAL;
    }
    RSB_TRY(ensure_cap(S, cfg->max_iters, cfg->estimator_delay));
    S->cfg = *cfg;
    S->k = k;
    S->started = false;
    const int64_t m = S->m, n = S->n;
    // B -> staging (fr) -> interleaved b; the unused slots are zero (their
    // z.z == 0 start leaves them stopped from the outset)
    RSB_TRY_CUDA(cudaMemcpyAsync(S->fr, B, (size_t)k * m * sizeof(double),
                                 where != RSB_HOST ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
    RSB_TRY(launch_bpack(ctx, S->b, S->fr, m, k));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < kB; ++r) {
        CglsState init{};
        init.norm_A = cfg->norm_A;
        init.delta = cfg->delta;
        init.max_iters = cfg->max_iters;
        init.d = cfg->estimator_delay;
        init.ratio_raw = cfg->ratio_raw;
        S->h_st[r] = init;
    }
    RSB_TRY_CUDA(cudaMemcpyAsync(S->st, S->h_st, kB * sizeof(CglsState), cudaMemcpyHostToDevice, ctx->stream));
    RSB_TRY_CUDA(cudaMemsetAsync(S->all_done, 0, sizeof(int), ctx->stream));
    CglsState *st = S->st;
    RSB_TRY(launch_bdot(ctx, S->ring, m, VecIn{S->b, nullptr, 0}, VecIn{S->b, nullptr, 0}, &st[0].b_norm, kSt, 1,
                        nullptr));
    RSB_TRY(launch_bfill(ctx, S->x, n, 0.0));
    RSB_TRY(launch_bcopy(ctx, S->r, VecIn{S->b, nullptr, 0}, m, none_g));
    RSB_TRY(launch_bspmv_t(ctx, S->A->csc(), VecIn{S->r, nullptr, 0}, S->z, EPI_STORE, VecIn{}, nullptr));
    RSB_TRY(launch_bdot(ctx, S->ring, n, VecIn{S->z, nullptr, 0}, VecIn{S->z, nullptr, 0}, &st[0].zz, kSt, 0, nullptr));
    kbc_start_check<<<1, kB, 0, ctx->stream>>>(st, S->all_done);
    RSB_TRY(cchk(ctx));
    RSB_TRY(b_precondition(S));
    RSB_TRY(launch_bdot(ctx, S->ring, n, VecIn{S->z, nullptr, 0}, VecIn{S->h, nullptr, 0}, &st[0].zh, kSt, 0,
                        S->all_done));
    kbc_start_rho<<<1, kB, 0, ctx->stream>>>(st, S->x_norms, S->cap + 1);
    RSB_TRY(cchk(ctx));
    RSB_TRY(launch_bcopy(ctx, S->p, VecIn{S->h, nullptr, 0}, n, st_gate(S)));
    RSB_TRY(read_bstate(S));
    for (int r = 0; r < k; ++r) {
        if (S->h_st[r].status == ST_ERROR) {
            set_error("zero denominator in stopping ratio");
            return RSB_EINVAL;
        }
        status[r] = S->h_st[r].status;
    }
    S->started = true;
    return RSB_OK;
}

// up to kit iterations of every running RHS; *all_done once none runs
int rsb_bsolver_iterate(rsb_bsolver *S, int64_t kit, int *all_done) {
    rsb_ctx *ctx = S->ctx;
    if (!S->started) {
        set_error("rsb_bsolver_iterate before rsb_bsolver_start");
        return RSB_ESTATE;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    int64_t done = 0, batch = 4;
    int all = *S->h_all;
    while (!all && done < kit) {
        const int64_t nb = std::min(batch, kit - done);
        for (int64_t i = 0; i < nb; ++i) RSB_TRY_CUDA(cudaGraphLaunch(S->exec, ctx->stream));
        ctx->launches += nb * S->graph_kernels;
        done += nb;
        RSB_TRY(read_bstate(S));
        all = *S->h_all;
        batch = std::min<int64_t>(batch * 2, 64);
    }
    for (int r = 0; r < S->k; ++r)
        if (S->h_st[r].status == ST_ERROR) {
            set_error("zero denominator in stopping ratio");
            return RSB_EINVAL;
        }
    *all_done = all;
    return RSB_OK;
}

// per-RHS reports (sv.py:243-266) and X (k x n row-major)
int rsb_bsolver_finish(rsb_bsolver *S, double *X, int where, rsb_report *reps, double *history, int64_t history_cap) {
    rsb_ctx *ctx = S->ctx;
    if (!S->started) {
        set_error("rsb_bsolver_finish before rsb_bsolver_start");
        return RSB_ESTATE;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    RSB_TRY(read_bstate(S));
    std::vector<CglsState> sts(S->h_st, S->h_st + kB);
    const int64_t cap = S->cap, d = S->d;
    std::vector<double> al(kB * cap), sg(kB * cap), xn(kB * (cap + 1)), hi(kB * (cap + d + 1));
    RSB_TRY_CUDA(cudaMemcpyAsync(al.data(), S->alphas, al.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaMemcpyAsync(sg.data(), S->sigmas, sg.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaMemcpyAsync(xn.data(), S->x_norms, xn.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaMemcpyAsync(hi.data(), S->history, hi.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    // final residual and gradient for every RHS (sv.py:256-266)
    CglsState *dst = S->st;
    RSB_TRY(launch_bspmv(ctx, S->A->csr(), VecIn{S->x, nullptr, 0}, S->fr, EPI_SUB_FROM, VecIn{S->b, nullptr, 0},
                         nullptr));
    RSB_TRY(launch_bdot(ctx, S->ring, S->m, VecIn{S->fr, nullptr, 0}, VecIn{S->fr, nullptr, 0}, &dst[0].qq, kSt, 1,
                        nullptr));
    RSB_TRY(launch_bspmv_t(ctx, S->A->csc(), VecIn{S->fr, nullptr, 0}, S->g, EPI_STORE, VecIn{}, nullptr));
    RSB_TRY(launch_bdot(ctx, S->ring, S->n, VecIn{S->g, nullptr, 0}, VecIn{S->g, nullptr, 0}, &dst[0].zz, kSt, 1,
                        nullptr));
    // x out: interleaved -> row-major staging (fr holds >= k n doubles) -> X
    RSB_TRY(read_bstate(S));
    RSB_TRY(launch_bunpack(ctx, S->fr, S->x, S->n, S->k));
    RSB_TRY_CUDA(cudaMemcpyAsync(X, S->fr, (size_t)S->k * S->n * sizeof(double),
                                 where != RSB_HOST ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < S->k; ++r) {
        const CglsState &st = sts[r];
        rsb_report *rep = &reps[r];
        double *hist_out = history ? history + r * history_cap : nullptr;
        std::memset(rep, 0, sizeof *rep);
        const double res_norm = S->h_st[r].qq, grad_norm = S->h_st[r].zz;
        if (st.status == ST_ZERO_START) {  // sv.py:184-196
            rep->its = 0;
            rep->converged = 1;
            rep->residual_norm = st.b_norm;
            rep->history_len = 1;
            if (hist_out && history_cap > 0) hist_out[0] = 0.0;
            continue;
        }
        const long long it_run = st.iters_run;
        const double *a_r = al.data() + r * cap, *s_r = sg.data() + r * cap, *x_r = xn.data() + r * (cap + 1);
        std::vector<double> hist(hi.data() + r * (cap + d + 1), hi.data() + r * (cap + d + 1) + st.hist_len);
        bool converged = st.status == ST_CONVERGED;
        const bool stopped_early = st.status == ST_STOPPED;
        long long its_cert = st.its_certified;
        if (stopped_early && !converged) {  // sv.py:243-253
            const int dd = S->cfg.estimator_delay;
            for (long long i = std::max(0LL, it_run - dd + 1); i <= it_run; ++i) {
                const double estim = py_sum_products(a_r, s_r, i, it_run);
                int err = 0;
                const double ratio = py_stopping_ratio(estim, S->cfg.norm_A, x_r[i], st.b_norm, S->cfg.ratio_raw, &err);
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
        if (hist_out)
            for (int64_t i = 0; i < std::min<int64_t>(history_cap, (int64_t)hist.size()); ++i) hist_out[i] = hist[i];
    }
    return RSB_OK;
}

int rsb_pcgls_batch8(rsb_bsolver *S, int k, const double *B, int where, const rsb_cgls_cfg *cfg, double *X,
                     rsb_report *reps, double *history, int64_t history_cap) {
    int status[kB];
    RSB_TRY(rsb_bsolver_start(S, k, B, where, cfg, status));
    int all = 0;
    RSB_TRY(rsb_bsolver_iterate(S, cfg->max_iters, &all));
    return rsb_bsolver_finish(S, X, where, reps, history, history_cap);
}

// Measurement: kit iterations, each one replay of an instrumented copy of the
// batch's iteration graph between events (L2 flushed before each, outside).
int rsb_bsolver_bench(rsb_bsolver *S, int64_t kit, int flush, double *iter_ms, double *tri_ms, int64_t *tri_launches,
                      int64_t *kernels_per_iter, int *all_done) {
    rsb_ctx *ctx = S->ctx;
    if (!S->started) {
        set_error("rsb_bsolver_bench before rsb_bsolver_start");
        return RSB_ESTATE;
    }
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    if (!S->bexec) RSB_TRY(b_capture(S, true, &S->bgraph, &S->bexec, nullptr, &S->btrace));
    double it_total = 0.0, tri_total = 0.0;
    for (int64_t i = 0; i < kit; ++i) {
        if (flush) RSB_TRY(rsb_l2_flush(ctx));
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
    }
    RSB_TRY(read_bstate(S));
    *iter_ms = it_total;
    *tri_ms = tri_total;
    *tri_launches = kit * (S->btrace / 2);
    *kernels_per_iter = S->graph_kernels;
    *all_done = *S->h_all;
    return RSB_OK;
}

}  // extern "C"
