/*
 * rowsplit_b200.h -- C ABI of the B200-native solve phase of the
 * row-splitting ILU preconditioned CGLS method (arxiv 2603.28642).
 *
 * One shared library, librowsplit_b200.so, all entry points extern "C",
 * plain pointers and sizes, FP64 values, int64 host indices (int32 on the
 * device).  The reference (`rowsplit`, pure Python + numpy) has no FFI; the
 * interface this ABI replaces is its Python API, cited per entry point as
 * file:line under /root/reference/pkg/src/rowsplit/ (sc = sparse_core.py,
 * pc = precond.py, sv = solver.py, il = ilup.py).  The Python mirror in
 * paper_2603_28642_b200/ binds it with ctypes.
 *
 * Conventions
 *   - Every function returns RSB_OK (0) or an RSB_E* status; the message
 *     of the last failure on the calling thread is rsb_last_error().
 *     Status -> Python exception: EINVAL -> ValueError, ESINGULAR ->
 *     numpy.linalg.LinAlgError, ECUDA/ENOMEM/ESTATE -> RuntimeError.
 *   - `where` says whether vector arguments are host (RSB_HOST) or device
 *     (RSB_DEVICE) pointers.  Host buffers are borrowed for the call only;
 *     host-pointer calls return after the result is in host memory.
 *   - Handles own their device memory and are immutable after creation
 *     (reference: sc.py:7-8, pc.py:111-113).  One rsb_ctx = one CUDA
 *     stream; a context is not re-entrant, use one per thread.
 *   - Arithmetic follows the reference's operation order.  With
 *     RSB_DOT_EXACT (default) every reduction reproduces numpy/OpenBLAS's
 *     association, so results are bit-identical to the reference run
 *     single-threaded on its host.
 */
#ifndef ROWSPLIT_B200_H
#define ROWSPLIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSB_OK 0
#define RSB_EINVAL 1    /* ValueError */
#define RSB_ESINGULAR 2 /* numpy.linalg.LinAlgError */
#define RSB_ECUDA 3     /* RuntimeError: CUDA failure / no device */
#define RSB_ENOMEM 4    /* RuntimeError: allocation */
#define RSB_ESTATE 5    /* RuntimeError: call out of order */

#define RSB_HOST 0
#define RSB_DEVICE 1
/* device pointers, enqueued on the context's stream without synchronising:
 * the caller orders its own work after it on that stream (rsb_ctx_stream);
 * rsb_dot then writes its result to the device pointer `out` */
#define RSB_DEVICE_ASYNC 2

/* context flags: reduction order for dots and norms */
#define RSB_DOT_EXACT 0 /* reference (OpenBLAS ddot) association: bitwise parity */
#define RSB_DOT_TREE 1  /* fixed-order two-level tree: deterministic, faster for n >> 1e6 */
/* exact order of the reference's OpenBLAS running T threads (OPENBLAS_NUM_THREADS=T
 * on a host with >= T cores, T <= 64): a dot longer than 10000 is split into T
 * contiguous chunks of widths ceil(rest / threads left), each reduced in the
 * one-thread order, partials summed in chunk order.  T = 0 or 1: one thread. */
#define RSB_DOT_BLAS_THREADS(t) (((t) & 0xFF) << 8)

/* triangular solve kinds (sc.py:243-313) */
#define RSB_TRI_LOWER 0        /* sparse_lower_solve(L, b, unit_diag=False)  sc.py:243 */
#define RSB_TRI_LOWER_UNIT 1   /* sparse_lower_solve(L, b, unit_diag=True)   sc.py:243 */
#define RSB_TRI_UPPER 2        /* sparse_upper_solve(U, b)                   sc.py:266 */
#define RSB_TRI_LOWER_T 3      /* sparse_lower_solve_transpose(L, b, False)  sc.py:282 */
#define RSB_TRI_LOWER_T_UNIT 4 /* sparse_lower_solve_transpose(L, b, True)   sc.py:282 */
#define RSB_TRI_UPPER_T 5      /* sparse_upper_solve_transpose(U, b)         sc.py:301 */

/* SMode / YMode (pc.py:36-48) */
#define RSB_S_DENSE 0
#define RSB_S_CG 1
#define RSB_S_IDENTITY 2
#define RSB_Y_EXPLICIT 0
#define RSB_Y_IMPLICIT 1

typedef struct rsb_ctx rsb_ctx;
typedef struct rsb_mat rsb_mat;
typedef struct rsb_pre rsb_pre;
typedef struct rsb_solver rsb_solver;
typedef struct rsb_ilup rsb_ilup;
typedef struct rsb_bsolver rsb_bsolver;
typedef struct rsb_dbuild rsb_dbuild;

/* ---- library / context ------------------------------------------------ */
const char *rsb_last_error(void);
int rsb_version(void);
int rsb_device_count(int *count);
int rsb_ctx_create(int device, int flags, rsb_ctx **out);
int rsb_ctx_destroy(rsb_ctx *ctx);
int rsb_ctx_sync(rsb_ctx *ctx);
/* the context's CUDA stream (a cudaStream_t), for callers that enqueue their
 * own work -- e.g. NCCL collectives -- in order with RSB_DEVICE_ASYNC calls */
int rsb_ctx_stream(rsb_ctx *ctx, void **stream);
/* launches of this library's kernels since the counter was last reset */
int rsb_ctx_kernel_launches(rsb_ctx *ctx, int64_t *count, int reset);
/* device memory of this context (bytes currently allocated) */
int rsb_ctx_mem_bytes(rsb_ctx *ctx, int64_t *bytes);
/* pinned host staging + device scratch, for callers timing copies */
int rsb_host_alloc(int64_t bytes, void **ptr);
int rsb_host_free(void *ptr);
int rsb_device_alloc(rsb_ctx *ctx, int64_t bytes, void **ptr);
int rsb_device_free(rsb_ctx *ctx, void *ptr);
int rsb_memcpy(rsb_ctx *ctx, void *dst, const void *src, int64_t bytes, int kind /*0 h2d,1 d2h,2 d2d*/);
/* device timing on the context stream: elapsed ms between two marks */
int rsb_event_mark(rsb_ctx *ctx, int slot);
int rsb_event_elapsed(rsb_ctx *ctx, int slot0, int slot1, float *ms);

/* ---- matrices: CscMatrix (sc.py:27-131) --------------------------------- */
/* Uploads host CSC (int64 col_ptr/row_idx, f64 values) as device CSR+CSC. */
int rsb_mat_create(rsb_ctx *ctx, int64_t nrows, int64_t ncols, const int64_t *col_ptr,
                   const int64_t *row_idx, const double *values, rsb_mat **out);
int rsb_mat_destroy(rsb_mat *A);
int rsb_mat_info(const rsb_mat *A, int64_t *nrows, int64_t *ncols, int64_t *nnz);

/* y = A x      matvec            sc.py:212-221 */
int rsb_matvec(rsb_mat *A, const double *x, double *y, int where);
/* z = A^T y    matvec_transpose  sc.py:224-235 */
int rsb_matvec_transpose(rsb_mat *A, const double *y, double *z, int where);
/* triangular solves, kind = RSB_TRI_*  (sc.py:243-313).  Level analysis is
 * done on first use per (matrix, kind) and cached on the matrix. */
int rsb_trsv(rsb_mat *T, int kind, const double *b, double *x, int where);
/* diagnostics: per-phase cycle counters of the last staged solve of (matrix,
 * kind); only when the schedule was analysed with RSB_TRSV_PROFILE set */
int rsb_trsv_profile(rsb_mat *T, int kind, long long *counters);
/* diagnostics (wide solve, RSB_TRSV_PROFILE): stamps[0] = start, stamps[1 + l]
 * = %globaltimer when level l completed, for min(cap, 4097) entries */
int rsb_trsv_profile_levels(rsb_mat *T, int kind, long long *stamps, int64_t cap);
/* dependency levels of the (matrix, kind) solve DAG (analysing it if needed) */
int rsb_trsv_levels(rsb_mat *T, int kind, int64_t *nlevels, int64_t *max_width);
/* which kernel runs the (matrix, kind) solve: RSB_TRSV_GRID (sync-free
 * grid-wide, wide DAGs), RSB_TRSV_STAGED (one CTA, staged records),
 * RSB_TRSV_LEAN (one CTA, register-pipelined; *lean_n = its longest task,
 * else 0), RSB_TRSV_LEVELS (a grid launch per level: wide DAGs with few
 * levels) or RSB_TRSV_LSYNC (one persistent launch, items of one level
 * taken in level order, a level waits on the previous one's completion) */
#define RSB_TRSV_GRID 0
#define RSB_TRSV_STAGED 1
#define RSB_TRSV_LEAN 2
#define RSB_TRSV_LEVELS 3
#define RSB_TRSV_LSYNC 4 /* persistent level-synchronous grid solve, items taken in level order (option) */
#define RSB_TRSV_LEVELSYNC 5 /* cooperative grid solve walking the levels with grid barriers (wide DAGs; default) */
#define RSB_TRSV_NATURAL 6 /* sync-free grid solve in index order, entries read from the matrix's own arrays (wide DAGs with far dependencies; default there) */
int rsb_trsv_variant(rsb_mat *T, int kind, int *variant, int *lean_n);
/* power_method_norm2 (sc.py:428-454); v0 = default_rng(seed).standard_normal(n),
 * drawn by the caller (host RNG stays on the host). */
int rsb_power_norm2(rsb_mat *A, const double *v0, int iters, double *est);
/* dense_cholesky_solve (sc.py:607-622): S x = b with the lower s x s
 * column-major factor G (host or device pointers per `where`) */
int rsb_chol_solve(rsb_ctx *ctx, int64_t s, const double *G, const double *b, double *x, int where);
/* a @ b for device vectors in the context's dot order */
int rsb_dot(rsb_ctx *ctx, int64_t n, const double *a, const double *b, double *out, int where);

/* ---- preconditioner: RowSplitPreconditioner (pc.py:106-186) ------------- */
/* perm: row_perm.perm (length m); L1 n x n strict lower (unit diagonal
 * implied), L2 (m-n) x n, U n x n upper with the diagonal stored last;
 * Y ((m-n) x n) required for RSB_Y_EXPLICIT; S_factor (s x s lower,
 * column-major) required for RSB_S_DENSE.  Mirrors build_preconditioner's
 * checks (pc.py:337-346). */
int rsb_pre_create(rsb_ctx *ctx, int64_t m, int64_t n, const int64_t *perm, rsb_mat *L1,
                   rsb_mat *L2, rsb_mat *U, rsb_mat *Y, const double *S_factor, int64_t s,
                   int s_mode, int y_mode, int cg_iters, rsb_pre **out);
int rsb_pre_destroy(rsb_pre *pre);
/* h = apply(r1, r2)             pc.py:167-186 */
int rsb_pre_apply(rsb_pre *pre, const double *r1, const double *r2, double *h, int where);
/* Y r1 / Y^T w / S v            pc.py:135-154 */
int rsb_pre_y_apply(rsb_pre *pre, const double *r1, double *out, int where);
int rsb_pre_y_apply_transpose(rsb_pre *pre, const double *w, double *out, int where);
int rsb_pre_s_matvec(rsb_pre *pre, const double *v, double *out, int where);

/* ---- solver: pcgls (sv.py:120-268) -------------------------------------- */
typedef struct {
    double norm_A;
    double delta;
    int64_t max_iters;
    int32_t estimator_delay;
    int32_t ratio_raw;
} rsb_cgls_cfg; /* CglsConfig sv.py:33-49 */

typedef struct {
    int64_t its;
    int64_t iters_run;
    int32_t converged;
    int32_t breakdown;
    double ratio_pt_final;
    double residual_norm;
    double gradient_norm;
    int64_t history_len;
} rsb_report; /* SolveReport sv.py:52-85 (psize/nmod are host-side) */

/* A solver owns the iteration workspace for one (A, pre) pair and the
 * captured CUDA graph of one iteration.  pre may be NULL (plain CGLS). */
int rsb_solver_create(rsb_mat *A, rsb_pre *pre, rsb_solver **out);
/* the same, running on ctx's stream (same device as A and pre).  A and pre
 * are read-only during a solve, so solvers on different contexts may share
 * them and run concurrently: the batch of independent right-hand sides of
 * config 4. */
int rsb_solver_create_on(rsb_ctx *ctx, rsb_mat *A, rsb_pre *pre, rsb_solver **out);
int rsb_solver_destroy(rsb_solver *S);
/* x = 0, r = b, z = A^T r, h, rho, p (sv.py:147-200).  *status: 0 running,
 * 4 = z.z == 0 at the start (x = 0 is stationary, sv.py:184-196). */
int rsb_solver_start(rsb_solver *S, const double *b, int where, const rsb_cgls_cfg *cfg,
                     int *status);
/* runs up to k iterations (sv.py:202-241); *status: 0 running, 1 converged,
 * 2 stopped early, 3 iteration cap reached. */
int rsb_solver_iterate(rsb_solver *S, int64_t k, int64_t *iters_run, int *status);
int rsb_solver_get_x(rsb_solver *S, double *x, int where);
/* partial-window certification, final residual and gradient norms
 * (sv.py:243-266); history gets min(cap, history_len) ratios. */
int rsb_solver_finish(rsb_solver *S, rsb_report *rep, double *history, int64_t history_cap);
/* Measurement: k iterations, each a replay of an instrumented copy of the
 * iteration graph bracketed by CUDA events on the context stream (L2 flushed
 * before each when flush != 0, outside the bracket).  Outputs the summed
 * device ms of the iterations and of the triangular solves inside them. */
int rsb_solver_bench(rsb_solver *S, int64_t k, int flush, double *iter_ms, double *tri_ms,
                     int64_t *tri_launches, int64_t *kernels_per_iter, int *status);
/* the sparse products (A x, A^T y, L2 t, L2^T w; sc.py:212-235) of the last
 * rsb_solver_bench call: their summed device ms (A^T r runs on a side branch
 * concurrently with the preconditioner, so classes can overlap) and count */
int rsb_solver_bench_products(rsb_solver *S, double *prod_ms, int64_t *prod_launches);
/* overwrite a 320 MiB scratch buffer (> L2) on the context stream */
int rsb_l2_flush(rsb_ctx *ctx);
/* whole solve in one call: start + iterate + finish + get_x */
int rsb_pcgls(rsb_solver *S, const double *b, int where, const rsb_cgls_cfg *cfg, double *x,
              rsb_report *rep, double *history, int64_t history_cap);
/* count independent solves, S[i] on b[i] -> x[i], reps[i] and
 * history[i*history_cap ...], advanced together so they overlap on the
 * device.  Solvers must be on distinct contexts.  Each result equals
 * rsb_pcgls on that solver alone, bit for bit. */
int rsb_pcgls_many(int count, rsb_solver *const *S, const double *const *b, int where,
                   const rsb_cgls_cfg *cfg, double *const *x, rsb_report *reps, double *history,
                   int64_t history_cap);

/* ---- batched solve: up to 8 right-hand sides sharing A and pre ---------- */
/* config 4's 64 RHS run 8 per GPU with replicated factors.
 * The reference solves one b per pcgls call (sv.py:120-126); a batch solver
 * advances 1..8 of those solves together through kernels that read every
 * matrix and factor entry once for all of them (RHS-interleaved vectors).
 * Each RHS's x and report equal rsb_pcgls on that b, bit for bit.  Needs
 * the implicit Y with cg or identity coupling (or pre == NULL) and wide
 * (grid-schedule) triangular solves; EINVAL otherwise. */
int rsb_bsolver_create(rsb_mat *A, rsb_pre *pre, rsb_bsolver **out);
int rsb_bsolver_destroy(rsb_bsolver *S);
/* B: k x m row-major (host or device per `where`), 1 <= k <= 8; status[k] */
int rsb_bsolver_start(rsb_bsolver *S, int k, const double *B, int where, const rsb_cgls_cfg *cfg, int *status);
int rsb_bsolver_iterate(rsb_bsolver *S, int64_t kit, int *all_done);
/* X: k x n row-major; reps[k]; history[r * history_cap ...] */
int rsb_bsolver_finish(rsb_bsolver *S, double *X, int where, rsb_report *reps, double *history,
                       int64_t history_cap);
int rsb_pcgls_batch8(rsb_bsolver *S, int k, const double *B, int where, const rsb_cgls_cfg *cfg, double *X,
                     rsb_report *reps, double *history, int64_t history_cap);
/* measurement, as rsb_solver_bench, for the whole batch */
int rsb_bsolver_bench(rsb_bsolver *S, int64_t kit, int flush, double *iter_ms, double *tri_ms,
                      int64_t *tri_launches, int64_t *kernels_per_iter, int *all_done);

/* ---- dense-coupling preconditioner build on the device -- */
/* build_y_explicit (pc.py:55-82): Y = L2 L1^{-1}, one sparse-RHS L1^T solve
 * per row of L2 in the reference's DFS reach order (sc.py:328-397), zeros
 * dropped; bit-identical.  what >= 1 also forms S = I + Y Y^T (pc.py:85-92;
 * fixed-order FP64 product, within rounding of numpy's `yd @ yd.T`) and its
 * Cholesky factor (sc.py:585-604; bit-identical given S); what = 2 keeps S.
 * L1, L2: device matrices of one context (rsb_mat_create). */
int rsb_dense_build(rsb_mat *L1, rsb_mat *L2, int what, rsb_dbuild **out);
/* sizes and the seconds of the three phases (Y, S, factor) */
int rsb_dense_build_sizes(const rsb_dbuild *B, int64_t *s, int64_t *n, int64_t *nnz_y, double *seconds3);
/* Y as host CSC (y_ptr n + 1, y_idx / y_val nnz_y), S and the factor as s x s
 * column-major host arrays; any output may be NULL */
int rsb_dense_build_copy(const rsb_dbuild *B, int64_t *y_ptr, int64_t *y_idx, double *y_val, double *S,
                         double *S_factor);
int rsb_dense_build_destroy(rsb_dbuild *B);
/* dense_cholesky_factorize (sc.py:585-604) on the device, in place on an
 * s x s column-major array (host or device per `where`), bit-identical */
int rsb_cholesky_factorize_device(rsb_ctx *ctx, int64_t s, double *g, int where);

/* ---- host setup (stays on the CPU; timed separately) -------------------- */
/* ilup_factorize (il.py:211-368), bit-identical factors.  Inputs: scaled A
 * as host CSC.  Query sizes, then copy out. */
int rsb_ilup_factorize(int64_t m, int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                       const double *values, int64_t p, double tau, double mu, double small,
                       rsb_ilup **out);
int rsb_ilup_sizes(const rsb_ilup *F, int64_t *nnz_l1, int64_t *nnz_l2, int64_t *nnz_u,
                   int64_t *nmod);
int rsb_ilup_copy(const rsb_ilup *F, int64_t *perm, int64_t *l1_ptr, int64_t *l1_idx,
                  double *l1_val, int64_t *l2_ptr, int64_t *l2_idx, double *l2_val,
                  int64_t *u_ptr, int64_t *u_idx, double *u_val, int64_t *row_counts);
int rsb_ilup_destroy(rsb_ilup *F);
/* build_y_explicit (pc.py:55-82): Y = L2 L1^{-1}, host CSC out (two-phase:
 * call with y_idx == NULL to get *nnz_y, then again with buffers). */
int rsb_build_y_explicit(int64_t s, int64_t n, const int64_t *l1_ptr, const int64_t *l1_idx,
                         const double *l1_val, const int64_t *l2_ptr, const int64_t *l2_idx,
                         const double *l2_val, int64_t *nnz_y, int64_t *y_ptr, int64_t *y_idx,
                         double *y_val);
/* dense_cholesky_factorize (sc.py:585-604) in place on an s x s column-major array */
int rsb_cholesky_factorize(int64_t s, double *g);
/* column_scale (sc.py:405-425): norms out, scaled values out */
int rsb_column_scale(int64_t ncols, const int64_t *col_ptr, const double *values,
                     double *scaled_values, double *norms);

/* the same on the device (upload, one kernel, download): bit-identical */
int rsb_column_scale_device(rsb_ctx *ctx, int64_t ncols, const int64_t *col_ptr, const double *values,
                            double *scaled_values, double *norms);

#ifdef __cplusplus
}
#endif
#endif /* ROWSPLIT_B200_H */
