// Batched solve (kBatch right-hand sides sharing A and the preconditioner):
// shared declarations of bkernels.cu and bsolver.cu.
#pragma once
#include "control.cuh"
#include "rsb_internal.h"

namespace rsb {

constexpr int kBatch = 8;

// per-RHS skip predicate: RHS r is skipped when the int at a + r*sa (bytes)
// or at b + r*sb is nonzero (the per-RHS control blocks' status / stop words)
struct BGate {
    const int *a;
    int sa;
    const int *b;
    int sb;
};

// exact-order dot partials of a batched launch: T chunks x kBatch RHS
struct BDotChunks {
    int T;
    double *part;
    unsigned *cnt;
};
struct BDotRing {
    double *part = nullptr;  // kDotSlots * kMaxBlasThreads * kBatch
    unsigned *cnt = nullptr;  // kDotSlots
    int64_t next = 0;
};

// scratch of the batched sync-free triangular solve: per-row completion
// flags (epoch-tagged), the epoch, the ticket
struct BTriWs {
    int *flag = nullptr;
    unsigned *epoch = nullptr;
    unsigned long long *ticket = nullptr;
    int64_t n = 0;
};

int launch_bspmv(rsb_ctx *ctx, const Compressed &A, VecIn x, double *y, int epi, VecIn e, const int *all_done);
int launch_bspmv_t(rsb_ctx *ctx, const Compressed &At, VecIn y, double *z, int epi, VecIn e, const int *all_done);
// out[r * ostride bytes] = a_r . b_r; skipped when all of need[r * nstride] are 0
int launch_bdot(rsb_ctx *ctx, BDotRing &ring, int64_t n, VecIn a, VecIn b, double *out, int ostride, int sqrt_out,
                const int *all_done, const int *need = nullptr, int nstride = 0);
int launch_baxpy(rsb_ctx *ctx, double *y, const double *x, const double *scal, int sstride, int sign, int64_t n,
                 BGate g);
int launch_bxpby(rsb_ctx *ctx, double *p, const double *h, const double *beta, int bstride, const int *copy_flag,
                 int cstride, int64_t n, BGate g);
int launch_bcopy(rsb_ctx *ctx, double *dst, VecIn src, int64_t n, BGate g);
int launch_bfill(rsb_ctx *ctx, double *x, int64_t n, double v);
int launch_bcg_init(rsb_ctx *ctx, double *w, double *r, double *p, const double *u, int64_t s, BGate g);
int launch_bpack(rsb_ctx *ctx, double *dst, const double *src, int64_t len, int k);
int launch_bunpack(rsb_ctx *ctx, double *dst, const double *src, int64_t len, int k);
bool btrsv_supported(const TriSched &T);
int launch_btrsv(rsb_ctx *ctx, const TriSched &T, VecIn a, const double *c, double *x, BTriWs &ws,
                 const int *all_done);
// index-order batched solve (btrsv_nat.cu), for schedules the analysis gave the index order
bool btrsv_nat_supported(const TriSched &T);
int launch_btrsv_nat(rsb_ctx *ctx, const TriSched &T, VecIn a, const double *c, double *x, BTriWs &ws,
                     const int *all_done);
int bpost(rsb_ctx *ctx);

}  // namespace rsb
