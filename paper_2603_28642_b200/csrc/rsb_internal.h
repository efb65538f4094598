// Internal declarations of librowsplit_b200.so (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/rowsplit_b200.h"

namespace rsb {

void set_error(const char *fmt, ...);

#define RSB_TRY_CUDA(call)                                                                  \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) {                                                            \
            rsb::set_error("CUDA error %s in %s (%s:%d)", cudaGetErrorString(e_), #call,    \
                           __FILE__, __LINE__);                                             \
            return RSB_ECUDA;                                                               \
        }                                                                                   \
    } while (0)

#define RSB_TRY(call)                \
    do {                             \
        int rc_ = (call);            \
        if (rc_ != RSB_OK) return rc_; \
    } while (0)

// Sentinel marking "not yet solved" entries of a triangular-solve output.  A
// signalling-NaN payload: FP64 arithmetic only ever produces quiet NaNs, and
// the solve kernel rewrites a copied input that happens to carry these exact
// bits, so no finished entry can look unfinished.
constexpr unsigned long long kSentinel = 0xFFF4D15EA5E0C0DEull;

// Largest order solved by the single-CTA triangular kernel (one byte of
// shared memory per unknown) and the mean level width below which it is
// chosen over the grid-wide kernel.
constexpr int64_t kCtaTriMaxN = 1 << 20;
constexpr int64_t kCtaTriMaxMeanWidth = 4096;
// Single-CTA solve: values of recently solved tasks live in a shared-memory
// ring indexed by task position (kRing slots).  With one barrier per level, a
// slot written at position p is reused by position p + kRing, so a dependency
// at distance d is still live if d + (widest level) < kRing.
constexpr int kRing = 4096;
// lean staged solve: widest level (one task per consumer thread) and longest task
constexpr int64_t kLeanMaxWidth = 128;
constexpr int64_t kLeanMaxN = 16;
// grid-wide solves with at most this many levels launch one kernel per level
// (0: only on request, RSB_TRSV_GRID=levels)
constexpr int32_t kLevelLaunchMaxLevels = 0;
constexpr int kStageBufs = 4;
constexpr int kStageSmemBudget = 220 * 1024;
// shared-memory bytes of one staging buffer
inline int64_t stage_buf_bytes(int64_t ch, int64_t emax, bool diag) {
    // rhs (8 B), task meta {row, len, record offset, -} (16 B), [diag, 1/diag] (16 B),
    // entry records (16 B, contiguous per task)
    return ch * 8 + ch * 16 + (diag ? ch * 16 : 0) + emax * 16;
}

// One entry of a staged solve: the factor value and where its unknown is read
// from -- the byte offset of its ring slot (>= 0), or -(row + 2) for a
// dependency older than the ring.
struct alignas(16) StageRec {
    double v;
    int32_t src;
    int32_t pad;
};
// lean variant: every task owns ns = round4(N) entry slots (zero-padded);
// per position: rhs (8 B), row (4 B), [diag pair] (16 B), entry values
// (8 B each) and sources (4 B each)
inline int64_t lean_buf_bytes(int64_t ch, int64_t ns, bool diag) {
    return ch * (8 + 4 + (diag ? 16 : 0) + ns * 12);
}
// dynamic shared memory: staging buffers, mbarriers, level bounds (nlevels + 5,
// padded to 4), the producer's event list (2 per chunk + a sentinel); the
// value ring is a static array
inline int64_t lean_dyn_smem_bytes(int64_t ch, int64_t ns, bool diag, int64_t nlevels, int64_t nchunks) {
    return kStageBufs * lean_buf_bytes(ch, ns, diag) + 2 * kStageBufs * 8 + ((nlevels + 8) & ~3LL) * 4 +
           (2 * nchunks + 2) * 8;
}
constexpr int64_t kLeanRingBytes = (int64_t)(kRing + 2) * 8;  // ring + a zero slot (+ pad)
inline int64_t stage_smem_bytes(int64_t ch, int64_t emax, bool diag, int64_t nlevels, int64_t nchunks) {
    // ring, staging buffers, mbarriers, level bounds (padded to 4), chunk record counts
    return (int64_t)kRing * 8 + kStageBufs * stage_buf_bytes(ch, emax, diag) + 2 * kStageBufs * 8 +
           ((nlevels + 4) & ~3LL) * 4 + nchunks * 4;
}
// task metadata of a staged solve (position order)
struct alignas(16) StageMeta {
    int32_t row;  // unknown written
    int32_t len;  // entries
    int32_t roff; // first record, relative to the task's chunk
    int32_t pad;
};

// ---------------------------------------------------------------------------
// device-side views (passed by value to kernels)
// ---------------------------------------------------------------------------

// Compressed sparse rows (or columns, for the transposed product): entries of
// line i are idx/val[ptr[i] .. ptr[i+1]) in the order the reference adds them.
// Row-banded copy of a CSC matrix (devsetup.cu): the entries of every column
// split by row band -- band b holds rows [b*rows_per_band, (b+1)*...) --
// band-major, so the transposed product can form its products band by band
// with each band's slice of the gathered vector resident in L2, then sum
// each column's products in the original order (kernels.cu).
constexpr int kMaxBands = 8;
struct Banded {
    int nbands;
    int64_t rows_per_band;
    const int32_t *bptr[kMaxBands];  // ncols + 1 each, offsets into the band-major arrays
    const int32_t *idx;              // rows, band-major
    const double *val;
    double *prod;                    // products scratch (nnz), owned by the matrix's context
    const void *owner;               // rsb_ctx whose stream may use `prod`
};

struct Compressed {
    int32_t nlines;  // rows for CSR, columns for CSC
    int32_t nother;
    int64_t nnz;
    const int32_t *ptr;
    const int32_t *idx;
    const double *val;
    int32_t max_len;  // longest line
    const Banded *bands = nullptr;  // CSC only, large matrices (see Banded)
};

// A vector operand, optionally read through a gather: v(i) = p[g[i + off]]
// (g == nullptr: p[i + off]).  Used to fuse the residual's pivot-order split
// r[perm] (sv.py:159-161) into the consumers.
struct VecIn {
    const double *p;
    const int32_t *g;
    int64_t off;
};

// Skip predicate for kernels of a device-side control loop: a kernel does no
// work when *a != 0 or (b && *b != 0).  Used to reproduce the reference's
// `break`s (sv.py:211-213,229-237; pc.py:294-307) without host syncs.
struct Gate {
    const int *a;
    const int *b;
};

// Task t's entries in the reference's accumulation order, read from the
// matrix's own arrays: idx/val[base + step * k], k < len (column t of the CSC
// for the transposed solves, row t of the CSR -- columns ascending /
// descending -- otherwise; the diagonal excluded for the non-unit kinds).
struct TaskSrc {
    const int32_t *ptr, *idx;
    const double *val;
    int first_off, last_off, step;  // base = ptr[t] + first_off (step +1) or ptr[t+1] - 1 - last_off (step -1)
    int diag_at;                    // 0: ptr[t] (first), 1: ptr[t+1] - 1 (last), -1: unit
    int forward;                    // dependency order: t ascending (1) or descending (0)
    __device__ void task(int t, int64_t &base, int &len) const {
        const int lo = ptr[t], hi = ptr[t + 1];
        len = (hi - lo) - first_off - last_off;
        base = step > 0 ? (int64_t)lo + first_off : (int64_t)hi - 1 - last_off;
    }
};
using NatSrc = TaskSrc;

// Level-ordered triangular-solve schedule: task t solves unknown task_row[t];
// tasks are sorted by dependency level, so every dependency of task t is a task
// < t.  Warp slice w (tasks 32w..32w+31) stores its entries interleaved --
// entry k of lane l at slice_off[w] + 32k + l -- in the reference's
// accumulation order; padding has col == -1.
struct TriDev {
    int32_t n;
    int32_t mode;  // bit0: dot (FMA/BLAS order) instead of sequential axpy; bit1: divide by diag
    const int32_t *task_row;
    const int64_t *slice_off;
    const int32_t *ecol;
    const double *eval;
    const double *diag;  // per task, nullptr when unit
    unsigned long long *ticket;
    // single-CTA schedules: ecol holds the dependency's task position when
    // its ring slot is still live (>= 0), else -(row + 2); tasks of level l
    // are positions level_ptr[l] .. level_ptr[l+1]
    int32_t has_far;
    int32_t nlevels;
    const int32_t *level_ptr;
    // staged single-CTA solve: task data is streamed into shared memory in
    // chunks of stage_ch positions (TMA bulk copies, kStageBufs deep)
    int32_t stage_ch;     // positions per chunk (multiple of 128, >= widest level)
    int32_t stage_emax;   // max entry slots of a chunk
    int32_t nchunks;
    const int64_t *chunk_roff;  // first record of each chunk (nchunks + 1)
    double *bpos;               // right-hand side gathered into position order
    const StageRec *recs;       // entry records, contiguous per task in position order
    // lean staged solve (lean_n > 0): entry values in lane pairs and sources in
    // lane quads per 32-position slice (one 16-byte load per 2 / 4 entries)
    const double *rval;
    const int32_t *rsrc;
    int32_t stage_lgch;  // log2(stage_ch)
    // lean producer events {level, chunk (issue) or -(chunk + 1) (await)}, by level
    const int2 *lean_ev;
    int32_t lean_nev;
    const StageMeta *meta;      // per position (padded to nchunks * stage_ch)
    const double *ddiag;        // per position: {diag, RN(1/diag)} (staged solve's exact division)
    long long *prof;            // optional per-phase cycle counters (RSB_TRSV_PROFILE), else null
};

// ---------------------------------------------------------------------------
// host-side objects behind the opaque handles
// ---------------------------------------------------------------------------

struct Ctx;

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// level-synchronous wide solve (trsv_lsync.cu): items of up to kLsItem
// consecutive task positions of one level, taken by persistent warps in
// level order; per-level done counts replicated kLsRep times
constexpr int kLsBlock = 256;
constexpr int kLsItem = 32;
constexpr int kLsRep = 32;
constexpr int kLsMaxLevels = 4096;
struct LsyncDev {
    int32_t nitems;
    const int32_t *item_pos;     // nitems + 1 position bounds
    const int32_t *item_level;   // level of each item
    const int32_t *level_items;  // nlevels + 1: first item of each level
    unsigned *ticket;
    unsigned *done;              // nlevels * kLsRep
};

struct TriSched {
    int kind = -1;
    int32_t n = 0;
    int64_t nlevels = 0;
    int64_t max_width = 0;
    int64_t entries = 0;  // padded entry slots
    int32_t *task_row = nullptr;
    int64_t *slice_off = nullptr;
    int32_t *ecol = nullptr;
    double *eval = nullptr;
    double *diag = nullptr;
    unsigned long long *ticket = nullptr;
    int32_t mode = 0;
    bool single_cta = false;  // run on one CTA with a shared-memory value ring (narrow DAG)
    int32_t has_far = 0;
    int64_t far_entries = 0;
    int32_t *level_ptr = nullptr;  // nlevels + 1 task positions
    int32_t stage_ch = 0, stage_emax = 0, nchunks = 0;
    int64_t *chunk_roff = nullptr;
    double *bpos = nullptr;
    int64_t padded_n = 0;  // task_row / diag / bpos / meta lengths (nchunks * stage_ch when staged)
    StageRec *recs = nullptr;
    int64_t nrecs = 0;
    // lean variant: every task holds at most lean_n entries, levels are at most
    // kCtaTri wide and no dependency is older than the ring; 0 = not lean
    int32_t lean_n = 0;
    // wide DAGs with few levels: one grid launch per level instead of the
    // sync-free grid kernel; host copy of the level bounds
    bool level_launch = false;
    // longest task; the persistent wide kernel (trsv_wide.cu) runs the grid
    // schedule unless a dot-order task has >= 16 entries (blocked BLAS order)
    int32_t max_task = 0;
    int32_t wide_n = 12;  // entries per task the wide kernel holds in registers (4, 8 or 12)
    // static-schedule sync-free variant (trsv_wide.cu k_trsv_static) and its
    // register entries: chosen for sequential-order forward solves whose tasks
    // mostly hold <= 4 entries (config 4's L1 at n = 8e6: 0.53 -> 0.41 ms)
    bool wide_static = false;
    int32_t static_n = 4;
    bool wide = false;
    // index-order sync-free kernel (trsv_nat.cu) reading the matrix's own
    // arrays: chosen when few dependencies are near in index distance
    bool use_nat = false;
    NatSrc nat{};
    int32_t nat_cap = 0;      // entries of a warp's shared-memory window (>= the longest line)
    int32_t nat_max_line = 0; // longest line, diagonal included
    int64_t nat_near = 0;     // dependencies closer than kNatNear positions
    // level-synchronous variant of the wide solve (default for <= kLsMaxLevels levels)
    bool lsync = false;
    // wide DAGs: one cooperative kernel walking the levels with grid barriers
    // (trsv_ls.cu); false: the sync-free kernel (trsv_wide.cu)
    bool level_sync = false;
    int32_t ls_nitems = 0;
    int32_t *ls_item_pos = nullptr, *ls_item_level = nullptr, *ls_level_items = nullptr;
    unsigned *ls_cnt = nullptr;  // the schedule's own counters (calls without a workspace)
    std::vector<int32_t> h_level_ptr;
    double *rval = nullptr;
    int32_t *rsrc = nullptr;
    int2 *lean_ev = nullptr;
    int32_t lean_nev = 0;
    StageMeta *meta = nullptr;
    double *ddiag = nullptr;
    long long *prof = nullptr;  // 8 counters, allocated when RSB_TRSV_PROFILE is set
    int32_t lgch() const {
        int32_t k = 0;
        while (stage_ch > 0 && (1 << k) < stage_ch) ++k;
        return k;
    }
    TriDev view() const {
        return TriDev{n,       mode,       task_row, slice_off,  ecol, eval, diag,   ticket,
                      has_far, (int32_t)nlevels,     level_ptr, stage_ch, stage_emax, nchunks,
                      chunk_roff, bpos,    recs,     rval,       rsrc,  lgch(), lean_ev, lean_nev, meta, ddiag, prof};
    }
};

}  // namespace rsb

// OpenBLAS-thread emulation of the exact dot order (RSB_DOT_BLAS_THREADS):
// per launch, T chunk partials and a completion counter in a ring of slots
constexpr int kMaxBlasThreads = 64;  // OpenBLAS MAX_THREADS of the reference's numpy wheel
constexpr int kDotSlots = 256;
struct DotChunks {
    int T;            // chunks (1: the one-thread order, no combine)
    double *part;     // T partial results
    unsigned *cnt;    // blocks done (the last one combines and resets it)
};

struct rsb_ctx {
    int device = 0;
    int flags = 0;
    int blas_threads = 1;  // OpenBLAS threads the exact dot order reproduces
    double *d_dot_part = nullptr;
    unsigned *d_dot_cnt = nullptr;
    int64_t dot_slot = 0;
    cudaStream_t stream = nullptr;
    // a second stream for graph branches off the critical path (the pcgls
    // iteration's ||x|| and z.z dots), with the events that fork and join it
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev[3] = {};
    int64_t launches = 0;
    int64_t mem_bytes = 0;
    cudaEvent_t ev[16] = {};
    // small device scratch for standalone dots / scalars
    double *d_scalar = nullptr;
    double *h_scalar = nullptr;  // pinned
    // tree-dot partials
    double *d_partials = nullptr;
    int partial_cap = 0;
    // bench instrumentation: event-record nodes around every triangular
    // solve captured into an instrumented iteration graph
    bool tracing = false;
    int trace_n = 0;
    cudaEvent_t trace_ev[64] = {};
    // the same for the sparse products (A x, A^T y, L2 t, L2^T w), recorded on
    // whichever stream launches them (A^T r runs on the side branch)
    int ptrace_n = 0;
    cudaEvent_t ptrace_ev[64] = {};
    double last_prod_ms = 0.0;  // summed by the last rsb_solver_bench
    int64_t last_prod_launches = 0;
    // L2 flush buffer (bench only, allocated on first use)
    void *flush_buf = nullptr;
    size_t flush_bytes = 0;
};

struct rsb_mat {
    rsb_ctx *ctx = nullptr;
    int64_t nrows = 0, ncols = 0, nnz = 0;
    // CSR of A (row sequential order, sc.py:220) and CSC of A (sc.py:231-234)
    int32_t *r_ptr = nullptr, *r_idx = nullptr;
    double *r_val = nullptr;
    int32_t *c_ptr = nullptr, *c_idx = nullptr;
    double *c_val = nullptr;
    int32_t max_row_len = 0, max_col_len = 0;
    // host CSC kept for lazily analysed triangular schedules
    std::vector<int64_t> h_ptr, h_idx;
    std::vector<double> h_val;
    rsb::TriSched *tri[6] = {};
    rsb::Compressed csr() const {
        return rsb::Compressed{(int32_t)nrows, (int32_t)ncols, nnz, r_ptr, r_idx, r_val, max_row_len};
    }
    rsb::Compressed csc() const {
        return rsb::Compressed{(int32_t)ncols, (int32_t)nrows, nnz, c_ptr, c_idx, c_val, max_col_len,
                               bands.nbands ? &bands : nullptr};
    }
    // row bands of the CSC (large matrices: the gathered vector exceeds L2)
    rsb::Banded bands{};
    std::vector<std::pair<void *, size_t>> band_bufs;
};

namespace rsb {

// memory helpers (tracked per context)
int dev_alloc(rsb_ctx *ctx, void **p, size_t bytes);
void dev_free(rsb_ctx *ctx, void *p, size_t bytes);
template <class T>
int dev_upload(rsb_ctx *ctx, T **dst, const T *src, size_t count) {
    RSB_TRY(dev_alloc(ctx, (void **)dst, count * sizeof(T)));
    if (count) RSB_TRY_CUDA(cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return RSB_OK;
}

// Host-or-device vector staging for the standalone entry points (api.cu).
struct Staged {
    rsb_ctx *ctx = nullptr;
    double *d = nullptr;
    size_t n = 0;
    bool owned = false;
    ~Staged();
};
int stage_in(rsb_ctx *ctx, const double *p, int64_t n, int where, Staged &s);
int stage_out(rsb_ctx *ctx, double *p, int64_t n, int where, Staged &s);
int finish_out(rsb_ctx *ctx, double *p, int64_t n, int where, Staged &s);
// cached level-ordered schedule of (matrix, kind)
int get_tri(rsb_mat *T, int kind, TriSched **out);
// one-time kernel attribute setup for the single-CTA triangular solve of order n
int prepare_trsv_cta(int64_t n);
int prepare_trsv_lean(int64_t smem_bytes);
int launch_trsv_lean(rsb_ctx *ctx, const TriSched &T, const TriDev &v, double *x, Gate g);
int launch_trsv_wide(rsb_ctx *ctx, const TriSched &T, const TriDev &v, VecIn a, const double *c, double *x, Gate g);
// index-order sync-free solve (trsv_nat.cu); tri_setup_nat decides whether a
// wide schedule uses it (RSB_TRSV_ORDER=natural | level overrides)
constexpr int64_t kNatNear = 1 << 18;
constexpr int kNatMaxCap = 1024;
// prefilled: x already holds the sentinel (the previous solve of the chain
// wrote it); fill_next: an n-vector this launch also fills with the sentinel
// (the next solve's output), gate or no gate
int launch_trsv_nat(rsb_ctx *ctx, const TriSched &T, const TriDev &v, VecIn a, const double *c, double *x, Gate g,
                    bool prefilled = false, double *fill_next = nullptr, double *rhs_copy = nullptr);
size_t trsv_nat_smem(int mode, int cap);
int tri_setup_nat(rsb_mat *T, int kind, TriSched *S);
TaskSrc tri_task_src(const rsb_mat *T, int kind);
// level-synchronous cooperative solve of a wide schedule for nb = 1 or 8
// interleaved right-hand sides (rstat: per-RHS status words, stride in ints)
int launch_trsv_ls(rsb_ctx *ctx, const TriSched &T, const TriDev &v, VecIn a, const double *c, double *x,
                   unsigned *bar, Gate g, int nb, const int *rstat, int rstride);
int launch_trsv_lsync(rsb_ctx *ctx, const TriSched &T, const TriDev &v, unsigned *counters, VecIn a,
                      const double *c, double *x, Gate g);
constexpr size_t kLsCounters = 32 + (size_t)kLsMaxLevels * kLsRep;
// one-time kernel attribute setup for the dense S solve of size s
int prepare_chol(int64_t s);
// one-time kernel attribute setup at context creation (dynamic shared memory)
int prepare_kernels();

// Per-stream scratch of triangular solves: the gathered right-hand side of the
// staged kernel and the block ticket of the grid kernel.  Owned by whoever
// launches (a preconditioner's workspace, a solver), never by the immutable
// schedule, so solves on different streams can share one schedule.
struct TriWs {
    double *bpos = nullptr;
    int64_t cap = 0;
    unsigned long long *ticket = nullptr;
    unsigned *ls_cnt = nullptr;  // kLsCounters
};
int tri_ws_alloc(rsb_ctx *ctx, TriWs &w, int64_t cap);
void tri_ws_free(rsb_ctx *ctx, TriWs &w);

// triangular-solve analysis (analysis.cpp)
int tri_analyse(rsb_mat *T, int kind, TriSched **out);
// device-side setup (devsetup.cu): matrices of at least kDeviceUploadMinNnz
// entries are checked and converted (CSR included) on the device; wide
// schedules (order > kCtaTriMaxN) are analysed there
constexpr int64_t kDeviceUploadMinNnz = 1 << 22;
int mat_upload_device(rsb_mat *A, const int64_t *col_ptr, const int64_t *row_idx, const double *values);
int mat_host_copy(rsb_mat *A);
// row bands of A's CSC when its gathered vector (8 * nrows bytes) exceeds
// kBandBytes and RSB_BANDS=1 (opt-in: measured slower); frees with the matrix
constexpr int64_t kBandBytes = 40ll << 20;
int mat_build_bands(rsb_mat *A);
int tri_analyse_device(rsb_mat *T, int kind, TriSched **out);
void tri_free(rsb_ctx *ctx, TriSched *s);

// ---------------------------------------------------------------------------
// kernel launchers (kernels.cu); all enqueue on ctx->stream
// ---------------------------------------------------------------------------
enum EpiOp { EPI_STORE = 0, EPI_ADD = 1, EPI_SUB_FROM = 2 };
// y(i) = acc (STORE) | e(i) + acc (ADD) | e(i) - acc (SUB_FROM),
// acc = sequential row sum of A x from 0.0 (sc.py:218-220)
int launch_spmv(rsb_ctx *ctx, const Compressed &A, VecIn x, double *y, int epi, VecIn e, Gate g);
// z(j) = acc | e(j) + acc, acc = p0 + pairwise(p1..), p = vals * y[rows] (sc.py:231-234)
int launch_spmv_t(rsb_ctx *ctx, const Compressed &At, VecIn y, double *z, int epi, VecIn e, Gate g);
// triangular solve of a schedule: x(row) = solve with rhs(row) = a(row) [+ c[row]]
// (ws: the launcher's scratch; nullptr uses the schedule's own, for standalone calls)
// A chain of solves whose outputs must hold the sentinel before they start
// (the sync-free kernels): a solve fills its successor's output while it runs
// -- the solves are latency-bound, the stores ride along -- instead of one
// fill launch per solve.  On return fill_next holds the sentinel whatever the
// gate says (by the solve kernel, or by a fill launch where the variant has
// no in-kernel fill).
struct TrsvChain {
    bool prefilled = false;       // x already holds the sentinel
    double *fill_next = nullptr;  // n-vector to fill with the sentinel (nullptr: none)
    // n-vector that receives the right-hand side a(row) as the solve reads it
    // (a permuted gather paid once for two solves); only where
    // trsv_wants_prefill(T) -- other variants ignore it
    double *rhs_copy = nullptr;
};
inline bool trsv_wants_prefill(const TriSched &T) { 
    return T.n > 0 && !T.single_cta && !T.level_launch && !T.lsync && T.wide && T.use_nat;  // launch_trsv's dispatch
}
int launch_trsv(rsb_ctx *ctx, const TriSched &T, VecIn a, const double *c, double *x, Gate g,
                const TriWs *ws = nullptr, TrsvChain chain = TrsvChain{});
// out[0] = a.b (sqrt_out: sqrt(a.b)) in the context's dot order; need: optional
// flag that must be nonzero for the dot to run
int launch_dot(rsb_ctx *ctx, int64_t n, VecIn a, VecIn b, double *out, int sqrt_out, Gate g,
               const int *need);
int launch_fill(rsb_ctx *ctx, double *x, int64_t n, unsigned long long bits, Gate g);
int launch_copy(rsb_ctx *ctx, double *dst, VecIn src, int64_t n, Gate g);
// y = y + s*x (sign=+1) or y = y - s*x (sign=-1), s = *scal
int launch_axpy(rsb_ctx *ctx, double *y, const double *x, const double *scal, int sign, int64_t n,
                Gate g);
// p = h + (*beta) * p, or p = h when *copy_flag != 0
int launch_xpby(rsb_ctx *ctx, double *p, const double *h, const double *beta, const int *copy_flag,
                int64_t n, Gate g);
// overwrite a buffer larger than L2 (bench: cold-cache iterations)
int launch_l2_flush(rsb_ctx *ctx);
// dense Cholesky solve with the lower column-major factor (sc.py:607-622)
int launch_chol_solve(rsb_ctx *ctx, const double *G, int64_t s, const double *u, double *w, Gate g);

}  // namespace rsb
