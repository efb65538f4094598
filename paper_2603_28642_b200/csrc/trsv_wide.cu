// Grid-wide sync-free triangular solve for wide DAGs (sm_100a): config-4
// structure at mu = 1 (n = 10^6, 23 / 66 levels of up to 236,578 unknowns).
//
// Persistent warps take 32-task slices in level order from an atomic ticket
// (a slice only depends on earlier positions, held by running warps or its
// own lanes, so the order cannot deadlock).  A lane loads its whole task at
// once -- its row and right-hand side (a gather through the row, in flight
// with the entry loads), its entries (up to N in registers) and the
// diagonal -- then polls only the operands still missing, all of them per
// round, through L2 with relaxed gpu-scope loads: a value is published by
// overwriting the output's sentinel, so a poll that finds it ready is also
// the operand load.  The ticket of the next slice is taken before the current
// one is worked on, hiding the atomic's latency.  The arithmetic is the
// reference's per-task order (the same as every other solve kernel here), so
// results are bit-identical.
//
// The previous grid kernel (k_trsv, one task per thread, a block per 128
// tasks) ran 8.8 waves at 37% occupancy (80 registers) and measured
// 110-510 GB/s on the config-4 structure (ncu: IPC 0.74, DRAM 8%).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kWideBlock = 256;
constexpr unsigned kWideMinBackoffNs = 32, kWideMaxBackoffNs = 128;
constexpr int kWideEvictFirst = 1;  // default of RSB_TRSV_EVICT (measured: L1 0.549 -> 0.526, U 0.796 -> 0.753 ms at n = 8e6)

__device__ __forceinline__ double ld_relaxed_f64(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double(v);
}

// predicated poll without a compiler memory barrier, so that all of a lane's
// polls of one round are in flight together (v keeps its value when !p)
__device__ __forceinline__ void poll_if(bool p, const double *a, unsigned long long &v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.relaxed.gpu.global.b64 %0, [%1];\n}"
                 : "+l"(v)
                 : "l"(a), "r"((int)p));
}

__device__ __forceinline__ void st_relaxed_f64(double *p, double v) {
    unsigned long long b = __double_as_longlong(v);
    if (b == kSentinel) b = 0x7FF8000000000000ull;  // a computed NaN with the sentinel's bits stays a NaN
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}

__device__ __forceinline__ bool is_sentinel(double v) { return __double_as_longlong(v) == (long long)kSentinel; }

// Entries past the N held in registers (U at mu = 1: ~10% of the rows have
// more than 12 entries, so most slices hold one).  They are handled in
// batches of kTailB with every load of a batch in flight together: a long
// task costs ceil((len - N) / kTailB) round trips instead of len - N.
constexpr int kTailB = 8;

// the task's entry count past `from` (entries are contiguous, then -1 padding)
__device__ __noinline__ int wide_tail_len(const TriDev &T, int64_t base, int lane, int from, int K) {
    int len = from;
    for (int q0 = from; q0 < K; q0 += kTailB) {
        int col[kTailB];
#pragma unroll
        for (int u = 0; u < kTailB; ++u) col[u] = q0 + u < K ? T.ecol[base + (int64_t)(q0 + u) * 32 + lane] : -1;
#pragma unroll
        for (int u = 0; u < kTailB; ++u) len += col[u] >= 0;
        if (col[kTailB - 1] < 0) break;
    }
    return len;
}

// are all entries past `from` published? (never blocks: a dependency may sit
// in another lane of the same warp)
__device__ __noinline__ bool wide_tail_ready(const TriDev &T, int64_t base, int lane, int from, int len,
                                             const double *x) {
    for (int q0 = from; q0 < len; q0 += kTailB) {
        int col[kTailB];
        unsigned long long v[kTailB];
#pragma unroll
        for (int u = 0; u < kTailB; ++u) col[u] = q0 + u < len ? T.ecol[base + (int64_t)(q0 + u) * 32 + lane] : -1;
#pragma unroll
        for (int u = 0; u < kTailB; ++u) {
            v[u] = 0;
            poll_if(col[u] >= 0, x + (col[u] >= 0 ? col[u] : 0), v[u]);
        }
#pragma unroll
        for (int u = 0; u < kTailB; ++u)
            if (col[u] >= 0 && v[u] == kSentinel) return false;
    }
    return true;
}

// entries past `from`, all published: the sequential order, out of line
template <int MODE>
__device__ __noinline__ double wide_tail(const TriDev &T, int64_t base, int lane, int from, int len, double acc,
                                         double dot, const double *x) {
    for (int q0 = from; q0 < len; q0 += kTailB) {
        int col[kTailB];
        double val[kTailB];
        unsigned long long v[kTailB];
#pragma unroll
        for (int u = 0; u < kTailB; ++u) {
            const bool in = q0 + u < len;
            col[u] = in ? T.ecol[base + (int64_t)(q0 + u) * 32 + lane] : -1;
            val[u] = in ? T.eval[base + (int64_t)(q0 + u) * 32 + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kTailB; ++u) {
            v[u] = 0;
            poll_if(col[u] >= 0, x + (col[u] >= 0 ? col[u] : 0), v[u]);
        }
#pragma unroll
        for (int u = 0; u < kTailB; ++u) {
            if (col[u] < 0) break;
            const double xj = __longlong_as_double((long long)v[u]);
            if (!(MODE & 1)) {
                if (xj != 0.0) acc = __dsub_rn(acc, __dmul_rn(val[u], xj));
            } else {
                dot = fma(val[u], xj, dot);
            }
        }
    }
    return (MODE & 1) ? __dsub_rn(acc, dot) : acc;
}

// resident blocks the register budget is sized for: fewer registers per lane
// (smaller N * P) buy more warps in flight
template <int R>
struct WideOcc {
    static constexpr int value = R <= 4 ? 6 : (R <= 8 ? 4 : 3);
};

// P consecutive slices per ticket, each lane holding one task of each: the
// tasks of a ticket are polled together (no slice waits behind another), and
// the ticket counter -- one address all warps hit -- sees P times fewer
// atomics.  A task may depend on an earlier task of its own ticket (even its
// own lane's): the warp-synchronous rounds publish it first.
template <int MODE, int N, bool TAIL, int P>
__global__ void __launch_bounds__(kWideBlock, WideOcc<N * P>::value) k_trsv_wide(TriDev T, VecIn a, const double *c,
                                                                               double *x, int first_slice, int nslices,
                                                                               unsigned max_backoff, Gate g, int ev) {
    if (gated(g)) return;
    const int lane = threadIdx.x & 31;
    // slices wholly inside level 0 were solved by the prologue
    const int ntickets = (nslices - first_slice + P - 1) / P;
    auto take = [&]() {
        int s = 0;
        if (lane == 0) s = (int)atomicAdd(T.ticket, 1ull);
        return __shfl_sync(0xffffffffu, s, 0);
    };
    int j = take();
    if (T.prof && j == 0 && lane == 0) {  // diagnostics: start stamp
        unsigned long long ts;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
        T.prof[7] = (long long)ts;
    }
    while (j < ntickets) {
        int row[P], len[P];
        double acc[P], d[P];
        int cols[P][N];
        double vals[P][N], xv[P][N];
        unsigned need[P], prev_need[P];
        bool done[P];
        int64_t base[P];
#pragma unroll
        for (int u = 0; u < P; ++u) {
            const int s = first_slice + j * P + u;
            const int t = s * 32 + lane;
            const bool valid = s < nslices && t < T.n;
            row[u] = -1;
            len[u] = 0;
            acc[u] = 0.0;
            d[u] = 1.0;
            need[u] = 0;
            prev_need[u] = ~0u;
            base[u] = 0;
            int K = 0;
            if (s < nslices) {
                base[u] = T.slice_off[s];
                K = (int)((T.slice_off[s + 1] - base[u]) >> 5);
            }
#pragma unroll
            for (int q = 0; q < N; ++q) {
                cols[u][q] = -1;
                vals[u][q] = 0.0;
                xv[u][q] = 0.0;
            }
            if (valid) {
                // the right-hand side a(row) [+ c[row]] is read here (the
                // permutation gather fused): its load overlaps the entry loads
                row[u] = ev ? __ldcs(T.task_row + t) : T.task_row[t];
                acc[u] = a.g ? a.p[a.g[row[u] + a.off]] : a.p[row[u] + a.off];
                if (c) acc[u] = __dadd_rn(acc[u], c[row[u]]);
                if (MODE & 2) d[u] = T.diag[t];
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (q < K) {
                        // ev: the entry stream is read evict-first, so it does not push the
                        // solved values (polled and gathered again) out of L2
                        const int64_t e = base[u] + (int64_t)q * 32 + lane;
                        cols[u][q] = ev ? __ldcs(T.ecol + e) : T.ecol[e];
                        vals[u][q] = ev ? __ldcs(T.eval + e) : T.eval[e];
                    }
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (cols[u][q] >= 0) {
                        need[u] |= 1u << q;
                        ++len[u];
                    }
                if (TAIL && len[u] == N && K > N)  // entries continue past the registers
                    len[u] = wide_tail_len(T, base[u], lane, N, K);
            }
            done[u] = !valid;
        }
        // warp-synchronous polling: every round each pending task loads all
        // of its missing operands; the ready ones compute and publish.  A
        // round without progress backs off, so that thousands of waiting warps
        // do not flood L2 with polls while the frontier level is computed.
        unsigned backoff = 0;
        for (;;) {
            bool pending = false, stalled = true;
#pragma unroll
            for (int u = 0; u < P; ++u) {
                pending |= !done[u];
                stalled &= done[u] || need[u] == prev_need[u];
            }
            if (!__any_sync(0xffffffffu, pending)) break;
            if (__all_sync(0xffffffffu, stalled) && backoff) __nanosleep(backoff);
            backoff = backoff ? min(backoff * 2, max_backoff) : kWideMinBackoffNs;
#pragma unroll
            for (int u = 0; u < P; ++u) {
                prev_need[u] = need[u];
                if (done[u]) continue;
                unsigned long long pv[N];
#pragma unroll
                for (int q = 0; q < N; ++q) {
                    pv[q] = kSentinel;
                    poll_if((need[u] >> q) & 1u, x + (cols[u][q] >= 0 ? cols[u][q] : 0), pv[q]);
                }
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (((need[u] >> q) & 1u) && pv[q] != kSentinel) {
                        xv[u][q] = __longlong_as_double((long long)pv[q]);
                        need[u] &= ~(1u << q);
                    }
                if (need[u] == 0 && (!TAIL || len[u] <= N || wide_tail_ready(T, base[u], lane, N, len[u], x))) {
                    double r = acc[u];
                    if (!(MODE & 1)) {
#pragma unroll
                        for (int q = 0; q < N; ++q)
                            if (q < len[u] && xv[u][q] != 0.0) r = __dsub_rn(r, __dmul_rn(vals[u][q], xv[u][q]));
                        if (TAIL && len[u] > N) r = wide_tail<MODE>(T, base[u], lane, N, len[u], r, 0.0, x);
                    } else if (len[u] > 0) {  // < 16 entries (the scalar OpenBLAS order; checked at analysis)
                        double dot = 0.0;
#pragma unroll
                        for (int q = 0; q < N; ++q)
                            if (q < len[u]) dot = fma(vals[u][q], xv[u][q], dot);
                        r = (TAIL && len[u] > N) ? wide_tail<MODE>(T, base[u], lane, N, len[u], r, dot, x)
                                                 : __dsub_rn(r, dot);
                    }
                    if (MODE & 2) r = __ddiv_rn(r, d[u]);
                    if (row[u] >= 0) st_relaxed_f64(x + row[u], r);
                    done[u] = true;
                }
            }
            __syncwarp();
        }
        j = take();
    }
}

// ---------------------------------------------------------------------------
// Static-schedule variant (RSB_TRSV_GRID=static): a cooperative launch (every
// warp resident) takes slices round-robin -- warp w owns slices w, w + W, ...
// of the non-level-0 range -- so a warp knows its next slices and runs a
// three-stage software pipeline across them:
//   A(s+2W): slice offset and task row        (independent loads)
//   B(s+W):  entries, diagonal, the right-hand side's gather index
//   C(s):    the right-hand side value and the dependencies (one round
//            trip), the chain, the store.
// Progress: the lowest unfinished slice's owner is working on it (all its
// earlier slices are finished) and its dependencies lie in lower slices.
// ---------------------------------------------------------------------------
template <int N>
struct StA {
    int64_t base;
    int K, row;
};
template <int N>
struct StB {
    int64_t base;
    int K, row, len;
    int64_t gi;  // index of the right-hand side in a.p
    double d;
    int cols[N];
    double vals[N];
};

template <int N>
__device__ __forceinline__ void st_a(const TriDev &T, int s, int nslices, int lane, StA<N> &A) {
    A.base = 0;
    A.K = 0;
    A.row = -1;
    if (s < nslices) {
        A.base = T.slice_off[s];
        A.K = (int)((T.slice_off[s + 1] - A.base) >> 5);
        const int t = s * 32 + lane;
        if (t < T.n) A.row = __ldcs(T.task_row + t);
    }
}

template <int MODE, int N, bool TAIL>
__device__ __forceinline__ void st_b(const TriDev &T, const VecIn &a, int s, int lane, const StA<N> &A, StB<N> &B) {
    B.base = A.base;
    B.K = A.K;
    B.row = A.row;
    B.len = 0;
    B.gi = 0;
    B.d = 1.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        B.cols[q] = -1;
        B.vals[q] = 0.0;
    }
    if (A.row < 0) return;
    B.gi = a.g ? (int64_t)a.g[A.row + a.off] : (int64_t)A.row + a.off;
    if (MODE & 2) B.d = T.diag[s * 32 + lane];
#pragma unroll
    for (int q = 0; q < N; ++q)
        if (q < A.K) {
            const int64_t e = A.base + (int64_t)q * 32 + lane;
            B.cols[q] = __ldcs(T.ecol + e);
            B.vals[q] = __ldcs(T.eval + e);
        }
}

// the gate, read once before the static solve: every warp of the launch must
// agree (a warp that skipped its slices would leave others waiting forever)
__global__ void k_gate_snap(Gate g, unsigned long long *snap) { *snap = gated(g) ? 1ull : 0ull; }

template <int MODE, int N, bool TAIL>
__global__ void __launch_bounds__(kWideBlock, 2) k_trsv_static(TriDev T, VecIn a, const double *c, double *x,
                                                                int first_slice, int nslices, unsigned max_backoff,
                                                                Gate g) {
    if (*(volatile const unsigned long long *)T.ticket) return;  // the snapshot of the gate (k_gate_snap)
    const int lane = threadIdx.x & 31;
    const int W = gridDim.x * (kWideBlock / 32);
    const int gw = blockIdx.x * (kWideBlock / 32) + (threadIdx.x >> 5);
    int s = first_slice + gw;
    StA<N> A0, A1;
    StB<N> B;
    st_a<N>(T, s, nslices, lane, A0);
    st_b<MODE, N, TAIL>(T, a, s, lane, A0, B);
    st_a<N>(T, s + W, nslices, lane, A1);
    while (s < nslices) {
        // next slices' stages first: their loads fly while this slice polls
        StB<N> Bn;
        st_b<MODE, N, TAIL>(T, a, s + W, lane, A1, Bn);
        StA<N> A2;
        st_a<N>(T, s + 2 * W, nslices, lane, A2);
        // C(s)
        int len = 0;
        unsigned need = 0;
#pragma unroll
        for (int q = 0; q < N; ++q)
            if (B.cols[q] >= 0) {
                need |= 1u << q;
                ++len;
            }
        if (TAIL && len == N && B.K > N) len = wide_tail_len(T, B.base, lane, N, B.K);
        double acc = 0.0;
        if (B.row >= 0) {
            acc = a.p[B.gi];
            if (c) acc = __dadd_rn(acc, c[B.row]);
        }
        bool done = B.row < 0;
        double xv[N];
#pragma unroll
        for (int q = 0; q < N; ++q) xv[q] = 0.0;
        unsigned prev = ~0u, backoff = 0;
        for (;;) {
            if (!__any_sync(0xffffffffu, !done)) break;
            const bool stalled = done || need == prev;
            if (__all_sync(0xffffffffu, stalled) && backoff) __nanosleep(backoff);
            backoff = backoff ? min(backoff * 2, max_backoff) : kWideMinBackoffNs;
            prev = need;
            if (!done) {
                unsigned long long pv[N];
#pragma unroll
                for (int q = 0; q < N; ++q) {
                    pv[q] = kSentinel;
                    poll_if((need >> q) & 1u, x + (B.cols[q] >= 0 ? B.cols[q] : 0), pv[q]);
                }
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (((need >> q) & 1u) && pv[q] != kSentinel) {
                        xv[q] = __longlong_as_double((long long)pv[q]);
                        need &= ~(1u << q);
                    }
                if (need == 0 && (!TAIL || len <= N || wide_tail_ready(T, B.base, lane, N, len, x))) {
                    double r = acc;
                    if (!(MODE & 1)) {
#pragma unroll
                        for (int q = 0; q < N; ++q)
                            if (q < len && xv[q] != 0.0) r = __dsub_rn(r, __dmul_rn(B.vals[q], xv[q]));
                        if (TAIL && len > N) r = wide_tail<MODE>(T, B.base, lane, N, len, r, 0.0, x);
                    } else if (len > 0) {
                        double dot = 0.0;
#pragma unroll
                        for (int q = 0; q < N; ++q)
                            if (q < len) dot = fma(B.vals[q], xv[q], dot);
                        r = (TAIL && len > N) ? wide_tail<MODE>(T, B.base, lane, N, len, r, dot, x) : __dsub_rn(r, dot);
                    }
                    if (MODE & 2) r = __ddiv_rn(r, B.d);
                    st_relaxed_f64(x + B.row, r);
                    done = true;
                }
            }
            __syncwarp();
        }
        s += W;
        B = Bn;
        A1 = A2;
    }
}

using StaticKernel = void (*)(TriDev, VecIn, const double *, double *, int, int, unsigned, Gate);

template <int MODE>
StaticKernel static_kernel(int n, bool tail) {
    if (n <= 4) return tail ? k_trsv_static<MODE, 4, true> : k_trsv_static<MODE, 4, false>;
    return tail ? k_trsv_static<MODE, 8, true> : k_trsv_static<MODE, 8, false>;
}

// Prologue of a wide solve: every unknown is set to the sentinel the main
// kernel polls, then the level-0 tasks, which have no dependencies, are
// solved (x = rhs, divided by the diagonal for the non-unit kinds -- the same
// operations as the main kernel).  The main
// kernel then skips the slices that lie wholly in level 0 (on config 4 at
// mu = 1 a quarter of L1's unknowns).
//
// Two launches: the sentinel fill runs over x in row order (coalesced), then
// the level-0 pass writes only the level-0 rows.  One pass over all positions
// writing x[task_row[t]] scattered every 8-byte store into its own 32-byte
// sector: at n = 8e6 (x = 64 MB, past what L2 absorbs) that cost ~70 us per
// solve (kernel table: U 0.78 -> 0.85 ms).
template <int MODE>
__global__ void k_wide_prologue(TriDev T, VecIn a, const double *c, double *x, int32_t lvl1, Gate g) {
    if (gated(g)) return;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < lvl1; t += (int64_t)gridDim.x * blockDim.x) {
        const int row = T.task_row[t];
        double r = a.g ? a.p[a.g[row + a.off]] : a.p[row + a.off];
        if (c) r = __dadd_rn(r, c[row]);
        if (MODE & 2) r = __ddiv_rn(r, T.diag[t]);
        unsigned long long bits = __double_as_longlong(r);
        if (bits == kSentinel) bits = 0x7FF8000000000000ull;
        reinterpret_cast<unsigned long long *>(x)[row] = bits;
    }
}

using WideKernel = void (*)(TriDev, VecIn, const double *, double *, int, int, unsigned, Gate, int);

template <int MODE, int P>
WideKernel wide_kernel(int n, bool tail) {
    if (n <= 4) return tail ? k_trsv_wide<MODE, 4, true, P> : k_trsv_wide<MODE, 4, false, P>;
    if (n <= 8) return tail ? k_trsv_wide<MODE, 8, true, P> : k_trsv_wide<MODE, 8, false, P>;
    return tail ? k_trsv_wide<MODE, 12, true, P> : k_trsv_wide<MODE, 12, false, P>;
}

WideKernel wide_kernel_for(int mode, int n, bool tail, int p) {
    if (p == 2) switch (mode) {
            case 0: return wide_kernel<0, 2>(n, tail);
            case 1: return wide_kernel<1, 2>(n, tail);
            case 2: return wide_kernel<2, 2>(n, tail);
            default: return wide_kernel<3, 2>(n, tail);
        }
    switch (mode) {
        case 0: return wide_kernel<0, 1>(n, tail);
        case 1: return wide_kernel<1, 1>(n, tail);
        case 2: return wide_kernel<2, 1>(n, tail);
        default: return wide_kernel<3, 1>(n, tail);
    }
}

}  // namespace

int launch_trsv_wide(rsb_ctx *ctx, const TriSched &T, const TriDev &v, VecIn a, const double *c, double *x, Gate g) {
    // registers hold wide_n entries per task (most tasks fit);
    // longer tasks take the batched out-of-line tail.  RSB_WIDE_P: slices per
    // ticket (experiments)
    const bool tail = T.max_task > T.wide_n;
    const char *ep = getenv("RSB_WIDE_P");
    const int p = (ep && atoi(ep) == 2) ? 2 : 1;
    WideKernel k = wide_kernel_for(T.mode, T.wide_n, tail, p);
    static int per_sm[4][3][2][2] = {};  // occupancy of each instantiation, queried once
    const int ni = T.wide_n <= 4 ? 0 : (T.wide_n <= 8 ? 1 : 2);
    int &occ = per_sm[T.mode & 3][ni][tail ? 1 : 0][p - 1];
    if (occ == 0) {
        RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWideBlock, 0));
        occ = std::max(occ, 1);
    }
    int sms = 0;
    RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const int nslices = (T.n + 31) / 32;
    const int32_t lvl1 = T.h_level_ptr.size() > 1 ? T.h_level_ptr[1] : T.n;  // level-0 positions
    const int first_slice = lvl1 / 32;
    RSB_TRY(launch_fill(ctx, x, T.n, kSentinel, g));
    if (lvl1 > 0) {
        const int pg = (int)std::min<int64_t>(((int64_t)lvl1 + 255) / 256, (int64_t)sms * 8);
        switch (T.mode & 3) {
            case 0: k_wide_prologue<0><<<pg, 256, 0, ctx->stream>>>(v, a, c, x, lvl1, g); break;
            case 1: k_wide_prologue<1><<<pg, 256, 0, ctx->stream>>>(v, a, c, x, lvl1, g); break;
            case 2: k_wide_prologue<2><<<pg, 256, 0, ctx->stream>>>(v, a, c, x, lvl1, g); break;
            default: k_wide_prologue<3><<<pg, 256, 0, ctx->stream>>>(v, a, c, x, lvl1, g); break;
        }
        RSB_TRY_CUDA(cudaGetLastError());
    }
    // experiments: RSB_WIDE_OCC caps the resident blocks per SM, RSB_WIDE_BACKOFF
    // sets the longest back-off (ns) of a waiting warp
    const char *eo = getenv("RSB_WIDE_OCC"), *eb = getenv("RSB_WIDE_BACKOFF");
    const int use_occ = eo ? std::max(1, std::min(occ, atoi(eo))) : occ;
    const unsigned max_backoff = eb ? (unsigned)std::max(kWideMinBackoffNs, (unsigned)atoi(eb)) : kWideMaxBackoffNs;
    const int grid = (int)std::min<int64_t>((int64_t)sms * use_occ,
                                            ((int64_t)(nslices - first_slice) * 32 / p + kWideBlock - 1) / kWideBlock);
    // the static-schedule variant: chosen by the analysis (T.wide_static) or
    // forced (RSB_TRSV_GRID=static / syncfree)
    const char *gvs = getenv("RSB_TRSV_GRID");
    const bool want_static = gvs ? std::strcmp(gvs, "static") == 0 : T.wide_static;
    if (want_static) {
        const char *wn = getenv("RSB_WIDE_N");
        const int sn = (wn ? atoi(wn) <= 4 : (T.wide_static || T.wide_n <= 4)) ? 4 : 8;
        const bool stail = T.max_task > sn;
        StaticKernel sk;
        switch (T.mode & 3) {
            case 0: sk = static_kernel<0>(sn, stail); break;
            case 1: sk = static_kernel<1>(sn, stail); break;
            case 2: sk = static_kernel<2>(sn, stail); break;
            default: sk = static_kernel<3>(sn, stail); break;
        }
        static int socc[4][2][2] = {};
        int &so = socc[T.mode & 3][sn == 8][stail];
        if (so == 0) {
            RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&so, sk, kWideBlock, 0));
            so = std::max(so, 1);
        }
        const int sgrid = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)sms * so, ((int64_t)(nslices - first_slice) * 32 + kWideBlock - 1) / kWideBlock));
        k_gate_snap<<<1, 1, 0, ctx->stream>>>(g, T.ticket == v.ticket ? v.ticket : v.ticket);
        RSB_TRY_CUDA(cudaGetLastError());
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sgrid);
        cfg.blockDim = dim3(kWideBlock);
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // every warp resident: the round-robin schedule needs it
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        RSB_TRY_CUDA(cudaLaunchKernelEx(&cfg, sk, v, a, c, x, first_slice, nslices, max_backoff, g));
        return RSB_OK;
    }
    const char *ee = getenv("RSB_TRSV_EVICT");
    const int ev = ee ? atoi(ee) != 0 : kWideEvictFirst;
    const char *pe = getenv("RSB_TRSV_PERSIST");  // experiments: keep x resident in L2
    if (pe && atoi(pe) != 0) {
        static size_t limit_set = 0;
        int maxw = 0, maxp = 0;
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
        const size_t want = std::min<size_t>((size_t)maxp, (size_t)T.n * sizeof(double));
        if (limit_set < want) {
            RSB_TRY_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
            limit_set = want;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(std::max(grid, 1));
        cfg.blockDim = dim3(kWideBlock);
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = x;
        attr[0].val.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)maxw, (size_t)T.n * sizeof(double));
        attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        RSB_TRY_CUDA(cudaLaunchKernelEx(&cfg, k, v, a, c, x, first_slice, nslices, max_backoff, g, ev));
        return RSB_OK;
    }
    k<<<std::max(grid, 1), kWideBlock, 0, ctx->stream>>>(v, a, c, x, first_slice, nslices, max_backoff, g, ev);
    return RSB_OK;
}

}  // namespace rsb
