// Grid-wide sync-free triangular solve for wide DAGs (sm_100a): config-4
// structure at mu = 1 (n = 10^6, 23 / 66 levels of up to 236,578 unknowns).
//
// Persistent warps take 32-task slices in level order from an atomic ticket
// (a slice only depends on earlier positions, held by running warps or its
// own lanes, so the order cannot deadlock).  A lane loads its whole task at
// once -- the right-hand side pre-gathered into position order (one coalesced
// load, no row -> rhs dependency), its entries (up to N in registers) and the
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

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kWideBlock = 256;
constexpr unsigned kWideMinBackoffNs = 32, kWideMaxBackoffNs = 128;

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

// resident blocks the register budget is sized for: fewer registers per task
// (smaller N) buy more warps in flight, which is what the solve is bound by
template <int N>
struct WideOcc {
    static constexpr int value = N <= 4 ? 6 : (N <= 8 ? 4 : 3);
};

template <int MODE, int N, bool TAIL>
__global__ void __launch_bounds__(kWideBlock, WideOcc<N>::value) k_trsv_wide(TriDev T, const double *bpos, double *x, int nslices,
                                                          unsigned max_backoff, int EARLY, Gate g) {
    if (gated(g)) return;
    const int lane = threadIdx.x & 31;
    auto take = [&]() {
        int s = 0;
        if (lane == 0) s = (int)atomicAdd(T.ticket, 1ull);
        return __shfl_sync(0xffffffffu, s, 0);
    };
    int s = take();
    if (T.prof && s == 0 && lane == 0) {  // diagnostics: start stamp
        unsigned long long ts;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
        T.prof[7] = (long long)ts;
    }
    // Optional software pipelining over slices (EARLY): the next slice's
    // ticket is taken while this slice's task loads are in flight, and its
    // entry offsets are loaded while this slice polls.  Holding the next
    // ticket cannot deadlock (it is started after the current slice, whose
    // dependencies all precede it), but measured slower: the held slice
    // waits behind the current one instead of being taken by a free warp.
    int64_t base = 0, base_end = 0;
    if (s < nslices) {
        base = T.slice_off[s];
        base_end = T.slice_off[s + 1];
    }
    while (s < nslices) {
        int nxt_raw = 0;
        if (EARLY && lane == 0) nxt_raw = (int)atomicAdd(T.ticket, 1ull);
        const int t = s * 32 + lane;
        const bool valid = t < T.n;
        const int K = (int)((base_end - base) >> 5);
        int row = -1, len = 0;
        double acc = 0.0, d = 1.0;
        int cols[N];
        double vals[N], xv[N];
        unsigned need = 0;
        if (valid) {
            row = T.task_row[t];
            acc = bpos[t];
            if (MODE & 2) d = T.diag[t];
#pragma unroll
            for (int q = 0; q < N; ++q) {
                cols[q] = -1;
                vals[q] = 0.0;
                xv[q] = 0.0;
                if (q < K) {
                    cols[q] = T.ecol[base + (int64_t)q * 32 + lane];
                    vals[q] = T.eval[base + (int64_t)q * 32 + lane];
                }
            }
#pragma unroll
            for (int q = 0; q < N; ++q)
                if (cols[q] >= 0) {
                    need |= 1u << q;
                    ++len;
                }
            if (TAIL && len == N && K > N)  // entries continue past the registers
                len = wide_tail_len(T, base, lane, N, K);
        }
        int nxt = 0;
        int64_t nbase = 0, nbase_end = 0;
        if (EARLY) {
            nxt = __shfl_sync(0xffffffffu, nxt_raw, 0);
            if (nxt < nslices) {
                nbase = T.slice_off[nxt];
                nbase_end = T.slice_off[nxt + 1];
            }
        }
        bool done = !valid;
        // warp-synchronous polling: every round each pending lane loads all
        // of its missing operands; the ready lanes compute and publish.  A
        // round without progress backs off, so that thousands of waiting warps
        // do not flood L2 with polls while the frontier level is computed.
        unsigned backoff = 0, prev_need = ~0u;
        while (__any_sync(0xffffffffu, !done)) {
            if (__all_sync(0xffffffffu, done || need == prev_need) && backoff) __nanosleep(backoff);
            prev_need = need;
            backoff = backoff ? min(backoff * 2, max_backoff) : kWideMinBackoffNs;
            if (!done) {
                unsigned long long pv[N];
#pragma unroll
                for (int q = 0; q < N; ++q) {
                    pv[q] = kSentinel;
                    poll_if((need >> q) & 1u, x + (cols[q] >= 0 ? cols[q] : 0), pv[q]);
                }
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (((need >> q) & 1u) && pv[q] != kSentinel) {
                        xv[q] = __longlong_as_double((long long)pv[q]);
                        need &= ~(1u << q);
                    }
                if (need == 0 && (!TAIL || len <= N || wide_tail_ready(T, base, lane, N, len, x))) {
                    double r = acc;
                    if (!(MODE & 1)) {
#pragma unroll
                        for (int q = 0; q < N; ++q)
                            if (q < len && xv[q] != 0.0) r = __dsub_rn(r, __dmul_rn(vals[q], xv[q]));
                        if (TAIL && len > N) r = wide_tail<MODE>(T, base, lane, N, len, r, 0.0, x);
                    } else if (len > 0) {  // < 16 entries (the scalar OpenBLAS order; checked at analysis)
                        double dot = 0.0;
#pragma unroll
                        for (int q = 0; q < N; ++q)
                            if (q < len) dot = fma(vals[q], xv[q], dot);
                        r = (TAIL && len > N) ? wide_tail<MODE>(T, base, lane, N, len, r, dot, x) : __dsub_rn(r, dot);
                    }
                    if (MODE & 2) r = __ddiv_rn(r, d);
                    if (row >= 0) st_relaxed_f64(x + row, r);
                    done = true;
                }
            }
            __syncwarp();
        }
        if (EARLY) {
            s = nxt;
            base = nbase;
            base_end = nbase_end;
        } else {
            s = take();
            if (s < nslices) {
                base = T.slice_off[s];
                base_end = T.slice_off[s + 1];
            }
        }
    }
}

using WideKernel = void (*)(TriDev, const double *, double *, int, unsigned, int, Gate);

template <int MODE>
WideKernel wide_kernel(int n, bool tail) {
    if (n <= 4) return tail ? k_trsv_wide<MODE, 4, true> : k_trsv_wide<MODE, 4, false>;
    if (n <= 8) return tail ? k_trsv_wide<MODE, 8, true> : k_trsv_wide<MODE, 8, false>;
    return tail ? k_trsv_wide<MODE, 12, true> : k_trsv_wide<MODE, 12, false>;
}

WideKernel wide_kernel_for(int mode, int n, bool tail) {
    switch (mode) {
        case 0: return wide_kernel<0>(n, tail);
        case 1: return wide_kernel<1>(n, tail);
        case 2: return wide_kernel<2>(n, tail);
        default: return wide_kernel<3>(n, tail);
    }
}

}  // namespace

int launch_trsv_wide(rsb_ctx *ctx, const TriSched &T, const TriDev &v, const double *bpos, double *x, Gate g) {
    // registers hold wide_n entries per task (most tasks fit);
    // longer tasks take the batched out-of-line tail
    const bool tail = T.max_task > T.wide_n;
    WideKernel k = wide_kernel_for(T.mode, T.wide_n, tail);
    static int per_sm[4][3][2] = {};  // occupancy of each instantiation, queried once
    const int ni = T.wide_n <= 4 ? 0 : (T.wide_n <= 8 ? 1 : 2);
    int &occ = per_sm[T.mode & 3][ni][tail ? 1 : 0];
    if (occ == 0) {
        RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWideBlock, 0));
        occ = std::max(occ, 1);
    }
    int sms = 0;
    RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const int nslices = (T.n + 31) / 32;
    // experiments: RSB_WIDE_OCC caps the resident blocks per SM, RSB_WIDE_BACKOFF
    // sets the longest back-off (ns) of a waiting warp
    const char *eo = getenv("RSB_WIDE_OCC"), *eb = getenv("RSB_WIDE_BACKOFF");
    const int use_occ = eo ? std::max(1, std::min(occ, atoi(eo))) : occ;
    const unsigned max_backoff = eb ? (unsigned)std::max(kWideMinBackoffNs, (unsigned)atoi(eb)) : kWideMaxBackoffNs;
    const int grid = (int)std::min<int64_t>((int64_t)sms * use_occ, (nslices * 32 + kWideBlock - 1) / kWideBlock);
    // RSB_WIDE_EARLY=1: software pipelining over slices (experiments; measured
    // slower on config 4 at n = 2e6: U 0.45 vs 0.30 ms -- a warp holding its
    // next slice delays that slice behind its current one)
    const char *ee = getenv("RSB_WIDE_EARLY");
    const int early = (ee && atoi(ee) == 1) ? 1 : 0;
    k<<<std::max(grid, 1), kWideBlock, 0, ctx->stream>>>(v, bpos, x, nslices, max_backoff, early, g);
    return RSB_OK;
}

}  // namespace rsb
