// Hot-path kernels of the B200 solve phase (sm_100a, FP64 CUDA cores).
//
// Every kernel reproduces the floating-point operation order of the
// reference's numpy/OpenBLAS code (pkg/src/rowsplit/sparse_core.py = sc.py),
// so results are bit-identical to it.  The file is compiled with
// -fmad=false: a*b+c is two roundings unless fma() is written out.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kBlock = 256;
constexpr int kSpmvHintDefault = 0;  // RSB_SPMV_HINT: L2 evict-first hint on k_spmv's matrix stream
constexpr int kTriBlock = 128;
constexpr int kCtaTri = 128;
constexpr int kStageRegs = 16;
constexpr int kDotChunk = 6144;  // elements per vector per stage of the staged exact dot (48 KB copies)
constexpr int kDotStages = 2;  // stages (a bulk copy occupies the SM's TMA ~900 cycles at any size up to 64 KB: few, large copies)


__device__ __forceinline__ double vin(const VecIn &v, int64_t i) {
    return v.g ? v.p[v.g[i + v.off]] : v.p[i + v.off];
}

// (Gathering the SpMV operand with an L2 evict_last policy and streaming the
// matrix evict-first was measured slower: config 4 at n = 8e6, A x 0.78 vs
// 0.55 ms, A^T y unchanged.)
// OpenBLAS with T threads (interface ddot, n > 10000): T contiguous chunks of
// widths ceil(rem / threads left), each reduced by the one-thread kernel
// above, the partial results summed in chunk order from 0.0
// (blas_level1_thread_with_return_value; verified bit for bit against numpy
// at OPENBLAS_NUM_THREADS = 2, 3, 4, 8 by tests/test_oracle_pin.py).
// Block t of the launch reduces chunk t.
__device__ __forceinline__ void dot_chunk(int64_t n, int T, int t, int64_t &lo, int64_t &w) {
    lo = 0;
    int64_t rem = n;
    for (int i = 0; i < t; ++i) {
        const int64_t wi = (rem + (T - i) - 1) / (T - i);
        lo += wi;
        rem -= wi;
    }
    w = (rem + (T - t) - 1) / (T - t);
}

// lane 0 of every block: publish this chunk's result; the last block to
// finish sums the partials in chunk order and writes the dot.  A gated block
// (skip) still counts itself, so the slot's counter is back at 0 after every
// launch even when the gate flips while the launch is being dispatched (the
// estimator on the side branch can stop the solve mid-launch); the value is
// then not written -- nothing downstream of a stop reads it.
__device__ __forceinline__ void dot_combine(double d, double *out, int sqrt_out, const DotChunks &c, bool skip) {
    if (c.T <= 1) {
        if (!skip) out[0] = sqrt_out ? sqrt(d) : d;
        return;
    }
    if (!skip) c.part[blockIdx.x] = d;
    __threadfence();
    const unsigned prev = atomicAdd(c.cnt, skip ? 0x10000u + 1u : 1u);
    if ((prev & 0xFFFFu) != (unsigned)c.T - 1) return;
    __threadfence();
    *c.cnt = 0;  // ready for the next replay of the graph
    if (skip || (prev >> 16)) return;  // some chunk was gated: no result
    double sum = 0.0;
    for (int i = 0; i < c.T; ++i) sum = __dadd_rn(sum, ((volatile const double *)c.part)[i]);
    out[0] = sqrt_out ? sqrt(sum) : sum;
}

__global__ void k_dot_exact(int64_t n, VecIn a, VecIn b, double *out, int sqrt_out, Gate g,
                            const int *need, DotChunks ch) {
    // `need` is set before the launch; only the gate can flip during it
    if (need && !*(volatile const int *)need) return;
    const bool skip = __shfl_sync(0xffffffffu, gated(g) ? 1 : 0, 0) != 0;
    int64_t lo = 0, w = n;
    if (ch.T > 1) dot_chunk(n, ch.T, blockIdx.x, lo, w);
    double d = 0.0;
    if (!skip)
        d = warp_blas_dot(
            w, [&](int64_t i) { return vin(a, lo + i); }, [&](int64_t i) { return vin(b, lo + i); });
    if (threadIdx.x == 0) dot_combine(d, out, sqrt_out, ch, skip);
}

// Fixed-shape two-level tree (RSB_DOT_TREE): block b sums a fixed chunk in a
// fixed order; the finisher sums the partials in index order.  Deterministic
// for a given n, not the reference's association.
__global__ void k_dot_tree_partial(int64_t n, VecIn a, VecIn b, double *partials, Gate g,
                                   const int *need) {
    if (gated(g) || (need && !*(volatile const int *)need)) return;
    __shared__ double sh[kBlock];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * chunk;
    const int64_t hi = min(n, lo + chunk);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kBlock) acc = fma(vin(a, i), vin(b, i), acc);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kBlock / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

__global__ void k_dot_tree_final(int nparts, const double *partials, double *out, int sqrt_out,
                                 Gate g, const int *need) {
    if (gated(g) || (need && !*(volatile const int *)need)) return;
    if (threadIdx.x == 0) {
        double d = 0.0;
        for (int i = 0; i < nparts; ++i) d = d + partials[i];
        out[0] = sqrt_out ? sqrt(d) : d;
    }
}

// ---------------------------------------------------------------------------
// y = A x: numpy's np.add.at scatter (sc.py:218-220) accumulates row i's
// contributions in ascending column order starting from 0.0, one rounding
// for the product and one for the add -- i.e. a CSR row-sequential sum.
// ---------------------------------------------------------------------------
template <int EPI>
__global__ void __launch_bounds__(kBlock) k_spmv(Compressed A, VecIn x, double *y, VecIn e, Gate g, int hint) {
    if (gated(g)) return;
    const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (i >= A.nlines) return;
    const int lo = A.ptr[i], hi = A.ptr[i + 1];
    double acc = 0.0;
    if (hint) {
        // the matrix stream marked evict-first in L2 (a cache-policy hint; L1
        // unchanged), so it does not push the gathered vector out of L2
        unsigned long long pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int k = lo; k < hi; ++k) {
            int c;
            double v;
            asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(c) : "l"(A.idx + k), "l"(pol));
            asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(A.val + k), "l"(pol));
            acc = __dadd_rn(acc, __dmul_rn(v, vin(x, c)));
        }
    } else {
        for (int k = lo; k < hi; ++k) acc = __dadd_rn(acc, __dmul_rn(A.val[k], vin(x, A.idx[k])));
    }
    if (EPI == EPI_ADD) acc = __dadd_rn(vin(e, i), acc);
    if (EPI == EPI_SUB_FROM) acc = __dsub_rn(vin(e, i), acc);
    y[i] = acc;
}

// products val[k]*y[idx[k]], k = lo .. lo+n-1 (n < 2^31)
__device__ __forceinline__ double pw_prod(const double *val, const int32_t *idx, const VecIn &y, int64_t lo,
                                          int64_t n) {
    struct Term {
        const double *val;
        const int32_t *idx;
        const VecIn *y;
        __device__ double operator()(int64_t k) const { return __dmul_rn(val[k], vin(*y, idx[k])); }
    };
    const Term t{val + lo, idx + lo, &y};
    if (n <= 128) return pw_leaf(t, 0, n);
    return Pairwise<25, Term>::sum(t, 0, n);
}

// already formed products p[0 .. n-1] (shared memory; n <= kSpCap < 128 * 2^5)
__device__ __forceinline__ double pw_smem(const double *p, int n) {
    struct Term {
        const double *p;
        __device__ double operator()(int64_t k) const { return p[k]; }
    };
    const Term t{p};
    if (n <= 128) return pw_leaf(t, 0, n);
    return Pairwise<5, Term>::sum(t, 0, n);
}

// ---------------------------------------------------------------------------
// Tiled SpMV (default).  A block owns kBlock consecutive lines (rows of the
// CSR / columns of the CSC).  Phase 1 streams the tile's entries with
// coalesced loads -- consecutive threads take consecutive entries, four in
// flight per thread -- and forms every product val * x[idx] (the products
// are independent: only the summation order is fixed), into shared memory.
// Phase 2: thread t sums line t's products in the reference's order
// (sequential from 0.0 for A x; p0 + pairwise for A^T y).  A tile whose
// entries exceed the staging buffer (a long line: config 2's dense rows)
// runs the thread-per-line loop instead, with the same order.
// ---------------------------------------------------------------------------
constexpr int kSpCap = 3072;  // staged products per tile (24 KB): 12 per line

__device__ __forceinline__ void stage_products(const Compressed &A, const VecIn &x, int lo, int hi,
                                               double *prod) {
    // a tile holds at most kSpCap = 12 kBlock entries: two fully predicated
    // rounds of 6 per thread, each with all its index, value and gather loads
    // in flight together
    constexpr int kHalf = kSpCap / kBlock / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k0 = lo + threadIdx.x + h * kHalf * kBlock;
        if (k0 >= hi) break;
        int c[kHalf];
        double v[kHalf], xv[kHalf];
#pragma unroll
        for (int u = 0; u < kHalf; ++u) {
            const int k = k0 + u * kBlock;
            c[u] = k < hi ? __ldcs(A.idx + k) : -1;
            v[u] = k < hi ? __ldcs(A.val + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kHalf; ++u) xv[u] = c[u] >= 0 ? vin(x, c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kHalf; ++u)
            if (c[u] >= 0) prod[k0 + u * kBlock - lo] = __dmul_rn(v[u], xv[u]);
    }
}

template <int EPI>
__global__ void __launch_bounds__(kBlock) k_spmv_tile(Compressed A, VecIn x, double *y, VecIn e, Gate g) {
    if (gated(g)) return;
    __shared__ double prod[kSpCap];
    const int64_t l0 = blockIdx.x * (int64_t)kBlock;
    const int64_t i = l0 + threadIdx.x;
    const bool valid = i < A.nlines;
    const int64_t lend = min((int64_t)A.nlines, l0 + kBlock);
    const int lo = A.ptr[l0], hi = A.ptr[lend];
    double acc = 0.0;
    if (hi - lo <= kSpCap) {
        stage_products(A, x, lo, hi, prod);
        __syncthreads();
        if (!valid) return;
        const int s = A.ptr[i] - lo, t = A.ptr[i + 1] - lo;
        for (int k = s; k < t; ++k) acc = __dadd_rn(acc, prod[k]);
    } else {
        if (!valid) return;
        const int s = A.ptr[i], t = A.ptr[i + 1];
        for (int k = s; k < t; ++k) acc = __dadd_rn(acc, __dmul_rn(A.val[k], vin(x, A.idx[k])));
    }
    if (EPI == EPI_ADD) acc = __dadd_rn(vin(e, i), acc);
    if (EPI == EPI_SUB_FROM) acc = __dsub_rn(vin(e, i), acc);
    y[i] = acc;
}

template <int EPI, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) k_spmv_t_tile(Compressed At, VecIn y, double *z, VecIn e, Gate g) {
    if (gated(g)) return;
    __shared__ double prod[kSpCap];
    const int64_t l0 = blockIdx.x * (int64_t)kBlock;
    const int64_t j = l0 + threadIdx.x;
    const bool valid = j < At.nlines;
    const int64_t lend = min((int64_t)At.nlines, l0 + kBlock);
    const int lo = At.ptr[l0], hi = At.ptr[lend];
    double acc = 0.0;
    if (hi - lo <= kSpCap) {
        stage_products(At, y, lo, hi, prod);
        __syncthreads();
        if (!valid) return;
        const int s = At.ptr[j] - lo, t = At.ptr[j + 1] - lo;
        if (t > s) acc = __dadd_rn(prod[s], pw_smem(prod + s + 1, t - s - 1));
    } else {
        if (!valid) return;
        const int s = At.ptr[j], t = At.ptr[j + 1];
        if (t > s) acc = __dadd_rn(__dmul_rn(At.val[s], vin(y, At.idx[s])), pw_prod(At.val, At.idx, y, s + 1, t - s - 1));
    }
    if (EPI == EPI_ADD) acc = __dadd_rn(vin(e, j), acc);
    z[j] = acc;
}

// z = A^T y: np.add.reduceat over the column's products (sc.py:231-234)
// gives z_j = p0 + pairwise(p1 .. p_{k-1}); empty columns stay 0.0.
template <int EPI>
__global__ void __launch_bounds__(kBlock) k_spmv_t(Compressed At, VecIn y, double *z, VecIn e, Gate g) {
    if (gated(g)) return;
    const int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (j >= At.nlines) return;
    const int lo = At.ptr[j], hi = At.ptr[j + 1];
    double acc = 0.0;
    if (hi > lo) {
        double p0 = __dmul_rn(At.val[lo], vin(y, At.idx[lo]));
        acc = __dadd_rn(p0, pw_prod(At.val, At.idx, y, lo + 1, hi - lo - 1));
    }
    if (EPI == EPI_ADD) acc = __dadd_rn(vin(e, j), acc);
    z[j] = acc;
}

// ---------------------------------------------------------------------------
// Sync-free level-ordered triangular solve.
//
// One thread per unknown.  Tasks are sorted by dependency level and blocks
// take consecutive task ranges in the order they start (atomic ticket), so a
// task only ever waits on tasks of blocks that are already running or done.
// The output vector itself is the completion flag: it is pre-filled with a
// sentinel NaN and a task spins (L2-coherent relaxed loads) until each of
// its inputs is no longer the sentinel.  Sequential mode reproduces the
// reference's column-oriented axpy (sc.py:253-262, 271-278):
//   x_i = b_i; for each dependency j in stored order: if x_j != 0: x_i -= l_ij*x_j
// then x_i /= d_i when a diagonal is stored.  Dot mode reproduces
// x_j -= vals @ x[rows] (sc.py:291,296,311): an OpenBLAS ddot of the gathered
// values (FMA chain below 16 entries, SkylakeX blocking above).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double wait_ready(const double *p) {
    unsigned long long v;
    do {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    } while (v == kSentinel);
    return __longlong_as_double(v);
}

__device__ __forceinline__ void publish(double *p, double v) {
    unsigned long long b = __double_as_longlong(v);
    if (b == kSentinel) b = 0x7FF8000000000000ull;
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}

// blas-order dot of a task's gathered entries, one thread (len >= 16 path)
template <class Wait>
__device__ double task_blas_dot(const TriDev &T, int64_t base, int lane, int len, Wait wait) {
    auto ent = [&](int k) { return base + (int64_t)k * 32 + lane; };
    const int n1 = len & ~15, n32 = n1 & ~31;
    double dot = 0.0;
    if (n1) {
        double a5[32];
        for (int q = 0; q < 32; ++q) a5[q] = 0.0;
        int i = 0;
        for (; i < n32; i += 32)
            for (int q = 0; q < 32; ++q) a5[q] = fma(T.eval[ent(i + q)], wait(T.ecol[ent(i + q)]), a5[q]);
        double a[16];
        for (int gq = 0; gq < 4; ++gq)
            for (int k = 0; k < 4; ++k) a[4 * gq + k] = a5[8 * gq + k] + a5[8 * gq + k + 4];
        for (; i < n1; i += 16)
            for (int q = 0; q < 16; ++q) a[q] = fma(T.eval[ent(i + q)], wait(T.ecol[ent(i + q)]), a[q]);
        double t[4];
        for (int k = 0; k < 4; ++k) t[k] = ((a[k] + a[4 + k]) + a[8 + k]) + a[12 + k];
        dot = (t[0] + t[2]) + (t[1] + t[3]);
    }
    for (int k = n1; k < len; ++k) dot = fma(wait(T.ecol[ent(k)]), T.eval[ent(k)], dot);
    return dot;
}

// One task's loads that do not depend on other unknowns (its first kPre
// entries, the right-hand side, the diagonal), issued before any wait.
constexpr int kPre = 12;

struct Task {
    int t, row, lane, K, len;  // len: number of real entries (K is the slice's padded width)
    int64_t base;
    int cols[kPre];
    double vals[kPre];
    double acc;  // right-hand side
    double d;    // diagonal (divide) or 1
};

template <int MODE>
__device__ __forceinline__ void load_task(const TriDev &T, int t, const VecIn &a, const double *c, Task &k) {
    k.t = t;
    k.lane = t & 31;
    k.row = T.task_row[t];
    const int w = t >> 5;
    k.base = T.slice_off[w];
    k.K = (int)((T.slice_off[w + 1] - k.base) >> 5);
#pragma unroll
    for (int q = 0; q < kPre; ++q) {
        k.cols[q] = -1;
        k.vals[q] = 0.0;
        if (q < k.K) {
            k.cols[q] = T.ecol[k.base + (int64_t)q * 32 + k.lane];
            k.vals[q] = T.eval[k.base + (int64_t)q * 32 + k.lane];
        }
    }
    double acc = vin(a, k.row);
    if (c) acc = __dadd_rn(acc, c[k.row]);
    k.acc = acc;
    k.d = (MODE & 2) ? T.diag[t] : 1.0;
    int len = 0;
#pragma unroll
    for (int q = 0; q < kPre; ++q) len += k.cols[q] >= 0;
    if (len == kPre)
        while (len < k.K && T.ecol[k.base + (int64_t)len * 32 + k.lane] >= 0) ++len;
    k.len = len;
}

// true when every dependency of the task is finished (never blocks)
template <class Ready>
__device__ __forceinline__ bool task_ready(const TriDev &T, const Task &k, Ready ready) {
    bool ok = true;
#pragma unroll
    for (int q = 0; q < kPre; ++q)
        if (k.cols[q] >= 0) ok &= ready(k.cols[q]);
    if (ok && k.len > kPre)
        for (int q = kPre; q < k.len; ++q) {
            if (!ready(T.ecol[k.base + (int64_t)q * 32 + k.lane])) return false;
        }
    return ok;
}

// The task's value, all dependencies finished; read(j) returns x_j.
// Sequential mode (sc.py:253-262, 271-278): acc -= l_ij * x_j in stored order,
// skipping x_j == 0.  Dot mode (sc.py:291,296,311): acc -= OpenBLAS ddot of
// the gathered values.  Then acc /= d for a stored diagonal.
template <int MODE, class Read>
__device__ __forceinline__ double task_value(const TriDev &T, const Task &k, Read read) {
    double acc = k.acc;
    if (!(MODE & 1)) {
#pragma unroll
        for (int q = 0; q < kPre; ++q) {
            if (q < k.len) {
                const double xj = read(k.cols[q]);
                if (xj != 0.0) acc = __dsub_rn(acc, __dmul_rn(k.vals[q], xj));
            }
        }
        for (int q = kPre; q < k.len; ++q) {
            const int64_t e = k.base + (int64_t)q * 32 + k.lane;
            const double xj = read(T.ecol[e]);
            if (xj != 0.0) acc = __dsub_rn(acc, __dmul_rn(T.eval[e], xj));
        }
    } else if (k.len > 0) {
        double dot = 0.0;
        if (k.len <= kPre) {
#pragma unroll
            for (int q = 0; q < kPre; ++q)
                if (q < k.len) dot = fma(k.vals[q], read(k.cols[q]), dot);
        } else if (k.len < 16) {
            for (int q = 0; q < k.len; ++q) {
                const int64_t e = k.base + (int64_t)q * 32 + k.lane;
                dot = fma(T.eval[e], read(T.ecol[e]), dot);
            }
        } else {
            dot = task_blas_dot(T, k.base, k.lane, k.len, read);
        }
        acc = __dsub_rn(acc, dot);
    }
    if (MODE & 2) acc = __ddiv_rn(acc, k.d);
    return acc;
}

__device__ __forceinline__ double ld_relaxed(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double(v);
}

// Grid-wide variant (wide DAGs): completion = the output entry is no longer
// the sentinel, observed through L2 with relaxed gpu-scope loads.  Blocks take
// consecutive task ranges in the order they start (atomic ticket), so a task
// only waits on blocks already resident or done.  Warp-synchronous polling:
// lanes never spin divergently; every round each pending lane checks all its
// dependencies, the ready ones compute and publish, and the warp reconverges.
// tasks longer than kPre (rare): out of line, keeps the fast path's registers low
template <int MODE>
__device__ __noinline__ double long_task_value(const TriDev &T, const Task &k, const double *x) {
    return task_value<MODE>(T, k, [&](int j) { return ld_relaxed(x + j); });
}

template <int MODE>
__global__ void __launch_bounds__(kTriBlock) k_trsv(TriDev T, VecIn a, const double *c, double *x,
                                                    Gate g) {
    if (gated(g)) return;
    __shared__ int s_blk;
    if (threadIdx.x == 0) s_blk = (int)atomicAdd(T.ticket, 1ull);
    __syncthreads();
    const int t = s_blk * kTriBlock + threadIdx.x;
    bool pending = t < T.n;
    Task k;
    if (pending) load_task<MODE>(T, t, a, c, k);
    auto ready = [&](int j) { return __double_as_longlong(ld_relaxed(x + j)) != (long long)kSentinel; };
    while (__any_sync(0xffffffffu, pending)) {
        if (pending) {
            if (k.len <= kPre) {
                // one L2 round trip per poll: the polled values are the operands
                double xv[kPre];
                bool ok = true;
#pragma unroll
                for (int q = 0; q < kPre; ++q) {
                    xv[q] = 0.0;
                    if (q < k.len) {
                        xv[q] = ld_relaxed(x + k.cols[q]);
                        ok &= __double_as_longlong(xv[q]) != (long long)kSentinel;
                    }
                }
                if (ok) {
                    double acc = k.acc;
                    if (!(MODE & 1)) {
#pragma unroll
                        for (int q = 0; q < kPre; ++q)
                            if (q < k.len && xv[q] != 0.0) acc = __dsub_rn(acc, __dmul_rn(k.vals[q], xv[q]));
                    } else if (k.len > 0) {
                        double dot = 0.0;
#pragma unroll
                        for (int q = 0; q < kPre; ++q)
                            if (q < k.len) dot = fma(k.vals[q], xv[q], dot);
                        acc = __dsub_rn(acc, dot);
                    }
                    if (MODE & 2) acc = __ddiv_rn(acc, k.d);
                    publish(x + k.row, acc);
                    pending = false;
                }
            } else if (task_ready(T, k, ready)) {
                publish(x + k.row, long_task_value<MODE>(T, k, x));
                pending = false;
            }
        }
        __syncwarp();
    }
}

// Level-synchronous grid solve (wide DAGs with few levels): one launch per
// level, one thread per task; every dependency was published by an earlier
// launch, so operands are plain loads and nothing polls.
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_trsv_level(TriDev T, VecIn a, const double *c, double *x, int lo, int hi,
                                                       Gate g) {
    if (gated(g)) return;
    for (int t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += gridDim.x * blockDim.x) {
        Task k;
        load_task<MODE>(T, t, a, c, k);
        x[k.row] = task_value<MODE>(T, k, [&](int j) { return x[j]; });
    }
}

__device__ __forceinline__ double canonical(double v) {
    return __double_as_longlong(v) == (long long)kSentinel ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

// ---- shared-memory staging primitives (sm_90+: mbarrier + 1-D TMA bulk copy)

// Exact-order dot for long contiguous vectors: the same single-warp OpenBLAS
// association as k_dot_exact, with both operands streamed through shared
// memory by TMA bulk copies (kDotStages-deep mbarrier pipeline) so the FMA
// chain waits on shared-memory, not global-memory, latency.
__global__ void __launch_bounds__(32) k_dot_exact_staged(int64_t n_all, const double *a_all, const double *b_all,
                                                         double *out, int sqrt_out, Gate g, const int *need,
                                                         DotChunks ch, int norm_stages) {
    if (need && !*(volatile const int *)need) return;
    if (__shfl_sync(0xffffffffu, gated(g) ? 1 : 0, 0)) {  // still count this chunk (dot_combine)
        if (threadIdx.x == 0) dot_combine(0.0, out, sqrt_out, ch, true);
        return;
    }
    extern __shared__ __align__(16) double dbuf[];
    constexpr int kBuf = kDotChunk + 2;  // one stage of one operand: a chunk shifted by <= 1 element
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(dbuf + kDotStages * 2 * kBuf);
    const int lane = threadIdx.x;
    // this block's chunk [lo, lo + n) of the operands (the whole vector when T = 1)
    int64_t lo = 0, n = n_all;
    if (ch.T > 1) dot_chunk(n_all, ch.T, blockIdx.x, lo, n);
    const double *a = a_all + lo, *b = b_all + lo;
    // bulk copies need 16-byte aligned sources and sizes: copy from the even
    // element below each stage's start (shift = lo & 1 elements into the
    // buffer) to the even element above its end, except past the end of the
    // vectors, where the last odd element is loaded by lane 0 instead
    const int shift = (int)(lo & 1);
    // a norm (a.a): one operand stream -- a chunk is bounded by its SM's
    // ingest rate (~16 B/cycle against the 64 the chain could use), so half
    // the bytes is close to half the time; same products, same order
    // and its buffers hold twice the stages
    const bool same = a_all == b_all && norm_stages > 0;
    const int nst = same ? norm_stages : kDotStages;
    const size_t sbuf = same ? kBuf : 2 * kBuf;  // doubles per stage
    const int64_t n32 = (n & ~(int64_t)15) & ~(int64_t)31;
    const int64_t nch = (n32 + kDotChunk - 1) / kDotChunk;
    if (lane == 0) {
        for (int st = 0; st < nst; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto span = [&](int64_t c, int64_t &c0, int64_t &c1, bool &patch) {
        const int64_t e0 = lo + c * kDotChunk, e1 = lo + min((int64_t)kDotChunk * (c + 1), n32);
        c0 = e0 & ~(int64_t)1;
        c1 = (e1 + 1) & ~(int64_t)1;
        patch = c1 > n_all;
        if (patch) c1 -= 2;
    };
    auto issue = [&](int64_t c) {
        const int st = (int)(c % nst);
        int64_t c0, c1;
        bool patch;
        span(c, c0, c1, patch);
        const unsigned bytes = (unsigned)((c1 - c0) * 8);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[st], same ? bytes : 2 * bytes);
        if (bytes) {
            bulk_g2s(dbuf + (size_t)st * sbuf, a_all + c0, bytes, &bar[st]);
            if (!same) bulk_g2s(dbuf + (size_t)st * sbuf + kBuf, b_all + c0, bytes, &bar[st]);
        }
    };
    if (lane == 0)
        for (int64_t c = 0; c < min((int64_t)nst, nch); ++c) issue(c);
    double acc = 0.0;
    for (int64_t c = 0; c < nch; ++c) {
        const int st = (int)(c % nst);
        mbar_wait_spin(&bar[st], (unsigned)((c / nst) & 1));
        double *buf_a = dbuf + (size_t)st * sbuf, *buf_b = same ? buf_a : buf_a + kBuf;
        {
            int64_t c0, c1;
            bool patch;
            span(c, c0, c1, patch);
            if (patch && lane == 0) {  // the vectors' last element (odd index) was not copied
                buf_a[c1 - c0] = a_all[c1];
                buf_b[c1 - c0] = b_all[c1];
            }
            __syncwarp();
        }
        const double *sa = buf_a + shift + lane, *sb = buf_b + shift + lane;
        const int steps = (int)min((int64_t)kDotChunk, n32 - c * kDotChunk) / 32;
        // the lane's FMA chain, 8 cycles a step: operands of the next 8 steps
        // are loaded while the current 8 issue, so the chain never waits on
        // shared-memory latency
        constexpr int G = 8;
        const int full_groups = steps / G;
        // two register sets, ping-pong: the loads of group g + 1 / g + 2 are in
        // flight while group g / g + 1 issues (pointer bumps only -- an index
        // select in the address made ptxas park a whole group's loads right in
        // front of their first use)
        double a0[G], b0[G], a1[G], b1[G];
        const double *pa = sa, *pb = sb;
        auto ld = [&](double(&ra)[G], double(&rb)[G], const double *qa, const double *qb) {
#pragma unroll
            for (int j = 0; j < G; ++j) {
                ra[j] = qa[32 * j];
                rb[j] = qb[32 * j];
            }
        };
        auto mac = [&](const double(&ra)[G], const double(&rb)[G]) {
#pragma unroll
            for (int j = 0; j < G; ++j) acc = fma(ra[j], rb[j], acc);
        };
        int gI = 0;
        if (full_groups > 0) ld(a0, b0, pa, pb);
        for (; gI + 3 <= full_groups; gI += 2) {
            ld(a1, b1, pa + 32 * G, pb + 32 * G);
            mac(a0, b0);
            ld(a0, b0, pa + 64 * G, pb + 64 * G);
            mac(a1, b1);
            pa += 64 * G;
            pb += 64 * G;
        }
        if (gI + 2 == full_groups) {
            ld(a1, b1, pa + 32 * G, pb + 32 * G);
            mac(a0, b0);
            mac(a1, b1);
        } else if (gI + 1 == full_groups) {
            mac(a0, b0);
        }
        for (int k = full_groups * G; k < steps; ++k) acc = fma(sa[32 * k], sb[32 * k], acc);
        __syncwarp();
        if (lane == 0 && c + nst < nch) issue(c + nst);
    }
    const double d = warp_blas_finish(acc, n, [&](int64_t i) { return a[i]; }, [&](int64_t i) { return b[i]; });
    if (lane == 0) dot_combine(d, out, sqrt_out, ch, false);
}

// (A variant with the operands brought into shared memory by all threads of
// a 256-thread block -- 16-byte cp.async, three stages of 4096 elements, two
// in flight -- and the chain on warp 0 measured slower: 0.084 vs 0.066 ms for
// the n = 8e6 dot, 0.144 vs 0.094 for m = 1.6e7; a chunk's 32 chains cannot be
// split, so one SM's ingest rate bounds a chunk either way.)

// right-hand side in task-position order: bpos[t] = a(row_t) [+ c[row_t]]
__global__ void k_gather_pos(int32_t n, int64_t padded, const int32_t *task_row, VecIn a, const double *c,
                             double *bpos, Gate g) {
    // let the solve that consumes bpos start its prologue (it waits for this
    // grid's completion before reading anything written here)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (gated(g)) return;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < padded; t += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        const int row = task_row[t];  // -1: padding task of the staged layout
        if (row >= 0) {
            v = vin(a, row);
            if (c) v = __dadd_rn(v, c[row]);
        }
        bpos[t] = v;
    }
}

// Single-CTA level-synchronous solve with shared-memory staging (narrow DAGs,
// e.g. config 1 at mu = 1: 1,290 / 2,806 levels of <= 66 unknowns).
//
// The dependency chain crosses one barrier per level and touches only
// shared memory:
//   - task data of positions [c*CH, (c+1)*CH) -- gathered right-hand sides,
//     diagonals, 16-byte entry records {value, source}, rows, lengths -- is
//     streamed into one of kStageBufs shared-memory buffers by 1-D TMA bulk
//     copies completing on an mbarrier, issued kStageBufs-1 chunks ahead;
//   - solved values go to a shared-memory ring indexed by task position; an
//     entry's source is the byte offset of its ring slot when the slot is
//     still live (distance + widest level < kRing), else -(row + 2) and the
//     value is read from the global output (FAR specialisation only);
//   - a task issues all its entry and ring loads before the ordered FP chain.
// Earlier designs measured 0.9-3 us per level (grid-wide sync-free, CTA
// spin-polling: spinning warps starved the critical warp of issue slots;
// per-thread prefetch: dependent global loads in front of every barrier);
// see profiles/.
// x[rows] @ vals in OpenBLAS association for a staged task with >= 16 entries
// (rare: L^T columns hold at most p entries); out of line to keep the fast
// path's registers free.
__device__ __noinline__ double rec_blas_dot(const StageRec *rec, int len, const unsigned char *ring,
                                            const double *x, bool far) {
    auto la = [&](int q) { return rec[q * 32].v; };
    auto lb = [&](int q) {
        const int s = rec[q * 32].src;
        return (!far || s >= 0) ? *reinterpret_cast<const double *>(ring + s) : x[-s - 2];
    };
    const int n1 = len & ~15, n32 = n1 & ~31;
    double dot = 0.0;
    if (n1) {
        double a5[32];
        for (int q = 0; q < 32; ++q) a5[q] = 0.0;
        int i = 0;
        for (; i < n32; i += 32)
            for (int q = 0; q < 32; ++q) a5[q] = fma(la(i + q), lb(i + q), a5[q]);
        double a4[16];
        for (int gq = 0; gq < 4; ++gq)
            for (int kk = 0; kk < 4; ++kk) a4[4 * gq + kk] = a5[8 * gq + kk] + a5[8 * gq + kk + 4];
        for (; i < n1; i += 16)
            for (int q = 0; q < 16; ++q) a4[q] = fma(la(i + q), lb(i + q), a4[q]);
        double tt[4];
        for (int kk = 0; kk < 4; ++kk) tt[kk] = ((a4[kk] + a4[4 + kk]) + a4[8 + kk]) + a4[12 + kk];
        dot = (tt[0] + tt[2]) + (tt[1] + tt[3]);
    }
    for (int q = n1; q < len; ++q) dot = fma(lb(q), la(q), dot);
    return dot;
}


// One staged task with at most N entries (N = the warp's longest task, so
// the loop is unrolled for exactly that many): all record and ring loads are
// issued first, products are formed off the chain, and the chain itself is
// one DSUB (sequential axpy order, sc.py:261-262) or one DFMA (OpenBLAS ddot
// order for < 16 entries, sc.py:291) per entry.  Entries past the lane's own
// length, and skipped ones (x_j == 0), contribute nothing: the DSUB chain
// subtracts +0.0 (identity for every acc, also -0.0), and fma(0, 0, dot) =
// dot because the FMA chain from +0.0 can never produce -0.0.
template <int N, int MODE, bool FAR>
__device__ __forceinline__ double stage_task(const StageRec *rec, int len, double acc, const unsigned char *ring,
                                             const double *x) {
    double v[N], xv[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
        v[q] = 0.0;
        xv[q] = 0.0;
        if (q < len) {
            const StageRec r = rec[q * 32];
            v[q] = r.v;
            xv[q] = (!FAR || r.src >= 0) ? *reinterpret_cast<const double *>(ring + r.src) : x[-r.src - 2];
        }
    }
    if (!(MODE & 1)) {
        double pr[N];
#pragma unroll
        for (int q = 0; q < N; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(v[q], xv[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) acc = __dsub_rn(acc, pr[q]);
    } else if (len > 0) {
        double dot = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) dot = fma(v[q], xv[q], dot);
        acc = __dsub_rn(acc, dot);
    }
    return acc;
}

// tasks with >= 16 entries (rare): streaming loop, BLAS-blocked dot order
template <int MODE, bool FAR>
__device__ __noinline__ double stage_task_long(const StageRec *rec, int len, double acc, const unsigned char *ring,
                                               const double *x) {
    auto src = [&](int s) -> double {
        return (!FAR || s >= 0) ? *reinterpret_cast<const double *>(ring + s) : x[-s - 2];
    };
    if (!(MODE & 1)) {
        for (int q = 0; q < len; ++q) {
            const StageRec r = rec[q * 32];
            const double xj = src(r.src);
            if (xj != 0.0) acc = __dsub_rn(acc, __dmul_rn(r.v, xj));
        }
    } else if (len > 0) {
        double dot = 0.0;
        if (len < 16) {
            for (int q = 0; q < len; ++q) {
                const StageRec r = rec[q * 32];
                dot = fma(r.v, src(r.src), dot);
            }
        } else {
            dot = rec_blas_dot(rec, len, ring, x, FAR);
        }
        acc = __dsub_rn(acc, dot);
    }
    return acc;
}

template <int MODE, bool FAR>
__global__ void __launch_bounds__(kCtaTri + 32) k_trsv_stage(TriDev T, double *x, Gate g) {
    if (gated(g)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool kDiag = (MODE & 2) != 0;
    constexpr int kConsumerWarps = kCtaTri / 32;
    const int CH = T.stage_ch, EM = T.stage_emax;
    unsigned char *ring = smem;
    unsigned char *bufs = smem + (size_t)kRing * 8;
    const size_t o_meta = (size_t)CH * 8, o_dd = o_meta + (size_t)CH * 16,
                 o_rec = o_dd + (kDiag ? (size_t)CH * 16 : 0), bb = o_rec + (size_t)EM * 16;
    unsigned long long *full = reinterpret_cast<unsigned long long *>(bufs + kStageBufs * bb);
    unsigned long long *empty = full + kStageBufs;
    int *lvl = reinterpret_cast<int *>(full + 2 * kStageBufs);
    const int nlev = T.nlevels, nch = T.nchunks, lgch = __ffs(CH) - 1;
    for (int i = threadIdx.x; i <= nlev; i += blockDim.x) lvl[i] = T.level_ptr[i];
    if (threadIdx.x == 0) {
        for (int b = 0; b < kStageBufs; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // the producer is warp 3 (SMSP 3); the consumer slice it displaces, the
    // rarely used 4th one, runs on warp 4 and shares SMSP 0 with the busiest
    const int warp = threadIdx.x >> 5;
    if (warp == 3) {
        // producer warp: chunk c goes to buffer c % kStageBufs once the
        // consumers released the chunk that held it; the consumers never issue
        if (threadIdx.x == 96) {
            for (int c = 0; c < nch; ++c) {
                const int b = c & (kStageBufs - 1);
                if (c >= kStageBufs) mbar_wait(&empty[b], (unsigned)(((c / kStageBufs) - 1) & 1));
                unsigned char *B = bufs + (size_t)b * bb;
                const int64_t r0 = T.chunk_roff[c];
                const int ne = (int)(T.chunk_roff[c + 1] - r0);
                const unsigned bytes = (unsigned)(CH * 8 + CH * 16 + (kDiag ? CH * 16 : 0) + ne * 16);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&full[b], bytes);
                bulk_g2s(B, T.bpos + (int64_t)c * CH, CH * 8, &full[b]);
                bulk_g2s(B + o_meta, T.meta + (int64_t)c * CH, CH * 16, &full[b]);
                if (kDiag) bulk_g2s(B + o_dd, T.ddiag + 2 * (int64_t)c * CH, CH * 16, &full[b]);
                if (ne) bulk_g2s(B + o_rec, T.recs + r0, (unsigned)ne * 16, &full[b]);
            }
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    const int slot = warp < 3 ? (int)threadIdx.x : (int)threadIdx.x - 32;
    int released = 0, ready = -1;
    long long pc[7] = {0, 0, 0, 0, 0, 0, 0}, tq = 0, tp = 0;
    const bool prof = T.prof && threadIdx.x == 0;
#define RSB_PROF(i)                 \
    if (prof) {                     \
        tq = clock64();             \
        pc[i] += tq - tp;           \
        tp = tq;                    \
    }
    if (prof) tp = clock64();
    for (int l = 0; l < nlev; ++l) {
        const int lo = lvl[l], hi = lvl[l + 1];
        const int first = lo >> lgch;       // refill buffers whose chunk lies wholly before this level
        const int last = (hi - 1) >> lgch;  // chunks this level reads must have landed
        for (; released < first; ++released)  // chunks wholly before this level are done
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                 smem_u32(&empty[released & (kStageBufs - 1)]))
                             : "memory");
        RSB_PROF(0)
        while (ready < last) {
            ++ready;
            mbar_wait(&full[ready & (kStageBufs - 1)], (unsigned)((ready / kStageBufs) & 1));
        }
        RSB_PROF(5)
        for (int t = lo + slot; t < hi; t += kCtaTri) {
            const int loc = t & (CH - 1);
            const unsigned char *B = bufs + (size_t)((t >> lgch) & (kStageBufs - 1)) * bb;
            const StageMeta m = reinterpret_cast<const StageMeta *>(B + o_meta)[loc];
            double acc = reinterpret_cast<const double *>(B)[loc];
            double2 dr = make_double2(1.0, 1.0);
            if (kDiag) dr = reinterpret_cast<const double2 *>(B + o_dd)[loc];
            const StageRec *rec = reinterpret_cast<const StageRec *>(B + o_rec) + m.roff;
            RSB_PROF(1)
            // code path unrolled for exactly the slice's longest task (uniform per warp)
            const int wlen = m.pad;
            switch (wlen) {
                case 0: break;
                case 1: acc = stage_task<1, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 2: acc = stage_task<2, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 3: acc = stage_task<3, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 4: acc = stage_task<4, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 5: acc = stage_task<5, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 6: acc = stage_task<6, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 7: acc = stage_task<7, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 8: acc = stage_task<8, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 9: acc = stage_task<9, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 10: acc = stage_task<10, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 11: acc = stage_task<11, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 12: acc = stage_task<12, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 13: acc = stage_task<13, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 14: acc = stage_task<14, MODE, FAR>(rec, m.len, acc, ring, x); break;
                case 15: acc = stage_task<15, MODE, FAR>(rec, m.len, acc, ring, x); break;
                default: acc = stage_task_long<MODE, FAR>(rec, m.len, acc, ring, x); break;
            }
            RSB_PROF(2)
            if (kDiag && m.row >= 0) acc = exact_div(acc, dr.x, dr.y);
            *reinterpret_cast<double *>(ring + (size_t)(t & (kRing - 1)) * 8) = acc;
            if (m.row >= 0) x[m.row] = acc;
            RSB_PROF(3)
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kCtaTri) : "memory");  // consumers only
        RSB_PROF(4)
    }
#undef RSB_PROF
    if (prof) {
        for (int i = 0; i < 5; ++i) T.prof[i] = pc[i];
        T.prof[6] = pc[5];
        T.prof[5] = nlev;
    }
}

// ---------------------------------------------------------------------------
// small vector kernels
// ---------------------------------------------------------------------------
__global__ void k_fill(double *x, int64_t n, unsigned long long bits, Gate g) {
    if (gated(g)) return;
    const double v = __longlong_as_double(bits);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void k_copy(double *dst, VecIn src, int64_t n, Gate g) {
    if (gated(g)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = vin(src, i);
}

// y += s*x  /  y -= s*x   (x += alpha*p, r -= alpha*q: sv.py:215-216, pc.py:303-304)
template <int SIGN>
__global__ void k_axpy(double *y, const double *x, const double *scal, int64_t n, Gate g) {
    if (gated(g)) return;
    const double s = *scal;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double t = __dmul_rn(s, x[i]);
        y[i] = SIGN > 0 ? __dadd_rn(y[i], t) : __dsub_rn(y[i], t);
    }
}

// p = h + beta*p (sv.py:240, pc.py:308) or p = h.copy() when copy_flag set
__global__ void k_xpby(double *p, const double *h, const double *beta, const int *copy_flag,
                       int64_t n, Gate g) {
    if (gated(g)) return;
    const bool cp = copy_flag && *copy_flag;
    const double b = cp ? 0.0 : *beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = cp ? h[i] : __dadd_rn(h[i], __dmul_rn(b, p[i]));
}

// ---------------------------------------------------------------------------
// Dense Cholesky solve S w = u with the lower column-major factor G
// (sc.py:607-622), one CTA.  Forward: column axpy x[j+1:] -= g[j+1:,j]*x[j]
// (parallel over rows, sequential over j -- the reference's order for every
// element).  Backward: x[j] -= g[j+1:,j] @ x[j+1:] as a warp-level OpenBLAS
// ddot (same association as the host), then x[j] /= g[j,j].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_chol_solve(const double *G, int64_t s, const double *u,
                                                      double *w, int use_smem, Gate g) {
    if (gated(g)) return;
    extern __shared__ double sx[];
    double *x = use_smem ? sx : w;
    for (int64_t i = threadIdx.x; i < s; i += kBlock) x[i] = u[i];
    __syncthreads();
    for (int64_t j = 0; j < s; ++j) {
        const double xj = __ddiv_rn(x[j], G[j + j * s]);
        __syncthreads();
        if (threadIdx.x == 0) x[j] = xj;
        for (int64_t i = j + 1 + threadIdx.x; i < s; i += kBlock)
            x[i] = __dsub_rn(x[i], __dmul_rn(G[i + j * s], xj));
        __syncthreads();
    }
    if (threadIdx.x < 32) {
        for (int64_t j = s - 1; j >= 0; --j) {
            double xj = x[j];
            if (j + 1 < s) {
                const double *gc = G + (j + 1) + j * s;
                const double *xc = x + j + 1;
                const double d = warp_blas_dot(
                    s - j - 1, [&](int64_t i) { return gc[i]; }, [&](int64_t i) { return xc[i]; });
                xj = __dsub_rn(xj, d);
            }
            xj = __ddiv_rn(xj, G[j + j * s]);
            __syncwarp();
            if (threadIdx.x == 0) x[j] = xj;
            __syncwarp();
        }
    }
    __syncthreads();
    if (use_smem)
        for (int64_t i = threadIdx.x; i < s; i += kBlock) w[i] = x[i];
}

inline int grid_for(int64_t n, int block) {
    int64_t b = (n + block - 1) / block;
    return (int)(b < 1 ? 1 : (b > (1 << 30) ? (1 << 30) : b));
}

inline int grid_stride(int64_t n) {
    // elementwise kernels: up to 8 waves of 148 SMs x 8 resident blocks
    int64_t b = (n + kBlock - 1) / kBlock;
    int64_t cap = 148 * 8 * 8;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

inline int post_launch(rsb_ctx *ctx, int kernels = 1) {
    ctx->launches += kernels;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("kernel launch failed: %s", cudaGetErrorString(e));
        return RSB_ECUDA;
    }
    return RSB_OK;
}

}  // namespace

// RSB_SPMV=thread / tile forces the thread-per-line / tiled kernels (experiments)
static int spmv_force() {
    static const int force = [] {
        const char *v = getenv("RSB_SPMV");
        return v ? (strcmp(v, "thread") == 0 ? 1 : (strcmp(v, "tile") == 0 ? 2 : 0)) : 0;
    }();
    return force;
}
static bool spmv_tiled() { return spmv_force() != 1; }

static int spmv_impl(rsb_ctx *ctx, const Compressed &A, VecIn x, double *y, int epi, VecIn e, Gate g) {
    if (A.nlines == 0) return RSB_OK;
    const int grid = grid_for(A.nlines, kBlock);
    // rows of at most 8 entries (A of configs 0 / 4: 6 per row): one thread per
    // row keeps the loads of a warp's rows in the same few lines and measured
    // faster (config 4 at n = 8e6: 0.55 vs 0.66 ms); longer or uneven rows
    // take the tiled kernel
    const bool tiled = spmv_force() == 2 || (spmv_tiled() && A.max_len > 8);
    if (tiled) {
        switch (epi) {
            case EPI_STORE: k_spmv_tile<EPI_STORE><<<grid, kBlock, 0, ctx->stream>>>(A, x, y, e, g); break;
            case EPI_ADD: k_spmv_tile<EPI_ADD><<<grid, kBlock, 0, ctx->stream>>>(A, x, y, e, g); break;
            default: k_spmv_tile<EPI_SUB_FROM><<<grid, kBlock, 0, ctx->stream>>>(A, x, y, e, g); break;
        }
        return post_launch(ctx);
    }
    static const int hint = getenv("RSB_SPMV_HINT") ? atoi(getenv("RSB_SPMV_HINT")) : kSpmvHintDefault;
    switch (epi) {
        case EPI_STORE: k_spmv<EPI_STORE><<<grid, kBlock, 0, ctx->stream>>>(A, x, y, e, g, hint); break;
        case EPI_ADD: k_spmv<EPI_ADD><<<grid, kBlock, 0, ctx->stream>>>(A, x, y, e, g, hint); break;
        default: k_spmv<EPI_SUB_FROM><<<grid, kBlock, 0, ctx->stream>>>(A, x, y, e, g, hint); break;
    }
    return post_launch(ctx);
}

// ---- row-banded transposed product (Banded, devsetup.cu mat_build_bands).
// Phase 1: every product val * y[row], one thread per entry over the
// band-major arrays, so the blocks run band by band and each band's slice of
// y stays in L2 (the plain kernel's gathers of a 128 MB y miss L2: 7.3 GB of
// DRAM reads for 1.4 GB of algorithmic bytes at config 4).  Phase 2: column
// j's products are its band segments in band order -- its original entry
// order -- summed p0 + pairwise(p1..) exactly as k_spmv_t_tile does.
__global__ void __launch_bounds__(kBlock) k_band_prod(Banded B, int64_t nnz, VecIn y, Gate g) {
    if (gated(g)) return;
    const int64_t e = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    // the products stream out (768 MB at config 4, read back once by the sum
    // pass): evict-first, so that the band of y stays in L2
    if (e < nnz) __stcs(B.prod + e, __dmul_rn(__ldcs(B.val + e), vin(y, __ldcs(B.idx + e))));
}

struct BandTerm {
    const double *prod;
    int nb;
    int lo[kMaxBands], cnt[kMaxBands];
    __device__ double operator()(int64_t k) const {
        for (int b = 0; b < nb; ++b) {
            if (k < cnt[b]) return prod[lo[b] + k];
            k -= cnt[b];
        }
        return 0.0;
    }
};

template <int EPI>
__global__ void __launch_bounds__(kBlock) k_band_sum(Banded B, int32_t ncols, double *z, VecIn e, Gate g) {
    if (gated(g)) return;
    const int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (j >= ncols) return;
    BandTerm t;
    t.prod = B.prod;
    t.nb = B.nbands;
    int n = 0;
    for (int b = 0; b < B.nbands; ++b) {
        t.lo[b] = B.bptr[b][j];
        t.cnt[b] = B.bptr[b][j + 1] - t.lo[b];
        n += t.cnt[b];
    }
    double acc = 0.0;
    if (n > 0) acc = __dadd_rn(t(0), n - 1 <= 128 ? pw_leaf(t, 1, n - 1) : Pairwise<25, BandTerm>::sum(t, 1, n - 1));
    if (EPI == EPI_ADD) acc = __dadd_rn(vin(e, j), acc);
    z[j] = acc;
}

// Tiled sum pass: a block owns kBlock consecutive columns; their products of
// band b are one contiguous run of the band-major array, staged into shared
// memory with coalesced loads (the per-column segments read straight from
// HBM are ~24-byte pieces: k_band_sum measured 2.17 ms for A^T y at config 4).
constexpr int kBandCap = 4608;  // staged products per tile (2 x 36 KB): 18 per column
template <int EPI>
__global__ void __launch_bounds__(kBlock) k_band_sum_tile(Banded B, int32_t ncols, double *z, VecIn e, Gate g) {
    if (gated(g)) return;
    extern __shared__ double band_smem[];
    double *sp = band_smem;            // band-major, as loaded
    double *sq = band_smem + kBandCap; // column-major: each column's products in entry order
    const int64_t l0 = blockIdx.x * (int64_t)kBlock;
    const int64_t lend = min((int64_t)ncols, l0 + kBlock);
    const int64_t j = l0 + threadIdx.x;
    const bool valid = j < ncols;
    // band b of the tile: global run [g0[b], g0[b] + cnt), staged at sp + off[b]
    int off = 0, start = 0, n = 0;
    int my_lo[kMaxBands], my_cnt[kMaxBands], my_off[kMaxBands];
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b) {
        my_lo[b] = my_cnt[b] = my_off[b] = 0;
        if (b < B.nbands) {
            const int32_t *bp = B.bptr[b];
            const int g0 = bp[l0], g1 = bp[lend];
            if (valid) {
                my_lo[b] = bp[j];
                my_cnt[b] = bp[j + 1] - my_lo[b];
            }
            my_off[b] = off + (my_lo[b] - g0);
            start += valid ? my_lo[b] - g0 : 0;
            n += my_cnt[b];
            if (off + (g1 - g0) <= kBandCap)
                for (int i = threadIdx.x; i < g1 - g0; i += kBlock) sp[off + i] = __ldcs(B.prod + g0 + i);
            off += g1 - g0;
        }
    }
    const bool staged = off <= kBandCap;  // uniform over the block
    double acc = 0.0;
    if (staged) {
        __syncthreads();
        int pos = start;
#pragma unroll
        for (int b = 0; b < kMaxBands; ++b)
            if (b < B.nbands)
                for (int k = 0; k < my_cnt[b]; ++k) sq[pos++] = sp[my_off[b] + k];
        if (n > 0) acc = __dadd_rn(sq[start], pw_smem(sq + start + 1, n - 1));
    } else if (valid) {  // a tile past the staging buffer: straight from the band-major array
        BandTerm t;
        t.prod = B.prod;
        t.nb = B.nbands;
#pragma unroll
        for (int b = 0; b < kMaxBands; ++b) {
            t.lo[b] = my_lo[b];
            t.cnt[b] = my_cnt[b];
        }
        if (n > 0) acc = __dadd_rn(t(0), n - 1 <= 128 ? pw_leaf(t, 1, n - 1) : Pairwise<25, BandTerm>::sum(t, 1, n - 1));
    }
    if (!valid) return;
    if (EPI == EPI_ADD) acc = __dadd_rn(vin(e, j), acc);
    z[j] = acc;
}

static int spmv_t_impl(rsb_ctx *ctx, const Compressed &At, VecIn y, double *z, int epi, VecIn e, Gate g) {
    if (At.nlines == 0) return RSB_OK;
    const int grid = grid_for(At.nlines, kBlock);
    // the banded path uses the matrix's product scratch: only on the stream of
    // the context that owns it (concurrent solvers on other streams take the
    // plain kernel)
    if (At.bands && At.bands->owner == (const void *)ctx) {
        const Banded B = *At.bands;
        k_band_prod<<<(unsigned)((At.nnz + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(B, At.nnz, y, g);
        RSB_TRY(post_launch(ctx));
        static const bool flat = getenv("RSB_BANDS_FLAT") && atoi(getenv("RSB_BANDS_FLAT")) != 0;  // experiments
        if (flat) {
            if (epi == EPI_ADD)
                k_band_sum<EPI_ADD><<<grid, kBlock, 0, ctx->stream>>>(B, At.nlines, z, e, g);
            else
                k_band_sum<EPI_STORE><<<grid, kBlock, 0, ctx->stream>>>(B, At.nlines, z, e, g);
        } else {
            constexpr size_t smem = 2 * kBandCap * sizeof(double);
            static bool attr = false;
            if (!attr) {
                RSB_TRY_CUDA(cudaFuncSetAttribute(k_band_sum_tile<EPI_ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                RSB_TRY_CUDA(cudaFuncSetAttribute(k_band_sum_tile<EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                attr = true;
            }
            if (epi == EPI_ADD)
                k_band_sum_tile<EPI_ADD><<<grid, kBlock, smem, ctx->stream>>>(B, At.nlines, z, e, g);
            else
                k_band_sum_tile<EPI_STORE><<<grid, kBlock, smem, ctx->stream>>>(B, At.nlines, z, e, g);
        }
        return post_launch(ctx);
    }
    // (An L2 persisting window over 32 / 64 / 79 MB of the gathered vector did not
    // help A^T y at n = 8e6 -- 1.51 / 1.38 / 1.45 vs 1.39 ms -- and the set-aside
    // slowed every other kernel: profiles/r02b/kernel_table_spmv_t_persist64.json.)
    if (spmv_tiled()) {
        static const bool occ6 = getenv("RSB_SPMV_T_OCC") && atoi(getenv("RSB_SPMV_T_OCC")) == 6;  // experiments
        if (occ6) {
            if (epi == EPI_ADD)
                k_spmv_t_tile<EPI_ADD, 6><<<grid, kBlock, 0, ctx->stream>>>(At, y, z, e, g);
            else
                k_spmv_t_tile<EPI_STORE, 6><<<grid, kBlock, 0, ctx->stream>>>(At, y, z, e, g);
        } else if (epi == EPI_ADD) {
            k_spmv_t_tile<EPI_ADD, 4><<<grid, kBlock, 0, ctx->stream>>>(At, y, z, e, g);
        } else {
            k_spmv_t_tile<EPI_STORE, 4><<<grid, kBlock, 0, ctx->stream>>>(At, y, z, e, g);
        }
        return post_launch(ctx);
    }
    if (epi == EPI_ADD)
        k_spmv_t<EPI_ADD><<<grid, kBlock, 0, ctx->stream>>>(At, y, z, e, g);
    else
        k_spmv_t<EPI_STORE><<<grid, kBlock, 0, ctx->stream>>>(At, y, z, e, g);
    return post_launch(ctx);
}

int launch_fill(rsb_ctx *ctx, double *x, int64_t n, unsigned long long bits, Gate g) {
    if (n == 0) return RSB_OK;
    k_fill<<<grid_stride(n), kBlock, 0, ctx->stream>>>(x, n, bits, g);
    return post_launch(ctx);
}

// bench instrumentation: event pairs around every sparse product captured
// into an instrumented iteration graph (on the launching stream)
template <class F>
static int traced_product(rsb_ctx *ctx, F &&launch) {
    const bool trace = ctx->tracing && ctx->ptrace_n + 2 <= 64;
    if (trace)
        RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->ptrace_ev[ctx->ptrace_n++], ctx->stream, cudaEventRecordExternal));
    RSB_TRY(launch());
    if (trace)
        RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->ptrace_ev[ctx->ptrace_n++], ctx->stream, cudaEventRecordExternal));
    return RSB_OK;
}

int launch_spmv(rsb_ctx *ctx, const Compressed &A, VecIn x, double *y, int epi, VecIn e, Gate g) {
    return traced_product(ctx, [&] { return spmv_impl(ctx, A, x, y, epi, e, g); });
}

int launch_spmv_t(rsb_ctx *ctx, const Compressed &At, VecIn y, double *z, int epi, VecIn e, Gate g) {
    return traced_product(ctx, [&] { return spmv_t_impl(ctx, At, y, z, epi, e, g); });
}

int launch_trsv(rsb_ctx *ctx, const TriSched &T, VecIn a, const double *c, double *x, Gate g,
                const TriWs *ws, TrsvChain chain) {
    if (T.n == 0) return RSB_OK;
    const bool nat = trsv_wants_prefill(T);
    if (chain.fill_next && !nat) {  // no in-kernel fill in this variant
        RSB_TRY(launch_fill(ctx, chain.fill_next, T.n, kSentinel, Gate{}));
        chain.fill_next = nullptr;
    }
    const bool trace = ctx->tracing && ctx->trace_n + 2 <= 64;
    if (trace)
        RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->trace_ev[ctx->trace_n++], ctx->stream, cudaEventRecordExternal));
    TriDev v = T.view();
    if (ws) {
        if (T.single_cta && ws->cap < T.padded_n) {
            set_error("triangular-solve scratch too small (%lld < %lld)", (long long)ws->cap, (long long)T.padded_n);
            return RSB_ESTATE;
        }
        v.bpos = ws->bpos;
        v.ticket = ws->ticket;
    }
    if (T.single_cta) {
        const size_t smem = (size_t)stage_smem_bytes(T.stage_ch, T.stage_emax, T.diag != nullptr, T.nlevels, T.nchunks);
        k_gather_pos<<<grid_stride(T.padded_n), kBlock, 0, ctx->stream>>>(T.n, T.padded_n, T.task_row, a, c,
                                                                          v.bpos, g);
        RSB_TRY(post_launch(ctx));
        const int sel = T.mode + (T.has_far ? 4 : 0);
        if (T.lean_n) {
            RSB_TRY(launch_trsv_lean(ctx, T, v, x, g));
        } else switch (sel) {
            case 0: k_trsv_stage<0, false><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            case 1: k_trsv_stage<1, false><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            case 2: k_trsv_stage<2, false><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            case 3: k_trsv_stage<3, false><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            case 4: k_trsv_stage<0, true><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            case 5: k_trsv_stage<1, true><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            case 6: k_trsv_stage<2, true><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
            default: k_trsv_stage<3, true><<<1, kCtaTri + 32, smem, ctx->stream>>>(v, x, g); break;
        }
    } else if (T.level_launch) {
        for (int32_t l = 0; l + 1 < (int32_t)T.h_level_ptr.size(); ++l) {
            const int lo = T.h_level_ptr[l], hi = T.h_level_ptr[l + 1];
            const int grid = (int)std::min<int64_t>((hi - lo + kBlock - 1) / kBlock, 148 * 16);
            switch (T.mode) {
                case 0: k_trsv_level<0><<<grid, kBlock, 0, ctx->stream>>>(v, a, c, x, lo, hi, g); break;
                case 1: k_trsv_level<1><<<grid, kBlock, 0, ctx->stream>>>(v, a, c, x, lo, hi, g); break;
                case 2: k_trsv_level<2><<<grid, kBlock, 0, ctx->stream>>>(v, a, c, x, lo, hi, g); break;
                default: k_trsv_level<3><<<grid, kBlock, 0, ctx->stream>>>(v, a, c, x, lo, hi, g); break;
            }
            if (l + 2 < (int32_t)T.h_level_ptr.size()) RSB_TRY(post_launch(ctx));
        }
    } else if (T.lsync) {
        RSB_TRY(launch_trsv_lsync(ctx, T, v, ws ? ws->ls_cnt : T.ls_cnt, a, c, x, g));
    } else if (T.wide && T.use_nat) {
        RSB_TRY_CUDA(cudaMemsetAsync(v.ticket, 0, sizeof(unsigned long long), ctx->stream));
        // sentinel fill unless the chain's previous solve did it, then the solve (counted below)
        RSB_TRY(launch_trsv_nat(ctx, T, v, a, c, x, g, chain.prefilled, chain.fill_next, chain.rhs_copy));
    } else if (T.wide && T.level_sync) {
        // level-synchronous cooperative solve (trsv_ls.cu), the default for wide DAGs
        RSB_TRY(launch_trsv_ls(ctx, T, v, a, c, x, reinterpret_cast<unsigned *>(v.ticket), g, 1, nullptr, 0));
        ctx->launches += 1;  // the barrier-counter memset is not a kernel; the solve is counted below
    } else if (T.wide) {
        RSB_TRY_CUDA(cudaMemsetAsync(v.ticket, 0, sizeof(unsigned long long), ctx->stream));
        RSB_TRY(launch_trsv_wide(ctx, T, v, a, c, x, g));  // sentinel fill, level 0, then the solve
        ctx->launches += 1;  // level 0 (the fill counted itself; the solve is counted below)
    } else {
        RSB_TRY(launch_fill(ctx, x, T.n, kSentinel, g));
        // blocks number themselves in start order from this counter
        RSB_TRY_CUDA(cudaMemsetAsync(v.ticket, 0, sizeof(unsigned long long), ctx->stream));
        const int grid = grid_for(T.n, kTriBlock);
        switch (T.mode) {
            case 0: k_trsv<0><<<grid, kTriBlock, 0, ctx->stream>>>(v, a, c, x, g); break;
            case 1: k_trsv<1><<<grid, kTriBlock, 0, ctx->stream>>>(v, a, c, x, g); break;
            case 2: k_trsv<2><<<grid, kTriBlock, 0, ctx->stream>>>(v, a, c, x, g); break;
            default: k_trsv<3><<<grid, kTriBlock, 0, ctx->stream>>>(v, a, c, x, g); break;
        }
    }
    RSB_TRY(post_launch(ctx));
    if (trace)
        RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->trace_ev[ctx->trace_n++], ctx->stream, cudaEventRecordExternal));
    return RSB_OK;
}

int tri_ws_alloc(rsb_ctx *ctx, TriWs &w, int64_t cap) {
    RSB_TRY(dev_alloc(ctx, (void **)&w.bpos, (size_t)std::max<int64_t>(cap, 1) * sizeof(double)));
    w.cap = cap;
    RSB_TRY(dev_alloc(ctx, (void **)&w.ticket, sizeof(unsigned long long)));
    RSB_TRY(dev_alloc(ctx, (void **)&w.ls_cnt, kLsCounters * sizeof(unsigned)));
    RSB_TRY_CUDA(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned long long), ctx->stream));
    return RSB_OK;
}

void tri_ws_free(rsb_ctx *ctx, TriWs &w) {
    if (w.bpos) dev_free(ctx, w.bpos, (size_t)std::max<int64_t>(w.cap, 1) * sizeof(double));
    if (w.ticket) dev_free(ctx, w.ticket, sizeof(unsigned long long));
    if (w.ls_cnt) dev_free(ctx, w.ls_cnt, kLsCounters * sizeof(unsigned));
    w = TriWs{};
}

int prepare_trsv_cta(int64_t smem_bytes) {
    static int granted = 48 * 1024;  // attributes only ever grow: every schedule keeps its launch valid
    const int smem = (int)smem_bytes;
    if (smem > granted) {
        granted = smem;
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_trsv_stage<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    return RSB_OK;
}

namespace {
__global__ void k_flush(double *buf, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = (double)i;
}
}  // namespace

int launch_l2_flush(rsb_ctx *ctx) {
    const size_t bytes = 320ull << 20;  // > 2.5x the 126 MB L2
    if (!ctx->flush_buf) {
        RSB_TRY(dev_alloc(ctx, &ctx->flush_buf, bytes));
        ctx->flush_bytes = bytes;
    }
    k_flush<<<148 * 8, kBlock, 0, ctx->stream>>>((double *)ctx->flush_buf, (int64_t)(bytes / 8));
    return post_launch(ctx);
}

int launch_dot(rsb_ctx *ctx, int64_t n, VecIn a, VecIn b, double *out, int sqrt_out, Gate g,
               const int *need) {
    if ((ctx->flags & RSB_DOT_TREE) && n > 4096) {
        int parts = (int)std::min<int64_t>((n + 8191) / 8192, 2 * 148 * 4);
        if (parts > ctx->partial_cap) {
            set_error("tree-dot partial buffer too small");
            return RSB_ESTATE;
        }
        k_dot_tree_partial<<<parts, kBlock, 0, ctx->stream>>>(n, a, b, ctx->d_partials, g, need);
        RSB_TRY(post_launch(ctx));
        k_dot_tree_final<<<1, 32, 0, ctx->stream>>>(parts, ctx->d_partials, out, sqrt_out, g, need);
        return post_launch(ctx);
    }
    // the reference's OpenBLAS runs dots longer than 10000 on T threads
    DotChunks ch{1, nullptr, nullptr};
    if (ctx->blas_threads > 1 && n > 10000) {
        const int slot = ctx->dot_slot++ % kDotSlots;
        ch = DotChunks{ctx->blas_threads, ctx->d_dot_part + (size_t)slot * kMaxBlasThreads, ctx->d_dot_cnt + slot};
    }
    const int64_t per_chunk = n / ch.T;
    const bool plain = !a.g && !b.g && !a.off && !b.off && ((uintptr_t)a.p % 16 == 0) && ((uintptr_t)b.p % 16 == 0);
    if (plain && per_chunk >= 2 * kDotChunk) {
        const size_t smem = (size_t)kDotStages * 2 * (kDotChunk + 2) * 8 + 2 * kDotStages * 8;
        static const int norm_stages = [] {  // experiments: stages of the one-stream norm (2 .. 2 * kDotStages)
            const char *e = getenv("RSB_DOT_NORM_STAGES");
            return e ? std::max(0, std::min(2 * kDotStages, atoi(e))) : 2 * kDotStages;  // 0: two streams
        }();
        k_dot_exact_staged<<<ch.T, 32, smem, ctx->stream>>>(n, a.p, b.p, out, sqrt_out, g, need, ch, norm_stages);
        return post_launch(ctx);
    }
    k_dot_exact<<<ch.T, 32, 0, ctx->stream>>>(n, a, b, out, sqrt_out, g, need, ch);
    return post_launch(ctx);
}

int prepare_kernels() {
    const int smem = kDotStages * 2 * (kDotChunk + 2) * 8 + 2 * kDotStages * 8;
    RSB_TRY_CUDA(cudaFuncSetAttribute(k_dot_exact_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return RSB_OK;
}

int launch_copy(rsb_ctx *ctx, double *dst, VecIn src, int64_t n, Gate g) {
    if (n == 0) return RSB_OK;
    k_copy<<<grid_stride(n), kBlock, 0, ctx->stream>>>(dst, src, n, g);
    return post_launch(ctx);
}

int launch_axpy(rsb_ctx *ctx, double *y, const double *x, const double *scal, int sign, int64_t n,
                Gate g) {
    if (n == 0) return RSB_OK;
    if (sign > 0)
        k_axpy<1><<<grid_stride(n), kBlock, 0, ctx->stream>>>(y, x, scal, n, g);
    else
        k_axpy<-1><<<grid_stride(n), kBlock, 0, ctx->stream>>>(y, x, scal, n, g);
    return post_launch(ctx);
}

int launch_xpby(rsb_ctx *ctx, double *p, const double *h, const double *beta, const int *copy_flag,
                int64_t n, Gate g) {
    if (n == 0) return RSB_OK;
    k_xpby<<<grid_stride(n), kBlock, 0, ctx->stream>>>(p, h, beta, copy_flag, n, g);
    return post_launch(ctx);
}

int prepare_chol(int64_t s) {
    // grow-only, like prepare_trsv_cta: a smaller s must not shrink the limit
    // an earlier (larger) preconditioner's launches rely on
    static size_t granted = 48 * 1024;
    const size_t smem = (size_t)s * sizeof(double);
    if (smem > granted && smem <= 200 * 1024) {
        RSB_TRY_CUDA(cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        granted = smem;
    }
    return RSB_OK;
}

int launch_chol_solve(rsb_ctx *ctx, const double *G, int64_t s, const double *u, double *w, Gate g) {
    if (s == 0) return RSB_OK;
    const size_t smem = (size_t)s * sizeof(double);
    const int use_smem = smem <= 200 * 1024;
    k_chol_solve<<<1, kBlock, use_smem ? smem : 0, ctx->stream>>>(G, s, u, w, use_smem, g);
    return post_launch(ctx);
}

}  // namespace rsb
