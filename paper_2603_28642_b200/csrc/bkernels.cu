// Kernels of the batched solve: kBatch = 8 right-hand sides that share A and
// the preconditioner (config 4: 8 RHS per GPU).
//
// Vectors are RHS-interleaved, v[i * 8 + r], so one matrix or factor entry
// is read once and applied to 8 independent chains, and every gathered
// operand is one 64-byte row instead of an 8-byte piece of a 32-byte
// sector.  Per right-hand side the arithmetic is exactly the single-RHS
// kernels' (the reference's order), so every RHS of the batch is bit-
// identical to its own pcgls run.
//
// Heavy kernels (products, solves, dots) compute all 8 right-hand sides
// unconditionally -- a stopped RHS's scratch vectors are never read again --
// and skip only when the whole batch has stopped; the updates of persistent
// state (x, r, p, w of the inner CG) are gated per RHS.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "bsolver.cuh"
#include "device_common.cuh"

namespace rsb {

namespace {

constexpr int kB = kBatch;
constexpr int kBlk = 256;

__device__ __forceinline__ int64_t bidx(const VecIn &v, int64_t i) {
    return v.g ? (int64_t)v.g[i + v.off] : i + v.off;
}
__device__ __forceinline__ bool all_off(const int *all_done) {
    return all_done && *(volatile const int *)all_done != 0;
}
__device__ __forceinline__ bool rhs_off(const BGate &g, int r) {
    return (g.a && *(volatile const int *)((const char *)g.a + (size_t)r * g.sa)) ||
           (g.b && *(volatile const int *)((const char *)g.b + (size_t)r * g.sb));
}
__device__ __forceinline__ const double *bscal(const double *p, int stride, int r) {
    return (const double *)((const char *)p + (size_t)r * stride);
}

inline int grid_stride_n(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlk - 1) / kBlk, 148 * 32));
}

// ---- y = A x (CSR, row-sequential from 0.0; sc.py:212-221): one line by
// an octet of lanes (lane r: RHS r), the gathers four at a time
__device__ __forceinline__ double bline_seq(const Compressed &A, const VecIn &x, int64_t i, int r) {
    const int lo = A.ptr[i], hi = A.ptr[i + 1];
    double acc = 0.0;
    int k = lo;
    for (; k + 4 <= hi; k += 4) {
        int c[4];
        double v[4], xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            c[u] = A.idx[k + u];
            v[u] = A.val[k + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = x.p[bidx(x, c[u]) * kB + r];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    for (; k < hi; ++k) acc = __dadd_rn(acc, __dmul_rn(A.val[k], x.p[bidx(x, A.idx[k]) * kB + r]));
    return acc;
}

// ---- z = A^T y (CSC, z_j = p0 + pairwise(p1..); sc.py:224-235), octet per column
struct BProd {
    const double *val;
    const int32_t *idx;
    const VecIn *y;
    int r;
    __device__ double operator()(int64_t k) const { return __dmul_rn(val[k], y->p[bidx(*y, idx[k]) * kB + r]); }
};

// eight products of a column (entries k0 .. k0+7 below `lim`), every index,
// value and gather in flight together
__device__ __forceinline__ void prod8(const Compressed &A, int lo, int k0, int lim, const VecIn &y, int r,
                                      double (&p)[8]) {
    int c[8];
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        c[u] = k0 + u < lim ? __ldcs(A.idx + lo + k0 + u) : 0;
        v[u] = k0 + u < lim ? __ldcs(A.val + lo + k0 + u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = k0 + u < lim ? __dmul_rn(v[u], y.p[bidx(y, c[u]) * kB + r]) : 0.0;
}

// z_j = p0 + pairwise(p1 .. p_{n-1}) streamed in chunks of 8 products (the
// 8 strided accumulators of numpy's pairwise leaf take one chunk per step)
__device__ __noinline__ double bline_pw(const Compressed &A, const VecIn &y, int64_t j, int r) {
    const int lo = A.ptr[j], n = A.ptr[j + 1] - lo;
    double acc = 0.0;
    const int m = n - 1;  // terms of the pairwise part
    if (n > 0 && m <= 128) {
        double p[8];
        prod8(A, lo, 0, n, y, r, p);  // p0 .. p7
        const double p0 = p[0];
        double rest;
        if (m < 8) {
            rest = -0.0;
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u <= m) rest = __dadd_rn(rest, p[u]);
        } else {
            double q[8];
            prod8(A, lo, 8, n, y, r, q);  // p8 .. p15
            double acc8[8];
            acc8[0] = p[1], acc8[1] = p[2], acc8[2] = p[3], acc8[3] = p[4];
            acc8[4] = p[5], acc8[5] = p[6], acc8[6] = p[7], acc8[7] = q[0];
            // terms t = 8 .. mb-1 (entries 9 .. mb) in chunks of 8
            const int mb = m - (m % 8);
            int t = 8;
            double cur[8];  // entries t+1 .. t+8
#pragma unroll
            for (int u = 0; u < 7; ++u) cur[u] = q[u + 1];
            {
                double nx[8];
                prod8(A, lo, 16, n, y, r, nx);
                cur[7] = nx[0];
                while (t < mb) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc8[k] = __dadd_rn(acc8[k], cur[k]);
                    t += 8;
#pragma unroll
                    for (int u = 0; u < 7; ++u) cur[u] = nx[u + 1];
                    if (t < m) {
                        prod8(A, lo, t + 8, n, y, r, nx);
                        cur[7] = nx[0];
                    }
                }
            }
            rest = __dadd_rn(__dadd_rn(__dadd_rn(acc8[0], acc8[1]), __dadd_rn(acc8[2], acc8[3])),
                             __dadd_rn(__dadd_rn(acc8[4], acc8[5]), __dadd_rn(acc8[6], acc8[7])));
            // tail terms mb .. m-1 (entries mb+1 .. m): cur[0 .. m-mb-1]
#pragma unroll
            for (int u = 0; u < 7; ++u)
                if (mb + u < m) rest = __dadd_rn(rest, cur[u]);
        }
        acc = __dadd_rn(p0, rest);
    } else if (n > 0) {
        const BProd t{A.val + lo, A.idx + lo, &y, r};
        acc = __dadd_rn(t(0), Pairwise<25, BProd>::sum(t, 1, n - 1));
    }
    return acc;
}


// ---- Tiled batched SpMV, both directions.  A block owns 32 consecutive
// lines (an octet of lanes per line, lane r = RHS r).  Phase 1 forms every
// product of the tile -- each entry's index and value are loaded once for
// its octet, all gathers of a thread in flight together -- into shared
// memory; phase 2 sums each line's products in the reference's order:
// sequentially from 0.0 for A x (np.add.at), p0 + pairwise(p1..) for A^T y
// (np.add.reduceat).  A tile with more entries than the buffer (dense rows)
// runs the per-line code instead.
constexpr int kBTile = 32;
constexpr int kBTileCap = 512;
constexpr int kBTileRounds = 2;  // measured at n = 8e6: 35.1 -> 32.9 ms per 8-RHS iteration (A^T 3.32 -> 3.03, L2^T -> 2.07 ms)

template <bool TRANS>
struct BTerm {
    const double *p;
    int r;
    __device__ double operator()(int64_t k) const { return p[k * kB + r]; }
};

// ROUNDS: the tile's products are formed in ROUNDS passes of kBTileCap /
// kBTile / ROUNDS entries per octet (1: 16 gathers in flight per thread, 80
// registers, 3 blocks per SM; 2: 8 in flight, more resident blocks)
template <bool TRANS, int EPI, int ROUNDS>
__global__ void __launch_bounds__(kBlk, ROUNDS == 1 ? 3 : (ROUNDS == 2 ? 5 : 6)) kb_spmv_tile(Compressed A, VecIn x, double *y, VecIn e,
                                                                        const int *all_done) {
    if (all_off(all_done)) return;
    __shared__ double prod[kBTileCap * kB];
    const int oct = threadIdx.x >> 3, r = threadIdx.x & 7;
    const int64_t l0 = blockIdx.x * (int64_t)kBTile;
    const int64_t i = l0 + oct;
    const bool valid = i < A.nlines;
    const int64_t lend = min((int64_t)A.nlines, l0 + kBTile);
    const int lo = A.ptr[l0], hi = A.ptr[lend];
    double acc = 0.0;
    if (hi - lo <= kBTileCap) {
        constexpr int U = kBTileCap / kBTile / ROUNDS;
#pragma unroll
        for (int h = 0; h < ROUNDS; ++h) {
            if (h > 0 && lo + kBTile * U * h >= hi) break;
            int c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = lo + oct + kBTile * (u + U * h);
                c[u] = k < hi ? __ldcs(A.idx + k) : -1;
                v[u] = k < hi ? __ldcs(A.val + k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? x.p[bidx(x, c[u]) * kB + r] : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c[u] >= 0) prod[(oct + kBTile * (u + U * h)) * kB + r] = __dmul_rn(v[u], xv[u]);
        }
        __syncthreads();
        if (!valid) return;
        const int s0 = A.ptr[i] - lo, t0 = A.ptr[i + 1] - lo;
        if (!TRANS) {
            for (int k = s0; k < t0; ++k) acc = __dadd_rn(acc, prod[k * kB + r]);
        } else if (t0 > s0) {
            const BTerm<TRANS> t{prod + (size_t)(s0 + 1) * kB, r};
            const int m = t0 - s0 - 1;
            acc = __dadd_rn(prod[s0 * kB + r], m <= 128 ? pw_leaf(t, 0, m) : Pairwise<3, BTerm<TRANS>>::sum(t, 0, m));
        }
    } else {
        if (!valid) return;
        acc = TRANS ? bline_pw(A, x, i, r) : bline_seq(A, x, i, r);
    }
    if (EPI == EPI_ADD) acc = __dadd_rn(e.p[bidx(e, i) * kB + r], acc);
    if (EPI == EPI_SUB_FROM) acc = __dsub_rn(e.p[bidx(e, i) * kB + r], acc);
    y[i * kB + r] = acc;
}


// (A persistent CSC variant staging each tile's indices and values by TMA
// two tiles ahead measured slower: 3.65 vs 2.88 ms per launch at n = 8e6 --
// two bulk copies per ~5 KB tile keep the SM's TMA unit busy longer than the
// index round trip they hide.)

// CSR products (A p, L2 t): an octet of lanes per row straight from global
// memory.  Rows here are short (6-7 entries); on config 4 at n = 8e6 this
// measured 2.1 ms for A p against 4.2 ms for the tiled kernel.
template <int EPI>
__global__ void __launch_bounds__(kBlk) kb_spmv_rows(Compressed A, VecIn x, double *y, VecIn e, const int *all_done) {
    if (all_off(all_done)) return;
    const int64_t tid = blockIdx.x * (int64_t)kBlk + threadIdx.x;
    const int64_t i = tid >> 3;
    const int r = (int)(tid & 7);
    if (i >= A.nlines) return;
    double acc = bline_seq(A, x, i, r);
    if (EPI == EPI_ADD) acc = __dadd_rn(e.p[bidx(e, i) * kB + r], acc);
    if (EPI == EPI_SUB_FROM) acc = __dsub_rn(e.p[bidx(e, i) * kB + r], acc);
    y[i * kB + r] = acc;
}

// (CSC products with an octet of lanes per column straight from global
// memory, the CSR kernel's scheme, measured slower than the tiled kernel twice:
// through bline_pw 87 vs 36.5 ms per batched iteration at n = 8e6, and with a
// register version for columns of <= 16 entries (L2^T w only) 37.4 vs 32.6.)

// ---- a @ b per RHS in the context's OpenBLAS order.  Block = 256 threads:
// thread t runs accumulator chain t >> 3 (of the 32 the OpenBLAS kernel
// keeps) of RHS t & 7, so a warp's loads are 4 whole 64-byte rows; at the
// end the 32 chains of each RHS are moved into warp r through shared
// memory for the fold (warp_blas_finish).  grid = T chunks; partials
// combined by the last block in chunk order (every block counts itself, so
// the slot is reset even when the batch stops mid-launch).
__global__ void __launch_bounds__(kBlk) kb_dot(int64_t n, VecIn a, VecIn b, double *out, int ostride, int sqrt_out,
                                                 const int *all_done, const int *need, int nstride, BDotChunks ch) {
    __shared__ int s_skip;
    __shared__ double s_acc[kB][33];
    if (threadIdx.x == 0) {
        int sk = all_off(all_done) ? 1 : 0;
        if (need && !sk) {  // only when some RHS needs it (z.p: rho <= 0, sv.py:203)
            int any = 0;
            for (int q = 0; q < kB; ++q) any |= *(volatile const int *)((const char *)need + (size_t)q * nstride);
            sk = !any;
        }
        s_skip = sk;
    }
    __syncthreads();
    const bool skip = s_skip != 0;
    int64_t lo = 0, w = n;
    if (ch.T > 1) {
        int64_t rem = n;
        for (int i = 0; i < (int)blockIdx.x; ++i) {
            const int64_t wi = (rem + (ch.T - i) - 1) / (ch.T - i);
            lo += wi;
            rem -= wi;
        }
        w = (rem + (ch.T - (int)blockIdx.x) - 1) / (ch.T - (int)blockIdx.x);
    }
    const int cr = threadIdx.x & 7, cc = threadIdx.x >> 3;  // this thread's (RHS, chain)
    const int64_t n32 = (w & ~(int64_t)15) & ~(int64_t)31;
    double acc = 0.0;
    if (!skip) {
        int64_t i = cc;
        auto la = [&](int64_t k) { return a.p[bidx(a, lo + k) * kB + cr]; };
        auto lb = [&](int64_t k) { return b.p[bidx(b, lo + k) * kB + cr]; };
        for (; i + 15 * 32 < n32; i += 16 * 32) {
            double xa[16], xb[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                xa[u] = la(i + u * 32);
                xb[u] = lb(i + u * 32);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = fma(xa[u], xb[u], acc);
        }
        for (; i < n32; i += 32) acc = fma(la(i), lb(i), acc);
    }
    s_acc[cr][cc] = acc;
    __syncthreads();
    const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double d = 0.0;
    if (!skip)
        d = warp_blas_finish(
            s_acc[r][lane], w, [&](int64_t k) { return a.p[bidx(a, lo + k) * kB + r]; },
            [&](int64_t k) { return b.p[bidx(b, lo + k) * kB + r]; });
    double *o = (double *)((char *)out + (size_t)r * ostride);
    if (ch.T <= 1) {
        if (!skip && lane == 0) *o = sqrt_out ? sqrt(d) : d;
        return;
    }
    if (!skip && lane == 0) ch.part[blockIdx.x * kB + r] = d;
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(ch.cnt, skip ? 0x10000u + 1u : 1u);
        last = (prev & 0xFFFFu) == (unsigned)ch.T - 1;
        if (last) {
            __threadfence();
            *ch.cnt = 0;
            if (skip || (prev >> 16)) last = false;
        }
    }
    __syncthreads();
    if (!last) return;
    if (lane == 0) {
        double sum = 0.0;
        for (int i = 0; i < ch.T; ++i) sum = __dadd_rn(sum, ((volatile const double *)ch.part)[i * kB + r]);
        *o = sqrt_out ? sqrt(sum) : sum;
    }
}

// ---- the same dot with both operands streamed through shared memory by 1-D
// TMA bulk copies (a chunk's rows are contiguous: lo*8 .. (lo+w)*8 doubles):
// kBDotRows rows per stage, kBDotStages stages in flight, so each SM keeps
// ~128 KB of loads in flight instead of the ~16 KB the thread loads reach.
// Operands are read directly (no gather); the chains, their order and the
// finish are kb_dot's.
constexpr int kBDotRows = 512;  // rows per stage: 32 KB per operand
constexpr int kBDotStages = 2;

__global__ void __launch_bounds__(kBlk, 1) kb_dot_staged(int64_t n, const double *a, const double *b, double *out,
                                                          int ostride, int sqrt_out, const int *all_done,
                                                          const int *need, int nstride, BDotChunks ch) {
    extern __shared__ __align__(128) double sbuf[];  // [stage][a|b][kBDotRows * 8]
    __shared__ unsigned long long bar[kBDotStages];
    __shared__ int s_skip;
    __shared__ double s_acc[kB][33];
    if (threadIdx.x == 0) {
        int sk = all_off(all_done) ? 1 : 0;
        if (need && !sk) {
            int any = 0;
            for (int q = 0; q < kB; ++q) any |= *(volatile const int *)((const char *)need + (size_t)q * nstride);
            sk = !any;
        }
        s_skip = sk;
        for (int st = 0; st < kBDotStages; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const bool skip = s_skip != 0;
    int64_t lo = 0, w = n;
    if (ch.T > 1) {
        int64_t rem = n;
        for (int i = 0; i < (int)blockIdx.x; ++i) {
            const int64_t wi = (rem + (ch.T - i) - 1) / (ch.T - i);
            lo += wi;
            rem -= wi;
        }
        w = (rem + (ch.T - (int)blockIdx.x) - 1) / (ch.T - (int)blockIdx.x);
    }
    const int cr = threadIdx.x & 7, cc = threadIdx.x >> 3;
    const int64_t n32 = (w & ~(int64_t)15) & ~(int64_t)31;
    const int64_t nst = (n32 + kBDotRows - 1) / kBDotRows;
    double acc = 0.0;
    if (!skip && nst > 0) {
        auto issue = [&](int64_t c) {
            const int st = (int)(c % kBDotStages);
            const int64_t r0 = c * kBDotRows, r1 = min(n32, r0 + kBDotRows);
            const unsigned bytes = (unsigned)((r1 - r0) * kB * sizeof(double));
            double *da = sbuf + (size_t)st * 2 * kBDotRows * kB;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[st], 2 * bytes);
            bulk_g2s(da, a + (lo + r0) * kB, bytes, &bar[st]);
            bulk_g2s(da + kBDotRows * kB, b + (lo + r0) * kB, bytes, &bar[st]);
        };
        if (threadIdx.x == 0)
            for (int64_t c = 0; c < min((int64_t)kBDotStages, nst); ++c) issue(c);
        for (int64_t c = 0; c < nst; ++c) {
            const int st = (int)(c % kBDotStages);
            mbar_wait(&bar[st], (unsigned)((c / kBDotStages) & 1));
            const double *da = sbuf + (size_t)st * 2 * kBDotRows * kB, *db = da + kBDotRows * kB;
            const int rows = (int)(min(n32, (c + 1) * kBDotRows) - c * kBDotRows);
            for (int i = cc; i < rows; i += 32) acc = fma(da[i * kB + cr], db[i * kB + cr], acc);
            __syncthreads();  // every thread is done with this buffer
            if (threadIdx.x == 0 && c + kBDotStages < nst) issue(c + kBDotStages);
        }
    }
    s_acc[cr][cc] = acc;
    __syncthreads();
    const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double d = 0.0;
    if (!skip)
        d = warp_blas_finish(
            s_acc[r][lane], w, [&](int64_t k) { return a[(lo + k) * kB + r]; },
            [&](int64_t k) { return b[(lo + k) * kB + r]; });
    double *o = (double *)((char *)out + (size_t)r * ostride);
    if (ch.T <= 1) {
        if (!skip && lane == 0) *o = sqrt_out ? sqrt(d) : d;
        return;
    }
    if (!skip && lane == 0) ch.part[blockIdx.x * kB + r] = d;
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(ch.cnt, skip ? 0x10000u + 1u : 1u);
        last = (prev & 0xFFFFu) == (unsigned)ch.T - 1;
        if (last) {
            __threadfence();
            *ch.cnt = 0;
            if (skip || (prev >> 16)) last = false;
        }
    }
    __syncthreads();
    if (!last) return;
    if (lane == 0) {
        double sum = 0.0;
        for (int i = 0; i < ch.T; ++i) sum = __dadd_rn(sum, ((volatile const double *)ch.part)[i * kB + r]);
        *o = sqrt_out ? sqrt(sum) : sum;
    }
}

// ---- elementwise, per-RHS scalars and gates.  The launch width is a
// multiple of 8, so a thread always handles the same RHS r = i & 7: its
// gate and scalar are read once.
template <int SIGN>
__global__ void kb_axpy(double *y, const double *x, const double *scal, int sstride, int64_t n, BGate g) {
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int r = (int)(i0 & 7);
    if (rhs_off(g, r)) return;
    const double s = *bscal(scal, sstride, r);
    for (int64_t i = i0; i < n * kB; i += (int64_t)gridDim.x * blockDim.x) {
        const double t = __dmul_rn(s, x[i]);
        y[i] = SIGN > 0 ? __dadd_rn(y[i], t) : __dsub_rn(y[i], t);
    }
}

// p = h + beta*p, or p = h where copy flag set (per RHS)
__global__ void kb_xpby(double *p, const double *h, const double *beta, int bstride, const int *copy_flag,
                        int cstride, int64_t n, BGate g) {
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int r = (int)(i0 & 7);
    if (rhs_off(g, r)) return;
    const bool cp = copy_flag && *(const int *)((const char *)copy_flag + (size_t)r * cstride);
    const double bt = cp ? 0.0 : *bscal(beta, bstride, r);
    for (int64_t i = i0; i < n * kB; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = cp ? h[i] : __dadd_rn(h[i], __dmul_rn(bt, p[i]));
}

__global__ void kb_copy(double *dst, VecIn src, int64_t n, BGate g) {
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int r = (int)(i0 & 7);
    if (rhs_off(g, r)) return;
    for (int64_t i = i0; i < n * kB; i += (int64_t)gridDim.x * blockDim.x) dst[i] = src.p[bidx(src, i >> 3) * kB + r];
}

__global__ void kb_fill(double *x, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * kB; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

// w = 0, r = u, p = u (_cg_fixed_steps start, pc.py:291-293)
__global__ void kb_cg_init(double *w, double *rr, double *p, const double *u, int64_t s, BGate g) {
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (rhs_off(g, (int)(i0 & 7))) return;
    for (int64_t i = i0; i < s * kB; i += (int64_t)gridDim.x * blockDim.x) {
        const double uv = u[i];
        w[i] = 0.0;
        rr[i] = uv;
        p[i] = uv;
    }
}

// row-major k x len (host order) <-> interleaved len x 8; missing RHS are zero
__global__ void kb_pack(double *dst, const double *src, int64_t len, int k) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len * kB; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i & 7);
        dst[i] = r < k ? src[(size_t)r * len + (i >> 3)] : 0.0;
    }
}
__global__ void kb_unpack(double *dst, const double *src, int64_t len, int k) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len * k; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / len, j = i - r * len;
        dst[i] = src[j * kB + r];
    }
}

// ---------------------------------------------------------------------------
// Batched sync-free triangular solve (wide schedules).  A lane owns one task
// for all 8 right-hand sides: its entries are loaded once; the dependencies
// of one half (4 RHS) at a time are read as two 16-byte loads per entry.
// Completion is a per-row flag holding the launch's epoch (written after the
// row's 8 values, release), so no sentinel fill of the 8n outputs is needed;
// the epoch is bumped by a one-thread kernel before every solve.
// ---------------------------------------------------------------------------
constexpr unsigned kBtMinBackoff = 32, kBtMaxBackoff = 256;

// Flags are polled with acquire loads (LDG.STRONG.GPU + an L1 invalidate): a
// flag seen set orders the row reads after it, with no fence on the consumer
// side.  (Relaxed polls followed by __threadfence() -- MEMBAR.SC.GPU -- measured
// the same: 32.9 vs 33.1 ms per 8-RHS iteration at n = 8e6.)
__device__ __forceinline__ int ld_flag(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_flag_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 4 consecutive doubles (32-byte aligned: half of a 64-byte row), through L2,
// as ONE 256-bit load (sm_100 LDG.256): a warp whose lanes read 32 different
// rows pays 32 L1TEX wavefronts per load instruction, so two 16-byte loads per
// half cost twice the wavefronts for the same bytes
__device__ __forceinline__ void ld4(const double *p, double (&v)[4]) {
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void st4(double *p, const double (&v)[4]) {
    asm volatile("st.global.cg.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}

// entries of the task past `from` (contiguous, then -1 padding)
__device__ __noinline__ int bt_tail_len(const TriDev &T, int64_t base, int from, int K) {
    int len = from;
    for (int q = from; q < K; ++q) {
        if (T.ecol[base + (int64_t)q * 32] < 0) break;
        ++len;
    }
    return len;
}

__device__ __noinline__ bool bt_tail_ready(const TriDev &T, int64_t base, int from, int len, const int *flag, int E) {
    for (int q0 = from; q0 < len; q0 += 8) {
        int f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int c = q0 + u < len ? T.ecol[base + (int64_t)(q0 + u) * 32] : -1;
            f[u] = c >= 0 ? ld_flag(flag + c) : E;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (f[u] != E) return false;
    }
    return true;
}

// entries past `from`, all published: continue the 4 chains of half h
template <int MODE>
__device__ __noinline__ void bt_tail(const TriDev &T, int64_t base, int from, int len, int h, const double *x,
                                     double (&acc)[4], double (&dot)[4]) {
    for (int q0 = from; q0 < len; q0 += 4) {
        int c[4];
        double v[4], xv[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            c[u] = q0 + u < len ? T.ecol[base + (int64_t)(q0 + u) * 32] : -1;
            v[u] = q0 + u < len ? T.eval[base + (int64_t)(q0 + u) * 32] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (c[u] >= 0)
                ld4(x + (int64_t)c[u] * kB + 4 * h, xv[u]);
            else
                xv[u][0] = xv[u][1] = xv[u][2] = xv[u][3] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (c[u] < 0) break;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!(MODE & 1)) {
                    if (xv[u][q] != 0.0) acc[q] = __dsub_rn(acc[q], __dmul_rn(v[u], xv[u][q]));
                } else {
                    dot[q] = fma(v[u], xv[u][q], dot[q]);
                }
            }
        }
    }
}

template <int MODE, int N, bool TAIL>
__global__ void __launch_bounds__(kBlk, 2) kb_trsv(TriDev T, VecIn a, const double *c, double *x, int *flag,
                                                    const unsigned *epoch, int first_slice, int nslices,
                                                    const int *all_done) {
    if (all_off(all_done)) return;
    const int E = (int)*(volatile const unsigned *)epoch;
    const int lane = threadIdx.x & 31;
    const int ntickets = nslices - first_slice;
    auto take = [&]() {
        int s = 0;
        if (lane == 0) s = (int)atomicAdd(T.ticket, 1ull);
        return __shfl_sync(0xffffffffu, s, 0);
    };
    int j = take();
    while (j < ntickets) {
        const int s = first_slice + j;
        const int t = s * 32 + lane;
        const bool valid = t < T.n;
        const int64_t base = T.slice_off[s] + lane;
        const int K = (int)((T.slice_off[s + 1] - T.slice_off[s]) >> 5);

        int row = -1, len = 0;
        int cols[N];
        double vals[N];
        double d = 1.0;
        int64_t ai = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            cols[q] = -1;
            vals[q] = 0.0;
        }
        unsigned need = 0;
        if (valid) {
            row = T.task_row[t];
            ai = a.g ? (int64_t)a.g[row + a.off] : (int64_t)row + a.off;
#pragma unroll
            for (int q = 0; q < N; ++q)
                if (q < K) {
                    cols[q] = T.ecol[base + (int64_t)q * 32];
                    vals[q] = T.eval[base + (int64_t)q * 32];
                }
#pragma unroll
            for (int q = 0; q < N; ++q)
                if (cols[q] >= 0) {
                    need |= 1u << q;
                    ++len;
                }
            if (TAIL && len == N && K > N) len = bt_tail_len(T, base, N, K);
            if (MODE & 2) d = T.diag[t];
        }
        bool done = !valid;
        unsigned prev = ~0u, backoff = 0;
        for (;;) {
            if (!__any_sync(0xffffffffu, !done)) break;
            const bool stalled = done || need == prev;
            if (__all_sync(0xffffffffu, stalled) && backoff) __nanosleep(backoff);
            backoff = backoff ? min(backoff * 2, kBtMaxBackoff) : kBtMinBackoff;
            prev = need;
            if (!done) {
                int f[N];
#pragma unroll
                for (int q = 0; q < N; ++q) f[q] = ((need >> q) & 1u) ? ld_flag(flag + cols[q]) : E;
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (f[q] == E) need &= ~(1u << q);
                if (need == 0 && (!TAIL || len <= N || bt_tail_ready(T, base, N, len, flag, E))) {
                    // both halves of every row at once, four entries per round: a task
                    // of <= 4 entries (most of L1's) costs one round trip of gathers
                    double acc[2][4], dot[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
                    ld4(a.p + ai * kB, acc[0]);
                    ld4(a.p + ai * kB + 4, acc[1]);
                    if (c) {
                        double cv[2][4];
                        ld4(c + (int64_t)row * kB, cv[0]);
                        ld4(c + (int64_t)row * kB + 4, cv[1]);
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int q = 0; q < 4; ++q) acc[h][q] = __dadd_rn(acc[h][q], cv[h][q]);
                    }
#pragma unroll
                    for (int e0 = 0; e0 < N; e0 += 4) {
                        if (e0 > 0 && e0 >= len) break;
                        double xv[4][2][4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (cols[e0 + u] >= 0) {
                                ld4(x + (int64_t)cols[e0 + u] * kB, xv[u][0]);
                                ld4(x + (int64_t)cols[e0 + u] * kB + 4, xv[u][1]);
                            } else {
#pragma unroll
                                for (int h = 0; h < 2; ++h) xv[u][h][0] = xv[u][h][1] = xv[u][h][2] = xv[u][h][3] = 0.0;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (e0 + u >= len) break;
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    if (!(MODE & 1)) {
                                        if (xv[u][h][q] != 0.0)
                                            acc[h][q] = __dsub_rn(acc[h][q], __dmul_rn(vals[e0 + u], xv[u][h][q]));
                                    } else {
                                        dot[h][q] = fma(vals[e0 + u], xv[u][h][q], dot[h][q]);
                                    }
                                }
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (TAIL && len > N) bt_tail<MODE>(T, base, N, len, h, x, acc[h], dot[h]);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if ((MODE & 1) && len > 0) acc[h][q] = __dsub_rn(acc[h][q], dot[h][q]);
                            if (MODE & 2) acc[h][q] = __ddiv_rn(acc[h][q], d);
                        }
                    }
                    st4(x + (int64_t)row * kB, acc[0]);
                    st4(x + (int64_t)row * kB + 4, acc[1]);
                    st_flag_release(flag + row, E);
                    done = true;
                }
            }
            __syncwarp();
        }
        // (taking the next ticket before this slice measured slower: U 4.2 vs
        // 2.8 ms at n = 8e6 -- a held slice waits behind this one)
        j = take();
    }
}

// (A pair variant -- two lanes per task, each carrying 4 right-hand sides, so
// that the halves of a dependency's row are read by adjacent lanes as one
// L1TEX wavefront and advance together -- measured slower: 35.4 vs 32.9 ms per
// 8-RHS iteration at n = 8e6; at 80 registers it spills and holds half as many
// tasks per warp.)

// Static-schedule batched solve for short-task forward solves (the single-RHS
// k_trsv_static's scheme): a cooperative launch, warp w owns slices w, w + W,
// ...; the next slice's row, offsets, entries and right-hand-side index are
// loaded while this slice waits, and all 8 right-hand sides' dependencies of
// a ready task are read at once (4 register entries; longer tasks take the
// tail per half).
template <int MODE, bool TAIL>
__global__ void __launch_bounds__(kBlk, 2) kb_trsv_static(TriDev T, VecIn a, const double *c, double *x, int *flag,
                                                          const unsigned *epoch, int first_slice, int nslices,
                                                          const int *all_done) {
    constexpr int N = 4;
    if (all_off(all_done)) return;  // set only between iterations: uniform over the launch
    const int E = (int)*(volatile const unsigned *)epoch;
    const int lane = threadIdx.x & 31;
    const int W = gridDim.x * (kBlk / 32);
    const int gw = blockIdx.x * (kBlk / 32) + (threadIdx.x >> 5);
    struct Pre {
        int64_t base;
        int K, row;
    };
    struct Task {
        int64_t base, ai;
        int K, row;
        double d;
        int cols[N];
        double vals[N];
    };
    auto stage_a = [&](int s, Pre &P) {
        P.base = 0;
        P.K = 0;
        P.row = -1;
        if (s < nslices) {
            P.base = T.slice_off[s] + lane;
            P.K = (int)((T.slice_off[s + 1] - T.slice_off[s]) >> 5);
            const int t = s * 32 + lane;
            if (t < T.n) P.row = __ldcs(T.task_row + t);
        }
    };
    auto stage_b = [&](int s, const Pre &P, Task &k) {
        k.base = P.base;
        k.K = P.K;
        k.row = P.row;
        k.ai = 0;
        k.d = 1.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            k.cols[q] = -1;
            k.vals[q] = 0.0;
        }
        if (P.row < 0) return;
        k.ai = a.g ? (int64_t)a.g[P.row + a.off] : (int64_t)P.row + a.off;
        if (MODE & 2) k.d = T.diag[s * 32 + lane];
#pragma unroll
        for (int q = 0; q < N; ++q)
            if (q < P.K) {
                k.cols[q] = __ldcs(T.ecol + P.base + (int64_t)q * 32);
                k.vals[q] = __ldcs(T.eval + P.base + (int64_t)q * 32);
            }
    };
    int s = first_slice + gw;
    Pre A1;
    Task cur;
    {
        Pre A0;
        stage_a(s, A0);
        stage_b(s, A0, cur);
    }
    stage_a(s + W, A1);
    while (s < nslices) {
        Task nxt;
        stage_b(s + W, A1, nxt);
        Pre A2;
        stage_a(s + 2 * W, A2);
        int len = 0;
        unsigned need = 0;
#pragma unroll
        for (int q = 0; q < N; ++q)
            if (cur.cols[q] >= 0) {
                need |= 1u << q;
                ++len;
            }
        if (TAIL && len == N && cur.K > N) len = bt_tail_len(T, cur.base, N, cur.K);
        bool done = cur.row < 0;
        unsigned prev = ~0u, backoff = 0;
        for (;;) {
            if (!__any_sync(0xffffffffu, !done)) break;
            const bool stalled = done || need == prev;
            if (__all_sync(0xffffffffu, stalled) && backoff) __nanosleep(backoff);
            backoff = backoff ? min(backoff * 2, kBtMaxBackoff) : kBtMinBackoff;
            prev = need;
            if (!done) {
                int f[N];
#pragma unroll
                for (int q = 0; q < N; ++q) f[q] = ((need >> q) & 1u) ? ld_flag(flag + cur.cols[q]) : E;
#pragma unroll
                for (int q = 0; q < N; ++q)
                    if (f[q] == E) need &= ~(1u << q);
                if (need == 0 && (!TAIL || len <= N || bt_tail_ready(T, cur.base, N, len, flag, E))) {
                    double xv[N][8], acc[8], cv[8];
#pragma unroll
                    for (int e = 0; e < N; ++e) {
                        if (cur.cols[e] >= 0) {
                            double h0[4], h1[4];
                            ld4(x + (int64_t)cur.cols[e] * kB, h0);
                            ld4(x + (int64_t)cur.cols[e] * kB + 4, h1);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                xv[e][q] = h0[q];
                                xv[e][4 + q] = h1[q];
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < 8; ++q) xv[e][q] = 0.0;
                        }
                    }
                    {
                        double h0[4], h1[4];
                        ld4(a.p + cur.ai * kB, h0);
                        ld4(a.p + cur.ai * kB + 4, h1);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            acc[q] = h0[q];
                            acc[4 + q] = h1[q];
                        }
                    }
                    if (c) {
                        double h0[4], h1[4];
                        ld4(c + (int64_t)cur.row * kB, h0);
                        ld4(c + (int64_t)cur.row * kB + 4, h1);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            cv[q] = h0[q];
                            cv[4 + q] = h1[q];
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc[q] = __dadd_rn(acc[q], cv[q]);
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        double ah[4], dot[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                        for (int q = 0; q < 4; ++q) ah[q] = acc[4 * h + q];
#pragma unroll
                        for (int e = 0; e < N; ++e) {
                            if (e >= len) break;
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (!(MODE & 1)) {
                                    if (xv[e][4 * h + q] != 0.0)
                                        ah[q] = __dsub_rn(ah[q], __dmul_rn(cur.vals[e], xv[e][4 * h + q]));
                                } else {
                                    dot[q] = fma(cur.vals[e], xv[e][4 * h + q], dot[q]);
                                }
                            }
                        }
                        if (TAIL && len > N) bt_tail<MODE>(T, cur.base, N, len, h, x, ah, dot);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if ((MODE & 1) && len > 0) ah[q] = __dsub_rn(ah[q], dot[q]);
                            if (MODE & 2) ah[q] = __ddiv_rn(ah[q], cur.d);
                        }
                        st4(x + (int64_t)cur.row * kB + 4 * h, ah);
                    }
                    st_flag_release(flag + cur.row, E);
                    done = true;
                }
            }
            __syncwarp();
        }
        s += W;
        cur = nxt;
        A1 = A2;
    }
}

// level 0 of a batched solve: no dependencies.  An octet of lanes per task
// (lane r: RHS r); after the octet's 8 stores, its first lane publishes the
// row's flag (the octet barrier orders the stores before the release).
template <int MODE>
__global__ void kb_trsv_level0(TriDev T, VecIn a, const double *c, double *x, int *flag, const unsigned *epoch,
                               int32_t lvl1, const int *all_done) {
    if (all_off(all_done)) return;
    const int E = (int)*(volatile const unsigned *)epoch;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int r = (int)(gt & 7);
    const unsigned octet = 0xFFu << (threadIdx.x & 24);
    for (int64_t t = gt >> 3; t < lvl1; t += ((int64_t)gridDim.x * blockDim.x) >> 3) {
        const int row = T.task_row[t];
        double v = a.p[bidx(a, row) * kB + r];
        if (c) v = __dadd_rn(v, c[(int64_t)row * kB + r]);
        if (MODE & 2) v = __ddiv_rn(v, T.diag[t]);
        x[(int64_t)row * kB + r] = v;
        __syncwarp(octet);
        if (r == 0) {
            __threadfence();
            st_flag_release(flag + row, E);
        }
    }
}

__global__ void kb_bump(unsigned *epoch) { *epoch += 1u; }

using BtKernel = void (*)(TriDev, VecIn, const double *, double *, int *, const unsigned *, int, int, const int *);

template <int MODE>
BtKernel bt_kernel(int n, bool tail) {
    if (n <= 4) return tail ? kb_trsv<MODE, 4, true> : kb_trsv<MODE, 4, false>;
    return tail ? kb_trsv<MODE, 8, true> : kb_trsv<MODE, 8, false>;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int bpost(rsb_ctx *ctx) {
    ctx->launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("kernel launch failed: %s", cudaGetErrorString(e));
        return RSB_ECUDA;
    }
    return RSB_OK;
}

int launch_bspmv(rsb_ctx *ctx, const Compressed &A, VecIn x, double *y, int epi, VecIn e, const int *all_done) {
    if (A.nlines == 0) return RSB_OK;
    const int grid = (int)((A.nlines * kB + kBlk - 1) / kBlk);
    switch (epi) {
        case EPI_ADD: kb_spmv_rows<EPI_ADD><<<grid, kBlk, 0, ctx->stream>>>(A, x, y, e, all_done); break;
        case EPI_SUB_FROM: kb_spmv_rows<EPI_SUB_FROM><<<grid, kBlk, 0, ctx->stream>>>(A, x, y, e, all_done); break;
        default: kb_spmv_rows<EPI_STORE><<<grid, kBlk, 0, ctx->stream>>>(A, x, y, e, all_done); break;
    }
    return bpost(ctx);
}

int launch_bspmv_t(rsb_ctx *ctx, const Compressed &At, VecIn y, double *z, int epi, VecIn e, const int *all_done) {
    if (At.nlines == 0) return RSB_OK;
    const int grid = (int)((At.nlines + kBTile - 1) / kBTile);
    const char *er = getenv("RSB_BTILE_ROUNDS");  // experiments
    const int rounds = er ? atoi(er) : kBTileRounds;
    if (rounds == 4) {
        if (epi == EPI_ADD)
            kb_spmv_tile<true, EPI_ADD, 4><<<grid, kBlk, 0, ctx->stream>>>(At, y, z, e, all_done);
        else
            kb_spmv_tile<true, EPI_STORE, 4><<<grid, kBlk, 0, ctx->stream>>>(At, y, z, e, all_done);
    } else if (rounds == 2) {
        if (epi == EPI_ADD)
            kb_spmv_tile<true, EPI_ADD, 2><<<grid, kBlk, 0, ctx->stream>>>(At, y, z, e, all_done);
        else
            kb_spmv_tile<true, EPI_STORE, 2><<<grid, kBlk, 0, ctx->stream>>>(At, y, z, e, all_done);
    } else if (epi == EPI_ADD)
        kb_spmv_tile<true, EPI_ADD, 1><<<grid, kBlk, 0, ctx->stream>>>(At, y, z, e, all_done);
    else
        kb_spmv_tile<true, EPI_STORE, 1><<<grid, kBlk, 0, ctx->stream>>>(At, y, z, e, all_done);
    return bpost(ctx);
}

int launch_bdot(rsb_ctx *ctx, BDotRing &ring, int64_t n, VecIn a, VecIn b, double *out, int ostride, int sqrt_out,
                const int *all_done, const int *need, int nstride) {
    const int T = (ctx->blas_threads > 1 && n > 10000) ? ctx->blas_threads : 1;
    BDotChunks ch{T, nullptr, nullptr};
    if (T > 1) {
        const int slot = (int)(ring.next++ % kDotSlots);
        ch.part = ring.part + (size_t)slot * kMaxBlasThreads * kB;
        ch.cnt = ring.cnt + slot;
    }
    static const bool staged = !(getenv("RSB_BDOT_STAGED") && atoi(getenv("RSB_BDOT_STAGED")) == 0);
    if (staged && !a.g && !b.g && a.off == 0 && b.off == 0) {
        constexpr size_t smem = (size_t)kBDotStages * 2 * kBDotRows * kB * sizeof(double);
        static bool attr = false;
        if (!attr) {
            RSB_TRY_CUDA(cudaFuncSetAttribute(kb_dot_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = true;
        }
        kb_dot_staged<<<T, kBlk, smem, ctx->stream>>>(n, a.p, b.p, out, ostride, sqrt_out, all_done, need, nstride, ch);
        return bpost(ctx);
    }
    kb_dot<<<T, kBlk, 0, ctx->stream>>>(n, a, b, out, ostride, sqrt_out, all_done, need, nstride, ch);
    return bpost(ctx);
}

int launch_baxpy(rsb_ctx *ctx, double *y, const double *x, const double *scal, int sstride, int sign, int64_t n,
                 BGate g) {
    if (sign > 0)
        kb_axpy<1><<<grid_stride_n(n * kB), kBlk, 0, ctx->stream>>>(y, x, scal, sstride, n, g);
    else
        kb_axpy<-1><<<grid_stride_n(n * kB), kBlk, 0, ctx->stream>>>(y, x, scal, sstride, n, g);
    return bpost(ctx);
}

int launch_bxpby(rsb_ctx *ctx, double *p, const double *h, const double *beta, int bstride, const int *copy_flag,
                 int cstride, int64_t n, BGate g) {
    kb_xpby<<<grid_stride_n(n * kB), kBlk, 0, ctx->stream>>>(p, h, beta, bstride, copy_flag, cstride, n, g);
    return bpost(ctx);
}

int launch_bcopy(rsb_ctx *ctx, double *dst, VecIn src, int64_t n, BGate g) {
    kb_copy<<<grid_stride_n(n * kB), kBlk, 0, ctx->stream>>>(dst, src, n, g);
    return bpost(ctx);
}

int launch_bfill(rsb_ctx *ctx, double *x, int64_t n, double v) {
    kb_fill<<<grid_stride_n(n * kB), kBlk, 0, ctx->stream>>>(x, n, v);
    return bpost(ctx);
}

int launch_bcg_init(rsb_ctx *ctx, double *w, double *r, double *p, const double *u, int64_t s, BGate g) {
    kb_cg_init<<<grid_stride_n(s * kB), kBlk, 0, ctx->stream>>>(w, r, p, u, s, g);
    return bpost(ctx);
}

int launch_bpack(rsb_ctx *ctx, double *dst, const double *src, int64_t len, int k) {
    kb_pack<<<grid_stride_n(len * kB), kBlk, 0, ctx->stream>>>(dst, src, len, k);
    return bpost(ctx);
}

int launch_bunpack(rsb_ctx *ctx, double *dst, const double *src, int64_t len, int k) {
    kb_unpack<<<grid_stride_n(len * k), kBlk, 0, ctx->stream>>>(dst, src, len, k);
    return bpost(ctx);
}

bool btrsv_supported(const TriSched &T) { return T.wide && T.max_task < (1 << 20); }

int launch_btrsv(rsb_ctx *ctx, const TriSched &T, VecIn a, const double *c, double *x, BTriWs &ws,
                 const int *all_done) {
    if (T.n == 0) return RSB_OK;
    if (!btrsv_supported(T)) {
        set_error("batched triangular solve needs a wide (grid) schedule");
        return RSB_ESTATE;
    }
    const bool trace = ctx->tracing && ctx->trace_n + 2 <= 64;
    if (trace)
        RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->trace_ev[ctx->trace_n++], ctx->stream, cudaEventRecordExternal));
    TriDev v = T.view();
    v.ticket = ws.ticket;
    kb_bump<<<1, 1, 0, ctx->stream>>>(ws.epoch);
    RSB_TRY(bpost(ctx));
    RSB_TRY_CUDA(cudaMemsetAsync(ws.ticket, 0, sizeof(unsigned long long), ctx->stream));
    if (btrsv_nat_supported(T)) {
        RSB_TRY(launch_btrsv_nat(ctx, T, a, c, x, ws, all_done));
        if (trace)
            RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->trace_ev[ctx->trace_n++], ctx->stream, cudaEventRecordExternal));
        return RSB_OK;
    }
    const int32_t lvl1 = T.h_level_ptr.size() > 1 ? T.h_level_ptr[1] : T.n;
    if (lvl1 > 0) {
        const int g0 = grid_stride_n((int64_t)lvl1 * kB);
        switch (T.mode & 3) {
            case 0: kb_trsv_level0<0><<<g0, kBlk, 0, ctx->stream>>>(v, a, c, x, ws.flag, ws.epoch, lvl1, all_done); break;
            case 1: kb_trsv_level0<1><<<g0, kBlk, 0, ctx->stream>>>(v, a, c, x, ws.flag, ws.epoch, lvl1, all_done); break;
            case 2: kb_trsv_level0<2><<<g0, kBlk, 0, ctx->stream>>>(v, a, c, x, ws.flag, ws.epoch, lvl1, all_done); break;
            default: kb_trsv_level0<3><<<g0, kBlk, 0, ctx->stream>>>(v, a, c, x, ws.flag, ws.epoch, lvl1, all_done); break;
        }
        RSB_TRY(bpost(ctx));
    }
    const int nslices = (T.n + 31) / 32;
    const int first_slice = lvl1 / 32;
    const char *gvs = getenv("RSB_TRSV_GRID");
    // the static-schedule variant is opt-in here (RSB_TRSV_GRID=static): with 8
    // right-hand sides per task it measured slower than the ticket kernel
    // (L1 at n = 8e6: 1.76 vs 1.53 ms; 128 registers with spills)
    const bool want_static = gvs && std::strcmp(gvs, "static") == 0;
    if (first_slice < nslices && want_static) {
        const bool tail = T.max_task > 4;
        auto k = (T.mode & 3) == 0 ? (tail ? kb_trsv_static<0, true> : kb_trsv_static<0, false>)
                 : (T.mode & 3) == 1 ? (tail ? kb_trsv_static<1, true> : kb_trsv_static<1, false>)
                 : (T.mode & 3) == 2 ? (tail ? kb_trsv_static<2, true> : kb_trsv_static<2, false>)
                                     : (tail ? kb_trsv_static<3, true> : kb_trsv_static<3, false>);
        static int socc[4][2] = {};
        int &so = socc[T.mode & 3][tail];
        if (so == 0) {
            RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&so, k, kBlk, 0));
            so = std::max(so, 1);
        }
        int sms = 0;
        RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int grid = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)sms * so, ((int64_t)(nslices - first_slice) * 32 + kBlk - 1) / kBlk));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kBlk);
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // round-robin slices: every warp must be resident
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        RSB_TRY_CUDA(cudaLaunchKernelEx(&cfg, k, v, a, c, x, ws.flag, (const unsigned *)ws.epoch, first_slice, nslices,
                                        all_done));
        RSB_TRY(bpost(ctx));
    } else if (first_slice < nslices) {
        const int wn = T.wide_n <= 4 ? 4 : 8;
        const bool tail = T.max_task > wn;
        BtKernel k;
        switch (T.mode & 3) {
            case 0: k = bt_kernel<0>(wn, tail); break;
            case 1: k = bt_kernel<1>(wn, tail); break;
            case 2: k = bt_kernel<2>(wn, tail); break;
            default: k = bt_kernel<3>(wn, tail); break;
        }
        static int occ_cache[4][2][2] = {};
        int &occ = occ_cache[T.mode & 3][wn == 8][tail];
        if (occ == 0) {
            RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBlk, 0));
            occ = std::max(occ, 1);
        }
        int sms = 0;
        RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int grid = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)sms * occ, ((int64_t)(nslices - first_slice) * 32 + kBlk - 1) / kBlk));
        k<<<grid, kBlk, 0, ctx->stream>>>(v, a, c, x, ws.flag, ws.epoch, first_slice, nslices, all_done);
        RSB_TRY(bpost(ctx));
    }
    if (trace)
        RSB_TRY_CUDA(cudaEventRecordWithFlags(ctx->trace_ev[ctx->trace_n++], ctx->stream, cudaEventRecordExternal));
    return RSB_OK;
}

}  // namespace rsb
