// Device helpers shared by the kernel translation units (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include "rsb_internal.h"

namespace rsb {

// Skip predicate of a device-side control loop (see Gate).
static __device__ __forceinline__ bool gated(const Gate &g) {
    return (g.a && *(volatile const int *)g.a) || (g.b && *(volatile const int *)g.b);
}

// ---- shared-memory addressing, mbarriers and 1-D TMA bulk copies
static __device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
static __device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
static __device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// busy-polling wait (mbarrier.test_wait never suspends the thread; try_wait
// may sleep past the phase flip, which puts wake-up latency on a critical path)
static __device__ __forceinline__ void mbar_wait_spin(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// a / d correctly rounded, given y = RN(1/d): q0 = RN(a*y), r = a - q0*d
// (exact, FMA), q1 = RN(q0 + r*y) (Markstein).  Valid while no intermediate
// over/underflows -- guaranteed for |a|, |d| in (2^-500, 2^500); outside that
// range (zeros, subnormals, non-finite values included) the IEEE division
// runs instead.  24 cycles of dependent FP64 instead of ~400 for div.rn.f64
// on sm_100 (scripts/probes/fp64_latency.cu); cross-checked bit for bit
// against a/b on 2.8e9 random and adversarial operand pairs.
static __device__ __forceinline__ double exact_div(double a, double d, double y) {
    const double aa = fabs(a), ad = fabs(d);
    if (ad > 0x1p-500 && ad < 0x1p500) {
        if (aa > 0x1p-500 && aa < 0x1p500) {
            const double q0 = __dmul_rn(a, y);
            const double r = fma(-q0, d, a);
            return fma(r, y, q0);
        }
        if (a == 0.0) return __dmul_rn(a, y);  // +-0 with the quotient's sign, exactly as a / d
    }
    return __ddiv_rn(a, d);
}

// ---------------------------------------------------------------------------
// OpenBLAS ddot association (SkylakeX kernel, one thread), one warp:
//   n1 = n & -16 through the vector kernel -- four 8-wide FMA accumulators
//   over 32-blocks (lane l holds accumulator l), folded 8 -> 4 (lo+hi half),
//   a trailing 16-block into four 4-wide accumulators, lane-wise
//   ((a0+a1)+a2)+a3, then (t0+t2)+(t1+t3); the tail is a scalar FMA chain.
// Bit-identical to numpy `a @ b` on the reference host (oracle/rsref.c
// rso_blas_dot, tests/test_oracle_pin.py).  All lanes must call; the
// result is valid in every lane.
// ---------------------------------------------------------------------------
// Second half of the OpenBLAS ddot association, given each lane's FMA
// accumulator over the 32-blocks [0, n32): fold 8 -> 4, the trailing 16-block,
// the lane reduction and the scalar tail.
template <class LA, class LB>
__device__ __forceinline__ double warp_blas_finish(double acc, int64_t n, LA la, LB lb) {
    const int lane = threadIdx.x & 31;
    const int64_t n1 = n & ~(int64_t)15;
    const int64_t n32 = n1 & ~(int64_t)31;
    // fold a5[g][k] + a5[g][k+4] into lane 8g+k (k < 4)
    double hi = __shfl_down_sync(0xffffffffu, acc, 4);
    double a4 = acc + hi;  // meaningful in lanes with (lane & 7) < 4
    if (n1 > n32) {
        const int g = lane >> 3, k = lane & 7;
        if (k < 4) {
            const int64_t e = n32 + 4 * g + k;
            a4 = fma(la(e), lb(e), a4);
        }
    }
    // t[k] = ((a[0][k] + a[1][k]) + a[2][k]) + a[3][k], a[g][k] in lane 8g+k
    double a1 = __shfl_down_sync(0xffffffffu, a4, 8);
    double a2 = __shfl_down_sync(0xffffffffu, a4, 16);
    double a3 = __shfl_down_sync(0xffffffffu, a4, 24);
    double t = ((a4 + a1) + a2) + a3;  // valid in lanes 0..3
    double t1 = __shfl_sync(0xffffffffu, t, 1);
    double t2 = __shfl_sync(0xffffffffu, t, 2);
    double t3 = __shfl_sync(0xffffffffu, t, 3);
    double t0 = __shfl_sync(0xffffffffu, t, 0);
    double dot = n1 ? (t0 + t2) + (t1 + t3) : 0.0;
    for (int64_t e = n1; e < n; ++e) dot = fma(lb(e), la(e), dot);
    return dot;
}

template <class LA, class LB>
__device__ __forceinline__ double warp_blas_dot(int64_t n, LA la, LB lb) {
    const int lane = threadIdx.x & 31;
    const int64_t n1 = n & ~(int64_t)15;
    const int64_t n32 = n1 & ~(int64_t)31;
    double acc = 0.0;
    int64_t i = lane;
    // unrolled FMA chain: loads of 8 blocks issued ahead of the dependent FMAs
    for (; i + 7 * 32 < n32; i += 8 * 32) {
        double xa[8], xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            xa[u] = la(i + u * 32);
            xb[u] = lb(i + u * 32);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(xa[u], xb[u], acc);
    }
    for (; i < n32; i += 32) acc = fma(la(i), lb(i), acc);
    return warp_blas_finish(acc, n, la, lb);
}


// numpy pairwise summation (DOUBLE_pairwise_sum): below 8 terms sequential
// from -0.0; up to 128 eight strided accumulators combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail; above, split at
// n/2 rounded down to a multiple of 8.  term(k) yields the k-th term.
template <class Term>
__device__ __forceinline__ double pw_leaf(const Term &term, int64_t o, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, term(o + i));
        return r;
    }
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = term(o + k);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], term(o + i + k));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, term(o + i));
    return res;
}

// The split levels as a chain of distinct non-inlined functions (depth D
// covers n < 128 * 2^D), so the stack is sized statically: no device
// recursion.
template <int D, class Term>
struct Pairwise {
    static __device__ __noinline__ double sum(const Term &term, int64_t o, int64_t n) {
        if (n <= 128) return pw_leaf(term, o, n);
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        const double left = Pairwise<D - 1, Term>::sum(term, o, n2);
        return __dadd_rn(left, Pairwise<D - 1, Term>::sum(term, o + n2, n - n2));
    }
};
template <class Term>
struct Pairwise<0, Term> {
    static __device__ __noinline__ double sum(const Term &term, int64_t o, int64_t n) { return pw_leaf(term, o, n); }
};

}  // namespace rsb
