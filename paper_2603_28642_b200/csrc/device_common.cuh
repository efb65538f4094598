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

}  // namespace rsb
