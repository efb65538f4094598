// Split exact-dot probe: 4 CTAs x 8 FMA chains (chains c0..c0+7 of the
// OpenBLAS 32-chain order); warps 1-3 copy the CTA's columns of a and b into
// a 4-stage ring of 256-step chunks with cp.async, warp 0 runs the chains.
// Variants:
//   copy   8: 8-byte cp.async.ca into {a, b} pairs per chain
//         16: 16-byte cp.async.cg into [a chains][b chains] per step
//   chain  0: waits/arrivals only (measures the copy)
//          1: register operands only (the DFMA floor)
//          2: smem operands, 16-step blocks, loads 8 steps ahead, chunk wait
//             hoisted to the chunk start (no barrier inside the inner loop)
//          4: copy 16 layout, a lane runs two chains: two LDS.128 + two DFMA per step
//          3: as 2, but the next block's loads are fenced off from the
//             current block's FMAs by a __syncwarp (ptxas otherwise sinks
//             the loads next to their consumers)
// Reports kernel time and the chain warp's cycles per step.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ds dot_split.cu && /tmp/ds
#include <cstdio>
#include <cuda_runtime.h>

constexpr int P = 4, C = 8, K = 256, S = 4, NCOPY = 96, SD = 16;
constexpr size_t SMEM = (size_t)S * K * SD * 8 + 2 * S * 8;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_spin(unsigned long long *bar, unsigned par) {
    asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(su32(bar)), "r"(par) : "memory");
}
__device__ __forceinline__ void wait_try(unsigned long long *bar, unsigned par) {
    asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(su32(bar)), "r"(par) : "memory");
}

template <int COPY, int CHAIN>
__global__ void __launch_bounds__(128) k(long long T, const double *a, const double *b, double *out, long long *cyc) {
    extern __shared__ __align__(16) double ring[];
    unsigned long long *full = (unsigned long long *)(ring + S * K * SD), *empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nch = T / K;  // full chunks only
    const int c0 = blockIdx.x * C;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(NCOPY));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp > 0) {
        if (CHAIN == 1) return;
        const int t = threadIdx.x - 32;
        for (long long c = 0; c < nch; ++c) {
            const int st = (int)(c % S);
            if (c >= S) wait_try(&empty[st], (unsigned)(((c / S) - 1) & 1));
            const long long s0 = c * K;
            double *dst = ring + (size_t)st * K * SD;
            if (COPY == 8) {
                for (int i = t; i < K * SD; i += NCOPY) {
                    const int l = i % C, v = (i / C) & 1, s = i / SD;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst + s * SD + 2 * l + v)),
                                 "l"((v ? b : a) + (s0 + s) * 32 + c0 + l)
                                 : "memory");
                }
            } else {
                for (int i = t; i < K * SD / 2; i += NCOPY) {
                    const int p = i % 8, s = i / 8, v = p / 4, q = p % 4;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + s * SD + v * C + 2 * q)),
                                 "l"((v ? b : a) + (s0 + s) * 32 + c0 + 2 * q)
                                 : "memory");
                }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
        }
        return;
    }
    const int l = lane & (C - 1);
    // operand addresses of step 0 for this lane
    const double *pa = ring + (COPY == 8 ? 2 * l : l), *pb = ring + (COPY == 8 ? 2 * l + 1 : C + l);
    double acc = 0.0;
    const long long t0 = clock64();
    if (CHAIN == 1) {
        double x = 1.0 + lane, y = 0.5;
        for (long long s = 0; s < T; s += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = fma(x + j, y, acc);
        }
    } else {
        wait_spin(&full[0], 0);
        double acc2 = 0.0, za[16], zb[16];
        double wa[16], wb[16], xa[16], ya[16], xb[16], yb[16];
        if (CHAIN == 3) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                xa[j] = pa[j * SD];
                ya[j] = pb[j * SD];
            }
        }
        if (CHAIN == 4) {
            const double2 *pp = reinterpret_cast<const double2 *>(ring) + (lane & 3);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double2 u = pp[j * 8], w = pp[j * 8 + 4];
                wa[j] = u.x, za[j] = u.y, wb[j] = w.x, zb[j] = w.y;
            }
        }
        if (CHAIN == 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                wa[j] = pa[j * SD];
                wb[j] = pb[j * SD];
            }
        }
        for (long long c = 0; c < nch; ++c) {
            if (c + 1 < nch) wait_spin(&full[(c + 1) % S], (unsigned)(((c + 1) / S) & 1));
            if (CHAIN == 2) {
                const int base = (int)((c % S) * K);
                const double2 *pp = reinterpret_cast<const double2 *>(ring) + l;
                for (int blk = 0; blk < K; blk += 16) {
                    const int r0 = base + blk, r1 = (r0 + 16) & (S * K - 1);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (COPY == 8) {
                            const double2 v = pp[(r0 + 8 + j) * (SD / 2)];
                            wa[8 + j] = v.x;
                            wb[8 + j] = v.y;
                        } else {
                            wa[8 + j] = pa[(r0 + 8 + j) * SD];
                            wb[8 + j] = pb[(r0 + 8 + j) * SD];
                        }
                        acc = fma(wa[j], wb[j], acc);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (COPY == 8) {
                            const double2 v = pp[(r1 + j) * (SD / 2)];
                            wa[j] = v.x;
                            wb[j] = v.y;
                        } else {
                            wa[j] = pa[(r1 + j) * SD];
                            wb[j] = pb[(r1 + j) * SD];
                        }
                        acc = fma(wa[8 + j], wb[8 + j], acc);
                    }
                }
            }
            if (CHAIN == 4) {
                const int base = (int)((c % S) * K);
                const double2 *pp = reinterpret_cast<const double2 *>(ring) + (lane & 3);
                for (int blk = 0; blk < K; blk += 16) {
                    const int r0 = base + blk, r1 = (r0 + 16) & (S * K - 1);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const double2 u = pp[(r0 + 8 + j) * 8], w = pp[(r0 + 8 + j) * 8 + 4];
                        wa[8 + j] = u.x, za[8 + j] = u.y, wb[8 + j] = w.x, zb[8 + j] = w.y;
                        acc = fma(wa[j], wb[j], acc);
                        acc2 = fma(za[j], zb[j], acc2);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const double2 u = pp[(r1 + j) * 8], w = pp[(r1 + j) * 8 + 4];
                        wa[j] = u.x, za[j] = u.y, wb[j] = w.x, zb[j] = w.y;
                        acc = fma(wa[8 + j], wb[8 + j], acc);
                        acc2 = fma(za[8 + j], zb[8 + j], acc2);
                    }
                }
            }
            if (CHAIN == 3) {
                const int base = (int)((c % S) * K);
                const double2 *pp = reinterpret_cast<const double2 *>(ring) + l;
                for (int blk = 0; blk < K; blk += 32) {
                    const int r1 = base + blk + 16, r2 = (base + blk + 32) & (S * K - 1);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (COPY == 8) {
                            const double2 v = pp[(r1 + j) * (SD / 2)];
                            xb[j] = v.x;
                            yb[j] = v.y;
                        } else {
                            xb[j] = pa[(r1 + j) * SD];
                            yb[j] = pb[(r1 + j) * SD];
                        }
                    }
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc = fma(xa[j], ya[j], acc);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (COPY == 8) {
                            const double2 v = pp[(r2 + j) * (SD / 2)];
                            xa[j] = v.x;
                            ya[j] = v.y;
                        } else {
                            xa[j] = pa[(r2 + j) * SD];
                            ya[j] = pb[(r2 + j) * SD];
                        }
                    }
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc = fma(xb[j], yb[j], acc);
                }
            }
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[c % S])) : "memory");
        }
        acc += acc2;
    }
    const long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = acc;
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int COPY, int CHAIN>
void run(long long n, double *a, double *b, double *o, long long *c) {
    const long long T = n / 32;
    cudaFuncSetAttribute(k<COPY, CHAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    long long h[P];
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k<COPY, CHAIN><<<P, 128, SMEM>>>(T, a, b, o, c);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, c, 8 * P, cudaMemcpyDeviceToHost);
    printf("copy%-2d chain%d n=%lld: %7.1f us, %.2f cycles/step\n", COPY, CHAIN, n, ms * 1e3, h[0] / (double)T);
}

int main() {
    const long long n = 1 << 20;
    double *a, *b, *o;
    long long *c;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    cudaMemset(b, 0, n * 8);
    cudaMalloc(&o, 8 * 32 * P);
    cudaMalloc(&c, 8 * P);
    run<8, 1>(n, a, b, o, c);
    run<8, 0>(n, a, b, o, c);
    run<16, 0>(n, a, b, o, c);
    run<8, 2>(n, a, b, o, c);
    run<16, 2>(n, a, b, o, c);
    run<16, 4>(n, a, b, o, c);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
