// FP64 dependent-chain latency and independent-op throughput as a function
// of active lanes (one warp on one SM).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/fpw fp64_warp.cu && /tmp/fpw
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double *out, long long *cyc, int active, int iters) {
    const int lane = threadIdx.x;
    if (lane >= active) return;
    double a = 1.0 + lane * 1e-3, b = 1e-9, c0 = 0.5, c1 = 0.25, c2 = 0.125, c3 = 0.0625;
    const long long t0 = clock64();
    if (MODE == 0) {  // dependent DADD chain
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j) a = __dadd_rn(a, b);
        }
    } else {  // 4 independent DMUL chains (throughput)
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                c0 = __dmul_rn(c0, 1.0000001);
                c1 = __dmul_rn(c1, 1.0000001);
                c2 = __dmul_rn(c2, 1.0000001);
                c3 = __dmul_rn(c3, 1.0000001);
            }
        }
    }
    const long long t1 = clock64();
    out[lane] = a + c0 + c1 + c2 + c3;
    if (lane == 0) cyc[0] = t1 - t0;
}

int main() {
    double *o;
    long long *c, h;
    cudaMalloc(&o, 32 * 8);
    cudaMalloc(&c, 8);
    const int iters = 4096;
    printf("{");
    for (int mode = 0; mode < 2; ++mode)
        for (int act : {1, 4, 8, 16, 32}) {
            for (int r = 0; r < 2; ++r) {
                if (mode == 0) k<0><<<1, 32>>>(o, c, act, iters);
                else k<1><<<1, 32>>>(o, c, act, iters);
            }
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("\"%s_lanes%d\": %.2f, ", mode == 0 ? "dadd_chain_cyc_per_op" : "dmul_4chains_cyc_per_op", act,
                   h / (double)(iters * 16));
        }
    printf("\"ok\": 1}\n");
    return 0;
}
