// Cycles per step of one lane's FMA chain fed from shared memory, as in the
// exact dot kernels: 8 lanes (or 32) each run a dependent DFMA chain over
// operands read with LDS.64, loads issued G steps ahead.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fcs fma_chain_smem.cu && /tmp/fcs
#include <cstdio>
#include <cuda_runtime.h>

template <int G, int STRIDE>
__global__ void k(double *out, long long *cyc, int steps, int active) {
    __shared__ double sa[2048], sb[2048];
    const int lane = threadIdx.x;
    for (int i = lane; i < 2048; i += 32) {
        sa[i] = 1.0 + 1e-9 * i;
        sb[i] = 1.0 - 1e-9 * i;
    }
    __syncwarp();
    double acc = 0.0;
    const long long t0 = clock64();
    if (lane < active) {
        const double *pa = sa + lane, *pb = sb + lane;
        double ra[G], rb[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            ra[j] = pa[STRIDE * j];
            rb[j] = pb[STRIDE * j];
        }
        for (int s = 0; s < steps; s += G) {
            double na[G], nb[G];
            const int base = ((s + G) * STRIDE) & 2047 & ~31;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                na[j] = pa[(base + STRIDE * j) & 2015];
                nb[j] = pb[(base + STRIDE * j) & 2015];
            }
#pragma unroll
            for (int j = 0; j < G; ++j) acc = fma(ra[j], rb[j], acc);
#pragma unroll
            for (int j = 0; j < G; ++j) {
                ra[j] = na[j];
                rb[j] = nb[j];
            }
        }
    }
    const long long t1 = clock64();
    out[lane] = acc;
    if (lane == 0) cyc[0] = t1 - t0;
}

int main() {
    double *o;
    long long *c, h;
    cudaMalloc(&o, 256);
    cudaMalloc(&c, 8);
    const int steps = 1 << 16;
    printf("{");
    for (int act : {8, 32}) {
        k<8, 8><<<1, 32>>>(o, c, steps, act);
        k<8, 8><<<1, 32>>>(o, c, steps, act);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("\"G8_stride8_active%d\": %.2f, ", act, h / (double)steps);
        k<16, 8><<<1, 32>>>(o, c, steps, act);
        k<16, 8><<<1, 32>>>(o, c, steps, act);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("\"G16_stride8_active%d\": %.2f, ", act, h / (double)steps);
        k<8, 32><<<1, 32>>>(o, c, steps, act);
        k<8, 32><<<1, 32>>>(o, c, steps, act);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("\"G8_stride32_active%d\": %.2f, ", act, h / (double)steps);
    }
    printf("\"ok\": 1}\n");
    return 0;
}
