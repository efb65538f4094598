// Dependent-chain latency of FP64 ops and shared-memory loads on this GPU
// (clock64 around 4096-long chains, one thread).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
    __syncthreads();
    if (threadIdx.x) return;
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < 4096; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    for (int i = 0; i < 4096; ++i) x = __dadd_rn(x, b);
    long long t2 = clock64();
    for (int i = 0; i < 4096; ++i) x = __dmul_rn(x, b);
    long long t3 = clock64();
    int idx = (int)x & 1023;
    for (int i = 0; i < 4096; ++i) idx = ((int)sm[idx] + i) & 1023;  // dependent LDS.64 + convert
    long long t4 = clock64();
    for (int i = 0; i < 1024; ++i) x = __ddiv_rn(x, b + i);
    long long t5 = clock64();
    for (int i = 0; i < 4096; ++i) { double s = x - b; x = (s != 0.0) ? s : x; }
    long long t6 = clock64();
    out[0] = x + idx;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}
int main() {
    double *o; long long *c, h[6];
    cudaMalloc(&o, 8); cudaMalloc(&c, 48);
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
    cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("{\"dfma\": %.2f, \"dadd\": %.2f, \"dmul\": %.2f, \"lds64_f2i_chain\": %.2f, \"ddiv\": %.2f, \"dsub_fsel\": %.2f}\n",
           h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0, h[3] / 4096.0, h[4] / 1024.0, h[5] / 4096.0);
    return 0;
}
