// Per-level cost of minimal level-synchronous skeletons on one CTA of 128
// threads, 2048 levels, one task per level on thread 0..w-1 (w = 32).
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(double *out, long long *cyc, const int *lvlg, int nlev) {
    __shared__ double ring[4096];
    __shared__ int lvl[2056];
    for (int i = threadIdx.x; i <= nlev; i += blockDim.x) lvl[i] = lvlg[i];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) ring[i] = 1.0 + i;
    __syncthreads();
    long long t0 = clock64();
    double acc = 0.5;
    for (int l = 0; l < nlev; ++l) {
        const int lo = lvl[l], hi = lvl[l + 1];
        const int t = lo + threadIdx.x;
        if (t < hi) {
            double a = ring[(t - 32) & 4095];                      // one dependency from the previous level
            if (V >= 1) a = ring[(t - 31) & 4095] - a * 0.5;        // two deps
            if (V >= 2) { for (int q = 0; q < 4; ++q) a = a - ring[(t - 33 - q) & 4095] * 0.25; }
            ring[t & 4095] = a + acc;
            if (V >= 3) out[t & 1023] = a;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { cyc[V] = clock64() - t0; out[0] += acc; }
}
int main() {
    const int nlev = 2048;
    int *hl = new int[nlev + 1]; for (int i = 0; i <= nlev; ++i) hl[i] = 32 * i;
    int *dl; double *o; long long *c, h[4];
    cudaMalloc(&dl, 4 * (nlev + 1)); cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 32);
    cudaMemcpy(dl, hl, 4 * (nlev + 1), cudaMemcpyHostToDevice);
    for (int r = 0; r < 2; ++r) { k<0><<<1, 128>>>(o, c, dl, nlev); k<1><<<1, 128>>>(o, c, dl, nlev); k<2><<<1, 128>>>(o, c, dl, nlev); k<3><<<1, 128>>>(o, c, dl, nlev); }
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("{\"cycles_per_level\": [%.1f, %.1f, %.1f, %.1f]}\n", h[0] / (double)nlev, h[1] / (double)nlev, h[2] / (double)nlev, h[3] / (double)nlev);
    return 0;
}
