// Single-CTA TMA ingest rate: one warp streams `total` bytes from global
// memory through `stages` shared-memory buffers of `chunk` bytes, each buffer
// filled by `split` 1-D bulk copies completing on one mbarrier.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma tma_ingest.cu && /tmp/tma
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const char *src, long long total, int chunk, int stages, int split, int fence, long long *cyc,
                  double *sink) {
    const int lanes_issue = 0;
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm + (size_t)stages * chunk);
    const int lane = threadIdx.x;
    if (lane == 0)
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long nch = total / chunk;
    auto issue = [&](long long c) {
        const int s = (int)(c % stages);
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk));
        __syncwarp();
        const int part = chunk / split;
        for (int p = 0; p < split; ++p)
            if (lanes_issue ? (lane == p) : (lane == 0)) {
                if (fence)
                    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     su32(sm + (size_t)s * chunk + p * part)),
                                 "l"(src + c * chunk + p * part), "r"(part), "r"(su32(&bar[s]))
                                 : "memory");
                else
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     su32(sm + (size_t)s * chunk + p * part)),
                                 "l"(src + c * chunk + p * part), "r"(part), "r"(su32(&bar[s]))
                                 : "memory");
            }
    };
    const long long t0 = clock64();
    for (long long c = 0; c < stages && c < nch; ++c) issue(c);
    double acc = 0.0;
    for (long long c = 0; c < nch; ++c) {
        const int s = (int)(c % stages);
        asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
                         su32(&bar[s])),
                     "r"((unsigned)((c / stages) & 1))
                     : "memory");
        acc += reinterpret_cast<const double *>(sm + (size_t)s * chunk)[lane];
        __syncwarp();
        if (c + stages < nch) {
            issue(c + stages);
        }
    }
    if (lane == 0) *cyc = clock64() - t0;
    sink[lane] = acc;
}

int main() {
    const long long total = 64ll << 20;
    char *src;
    double *sink;
    long long *c, h;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    cudaMalloc(&sink, 256);
    cudaMalloc(&c, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("{");
    bool first = true;
    for (int chunk : {4096, 16384})
        for (int stages : {1, 2, 4})
            for (int split : {1})
                for (int li : {0, 1}) {
                    if ((long long)chunk * stages > 200 * 1024) continue;
                    const size_t smem = (size_t)chunk * stages + 64;
                    for (int r = 0; r < 2; ++r) k<<<1, 32, smem>>>(src, total, chunk, stages, split, li, c, sink);
                    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
                    printf("%s\"c%d_s%d_x%d_%s\": %.1f", first ? "" : ", ", chunk, stages, split, li ? "cta" : "cluster",
                           total / (double)h);
                    first = false;
                }
    printf("}\n");
    cudaError_t e = cudaDeviceSynchronize();
    fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return 0;
}
