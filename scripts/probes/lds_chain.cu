// Cost of shared-memory operand loads interleaved with one lane-group's
// dependent DFMA chain (data resident in shared memory, loads 8 steps
// ahead, 16-step unrolled blocks).  Variant v:
//   0: no loads (register operands)        1: one LDS.64 per step
//   2: one LDS.128 per step ({a, b} pair)  3: two LDS.64 per step
//   4: one LDS.128 per two steps ({a_s, a_s+1}; b from registers)
//   5: two chains per lane: two LDS.128 ({a_2m, a_2m+1}, {b_2m, b_2m+1}) and two DFMAs per step
// active lanes: all 32 with 8 distinct addresses (lanes l, l+8, ... share)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lc lds_chain.cu && /tmp/lc
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(int steps, double *out, long long *cyc) {
    __shared__ double2 sm[2048];
    const int lane = threadIdx.x, l = lane & 7;
    for (int i = lane; i < 2048; i += 32) sm[i] = make_double2(1.0 + 1e-9 * i, 1.0 - 1e-9 * i);
    __syncwarp();
    const double2 *p = sm + l;
    const double *q = reinterpret_cast<const double *>(sm) + l;
    double acc = 0.0, acc2 = 0.0, cb = 0.75;
    double ya[16], yb[16];
    double xa[16], xb[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) xa[j] = xb[j] = ya[j] = yb[j] = 1.0 + j;
    const long long t0 = clock64();
    for (int s = 0; s < steps; s += 16) {
        const int r0 = (s * 8) & 2047 & ~127, r1 = ((s + 16) * 8) & 2047 & ~127;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int slot = (j + 8) & 15;
            const int r = (j < 8 ? r0 + (8 + j) * 8 : r1 + (j - 8) * 8);
            if (V == 1) xa[slot] = q[2 * r];
            if (V == 2) {
                const double2 v = p[r];
                xa[slot] = v.x;
                xb[slot] = v.y;
            }
            if (V == 3) {
                xa[slot] = q[2 * r];
                xb[slot] = q[2 * r + 1];
            }
            if (V == 4 && (j & 1) == 0) {
                const double2 v = p[r];
                xa[slot] = v.x;
                xa[slot + 1] = v.y;
            }
            if (V == 5) {
                const double2 u = p[2 * r], w = p[2 * r + 1];
                xa[slot] = u.x;
                ya[slot] = u.y;
                xb[slot] = w.x;
                yb[slot] = w.y;
                acc2 = fma(ya[j], yb[j], acc2);
            }
            acc = fma(xa[j], (V == 1 || V == 4) ? cb : xb[j], acc);
        }
    }
    const long long t1 = clock64();
    out[lane] = acc + acc2;
    if (lane == 0) cyc[0] = t1 - t0;
}

template <int V>
void run(double *o, long long *c) {
    long long h;
    const int steps = 1 << 16;
    k<V><<<1, 32>>>(steps, o, c);
    k<V><<<1, 32>>>(steps, o, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("v%d: %.2f cycles/step\n", V, h / (double)steps);
}

int main() {
    double *o;
    long long *c;
    cudaMalloc(&o, 256);
    cudaMalloc(&c, 8);
    run<0>(o, c);
    run<1>(o, c);
    run<2>(o, c);
    run<3>(o, c);
    run<4>(o, c);
    run<5>(o, c);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
