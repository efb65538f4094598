// Per-level cost ladder of the staged single-CTA triangular solve, one
// component at a time (synthetic level sets of 32 tasks x K entries, all
// task data resident in shared memory, 4 consumer warps + 1 idle warp).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/ladder level_ladder.cu && /tmp/ladder
//
// V0  meta LDS -> record LDS -> ring LDS -> fixed-N DSUB chain -> STS -> bar
// V1  V0 + switch on the slice's trip count (16 unrolled chains)
// V2  V1 + exact division (diag pair LDS)
// V3  V2 + global store of the result
// V4  V0 with the next level's meta and records prefetched into registers
// V5  V0 with sources and values in registers from a constant pattern
//     (no record loads: ring LDS -> chain -> STS -> bar)
// V6  V0 without the bar.sync (one warp, __syncwarp)
// V7  pipelined: meta 2 levels ahead, records 1 level ahead, ring loads first, fixed-K chain
// V8  V7 with an if-ladder dispatch on the trip count
// V9  V7 with a fixed 16-step chain
// V10 V7 with the switch dispatch
// V11 V7 + exact division
// V12 V7 with exactly K record and ring loads (no predicated-off loads)
// V13 V12 with the ring loads also predicated on the lane's length
// V14 V7 with loads in groups of 4 under warp-uniform branches, fixed-K chain
// V15 V14 with the chain also in groups of 4 (trip count rounded up to 4)
// V16 V7 with conflict-free (lane-consecutive) ring addresses
// V17 V7 with exactly K ring loads and a 16-step chain (zeros past K)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int K = 6;        // entries per task
constexpr int NLEV = 2048;  // levels (32 tasks each)
constexpr int RING = 4096;
constexpr int CYC = 16;     // task data cycles through CYC levels' worth of storage

struct __align__(16) Rec { double v; int src; int pad; };
struct __align__(16) Meta { int row, len, roff, pad; };

__device__ __forceinline__ double exact_div(double a, double d, double y) {
    const double aa = fabs(a), ad = fabs(d);
    if (ad > 0x1p-500 && ad < 0x1p500) {
        if (aa > 0x1p-500 && aa < 0x1p500) {
            const double q0 = __dmul_rn(a, y);
            const double r = fma(-q0, d, a);
            return fma(r, y, q0);
        }
        if (a == 0.0) return __dmul_rn(a, y);
    }
    return __ddiv_rn(a, d);
}

template <int N>
__device__ __forceinline__ double chain(const Rec *rec, int len, double acc, const double *ring) {
    double v[N], xv[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
        v[q] = 0.0; xv[q] = 0.0;
        if (q < len) { const Rec r = rec[q * 32]; v[q] = r.v; xv[q] = ring[r.src]; }
    }
    double pr[N];
#pragma unroll
    for (int q = 0; q < N; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(v[q], xv[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) acc = __dsub_rn(acc, pr[q]);
    return acc;
}

template <int V>
__global__ void __launch_bounds__(160) k(const Meta *gm, const Rec *gr, const double2 *gdd, double *x,
                                         long long *cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *ring = reinterpret_cast<double *>(sm);
    Meta *meta = reinterpret_cast<Meta *>(ring + RING);           // NLEV*32
    double2 *dd = reinterpret_cast<double2 *>(meta + CYC * 32);
    Rec *rec = reinterpret_cast<Rec *>(dd + CYC * 32);
    int *lvl = reinterpret_cast<int *>(rec + CYC * K * 32);
    const int tid = threadIdx.x;
    for (int i = tid; i < CYC * 32; i += blockDim.x) { meta[i] = gm[i]; dd[i] = gdd[i]; }
    for (int i = tid; i < CYC * K * 32; i += blockDim.x) rec[i] = gr[i];
    for (int i = tid; i <= NLEV; i += blockDim.x) lvl[i] = 32 * i;
    for (int i = tid; i < RING; i += blockDim.x) ring[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    if (tid >= 128) return;
    const long long t0 = clock64();
    if (V == 6 && tid >= 32) return;
    if (V == 4) {
        // prefetch: next level's meta + records in registers
        Meta nm = meta[tid];
        Rec nr[K];
#pragma unroll
        for (int q = 0; q < K; ++q) nr[q] = rec[(nm.roff + q * 32) % (CYC * K * 32)];
        for (int l = 0; l < NLEV; ++l) {
            const int lo = lvl[l], hi = lvl[l + 1];
            const int t = lo + tid;
            const Meta m = nm;
            Rec r[K];
#pragma unroll
            for (int q = 0; q < K; ++q) r[q] = nr[q];
            double acc = 1.0;
            if (t < hi) {
                double xv[K];
#pragma unroll
                for (int q = 0; q < K; ++q) xv[q] = q < m.len ? ring[r[q].src] : 0.0;
                const int tn = hi + tid;
                if (tn < lvl[l + 2 <= NLEV ? l + 2 : NLEV]) {
                    nm = meta[tn & (CYC * 32 - 1)];
#pragma unroll
                    for (int q = 0; q < K; ++q) nr[q] = rec[(nm.roff + q * 32) % (CYC * K * 32)];
                }
                double pr[K];
#pragma unroll
                for (int q = 0; q < K; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(r[q].v, xv[q]) : 0.0;
#pragma unroll
                for (int q = 0; q < K; ++q) acc = __dsub_rn(acc, pr[q]);
                ring[t & (RING - 1)] = acc;
            } else {
                const int tn = hi + tid;
                if (tn < lvl[l + 2 <= NLEV ? l + 2 : NLEV]) {
                    nm = meta[tn & (CYC * 32 - 1)];
#pragma unroll
                    for (int q = 0; q < K; ++q) nr[q] = rec[(nm.roff + q * 32) % (CYC * K * 32)];
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
    } else {
        for (int l = 0; l < NLEV; ++l) {
            const int lo = lvl[l], hi = lvl[l + 1];
            for (int t = lo + tid; t < hi; t += 128) {
                double acc;
                int row;
                if (V == 5) {
                    acc = 1.0;
                    row = t;
                    double xv[K];
#pragma unroll
                    for (int q = 0; q < K; ++q) xv[q] = ring[(t - 32 - 5 * q) & (RING - 1)];
#pragma unroll
                    for (int q = 0; q < K; ++q) acc = __dsub_rn(acc, __dmul_rn(0.125 * (q + 1), xv[q]));
                } else {
                    const Meta m = meta[t & (CYC * 32 - 1)];
                    row = m.row;
                    acc = 1.0;
                    const Rec *rp = rec + (m.roff % (CYC * K * 32));
                    if (V >= 1 && V <= 3) {
                        switch (m.pad) {
                            case 1: acc = chain<1>(rp, m.len, acc, ring); break;
                            case 2: acc = chain<2>(rp, m.len, acc, ring); break;
                            case 3: acc = chain<3>(rp, m.len, acc, ring); break;
                            case 4: acc = chain<4>(rp, m.len, acc, ring); break;
                            case 5: acc = chain<5>(rp, m.len, acc, ring); break;
                            case 6: acc = chain<6>(rp, m.len, acc, ring); break;
                            case 7: acc = chain<7>(rp, m.len, acc, ring); break;
                            case 8: acc = chain<8>(rp, m.len, acc, ring); break;
                            case 9: acc = chain<9>(rp, m.len, acc, ring); break;
                            case 10: acc = chain<10>(rp, m.len, acc, ring); break;
                            case 11: acc = chain<11>(rp, m.len, acc, ring); break;
                            case 12: acc = chain<12>(rp, m.len, acc, ring); break;
                            case 13: acc = chain<13>(rp, m.len, acc, ring); break;
                            case 14: acc = chain<14>(rp, m.len, acc, ring); break;
                            case 15: acc = chain<15>(rp, m.len, acc, ring); break;
                            default: acc = chain<16>(rp, m.len, acc, ring); break;
                        }
                    } else {
                        acc = chain<K>(rp, m.len, acc, ring);
                    }
                    if (V >= 2 && V <= 3) {
                        const double2 d = dd[t & (CYC * 32 - 1)];
                        acc = exact_div(acc, d.x, d.y);
                    }
                }
                ring[t & (RING - 1)] = acc;
                if (V == 3) x[row] = acc;
            }
            if (V == 6) __syncwarp();
            else asm volatile("bar.sync 1, 128;" ::: "memory");
        }
    }
    if (tid == 0) cyc[V] = clock64() - t0;
}


// ---- pipelined variants (V7..V10): meta two levels ahead, records one level
// ahead, ring loads first after the barrier; two task buffers alternate
struct Task { int4 m; double v[16]; int src[16]; };

template <int N>
__device__ __forceinline__ double chain_r(const double (&xv)[16], const double (&v)[16], double acc) {
    double pr[N];
#pragma unroll
    for (int q = 0; q < N; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(v[q], xv[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) acc = __dsub_rn(acc, pr[q]);
    return acc;
}

template <int V>
__global__ void __launch_bounds__(160) kp(const Meta *gm, const Rec *gr, const double2 *gdd, double *x,
                                          long long *cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *ring = reinterpret_cast<double *>(sm);
    Meta *meta = reinterpret_cast<Meta *>(ring + RING);
    double2 *dd = reinterpret_cast<double2 *>(meta + CYC * 32);
    Rec *rec = reinterpret_cast<Rec *>(dd + CYC * 32);
    int *lvl = reinterpret_cast<int *>(rec + CYC * K * 32);
    const int tid = threadIdx.x;
    for (int i = tid; i < CYC * 32; i += blockDim.x) { meta[i] = gm[i]; dd[i] = gdd[i]; }
    for (int i = tid; i < CYC * K * 32; i += blockDim.x) rec[i] = gr[i];
    for (int i = tid; i <= NLEV + 4; i += blockDim.x) lvl[i] = 32 * (i < NLEV ? i : NLEV);
    for (int i = tid; i < RING; i += blockDim.x) ring[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    if (tid >= 128) return;
    const long long t0 = clock64();
    auto meta_of = [&](int t, int hi) -> int4 {
        if (t < hi) { const Meta m = meta[t & (CYC * 32 - 1)]; return make_int4(m.row, m.len, m.roff, m.pad); }
        return make_int4(-2, 0, 0, 0);
    };
    auto load_recs = [&](Task &T) {
        const Rec *rp = rec + (T.m.z % (CYC * K * 32));
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            T.v[q] = 0.0; T.src[q] = 0;
            if (q < T.m.y) { const Rec r = rp[q * 32]; T.v[q] = r.v; T.src[q] = r.src; }
        }
    };
    // records of a task, only as many as the slice needs (groups of 4 under
    // a warp-uniform branch) -- V12+ (V12/V13: exactly K)
    auto load_recs_k = [&](Task &T) {
        const Rec *rp = rec + (T.m.z % (CYC * K * 32));
#pragma unroll
        for (int q = 0; q < 16; ++q) { T.v[q] = 0.0; T.src[q] = 0; }
        if (V == 12 || V == 13) {
#pragma unroll
            for (int q = 0; q < K; ++q) { const Rec r = rp[q * 32]; T.v[q] = r.v; T.src[q] = r.src; }
        } else {
            const int pad = T.m.w;
#pragma unroll
            for (int g4 = 0; g4 < 16; g4 += 4)
                if (pad > g4) {
#pragma unroll
                    for (int q = g4; q < g4 + 4; ++q)
                        if (q < T.m.y) { const Rec r = rp[q * 32]; T.v[q] = r.v; T.src[q] = r.src; }
                }
        }
    };
    Task A, B;
    A.m = meta_of(tid, 32);
    load_recs(A);
    B.m = meta_of(32 + tid, 64);
    int lo = 0;
    auto level = [&](int l, Task &C, Task &Nx) {
        const int hi = lvl[l + 1], hi1 = lvl[l + 2], hi2 = lvl[l + 3];
        double xv[16];
        if (V == 12) {
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = q < K ? ring[C.src[q]] : 0.0;
        } else if (V == 13) {
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = (q < K && q < C.m.y) ? ring[C.src[q]] : 0.0;
        } else if (V == 14 || V == 15) {
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = 0.0;
            const int pad = C.m.w;
#pragma unroll
            for (int g4 = 0; g4 < 16; g4 += 4)
                if (g4 == 0 || pad > g4) {
#pragma unroll
                    for (int q = g4; q < g4 + 4; ++q) xv[q] = q < C.m.y ? ring[C.src[q]] : 0.0;
                }
        } else if (V == 16) {  // conflict-free ring addresses (lane-consecutive)
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = q < C.m.y ? ring[(tid & 31) + 32 * q + (C.src[q] & 0) ] : 0.0;
        } else if (V == 17) {  // exactly K loads, 16-step chain
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = q < K ? ring[C.src[q]] : 0.0;
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) xv[q] = q < C.m.y ? ring[C.src[q]] : 0.0;
        }
        if (V >= 12 && V <= 15) load_recs_k(Nx);
        else load_recs(Nx);
        const int4 mm = meta_of(hi1 + tid, hi2);
        if (C.m.x != -2) {
            double acc = 1.0;
            const int pad = C.m.w;
            if (V == 7 || V == 11 || V == 12 || V == 13 || V == 14 || V == 16) {
                acc = chain_r<K>(xv, C.v, acc);
            } else if (V == 15) {
                // chain in groups of 4 under warp-uniform branches
                double pr[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(C.v[q], xv[q]) : 0.0;
#pragma unroll
                for (int g4 = 0; g4 < 16; g4 += 4)
                    if (g4 == 0 || pad > g4) {
#pragma unroll
                        for (int q = g4; q < g4 + 4; ++q) acc = __dsub_rn(acc, pr[q]);
                    }
            } else if (V == 8) {
                if (pad <= 2) acc = chain_r<2>(xv, C.v, acc);
                else if (pad <= 4) acc = chain_r<4>(xv, C.v, acc);
                else if (pad <= 6) acc = chain_r<6>(xv, C.v, acc);
                else if (pad <= 8) acc = chain_r<8>(xv, C.v, acc);
                else if (pad <= 12) acc = chain_r<12>(xv, C.v, acc);
                else acc = chain_r<16>(xv, C.v, acc);
            } else if (V == 9 || V == 17) {
                acc = chain_r<16>(xv, C.v, acc);
            } else {
                switch (pad) {
                    case 1: acc = chain_r<1>(xv, C.v, acc); break;
                    case 2: acc = chain_r<2>(xv, C.v, acc); break;
                    case 3: acc = chain_r<3>(xv, C.v, acc); break;
                    case 4: acc = chain_r<4>(xv, C.v, acc); break;
                    case 5: acc = chain_r<5>(xv, C.v, acc); break;
                    case 6: acc = chain_r<6>(xv, C.v, acc); break;
                    case 7: acc = chain_r<7>(xv, C.v, acc); break;
                    case 8: acc = chain_r<8>(xv, C.v, acc); break;
                    case 9: acc = chain_r<9>(xv, C.v, acc); break;
                    case 10: acc = chain_r<10>(xv, C.v, acc); break;
                    case 11: acc = chain_r<11>(xv, C.v, acc); break;
                    case 12: acc = chain_r<12>(xv, C.v, acc); break;
                    case 13: acc = chain_r<13>(xv, C.v, acc); break;
                    case 14: acc = chain_r<14>(xv, C.v, acc); break;
                    case 15: acc = chain_r<15>(xv, C.v, acc); break;
                    default: acc = chain_r<16>(xv, C.v, acc); break;
                }
            }
            if (V == 11) {
                const double2 d = dd[(lo + tid) & (CYC * 32 - 1)];
                acc = exact_div(acc, d.x, d.y);
            }
            ring[(lo + tid) & (RING - 1)] = acc;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        C.m = mm;
        lo = hi;
    };
    for (int l = 0; l < NLEV; l += 2) {
        level(l, A, B);
        level(l + 1, B, A);
    }
    if (tid == 0) cyc[V] = clock64() - t0;
}

int main() {
    const int npos = NLEV * 32;
    Meta *hm = new Meta[npos];
    Rec *hr = new Rec[CYC * K * 32];
    double2 *hd = new double2[npos];
    uint32_t st = 12345;
    auto rnd = [&]() { st = st * 1664525u + 1013904223u; return st >> 8; };
    for (int p = 0; p < npos; ++p) {
        const int l = p / 32;
        hm[p] = Meta{p, K, ((l % CYC) * K * 32) + (p & 31), K};
        const double d = 1.5 + (rnd() % 1000) * 1e-3;
        hd[p] = make_double2(d, 1.0 / d);
    }
    for (int i = 0; i < CYC * K * 32; ++i) hr[i] = Rec{0.01 * (1 + (int)(rnd() % 100)), (int)(rnd() % RING), 0};
    Meta *dm; Rec *dr; double2 *dd; double *x; long long *c;
    cudaMalloc(&dm, npos * sizeof(Meta)); cudaMalloc(&dr, CYC * K * 32 * sizeof(Rec)); cudaMalloc(&dd, npos * 16);
    cudaMalloc(&x, npos * 8); cudaMalloc(&c, 18 * 8);
    cudaMemcpy(dm, hm, npos * sizeof(Meta), cudaMemcpyHostToDevice);
    cudaMemcpy(dr, hr, CYC * K * 32 * sizeof(Rec), cudaMemcpyHostToDevice);
    cudaMemcpy(dd, hd, npos * 16, cudaMemcpyHostToDevice);
    const size_t smem = RING * 8 + (size_t)CYC * 32 * 32 + CYC * K * 32 * 16 + (NLEV + 8) * 4;
    auto setp = [&](auto kern) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); };
    printf("smem %zu\n", smem);
    setp(k<0>); setp(k<1>); setp(k<2>); setp(k<3>); setp(k<4>); setp(k<5>); setp(k<6>);
    setp(kp<7>); setp(kp<8>); setp(kp<9>); setp(kp<10>); setp(kp<11>);
    setp(kp<12>); setp(kp<13>); setp(kp<14>); setp(kp<15>); setp(kp<16>); setp(kp<17>);
    for (int r = 0; r < 2; ++r) {
        k<0><<<1, 160, smem>>>(dm, dr, dd, x, c); k<1><<<1, 160, smem>>>(dm, dr, dd, x, c);
        k<2><<<1, 160, smem>>>(dm, dr, dd, x, c); k<3><<<1, 160, smem>>>(dm, dr, dd, x, c);
        k<4><<<1, 160, smem>>>(dm, dr, dd, x, c); k<5><<<1, 160, smem>>>(dm, dr, dd, x, c);
        k<6><<<1, 160, smem>>>(dm, dr, dd, x, c);
        kp<7><<<1, 160, smem>>>(dm, dr, dd, x, c); kp<8><<<1, 160, smem>>>(dm, dr, dd, x, c);
        kp<9><<<1, 160, smem>>>(dm, dr, dd, x, c); kp<10><<<1, 160, smem>>>(dm, dr, dd, x, c);
        kp<11><<<1, 160, smem>>>(dm, dr, dd, x, c);
        kp<12><<<1, 160, smem>>>(dm, dr, dd, x, c); kp<13><<<1, 160, smem>>>(dm, dr, dd, x, c);
        kp<14><<<1, 160, smem>>>(dm, dr, dd, x, c); kp<15><<<1, 160, smem>>>(dm, dr, dd, x, c);
        kp<16><<<1, 160, smem>>>(dm, dr, dd, x, c); kp<17><<<1, 160, smem>>>(dm, dr, dd, x, c);
    }
    cudaError_t e = cudaDeviceSynchronize();
    long long h[18];
    cudaMemcpy(h, c, 144, cudaMemcpyDeviceToHost);
    printf("{\"err\": \"%s\", \"cycles_per_level\": {", cudaGetErrorString(e));
    for (int v = 0; v < 18; ++v) printf("\"V%d\": %.1f%s", v, h[v] / (double)NLEV, v < 17 ? ", " : "");
    printf("}}\n");
    return 0;
}
