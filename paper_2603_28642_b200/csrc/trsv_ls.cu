// Level-synchronous grid-wide triangular solve for wide DAGs (sm_100a).
//
// Config 4 at mu = 1 and n = 8e6: L1 has 27 levels (the first 1.9M wide), U
// 66 levels that are ALL 115k-477k wide.  Every level is a set of
// independent tasks whose operands were published by earlier levels, so a
// level is a streaming pass with no polling: one persistent cooperative
// kernel walks the levels with a grid barrier between them.  Per level a
// warp owns a static share of the level's items (32 tasks, or 4 tasks x 8
// right-hand sides in the batched form); before every barrier it has
// already loaded its first item of the next level -- the task's row,
// right-hand side, diagonal and entries do not depend on the level being
// finished -- so after the barrier the only loads on the critical path are
// the dependencies x[col], all issued at once.
//
// The arithmetic per task is the reference's order (the same sequence as
// every other solve kernel here: sequential axpy order for L and U solves,
// the scalar OpenBLAS FMA chain for the transposed solve's dots), so the
// results are bit-identical.
//
// Barriers: a monotonically increasing arrival counter (reset by a memset
// node before the launch); all blocks are co-resident (cooperative launch),
// and every block takes part in every barrier even when its work is gated
// off, so a gate that flips during the launch cannot strand a block.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kLsBlockT = 256;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

// one task of one right-hand side, loaded ahead of its dependencies
template <int N>
struct LsTask {
    int row;     // unknown written (-1: no task)
    int len;     // real entries
    int K;       // the slice's entry rows (entries continue past N when len > N)
    int64_t base;
    int cols[N];
    double vals[N];
    double acc;  // right-hand side
    double d;    // diagonal (MODE & 2)
};

template <int NB>
__device__ __forceinline__ double rhs_of(const VecIn &a, const double *c, int row, int r) {
    const int64_t i = a.g ? (int64_t)a.g[row + a.off] : (int64_t)row + a.off;
    double v = a.p[i * NB + r];
    if (c) v = __dadd_rn(v, c[(int64_t)row * NB + r]);
    return v;
}

template <int MODE, int N, int NB>
__device__ __forceinline__ void ls_load(const TriDev &T, const VecIn &a, const double *c, int q, int r,
                                        LsTask<N> &k) {
    k.row = -1;
    k.len = 0;
    k.K = 0;
    k.base = 0;
    k.acc = 0.0;
    k.d = 1.0;
#pragma unroll
    for (int e = 0; e < N; ++e) {
        k.cols[e] = -1;
        k.vals[e] = 0.0;
    }
    if (q < 0) return;
    const int s = q >> 5, ln = q & 31;
    k.base = T.slice_off[s] + ln;
    k.K = (int)((T.slice_off[s + 1] - T.slice_off[s]) >> 5);
    k.row = T.task_row[q];
#pragma unroll
    for (int e = 0; e < N; ++e)
        if (e < k.K) {
            k.cols[e] = __ldg(T.ecol + k.base + (int64_t)e * 32);
            k.vals[e] = __ldg(T.eval + k.base + (int64_t)e * 32);
        }
    k.acc = rhs_of<NB>(a, c, k.row, r);
    if (MODE & 2) k.d = T.diag[q];
}

// dependencies (all published by earlier levels): loads only, so that the
// loads of several items are in flight together
template <int N, int NB>
__device__ __forceinline__ void ls_deps(const LsTask<N> &k, int r, const double *x, double (&xv)[N]) {
#pragma unroll
    for (int e = 0; e < N; ++e) xv[e] = k.cols[e] >= 0 ? __ldcg(x + (int64_t)k.cols[e] * NB + r) : 0.0;
}

// the reference's order and the store.  Entries past N (long rows of U) in
// batches of 8 with their loads in flight together.
template <int MODE, int N, bool TAIL, int NB>
__device__ __forceinline__ void ls_compute(const TriDev &T, const LsTask<N> &k, const double (&xv)[N], int r,
                                           double *x) {
    if (k.row < 0) return;
    double acc = k.acc, dot = 0.0;
#pragma unroll
    for (int e = 0; e < N; ++e) {
        if (k.cols[e] < 0) break;
        if (!(MODE & 1)) {
            if (xv[e] != 0.0) acc = __dsub_rn(acc, __dmul_rn(k.vals[e], xv[e]));
        } else {
            dot = fma(k.vals[e], xv[e], dot);
        }
    }
    if (TAIL && k.K > N && k.cols[N - 1] >= 0) {
        for (int e0 = N; e0 < k.K; e0 += 8) {
            int cc[8];
            double vv[8], xx[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                cc[u] = e0 + u < k.K ? __ldg(T.ecol + k.base + (int64_t)(e0 + u) * 32) : -1;
                vv[u] = e0 + u < k.K ? __ldg(T.eval + k.base + (int64_t)(e0 + u) * 32) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) xx[u] = cc[u] >= 0 ? __ldcg(x + (int64_t)cc[u] * NB + r) : 0.0;
            bool end = false;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (cc[u] < 0) {
                    end = true;
                    break;
                }
                if (!(MODE & 1)) {
                    if (xx[u] != 0.0) acc = __dsub_rn(acc, __dmul_rn(vv[u], xx[u]));
                } else {
                    dot = fma(vv[u], xx[u], dot);
                }
            }
            if (end) break;
        }
    }
    if (MODE & 1) acc = (k.cols[0] >= 0) ? __dsub_rn(acc, dot) : acc;
    if (MODE & 2) acc = __ddiv_rn(acc, k.d);
    x[(int64_t)k.row * NB + r] = acc;
}

// Level-synchronous solve of levels [0, nlev): item i of a level covers task
// positions lp[l] + i * TPI .. + TPI - 1 (TPI = 32 / NB); warp w of the grid
// takes items w, w + W, ..., P of them at a time: the task data of P items is
// loaded together, then their dependencies together, then the P chains run.
// The first P items of the next level are loaded before each barrier.
template <int MODE, int N, bool TAIL, int NB, int P>
__global__ void __launch_bounds__(kLsBlockT, 2) k_trsv_ls(TriDev T, VecIn a, const double *c, double *x,
                                                          unsigned *bar, Gate g, const int *rstat, int rstride) {
    constexpr int TPI = 32 / NB;
    const int lane = threadIdx.x & 31;
    const int o = NB == 1 ? lane : lane >> 3;  // task of the item
    const int r = NB == 1 ? 0 : lane & 7;      // right-hand side
    const int W = gridDim.x * (kLsBlockT / 32);
    const int gw = blockIdx.x * (kLsBlockT / 32) + (threadIdx.x >> 5);
    // gated work is skipped, barriers are not (see the file comment)
    bool off = gated(g);
    if (NB > 1 && rstat) off = off || *(volatile const int *)(rstat + r * rstride) != 0;
    const int nlev = T.nlevels;
    auto pos_of = [&](int l, int i) -> int {  // -1: past the level
        const int lo = T.level_ptr[l], hi = T.level_ptr[l + 1];
        const int q = lo + i * TPI + o;
        return (!off && i * TPI < hi - lo && q < hi) ? q : -1;
    };
    auto items = [&](int l) { return (T.level_ptr[l + 1] - T.level_ptr[l] + TPI - 1) / TPI; };
    LsTask<N> k[P];
#pragma unroll
    for (int u = 0; u < P; ++u) ls_load<MODE, N, NB>(T, a, c, pos_of(0, gw + u * W), r, k[u]);
    for (int l = 0; l < nlev; ++l) {
        const int ni = items(l);
        for (int i = gw; i < ni; i += P * W) {
            if (i != gw) {
#pragma unroll
                for (int u = 0; u < P; ++u) ls_load<MODE, N, NB>(T, a, c, pos_of(l, i + u * W), r, k[u]);
            }
            double xv[P][N];
#pragma unroll
            for (int u = 0; u < P; ++u) ls_deps<N, NB>(k[u], r, x, xv[u]);
#pragma unroll
            for (int u = 0; u < P; ++u) ls_compute<MODE, N, TAIL, NB>(T, k[u], xv[u], r, x);
        }
        if (l + 1 < nlev) {
            // the next level's first items are loaded before the barrier
#pragma unroll
            for (int u = 0; u < P; ++u) ls_load<MODE, N, NB>(T, a, c, pos_of(l + 1, gw + u * W), r, k[u]);
            grid_barrier(bar, (unsigned)(l + 1) * gridDim.x);
        }
    }
}

using LsKernel = void (*)(TriDev, VecIn, const double *, double *, unsigned *, Gate, const int *, int);

// items in flight per warp: P = 4 / 2 / 1 for 4 / 8 / 12 register entries
// (RSB_LS_P caps it, experiments)
template <int MODE, int NB, int N, bool TAIL>
LsKernel ls_kernel_p(int pcap) {
    constexpr int PD = N <= 4 ? 4 : (N <= 8 ? 2 : 1);
    const int p = std::min(PD, pcap);
    if (p >= 4) return k_trsv_ls<MODE, N, TAIL, NB, (PD >= 4 ? 4 : 1)>;
    if (p >= 2) return k_trsv_ls<MODE, N, TAIL, NB, (PD >= 2 ? 2 : 1)>;
    return k_trsv_ls<MODE, N, TAIL, NB, 1>;
}

template <int MODE, int NB>
LsKernel ls_kernel(int n, bool tail, int pcap) {
    if (n <= 4) return tail ? ls_kernel_p<MODE, NB, 4, true>(pcap) : ls_kernel_p<MODE, NB, 4, false>(pcap);
    if (n <= 8) return tail ? ls_kernel_p<MODE, NB, 8, true>(pcap) : ls_kernel_p<MODE, NB, 8, false>(pcap);
    return tail ? ls_kernel_p<MODE, NB, 12, true>(pcap) : ls_kernel_p<MODE, NB, 12, false>(pcap);
}

template <int NB>
LsKernel ls_kernel_for(int mode, int n, bool tail, int pcap) {
    switch (mode & 3) {
        case 0: return ls_kernel<0, NB>(n, tail, pcap);
        case 1: return ls_kernel<1, NB>(n, tail, pcap);
        case 2: return ls_kernel<2, NB>(n, tail, pcap);
        default: return ls_kernel<3, NB>(n, tail, pcap);
    }
}

}  // namespace

// grid of the level-synchronous solve: every block co-resident
int launch_trsv_ls(rsb_ctx *ctx, const TriSched &T, const TriDev &v, VecIn a, const double *c, double *x,
                   unsigned *bar, Gate g, int nb, const int *rstat, int rstride) {
    const bool tail = T.max_task > T.wide_n;
    const char *ep = getenv("RSB_LS_P");
    const int pcap = ep ? std::max(1, atoi(ep)) : 4;
    const int pi = pcap >= 4 ? 2 : (pcap >= 2 ? 1 : 0);
    LsKernel k = nb == 8 ? ls_kernel_for<8>(T.mode, T.wide_n, tail, pcap)
                         : ls_kernel_for<1>(T.mode, T.wide_n, tail, pcap);
    static int occ_cache[2][4][3][2][3] = {};
    const int ni = T.wide_n <= 4 ? 0 : (T.wide_n <= 8 ? 1 : 2);
    int &occ = occ_cache[nb == 8][T.mode & 3][ni][tail][pi];
    if (occ == 0) {
        RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kLsBlockT, 0));
        occ = std::max(occ, 1);
    }
    int sms = 0;
    RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const char *eo = getenv("RSB_LS_OCC");  // experiments: fewer resident blocks per SM
    const int use_occ = eo ? std::max(1, std::min(occ, atoi(eo))) : occ;
    // no more warps than the widest level has items
    const int64_t tpi = 32 / nb;
    const int64_t max_items = (T.max_width + tpi - 1) / tpi;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * use_occ,
                                                                 (max_items + kLsBlockT / 32 - 1) / (kLsBlockT / 32)));
    RSB_TRY_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx->stream));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kLsBlockT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RSB_TRY_CUDA(cudaLaunchKernelEx(&cfg, k, v, a, c, x, bar, g, rstat, rstride));
    return RSB_OK;
}

}  // namespace rsb
