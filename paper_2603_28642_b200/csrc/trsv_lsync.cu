// Level-synchronous grid-wide triangular solve for wide, shallow DAGs
// (sm_100a): the config-4 structure at mu = 1 (n = 8e6: 27 / 66 levels of up
// to 1.9M unknowns).
//
// Each level's task positions are cut into items of up to kLsItem = 32
// consecutive positions; items are numbered in level order and persistent
// warps take them from an atomic ticket.  A warp first loads everything its
// item needs that does not depend on the solve -- row, right-hand side (the
// permutation gather fused), diagonal and up to N entries per task -- then
// waits until every item of the previous level has been counted done,
// gathers the dependencies (all complete, so no per-operand polling: one
// L2 round trip with all loads in flight), runs the reference's per-task
// arithmetic, stores, and counts its item done.  Counts are spread over
// kLsRep replicas per level so the completion atomics of a level's thousands
// of items do not serialise on one address.
//
// Warps that are not resident hold no item, so they never hold up a level:
// no co-residency assumption, safe beside concurrent solves on other streams.  The arithmetic per task is the one
// every solve kernel here uses (sc.py:243-313 order), so results are
// bit-identical to the other variants and to the reference.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

__device__ __forceinline__ double vin_l(const VecIn &v, int64_t i) { return v.g ? v.p[v.g[i + v.off]] : v.p[i + v.off]; }

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// one task of an item, everything that does not depend on the solve
template <int N>
struct LsTask {
    int row, len, K, sl;
    int64_t base;
    double acc, d;
    int cols[N];
    double vals[N];
};

template <int MODE, int N>
__device__ __forceinline__ void ls_load(const TriDev &T, const VecIn &a, const double *c, int p, bool valid,
                                        LsTask<N> &k) {
    k.row = 0;
    k.len = 0;
    k.K = 0;
    k.sl = p & 31;
    k.base = 0;
    k.acc = 0.0;
    k.d = 1.0;
    if (valid) {
        const int s = p >> 5;
        k.base = T.slice_off[s];
        k.K = (int)((T.slice_off[s + 1] - k.base) >> 5);
        k.row = T.task_row[p];
        k.acc = vin_l(a, k.row);
        if (c) k.acc = __dadd_rn(k.acc, c[k.row]);
        if (MODE & 2) k.d = T.diag[p];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        k.cols[q] = -1;
        k.vals[q] = 0.0;
        if (q < k.K) {
            k.cols[q] = __ldcs(T.ecol + k.base + (int64_t)q * 32 + k.sl);
            k.vals[q] = __ldcs(T.eval + k.base + (int64_t)q * 32 + k.sl);
        }
    }
}

template <int MODE, int N>
__device__ __forceinline__ void ls_solve(const TriDev &T, const LsTask<N> &k, double *x) {
    double xv[N];
    int len = 0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        len += k.cols[q] >= 0;
        xv[q] = k.cols[q] >= 0 ? __ldcg(x + k.cols[q]) : 0.0;  // all dependencies final: loads in flight together
    }
    double r = k.acc;
    if (!(MODE & 1)) {
#pragma unroll
        for (int q = 0; q < N; ++q)
            if (q < len && xv[q] != 0.0) r = __dsub_rn(r, __dmul_rn(k.vals[q], xv[q]));
        if (len == N)  // entries continue past the registers (rare)
            for (int q = N; q < k.K; ++q) {
                const int64_t e = k.base + (int64_t)q * 32 + k.sl;
                const int col = T.ecol[e];
                if (col < 0) break;
                const double xj = __ldcg(x + col);
                if (xj != 0.0) r = __dsub_rn(r, __dmul_rn(T.eval[e], xj));
            }
    } else {  // < 16 entries: the scalar OpenBLAS order (checked at analysis)
        double dot = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q)
            if (q < len) dot = fma(k.vals[q], xv[q], dot);
        if (len == N)
            for (int q = N; q < k.K; ++q) {
                const int64_t e = k.base + (int64_t)q * 32 + k.sl;
                const int col = T.ecol[e];
                if (col < 0) break;
                dot = fma(T.eval[e], __ldcg(x + col), dot);
            }
        r = __dsub_rn(r, dot);
    }
    if (MODE & 2) r = __ddiv_rn(r, k.d);
    x[k.row] = r;
}

// Warp items of 32 positions.  A warp takes its next item's ticket and
// issues that item's loads before it waits on and solves the current one,
// so a level's items start from data already in registers.  Tickets are
// taken in order and a warp's current item precedes its next, so the
// smallest unfinished item is always some warp's current item, whose lower
// levels are complete: no deadlock, no co-residency assumption.
template <int MODE, int N>
__global__ void __launch_bounds__(kLsBlock) k_trsv_lsync(TriDev T, LsyncDev P, VecIn a, const double *c, double *x,
                                                        Gate g) {
    if (gated(g)) return;
    const int lane = threadIdx.x & 31;
    auto take = [&]() {
        int s = 0;
        if (lane == 0) s = (int)atomicAdd(P.ticket, 1u);
        return __shfl_sync(0xffffffffu, s, 0);
    };
    int it = take();
    if (it >= P.nitems) return;
    LsTask<N> cur, nxt;
    int p = P.item_pos[it] + lane;
    ls_load<MODE, N>(T, a, c, p, p < P.item_pos[it + 1], cur);
    while (it < P.nitems) {
        const int L = P.item_level[it];
        const bool cur_valid = P.item_pos[it] + lane < P.item_pos[it + 1];
        const int nit = take();
        if (nit < P.nitems) {
            const int q = P.item_pos[nit] + lane;
            ls_load<MODE, N>(T, a, c, q, q < P.item_pos[nit + 1], nxt);
        }
        if (L > 0) {  // wait until every item of level L - 1 is counted done
            const unsigned want = (unsigned)(P.level_items[L] - P.level_items[L - 1]);
            const unsigned *cnt = P.done + (size_t)(L - 1) * kLsRep;
            for (;;) {
                unsigned v = ld_acquire_u32(cnt + lane);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (v >= want) break;
                __nanosleep(32);
            }
        }
        if (cur_valid) ls_solve<MODE, N>(T, cur, x);
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(P.done + (size_t)L * kLsRep + (it % kLsRep), 1u);
        }
        it = nit;
        cur = nxt;
    }
}

using LsyncKernel = void (*)(TriDev, LsyncDev, VecIn, const double *, double *, Gate);

template <int MODE>
LsyncKernel lsync_kernel(int n) {
    if (n <= 4) return k_trsv_lsync<MODE, 4>;
    if (n <= 8) return k_trsv_lsync<MODE, 8>;
    return k_trsv_lsync<MODE, 12>;
}

}  // namespace

int launch_trsv_lsync(rsb_ctx *ctx, const TriSched &T, const TriDev &v, unsigned *counters, VecIn a,
                      const double *c, double *x, Gate g) {
    LsyncKernel k;
    switch (T.mode) {
        case 0: k = lsync_kernel<0>(T.max_task); break;
        case 1: k = lsync_kernel<1>(T.max_task); break;
        case 2: k = lsync_kernel<2>(T.max_task); break;
        default: k = lsync_kernel<3>(T.max_task); break;
    }
    static int occ_cache[4][3] = {};
    const int ni = T.max_task <= 4 ? 0 : (T.max_task <= 8 ? 1 : 2);
    int &occ = occ_cache[T.mode & 3][ni];
    if (occ == 0) {
        RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kLsBlock, 0));
        occ = std::max(occ, 1);
    }
    int sms = 0;
    RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    // counters: [0] ticket, [32 ..) per-level replicated done counts
    const LsyncDev P{T.ls_nitems, T.ls_item_pos, T.ls_item_level, T.ls_level_items, counters, counters + 32};
    RSB_TRY_CUDA(cudaMemsetAsync(counters, 0, (32 + (size_t)T.nlevels * kLsRep) * sizeof(unsigned), ctx->stream));
    const int grid = (int)std::min<int64_t>((int64_t)sms * occ, T.ls_nitems);
    k<<<std::max(grid, 1), kLsBlock, 0, ctx->stream>>>(v, P, a, c, x, g);
    return RSB_OK;
}

}  // namespace rsb
