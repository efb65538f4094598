// Index-order sync-free triangular solve for 8 interleaved right-hand sides
// (the batched counterpart of trsv_nat.cu; config 4: 8 RHS per GPU).
//
// The level-ordered batched kernel (bkernels.cu kb_trsv) gives a lane one
// task and reads each dependency's 64-byte row x[col * 8 .. + 8) with four
// 16-byte loads per lane: 32 lanes touch 32 different rows, so every one of
// those loads costs 32 L1TEX wavefronts -- four wavefronts per entry plus one
// for its flag (ncu at n = 8e6: L1TEX-bound at 1.5 - 1.65 ms per L1 solve).
// Here a row is always moved by lanes that share it:
//   - a warp takes 32 consecutive unknowns (index order is a topological
//     order); their line pointers, right-hand-side rows and output rows are
//     contiguous, their entries one span of the matrix's own CSR / CSC arrays;
//   - the span is loaded entry-parallel (coalesced) and each dependency's
//     completion flag polled once (epoch-tagged flags, no fill of the 8n
//     outputs);
//   - the rows of the finished dependencies are copied into shared memory by
//     16-byte cp.async, four lanes per row (one wavefront per row, every
//     row of the span in flight at once, no registers held);
//   - the chains run a row per lane with its 8 right-hand sides side by side
//     (8 independent chains per lane) in the reference's per-task order; a
//     dependency that was not finished at the first poll (near in index
//     distance) is polled again there and read straight from global memory;
//   - a lane stores its output row, fences, and releases the row's flag.
// Per right-hand side the operation order is the single-RHS kernels', so
// every RHS stays bit-identical to its own solve.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "bsolver.cuh"
#include "device_common.cuh"

namespace rsb {

namespace {

constexpr int kB = kBatch;
constexpr int kBnBlock = 128;
constexpr int kBnWarps = kBnBlock / 32;
constexpr unsigned kBnMinBackoffNs = 32, kBnMaxBackoffNs = 256;

// acquire polls: a flag seen set orders the row reads after it (no consumer-side fence)
__device__ __forceinline__ int bn_ld_flag(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void bn_st_flag_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bn_cp16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void bn_cp_wait_all() {
    asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
}

// shared memory of one warp: x rows of the span (8 values padded to kRow = 10
// doubles, so lanes reading different rows spread over the banks), the
// slice's right-hand-side rows, entry values, entry columns
constexpr int kRow = 10;
__host__ __device__ constexpr size_t bn_warp_bytes(int cap) {
    return (size_t)cap * (kRow * 8 + 8 + 4) + 32 * kRow * 8;
}

__device__ __forceinline__ int bn_ld_flag_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(kBnBlock) kb_trsv_nat(NatSrc s, int n, VecIn a, const double *c, double *x, int *flag,
                                                      const unsigned *epoch, unsigned long long *ticket, int cap,
                                                      const int *all_done) {
    if (all_done && *(volatile const int *)all_done != 0) return;
    constexpr bool kDot = (MODE & 1) != 0;
    const int E = (int)*(volatile const unsigned *)epoch;
    extern __shared__ __align__(16) unsigned char bn_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char *wbase = bn_smem + (size_t)warp * bn_warp_bytes(cap);
    double *sx = reinterpret_cast<double *>(wbase);  // [cap][kRow]
    double *srhs = sx + (size_t)cap * kRow;           // [32][kRow]
    double *sv = srhs + 32 * kRow;                    // [cap]
    int *sc = reinterpret_cast<int *>(sv + cap);      // [cap]: column, or -(column + 1) once its row is staged
    const int nsl = (n + 31) / 32;
    const unsigned full = 0xffffffffu;
    const int cpe = lane >> 2, part = lane & 3;       // copy phase: entry of the group of 8, 16-byte piece
    for (;;) {
        int w = 0;
        if (lane == 0) w = (int)atomicAdd(ticket, 1ull);
        w = __shfl_sync(full, w, 0);
        if (w >= nsl) break;
        const int q = w * 32 + lane;
        const bool valid = q < n;
        const int t = s.forward ? q : n - 1 - q;
        const int tlo = s.forward ? w * 32 : n - 32 - w * 32, thi = tlo + 31;
        int elo, ehi;
        long long ai = 0;
        if (valid) {
            elo = __ldg(s.ptr + t);
            ehi = __ldg(s.ptr + t + 1);
            ai = a.g ? (long long)a.g[t + a.off] : (long long)t + a.off;
        } else {  // past the end (last slice only): an empty line at the span's edge
            elo = ehi = __ldg(s.ptr + (s.forward ? n : 0));
        }
        const int len = (ehi - elo) - s.first_off - s.last_off;
        const int base = s.step > 0 ? elo + s.first_off : ehi - 1 - s.last_off;  // entry k at base + step * k
        // the slice's right-hand-side rows, four lanes per row (completed with
        // the first pass's copies)
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int rho = it * 8 + cpe;
            const long long ar = __shfl_sync(full, ai, rho);
            const bool vr = __shfl_sync(full, (int)valid, rho) != 0;
            if (vr) bn_cp16(srhs + rho * kRow + part * 2, a.p + ar * kB + part * 2);
        }
        int la = 0;
        while (la < 32) {
            // lanes [la, lb): the longest run whose span fits the window
            const int a_lo = __shfl_sync(full, elo, la), a_hi = __shfl_sync(full, ehi, la);
            const int span_to_me = s.forward ? ehi - a_lo : a_hi - elo;
            const unsigned over = __ballot_sync(full, lane >= la && span_to_me > cap);
            const int lb = over ? __ffs(over) - 1 : 32;
            const int b_lo = __shfl_sync(full, elo, lb - 1), b_hi = __shfl_sync(full, ehi, lb - 1);
            const int S0 = s.forward ? a_lo : b_lo, S1 = s.forward ? b_hi : a_hi;
            const int32_t *gi = s.idx + S0;
            const double *gv = s.val + S0;
            const int span = S1 - S0;
            // the span, entry-parallel: coalesced loads, each dependency's flag polled
            // once (entries pointing into this slice -- its diagonals, dependencies
            // between its rows -- cannot be finished yet and are left for the chain)
            for (int i0 = lane; i0 < span; i0 += 128) {
                int ci[4], f[4];
                double vi[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool in = i0 + u * 32 < span;
                    ci[u] = in ? __ldcs(gi + i0 + u * 32) : -1;
                    vi[u] = in ? __ldcs(gv + i0 + u * 32) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool ask = ci[u] >= 0 && (ci[u] < tlo || ci[u] > thi);
                    f[u] = ask ? bn_ld_flag(flag + ci[u]) : E - 1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (i0 + u * 32 >= span) continue;
                    sc[i0 + u * 32] = f[u] == E ? -(ci[u] + 1) : ci[u];
                    sv[i0 + u * 32] = vi[u];
                }
            }
            __syncwarp();
            // rows of the finished dependencies: four lanes per 64-byte row, every
            // row of the span in flight at once
            for (int e0 = 0; e0 < span; e0 += 8) {
                const int e = e0 + cpe;
                if (e < span) {
                    const int cc = sc[e];
                    if (cc < 0) bn_cp16(sx + (size_t)e * kRow + part * 2, x + (size_t)(-cc - 1) * kB + part * 2);
                }
            }
            bn_cp_wait_all();
            __syncwarp();
            // the chains: lane = row, its 8 right-hand sides side by side (8
            // independent chains per lane), resumed each round where the first
            // unfinished dependency stopped it
            const bool mine = valid && lane >= la && lane < lb;
            bool done = !mine;
            int k = 0, sl = base - S0;
            double acc[kB], dot[kB];
#pragma unroll
            for (int r = 0; r < kB; ++r) {
                acc[r] = 0.0;
                dot[r] = 0.0;
            }
            if (mine) {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const double2 v2 = *reinterpret_cast<const double2 *>(srhs + lane * kRow + 2 * h);
                    acc[2 * h] = v2.x;
                    acc[2 * h + 1] = v2.y;
                }
                if (c) {
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const double2 v2 = __ldcg(reinterpret_cast<const double2 *>(c + (size_t)t * kB) + h);
                        acc[2 * h] = __dadd_rn(acc[2 * h], v2.x);
                        acc[2 * h + 1] = __dadd_rn(acc[2 * h + 1], v2.y);
                    }
                }
            }
            unsigned backoff = 0;
            for (;;) {
                bool progress = false;
                if (!done) {
                    const int kin = k;
                    while (k < len) {
                        const int cc = sc[sl];
                        const double v = sv[sl];
                        double xv[kB];
                        if (cc < 0) {
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                const double2 v2 = *reinterpret_cast<const double2 *>(sx + (size_t)sl * kRow + 2 * h);
                                xv[2 * h] = v2.x;
                                xv[2 * h + 1] = v2.y;
                            }
                        } else {
                            if (bn_ld_flag_acquire(flag + cc) != E) break;
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                const double2 v2 = __ldcg(reinterpret_cast<const double2 *>(x + (size_t)cc * kB) + h);
                                xv[2 * h] = v2.x;
                                xv[2 * h + 1] = v2.y;
                            }
                        }
#pragma unroll
                        for (int r = 0; r < kB; ++r) {
                            if (kDot) {
                                dot[r] = fma(v, xv[r], dot[r]);
                            } else {
                                // the reference skips zero operands (sc.py:262); acc - (+0.0) == acc
                                acc[r] = __dsub_rn(acc[r], xv[r] != 0.0 ? __dmul_rn(v, xv[r]) : 0.0);
                            }
                        }
                        ++k;
                        sl += s.step;
                    }
                    progress = k != kin;
                    if (k == len) {
                        double d = 1.0;
                        if (MODE & 2) d = sv[(s.diag_at == 0 ? elo : ehi - 1) - S0];
#pragma unroll
                        for (int r = 0; r < kB; ++r) {
                            if (kDot && len > 0) acc[r] = __dsub_rn(acc[r], dot[r]);  // < 16 entries: the scalar BLAS order
                            if (MODE & 2) acc[r] = __ddiv_rn(acc[r], d);
                        }
                        double2 *o2 = reinterpret_cast<double2 *>(x + (size_t)t * kB);
#pragma unroll
                        for (int h = 0; h < 4; ++h) __stcg(o2 + h, make_double2(acc[2 * h], acc[2 * h + 1]));
                        bn_st_flag_release(flag + t, E);  // the row was written by this lane: the release orders it
                        done = true;
                        progress = true;
                    }
                }
                if (!__any_sync(full, !done)) break;
                if (!__any_sync(full, progress)) {
                    backoff = backoff ? min(backoff * 2, kBnMaxBackoffNs) : kBnMinBackoffNs;
                    __nanosleep(backoff);
                } else {
                    backoff = 0;
                }
            }
            __syncwarp();
            la = lb;
        }
    }
}

// (An octet-per-row variant -- the batched CSR product's scheme with flags: rows
// in index order round-robin over a cooperative launch, no shared memory, each
// lane of the octet loading and polling one entry of a chunk of 8 -- measured
// 38.8 ms per 8-RHS iteration at n = 8e6 against 36.0 for the kernel above and
// 33.0 for the level-ordered one: one release fence per row instead of per
// 32 rows.)

using BnKernel = void (*)(NatSrc, int, VecIn, const double *, double *, int *, const unsigned *, unsigned long long *,
                          int, const int *);

BnKernel bn_kernel(int mode) {
    switch (mode & 3) {
        case 0: return kb_trsv_nat<0>;
        case 1: return kb_trsv_nat<1>;
        case 2: return kb_trsv_nat<2>;
        default: return kb_trsv_nat<3>;
    }
}

// window of the batched kernel: 92 bytes of shared memory per entry, so the
// single-RHS window is cut to keep three blocks per SM
constexpr int kBnCap = 160;

}  // namespace

bool btrsv_nat_supported(const TriSched &T) {
    // opt-in (RSB_BTRSV_NAT=1): 36.0 ms per 8-RHS iteration at n = 8e6 against 33.0 with the
    // level-ordered kernel (per launch 1.66 / 1.33 / 4.30 vs 1.55 / 1.31 / 2.79 ms for L1 /
    // L1^T / U before the acquire-load flags) -- 12 warps per SM (17 KB of shared memory per
    // warp) do not hide the slice's dependent round trips
    const char *eon = getenv("RSB_BTRSV_NAT");  // read per launch (launches happen at graph capture)
    const bool on = eon && atoi(eon) != 0;
    return on && T.use_nat && T.nat_max_line <= kBnCap;
}

int launch_btrsv_nat(rsb_ctx *ctx, const TriSched &T, VecIn a, const double *c, double *x, BTriWs &ws,
                     const int *all_done) {
    BnKernel k = bn_kernel(T.mode);
    const int cap = std::min<int>(T.nat_cap, kBnCap);
    const size_t smem = (size_t)kBnWarps * bn_warp_bytes(cap);
    static size_t granted[4] = {};  // grow-only opt-in above 48 KB
    if (smem > 48 * 1024 && smem > granted[T.mode & 3]) {
        RSB_TRY_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        granted[T.mode & 3] = smem;
    }
    int occ = 0, sms = 0;
    RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBnBlock, smem));
    RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    occ = std::max(occ, 1);
    if (const char *eo = getenv("RSB_BNAT_OCC")) occ = std::max(1, std::min(occ, atoi(eo)));  // experiments
    const int64_t nsl = ((int64_t)T.n + 31) / 32;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, (nsl + kBnWarps - 1) / kBnWarps));
    k<<<grid, kBnBlock, smem, ctx->stream>>>(T.nat, T.n, a, c, x, ws.flag, ws.epoch, ws.ticket, cap, all_done);
    return bpost(ctx);
}

}  // namespace rsb
