// Lean single-CTA triangular solve for narrow dependency DAGs (sm_100a).
//
// Used when every level is at most kLeanMaxWidth wide (one task per consumer
// thread), every task has at most N <= 16 entries (< 16 for the dot order),
// and every dependency is still in the shared-memory value ring -- config 1
// at mu = 1 (1,290 / 2,806 levels of <= 66 unknowns, <= 14 entries).
// Bit-identical to k_trsv_stage (kernels.cu) and to the reference solves
// (sc.py:253-300): the same per-task operation order, the same exact
// division.
//
// What makes it lean (measured with scripts/probes/level_ladder.cu on B200,
// cycles per level of a 32-wide, 6-entry synthetic level set): every
// dependent shared-memory load in front of the chain costs ~120 cycles
// (meta -> record -> ring: 449 vs 212 with ring loads only), a per-warp
// switch on the trip count ~210 (BRX), a warp-uniform branch with loads
// behind it ~100, and a predicated-off load whose result is consumed ~20.
// So the level loop has no branch but its own back edge:
//   - software pipeline across the barrier: at level l a thread holds its
//     whole level-l task in registers (entry sources and values, rhs,
//     diagonal) and the meta of its level-(l+1) task; right after the
//     barrier it issues the level-l ring loads -- the only loads on the
//     dependency chain -- then the 16-byte loads of level l+1's task and
//     the meta of level l+2, then runs the chain;
//   - the chain is unrolled for the schedule's longest task N (a kernel
//     template parameter): shorter tasks run zero entries, which leave the
//     result unchanged bit for bit (see fast_chain in kernels.cu);
//   - the division is Markstein's exact reciprocal division, branch-free;
//     the rare operand outside its range (zero excepted) takes IEEE division
//     behind one warp vote;
//   - task data arrives by 1-D TMA bulk copies into kStageBufs chunk buffers
//     (producer warp); the consumers release and await chunks only between
//     segments of levels that the resident chunks cover, never per level;
//   - two task buffers alternate (level loop unrolled by two), so nothing is
//     copied between registers.
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kLeanConsumers = 128;  // 4 consumer warps, one 32-position slice each per level
constexpr int kLeanThreads = kLeanConsumers + 32;
constexpr int kLeanProducerWarp = 3;  // SMSP 3; the rarely used 4th slice runs on warp 4
static_assert(kLeanMaxWidth == kLeanConsumers, "one task per consumer thread and level");

// predicated shared-memory accesses: the destination keeps its value when p
// is false (no branch)
__device__ __forceinline__ void lds_f64_if(bool p, unsigned a, double &v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}"
                 : "+d"(v)
                 : "r"(a), "r"((int)p));
}
__device__ __forceinline__ void lds_v2f64_if(bool p, unsigned a, double2 &v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q ld.shared.v2.f64 {%0, %1}, [%2];\n}"
                 : "+d"(v.x), "+d"(v.y)
                 : "r"(a), "r"((int)p));
}
__device__ __forceinline__ void lds_v4_if(bool p, unsigned a, int4 &v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];\n}"
                 : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
                 : "r"(a), "r"((int)p));
}
__device__ __forceinline__ void sts_f64_if(bool p, unsigned a, double v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}" ::"r"(a), "d"(v),
                 "r"((int)p)
                 : "memory");
}
__device__ __forceinline__ void stg_f64_if(bool p, double *a, double v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(a), "d"(v),
                 "r"((int)p)
                 : "memory");
}

// IEEE division for the rare operands outside the exact range, out of line
// so that the compiler cannot hoist its reciprocal iteration onto every
// level's critical path
__device__ __noinline__ double ieee_div(double a, double d) { return __ddiv_rn(a, d); }

template <int N>
struct LeanTask {
    int4 m;  // {row (-1 padding, -2 no task), len, slice base in its chunk, slice's longest task}
    int src[4 * ((N + 3) / 4)];
    double v[2 * ((N + 1) / 2)];
    double acc;  // right-hand side (gathered)
    double2 dr;  // {diag, RN(1/diag)}; 1/diag = 0 marks a diagonal outside the exact range
};

template <int MODE, int N>
__global__ void __launch_bounds__(kLeanThreads) k_trsv_lean(TriDev T, double *x, Gate g) {
    if (gated(g)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool kDiag = (MODE & 2) != 0;
    constexpr int NQ = (N + 3) / 4, NP = (N + 1) / 2;
    const int CH = T.stage_ch, EM = T.stage_emax;
    unsigned char *bufs = smem + (size_t)kRing * 8;
    const unsigned o_meta = (unsigned)CH * 8, o_dd = o_meta + (unsigned)CH * 16,
                   o_val = o_dd + (kDiag ? (unsigned)CH * 16 : 0u), o_src = o_val + (unsigned)EM * 8,
                   bb = o_src + (unsigned)EM * 4;
    unsigned long long *full = reinterpret_cast<unsigned long long *>(bufs + kStageBufs * (size_t)bb);
    unsigned long long *empty = full + kStageBufs;
    int *lvl = reinterpret_cast<int *>(empty + kStageBufs);
    const int nlev = T.nlevels, nch = T.nchunks, lgch = __ffs(CH) - 1;
    // level bounds, padded with the end so lvl[l + 3] is always valid
    for (int i = threadIdx.x; i <= nlev + 4; i += blockDim.x) lvl[i] = T.level_ptr[i < nlev ? i : nlev];
    if (threadIdx.x == 0) {
        for (int b = 0; b < kStageBufs; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], kLeanConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kLeanProducerWarp) {
        // chunk c goes to buffer c % kStageBufs once the consumers released
        // the chunk that held it
        if (lane == 0) {
            for (int c = 0; c < nch; ++c) {
                const int b = c & (kStageBufs - 1);
                if (c >= kStageBufs) mbar_wait(&empty[b], (unsigned)(((c / kStageBufs) - 1) & 1));
                unsigned char *B = bufs + (size_t)b * bb;
                const int64_t r0 = T.chunk_roff[c];
                const int ne = (int)(T.chunk_roff[c + 1] - r0);
                const unsigned bytes = (unsigned)(CH * 8 + CH * 16 + (kDiag ? CH * 16 : 0) + ne * 12);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&full[b], bytes);
                bulk_g2s(B, T.bpos + (int64_t)c * CH, CH * 8, &full[b]);
                bulk_g2s(B + o_meta, T.meta + (int64_t)c * CH, CH * 16, &full[b]);
                if (kDiag) bulk_g2s(B + o_dd, T.ddiag + 2 * (int64_t)c * CH, CH * 16, &full[b]);
                if (ne) {
                    bulk_g2s(B + o_val, T.rval + r0, (unsigned)ne * 8, &full[b]);
                    bulk_g2s(B + o_src, T.rsrc + r0, (unsigned)ne * 4, &full[b]);
                }
            }
        }
        return;
    }
    const int slot = warp < kLeanProducerWarp ? (int)threadIdx.x : (int)threadIdx.x - 32;
    // shared-window bases, opaque so they stay in registers (not
    // rematerialised from SR_CgaCtaId every level)
    unsigned s_ring, s_bufs;
    asm volatile("mov.u32 %0, %1;" : "=r"(s_ring) : "r"(smem_u32(smem)));
    asm volatile("mov.u32 %0, %1;" : "=r"(s_bufs) : "r"(smem_u32(bufs)));
    int released = 0, ready = -1;
    auto await_chunk = [&](int c) {
        for (; ready < c; ) {
            ++ready;
            mbar_wait(&full[ready & (kStageBufs - 1)], (unsigned)((ready / kStageBufs) & 1));
        }
    };
    auto release_below = [&](int c) {
        for (; released < c; ++released)
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                 smem_u32(&empty[released & (kStageBufs - 1)]))
                             : "memory");
    };
    auto sbuf = [&](int t) -> unsigned { return s_bufs + (unsigned)((t >> lgch) & (kStageBufs - 1)) * bb; };
    auto load_meta = [&](int t, int hi) -> int4 {
        int4 m = make_int4(-2, 0, 0, 0);
        lds_v4_if(t < hi, sbuf(t) + o_meta + (unsigned)(t & (CH - 1)) * 16, m);
        return m;
    };
    // the rest of task t (its meta already in S.m): sources in quads, values
    // in pairs, rhs, diagonal; nothing past the task's length is loaded
    auto load_task = [&](LeanTask<N> &S, int t) {
        const int len = S.m.y;
        const bool has = S.m.x != -2;
        const unsigned B = sbuf(t), loc = (unsigned)(t & (CH - 1));
        const unsigned sa = B + o_src + (unsigned)(S.m.z + lane * 4) * 4;
        const unsigned va = B + o_val + (unsigned)(S.m.z + lane * 2) * 8;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            int4 s4 = make_int4(0, 0, 0, 0);
            lds_v4_if(4 * q < len, sa + q * 512, s4);
            S.src[4 * q] = s4.x;
            S.src[4 * q + 1] = s4.y;
            S.src[4 * q + 2] = s4.z;
            S.src[4 * q + 3] = s4.w;
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double2 v2 = make_double2(0.0, 0.0);
            lds_v2f64_if(2 * q < len, va + q * 512, v2);
            S.v[2 * q] = v2.x;
            S.v[2 * q + 1] = v2.y;
        }
        S.acc = 0.0;
        lds_f64_if(has, B + loc * 8, S.acc);
        S.dr = make_double2(1.0, 1.0);
        if (kDiag) lds_v2f64_if(has, B + o_dd + loc * 16, S.dr);
    };

    int lo = lvl[0], hi = lvl[1], hi1 = lvl[2];
    auto level = [&](int l, LeanTask<N> &C, LeanTask<N> &Nx) {
        const int hi2 = lvl[l + 3];  // end of level l + 2
        const int t = lo + slot;
        // 1. this level's dependency loads
        double xv[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
            xv[q] = 0.0;
            lds_f64_if(q < C.m.y, s_ring + (unsigned)C.src[q], xv[q]);
        }
        // 2. the next levels' task data (independent of this level's values)
        load_task(Nx, hi + slot);
        const int4 mm = load_meta(hi1 + slot, hi2);
        // 3. the ordered chain (sc.py:261-262 sequential axpy order, or the
        //    OpenBLAS ddot order for < 16 entries, sc.py:291)
        double acc = C.acc;
        if (!(MODE & 1)) {
            double pr[N];
#pragma unroll
            for (int q = 0; q < N; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(C.v[q], xv[q]) : 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) acc = __dsub_rn(acc, pr[q]);
        } else {
            double dot = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) dot = fma(C.v[q], xv[q], dot);
            acc = __dsub_rn(acc, dot);  // len 0: acc - (+0) = acc, also for -0
        }
        // 4. exact division (see exact_div), branch-free
        if (kDiag) {
            const double d = C.dr.x, y = C.dr.y;
            const double q0 = __dmul_rn(acc, y);
            const double r = fma(-q0, d, acc);
            const double q1 = fma(r, y, q0);
            const unsigned e = ((unsigned)__double2hiint(acc) >> 20) & 0x7ffu;
            const bool aok = e - 524u <= 998u;  // 2^-499 <= |acc| < 2^500
            const bool bad = C.m.x >= 0 && (y == 0.0 || (!aok && acc != 0.0));
            double res = aok ? q1 : q0;  // acc == 0: q0 = +-0 with the quotient's sign
            if (__any_sync(0xffffffffu, bad)) {
                if (bad) res = ieee_div(acc, d);
            }
            if (C.m.x >= 0) acc = res;
        }
        // 5. publish
        sts_f64_if(C.m.x != -2, s_ring + (unsigned)(t & (kRing - 1)) * 8, acc);
        stg_f64_if(C.m.x >= 0, x + (C.m.x >= 0 ? C.m.x : 0), acc);
        asm volatile("bar.sync 1, %0;" ::"n"(kLeanConsumers) : "memory");
        C.m = mm;  // C now waits for level l + 2
        lo = hi;
        hi = hi1;
        hi1 = hi2;
    };

    LeanTask<N> A, Bt;
    await_chunk((lvl[2] - 1 >= 0 ? lvl[2] - 1 : 0) >> lgch);
    A.m = load_meta(lo + slot, hi);
    load_task(A, lo + slot);
    Bt.m = load_meta(hi + slot, hi1);
    int l = 0;
    while (l < nlev) {
        // segment: level l is in registers; iteration l' reads positions
        // below lvl[l' + 3].  Chunks wholly before level l + 1 are done with.
        release_below(hi >> lgch);
        await_chunk((lvl[l + 4] - 1) >> lgch);  // the next pair
        const int ready_end = (ready + 1) << lgch;
        int lend = l;
        while (lend + 2 <= nlev && lvl[lend + 4] <= ready_end) lend += 2;
        if (lend == l) {  // the last level (nlev odd)
            level(l, A, Bt);
            ++l;
            continue;
        }
        for (; l < lend; l += 2) {
            level(l, A, Bt);
            level(l + 1, Bt, A);
        }
    }
}

using LeanKernel = void (*)(TriDev, double *, Gate);

template <int MODE>
LeanKernel lean_kernel(int n) {
    switch (n) {
        case 1: return k_trsv_lean<MODE, 1>;
        case 2: return k_trsv_lean<MODE, 2>;
        case 3: return k_trsv_lean<MODE, 3>;
        case 4: return k_trsv_lean<MODE, 4>;
        case 5: return k_trsv_lean<MODE, 5>;
        case 6: return k_trsv_lean<MODE, 6>;
        case 7: return k_trsv_lean<MODE, 7>;
        case 8: return k_trsv_lean<MODE, 8>;
        case 9: return k_trsv_lean<MODE, 9>;
        case 10: return k_trsv_lean<MODE, 10>;
        case 11: return k_trsv_lean<MODE, 11>;
        case 12: return k_trsv_lean<MODE, 12>;
        case 13: return k_trsv_lean<MODE, 13>;
        case 14: return k_trsv_lean<MODE, 14>;
        case 15: return k_trsv_lean<MODE, 15>;
        case 16: return (MODE & 1) ? nullptr : k_trsv_lean<MODE, 16>;
        default: return nullptr;
    }
}

LeanKernel lean_kernel_for(int mode, int n) {
    switch (mode) {
        case 0: return lean_kernel<0>(n);
        case 1: return lean_kernel<1>(n);
        case 2: return lean_kernel<2>(n);
        default: return lean_kernel<3>(n);
    }
}

}  // namespace

int prepare_trsv_lean(int64_t smem_bytes) {
    static int granted = 48 * 1024;  // attributes only ever grow: every schedule keeps its launch valid
    const int smem = (int)smem_bytes;
    if (smem > granted) {
        for (int mode = 0; mode < 4; ++mode)
            for (int n = 1; n <= (int)kLeanMaxN; ++n) {
                LeanKernel k = lean_kernel_for(mode, n);
                if (k) RSB_TRY_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            }
        granted = smem;
    }
    return RSB_OK;
}

int launch_trsv_lean(rsb_ctx *ctx, const TriSched &T, const TriDev &v, double *x, Gate g) {
    LeanKernel k = lean_kernel_for(T.mode, T.lean_n);
    if (!k) {
        set_error("no lean triangular kernel for mode %d, n %d", T.mode, T.lean_n);
        return RSB_ESTATE;
    }
    const size_t smem = (size_t)lean_smem_bytes(T.stage_ch, T.stage_emax, T.diag != nullptr, T.nlevels);
    k<<<1, kLeanThreads, smem, ctx->stream>>>(v, x, g);
    return RSB_OK;
}

}  // namespace rsb
