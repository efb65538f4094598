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
//   - task data arrives by 1-D TMA bulk copies into kStageBufs chunk buffers,
//     issued by a producer warp that takes part in the level barrier: it
//     lets the consumers into a level only once the chunks that level
//     prefetches from have landed, and refills a buffer as soon as the
//     barriers show its chunk is done with -- the consumers never wait on
//     an mbarrier or release a buffer;
//   - two task buffers alternate (level loop unrolled by two), so nothing is
//     copied between registers.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

// W consumer warps (one 32-position slice each per level, W = widest level / 32)
// and one producer warp: warp W, or warp 3 when W = 4 (the rarely used 4th
// slice then runs on warp 4, sharing SMSP 0 instead of the busiest slice)
constexpr int kLeanConsumers = 128;
constexpr int kLeanThreads = kLeanConsumers + 32;
static_assert(kLeanMaxWidth == kLeanConsumers, "one task per consumer thread and level");

// predicated global store (no branch)
__device__ __forceinline__ void stg_f64_if(bool p, double *a, double v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(a), "d"(v),
                 "r"((int)p)
                 : "memory");
}

// IEEE division for the rare operands outside the exact range, out of line
// so that the compiler cannot hoist its reciprocal iteration onto every
// level's critical path
__device__ __noinline__ double ieee_div(double a, double d) { return __ddiv_rn(a, d); }

template <int NS>
struct LeanTask {
    int row;     // unknown written (-1 padding position, -2 no task)
    double acc;  // right-hand side (gathered)
    double2 dr;  // {diag, RN(1/diag)}; 1/diag = 0 marks a diagonal outside the exact range
    int src[NS];  // ring byte offsets (the zero slot past the task's length)
    double v[NS];
};

__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds_v4(unsigned a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// four ring offsets, rebased to absolute shared addresses inside the asm (the
// compiler cannot sink the adds back onto the loads that use them)
__device__ __forceinline__ int4 lds_v4_rebase(unsigned a, unsigned base) {
    int4 v;
    asm volatile(
        "{\n ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];\n add.s32 %0, %0, %5;\n add.s32 %1, %1, %5;\n"
        " add.s32 %2, %2, %5;\n add.s32 %3, %3, %5;\n}"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "r"(a), "r"(base));
    return v;
}
__device__ __forceinline__ void sts_f64_if(bool p, unsigned a, double v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}" ::"r"(a), "d"(v),
                 "r"((int)p)
                 : "memory");
}
// the same with a compile-time byte offset folded into the instruction
template <int OFF>
__device__ __forceinline__ int4 lds_v4_rebase_at(unsigned a, unsigned base) {
    int4 v;
    asm volatile(
        "{\n ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+%6];\n add.s32 %0, %0, %5;\n add.s32 %1, %1, %5;\n"
        " add.s32 %2, %2, %5;\n add.s32 %3, %3, %5;\n}"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "r"(a), "r"(base), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ double2 lds_v2f64_at(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ int4 lds_v4_at(unsigned a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a), "n"(OFF));
    return v;
}
template <int Q, int NQ_>
struct SrcQuads {
    template <class S>
    __device__ __forceinline__ static void run(S &st, unsigned a, unsigned base) {
        const int4 s4 = lds_v4_at<Q * 512>(a);
        st.src[4 * Q] = s4.x;
        st.src[4 * Q + 1] = s4.y;
        st.src[4 * Q + 2] = s4.z;
        st.src[4 * Q + 3] = s4.w;
        SrcQuads<Q + 1, NQ_>::run(st, a, base);
    }
};
template <int NQ_>
struct SrcQuads<NQ_, NQ_> {
    template <class S>
    __device__ __forceinline__ static void run(S &, unsigned, unsigned) {}
};
template <int Q, int NP_>
struct ValPairs {
    template <class S>
    __device__ __forceinline__ static void run(S &st, unsigned a) {
        const double2 v2 = lds_v2f64_at<Q * 512>(a);
        st.v[2 * Q] = v2.x;
        st.v[2 * Q + 1] = v2.y;
        ValPairs<Q + 1, NP_>::run(st, a);
    }
};
template <int NP_>
struct ValPairs<NP_, NP_> {
    template <class S>
    __device__ __forceinline__ static void run(S &, unsigned) {}
};
__device__ __forceinline__ double2 lds_v2f64(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
template <int MODE, int N>
__global__ void __launch_bounds__(kLeanThreads) k_trsv_lean(TriDev T, double *x, Gate g) {
    // Launched as a programmatic dependent of k_gather_pos: everything up to
    // griddepcontrol.wait below touches only the schedule (static since the
    // analysis) and shared memory, so it overlaps the gather; the gate, the
    // gathered right-hand side and x are touched only after the wait.
    constexpr bool kDiag = (MODE & 2) != 0;
    constexpr int NS = 4 * ((N + 3) / 4), NQ = NS / 4, NP = NS / 2;
    __shared__ __align__(16) double ring[kRing + 2];  // values by task position; ring[kRing] = 0
    __shared__ __align__(16) int zsrc[NS * 32];       // sources of a lane without a task: the zero slot
    extern __shared__ __align__(16) unsigned char smem[];
    const int CH = T.stage_ch, lgch = T.stage_lgch;
    unsigned char *bufs = smem;
    const unsigned o_row = (unsigned)CH * 8, o_dd = o_row + (unsigned)CH * 4,
                   o_val = o_dd + (kDiag ? (unsigned)CH * 16 : 0u), o_src = o_val + (unsigned)CH * NS * 8,
                   bb = o_src + (unsigned)CH * NS * 4;
    unsigned long long *full = reinterpret_cast<unsigned long long *>(bufs + kStageBufs * (size_t)bb);
    int *lvl = reinterpret_cast<int *>(full + 2 * kStageBufs);
    const int nlev = T.nlevels;
    int2 *ev = reinterpret_cast<int2 *>(lvl + ((nlev + 8) & ~3));
    const long long t_entry = T.prof ? clock64() : 0;
    // level bounds, padded with the end so lvl[l + 3] is always valid, and the
    // producer's event list: kPro loads in flight per thread before any store
    // (one global round trip per kPro * blockDim entries, not per blockDim --
    // U on config 1 has 2,806 levels)
    {
        constexpr int kPro = 8;
        const int nl = nlev + 5, ne = T.lean_nev, stride = (int)blockDim.x;
        for (int i0 = threadIdx.x; i0 < nl; i0 += kPro * stride) {
            int v[kPro];
#pragma unroll
            for (int u = 0; u < kPro; ++u) {
                const int i = i0 + u * stride;
                v[u] = i < nl ? __ldg(T.level_ptr + (i < nlev ? i : nlev)) : 0;
            }
#pragma unroll
            for (int u = 0; u < kPro; ++u)
                if (i0 + u * stride < nl) lvl[i0 + u * stride] = v[u];
        }
        for (int i0 = threadIdx.x; i0 < ne; i0 += kPro * stride) {
            int2 v[kPro];
#pragma unroll
            for (int u = 0; u < kPro; ++u) {
                const int i = i0 + u * stride;
                v[u] = i < ne ? __ldg(T.lean_ev + i) : make_int2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < kPro; ++u)
                if (i0 + u * stride < ne) ev[i0 + u * stride] = v[u];
        }
    }
    for (int i = threadIdx.x; i < NS * 32; i += blockDim.x) zsrc[i] = kRing * 8;
    if (threadIdx.x == 0) {
        ring[kRing] = 0.0;
        for (int b = 0; b < kStageBufs; ++b) mbar_init(&full[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_gather_pos (and all before it) complete
    if (gated(g)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = (int)(blockDim.x >> 5) - 1;  // consumer warps
    const int pwarp = nwarps == 4 ? 3 : nwarps;      // producer warp
    const unsigned nthreads = blockDim.x;            // the level barrier: consumers + producer
    if (warp == pwarp) {
        // Producer, in lockstep with the consumers' level barriers: it passes
        // barrier j only once the chunks that iteration j + 1 prefetches from
        // have landed, and refills a buffer as soon as the barriers show that
        // its chunk is done with -- the consumers never touch a chunk-level
        // barrier.  What to do before which barrier is the host's event list
        // (analysis.cpp), so a level without events costs a compare.
        auto issue = [&](int c) {
            if (lane == 0) {
                const int b = c & (kStageBufs - 1);
                unsigned char *B = bufs + (size_t)b * bb;
                const int64_t p0 = (int64_t)c * CH;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&full[b], bb);
                bulk_g2s(B, T.bpos + p0, CH * 8, &full[b]);
                bulk_g2s(B + o_row, T.task_row + p0, CH * 4, &full[b]);
                if (kDiag) bulk_g2s(B + o_dd, T.ddiag + 2 * p0, CH * 16, &full[b]);
                bulk_g2s(B + o_val, T.rval + p0 * NS, (unsigned)CH * NS * 8, &full[b]);
                bulk_g2s(B + o_src, T.rsrc + p0 * NS, (unsigned)CH * NS * 4, &full[b]);
            }
        };
        int e = 0;
        int2 cur = ev[0];
        long long pwait = 0;
        auto events_at = [&](int j) {
            while (cur.x == j) {
                if (cur.y >= 0) {
                    issue(cur.y);
                } else {
                    const int c = -cur.y - 1;
                    const long long tw = T.prof ? clock64() : 0;
                    mbar_wait_spin(&full[c & (kStageBufs - 1)], (unsigned)((c / kStageBufs) & 1));
                    if (T.prof) pwait += clock64() - tw;
                }
                cur = ev[++e];
            }
        };
        events_at(-1);  // the first buffers; levels 0 and 1 landed
        asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
        for (int j = 0; j < nlev; ++j) {
            events_at(j);
            asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
        }
        if (T.prof && lane == 0) T.prof[6] = pwait;
        return;
    }
    const int slot = warp < pwarp ? (int)threadIdx.x : (int)threadIdx.x - 32;
    // shared-window bases, opaque so they stay in registers (not
    // rematerialised from SR_CgaCtaId every level); the ring's own base is
    // left to the compiler, which keeps it in a uniform register
    unsigned s_ring, s_bufs, s_zsrc, s_lvl;
    asm volatile("mov.u32 %0, %1;" : "=r"(s_ring) : "r"(smem_u32(ring)));
    const unsigned u_ring = smem_u32(ring);
    auto ring_ld = [&](unsigned off) { return lds_f64(u_ring + off); };
    asm volatile("mov.u32 %0, %1;" : "=r"(s_bufs) : "r"(smem_u32(bufs)));
    asm volatile("mov.u32 %0, %1;" : "=r"(s_zsrc) : "r"(smem_u32(zsrc)));
    asm volatile("mov.u32 %0, %1;" : "=r"(s_lvl) : "r"(smem_u32(lvl)));
    // all of the task at position t, unconditionally; a lane without a task
    // (a position past the level) reads its sources from zsrc, the rest is
    // loaded and never published
    // A lane without a task (a position past the level) points every load at
    // zsrc with no lane offset: its warp's loads become single-wavefront
    // broadcasts instead of competing with the busy warps for shared-memory
    // bandwidth, and its sources are the ring's zero slot.
    auto load_task = [&](LeanTask<NS> &S, int t, bool has) {
        const unsigned B = s_bufs + (unsigned)((t >> lgch) & (kStageBufs - 1)) * bb;
        const unsigned loc = (unsigned)(t & (CH - 1)), base = (loc - (unsigned)lane) * NS;
        const int row = lds_s32(has ? B + o_row + loc * 4 : s_zsrc);
        S.row = has ? row : -2;
        S.acc = lds_f64(has ? B + loc * 8 : s_zsrc);
        S.dr = kDiag ? lds_v2f64(has ? B + o_dd + loc * 16 : s_zsrc) : make_double2(1.0, 1.0);
        // one base address per array, the 16-byte groups at immediate offsets;
        // sources stay ring offsets: the ring's base is a uniform register
        // that the ring loads add for free ([R + UR] addressing)
        const unsigned sa = has ? B + o_src + base * 4 + (unsigned)lane * 16 : s_zsrc;
        SrcQuads<0, NQ>::run(S, sa, s_ring);
        ValPairs<0, NP>::run(S, has ? B + o_val + base * 8 + (unsigned)lane * 16 : s_zsrc);
    };

    int lo = lvl[0], hi = lvl[1];
    auto level = [&](int l, LeanTask<NS> &C, LeanTask<NS> &Nx) {
        const int hi1 = lds_s32(s_lvl + (unsigned)(l + 2) * 4);  // end of level l + 1
        const int t = lo + slot;
        // 1. this level's dependency loads (the only loads on the chain)
        double xv[N];
#pragma unroll
        for (int q = 0; q < N; ++q) xv[q] = ring_ld((unsigned)C.src[q]);
        // 2. the next level's task (independent of this level's values)
        load_task(Nx, hi + slot, hi + slot < hi1);
        // 3. the ordered chain (sc.py:261-262 sequential axpy order, or the
        //    OpenBLAS ddot order for < 16 entries, sc.py:291); empty slots
        //    read the zero slot and change nothing
        double acc = C.acc;
        if (!(MODE & 1)) {
            // products off the chain; a skipped entry subtracts +0, which
            // leaves every acc unchanged (also -0 and NaN)
            double pr[N];
#pragma unroll
            for (int q = 0; q < N; ++q) pr[q] = xv[q] != 0.0 ? __dmul_rn(C.v[q], xv[q]) : 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) acc = __dsub_rn(acc, pr[q]);
        } else {
            double dot = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) dot = fma(C.v[q], xv[q], dot);
            acc = __dsub_rn(acc, dot);  // an empty task: acc - (+0) = acc, also for -0
        }
        // 4. exact division (see exact_div), branch-free
        if (kDiag) {
            const double d = C.dr.x, y = C.dr.y;
            const double q0 = __dmul_rn(acc, y);
            const double r = fma(-q0, d, acc);
            const double q1 = fma(r, y, q0);
            const unsigned e = ((unsigned)__double2hiint(acc) >> 20) & 0x7ffu;
            const bool aok = e - 524u <= 998u;  // 2^-499 <= |acc| < 2^500
            const bool bad = C.row >= 0 && (y == 0.0 || (!aok && acc != 0.0));
            double res = aok ? q1 : q0;  // acc == 0: q0 = +-0 with the quotient's sign
            if (__any_sync(0xffffffffu, bad)) {
                if (bad) res = ieee_div(acc, d);
            }
            if (C.row >= 0) acc = res;
        }
        // 5. publish
        sts_f64_if(C.row != -2, s_ring + (unsigned)(t & (kRing - 1)) * 8, acc);
        stg_f64_if(C.row >= 0, x + (C.row >= 0 ? C.row : 0), acc);
        asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
        lo = hi;
        hi = hi1;
    };

    LeanTask<NS> A, Bt;
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");  // levels 0 and 1 have landed
    load_task(A, lo + slot, lo + slot < hi);
    const bool prof = T.prof != nullptr && threadIdx.x == 0;
    const long long tp = prof ? clock64() : 0;
    int l = 0;
    for (; l + 1 < nlev; l += 2) {
        level(l, A, Bt);
        level(l + 1, Bt, A);
    }
    if (l < nlev) level(l, A, Bt);  // the last level when nlev is odd
    if (prof) {
        T.prof[7] = tp - t_entry;  // prologue: entry to the first level
        T.prof[0] = 0;
        T.prof[1] = clock64() - tp;
        T.prof[2] = 1;
        T.prof[3] = 0;
        T.prof[4] = T.nchunks;
        T.prof[5] = nlev;
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
    const size_t smem =
        (size_t)lean_dyn_smem_bytes(T.stage_ch, (T.lean_n + 3) & ~3, T.diag != nullptr, T.nlevels, T.nchunks);
    const int warps = (int)std::min<int64_t>(4, std::max<int64_t>(1, (T.max_width + 31) / 32));
    // programmatic dependent launch: the prologue runs while k_gather_pos
    // (which triggers its dependents on entry) is still working
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32 * (warps + 1));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RSB_TRY_CUDA(cudaLaunchKernelEx(&cfg, k, v, x, g));
    return RSB_OK;
}

}  // namespace rsb
