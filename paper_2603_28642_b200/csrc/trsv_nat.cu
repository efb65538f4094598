// Index-order sync-free triangular solve for wide DAGs whose dependencies are
// mostly far away (config 4: random structure, n = 8e6, 27 / 66 levels).
//
// The level-ordered grid kernel (trsv_wide.cu) visits the unknowns sorted by
// level, so its right-hand side reads and its output stores are 8-byte
// accesses scattered over 64 MB vectors: each costs a 64-byte DRAM access on
// this part (ncu at n = 8e6: 1.8 GB of DRAM traffic for an L1 solve of 0.43 GB
// algorithmic bytes, profiles/ncu_traffic.json).  Index order is a
// topological order too (forward solves ascending, backward descending), and
// in it everything except the dependency gathers streams:
//   - a warp takes 32 consecutive unknowns from a ticket;
//   - their line pointers, right-hand sides and outputs are contiguous;
//   - their entries are one contiguous span of the matrix's own CSR / CSC
//     arrays (no packed copy, no padding), loaded cooperatively into shared
//     memory with coalesced loads;
//   - each lane then polls its dependencies (an output entry is its own
//     completion flag: sentinel NaN filled before the solve), records the
//     values next to the entries in shared memory and, once all are there,
//     runs the reference's per-task chain in order and publishes.
// A span longer than the warp's shared-memory window is worked through in
// passes over consecutive lane ranges.  Deadlock-free: every dependency of a
// taken slice lies in a slice taken earlier (held by a resident warp) or in a
// lower lane of the same slice.
//
// Chosen by the analysis when few dependencies are near in index distance
// (devsetup.cu); bit-identical to every other solve kernel (same per-task
// operation order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device_common.cuh"
#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kNatBlock = 256;
constexpr int kNatWarps = kNatBlock / 32;
constexpr unsigned kNatMinBackoffNs = 32, kNatMaxBackoffNs = 256;

__device__ __forceinline__ void nat_poll_if(bool p, const double *a, unsigned long long &v) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.relaxed.gpu.global.b64 %0, [%1];\n}"
                 : "+l"(v)
                 : "l"(a), "r"((int)p));
}

__device__ __forceinline__ void nat_publish(double *p, double v) {
    unsigned long long b = __double_as_longlong(v);
    if (b == kSentinel) b = 0x7FF8000000000000ull;  // a computed NaN with the sentinel's bits stays a NaN
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}

// bytes of shared memory per staged entry: value, column, and for the dot
// order (FMA of the unrounded operands) the dependency's value; the
// sequential order stores the rounded product over the value instead
__host__ __device__ constexpr int nat_entry_bytes(int mode) { return (mode & 1) ? 20 : 12; }

// the gate, read once before a static-schedule solve: every warp of the launch
// must agree (a warp that skipped its slices would leave others waiting)
__global__ void k_nat_gate_snap(Gate g, unsigned long long *snap) { *snap = gated(g) ? 1ull : 0ull; }

// STATIC: slices round-robin over the launch's warps (cooperative launch,
// every warp resident) instead of a ticket, so a warp knows its next slice
// and loads that slice's line pointers and right-hand side while it works
// on the current one.  Progress: the lowest unfinished slice's owner is
// working on it, and its dependencies lie in lower slices.
struct NatSlice {
    int elo, ehi;  // the lane's line: entries [elo, ehi) of the matrix arrays
    double acc;    // its right-hand side
};

__device__ __forceinline__ NatSlice nat_slice_load(const NatSrc &s, int n, const VecIn &a, const double *c, int w,
                                                   int nsl, int lane, double *rhs_copy = nullptr) {
    NatSlice r{0, 0, 0.0};
    if (w >= nsl) return r;
    const int q = w * 32 + lane;
    if (q < n) {
        const int t = s.forward ? q : n - 1 - q;
        r.elo = __ldg(s.ptr + t);
        r.ehi = __ldg(s.ptr + t + 1);
        r.acc = a.g ? a.p[a.g[t + a.off]] : a.p[t + a.off];
        if (rhs_copy) rhs_copy[t] = r.acc;  // the gathered a(t), contiguous, for a later solve of the chain
        if (c) r.acc = __dadd_rn(r.acc, c[t]);
    } else {  // past the end (last slice only): an empty line at the span's edge
        r.elo = r.ehi = __ldg(s.ptr + (s.forward ? n : 0));
    }
    return r;
}

template <int MODE, int MINB, bool STATIC>
__global__ void __launch_bounds__(kNatBlock, MINB) k_trsv_nat(NatSrc s, int n, VecIn a, const double *c, double *x,
                                                          unsigned long long *ticket, int cap, unsigned max_backoff,
                                                          unsigned min_backoff, Gate g, double *fill,
                                                          double *rhs_copy) {
    if (fill) {
        // this block's share of the sentinel fill of the chain's next output
        // (TrsvChain): before the gate, so the vector is filled whatever the
        // status says; the stores drain while the slices below wait on their
        // dependencies
        const int64_t per = (((int64_t)n + gridDim.x - 1) / gridDim.x + 31) & ~(int64_t)31;
        const int64_t lo = blockIdx.x * per, hi = min((int64_t)n, lo + per);
        const double sent = __longlong_as_double((long long)kSentinel);
        for (int64_t i = lo + threadIdx.x; i < hi; i += kNatBlock) fill[i] = sent;
    }
    if (STATIC) {
        if (*(volatile const unsigned long long *)ticket) return;  // the gate's snapshot
    } else if (gated(g)) {
        return;
    }
    constexpr bool kKeepX = (MODE & 1) != 0;
    extern __shared__ __align__(16) unsigned char nat_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sv = reinterpret_cast<double *>(nat_smem) + (size_t)warp * cap * (kKeepX ? 2 : 1);
    double *sx = sv + cap;  // kKeepX only
    int *sc = reinterpret_cast<int *>(reinterpret_cast<double *>(nat_smem) + (size_t)kNatWarps * cap * (kKeepX ? 2 : 1)) +
              (size_t)warp * cap;
    const int nsl = (n + 31) / 32;
    const unsigned full = 0xffffffffu;
    const int wstride = gridDim.x * kNatWarps;
    int w = STATIC ? blockIdx.x * kNatWarps + warp : 0;
    NatSlice nx = STATIC ? nat_slice_load(s, n, a, c, w, nsl, lane, rhs_copy) : NatSlice{0, 0, 0.0};
    for (;; w += wstride) {
        if (!STATIC) {
            if (lane == 0) w = (int)atomicAdd(ticket, 1ull);
            w = __shfl_sync(full, w, 0);
        }
        if (w >= nsl) break;
        const NatSlice cur = STATIC ? nx : nat_slice_load(s, n, a, c, w, nsl, lane, rhs_copy);
        if (STATIC) nx = nat_slice_load(s, n, a, c, w + wstride, nsl, lane, rhs_copy);  // in flight during this slice
        const int q = w * 32 + lane;
        const bool valid = q < n;
        const int t = s.forward ? q : n - 1 - q;
        // unknowns of this slice: [tlo, thi]
        const int tlo = s.forward ? w * 32 : n - 32 - w * 32, thi = tlo + 31;
        const int elo = cur.elo, ehi = cur.ehi;
        const int len = (ehi - elo) - s.first_off - s.last_off;
        const int base = s.step > 0 ? elo + s.first_off : ehi - 1 - s.last_off;  // entry k at base + step * k
        int la = 0;
        while (la < 32) {
            // lanes [la, lb): the longest run whose span fits the window
            const int a_lo = __shfl_sync(full, elo, la), a_hi = __shfl_sync(full, ehi, la);
            const int span_to_me = s.forward ? ehi - a_lo : a_hi - elo;
            const unsigned over = __ballot_sync(full, lane >= la && span_to_me > cap);
            const int lb = over ? __ffs(over) - 1 : 32;
            const int b_lo = __shfl_sync(full, elo, lb - 1), b_hi = __shfl_sync(full, ehi, lb - 1);
            const int S0 = s.forward ? a_lo : b_lo, S1 = s.forward ? b_hi : a_hi;
            // The span, entry-parallel (lane i: entries i, i + 32, ...): coalesced
            // loads, then every dependency polled once -- most are ready (far
            // behind) and are recorded next to their entry.  Entries pointing into
            // this slice (its diagonals, dependencies between its lanes) cannot be
            // ready yet and are left for the chain.
            const int32_t *gi = s.idx + S0;
            const double *gv = s.val + S0;
            const int span = S1 - S0;
            constexpr int kU = MINB >= 8 ? 2 : 4;  // entries in flight per lane (fewer: fewer registers, more warps)
            for (int i0 = lane; i0 < span; i0 += 32 * kU) {
                int ci[kU];
                double vi[kU];
                unsigned long long pv[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const bool in = i0 + u * 32 < span;
                    ci[u] = in ? __ldcs(gi + i0 + u * 32) : -1;
                    vi[u] = in ? __ldcs(gv + i0 + u * 32) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    pv[u] = kSentinel;
                    const bool ask = ci[u] >= 0 && (ci[u] < tlo || ci[u] > thi);
                    nat_poll_if(ask, x + (ask ? ci[u] : 0), pv[u]);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if (i0 + u * 32 >= span) continue;
                    const bool got = pv[u] != kSentinel;
                    const double xv = __longlong_as_double((long long)pv[u]);
                    sc[i0 + u * 32] = got ? -1 : ci[u];
                    if (kKeepX) {
                        sv[i0 + u * 32] = vi[u];
                        if (got) sx[i0 + u * 32] = xv;
                    } else {
                        // the reference skips zero operands (sc.py:262); acc - (+0.0) == acc
                        // bit for bit, so a skipped entry's product is recorded as +0.0
                        sv[i0 + u * 32] = got ? (xv != 0.0 ? __dmul_rn(vi[u], xv) : 0.0) : vi[u];
                    }
                }
            }
            __syncwarp();
            // the reference's chain in entry order, resumed each round where the
            // first missing operand stopped it (polled again there)
            const bool mine = valid && lane >= la && lane < lb;
            bool done = !mine;
            int k = 0, sl = base - S0;
            double r = cur.acc, dot = 0.0;
            unsigned backoff = 0;
            for (;;) {
                bool progress = false;
                if (!done) {
                    const int kin = k;
                    while (k < len) {
                        const int cc = sc[sl];
                        double p = sv[sl];
                        if (kKeepX) {
                            double xv;
                            if (cc >= 0) {
                                unsigned long long pv = kSentinel;
                                nat_poll_if(true, x + cc, pv);
                                if (pv == kSentinel) break;
                                xv = __longlong_as_double((long long)pv);
                            } else {
                                xv = sx[sl];
                            }
                            dot = fma(p, xv, dot);
                        } else {
                            if (cc >= 0) {
                                unsigned long long pv = kSentinel;
                                nat_poll_if(true, x + cc, pv);
                                if (pv == kSentinel) break;
                                const double xv = __longlong_as_double((long long)pv);
                                p = xv != 0.0 ? __dmul_rn(p, xv) : 0.0;
                            }
                            r = __dsub_rn(r, p);
                        }
                        ++k;
                        sl += s.step;
                    }
                    progress = k != kin;
                    if (k == len) {
                        if (kKeepX && len > 0) r = __dsub_rn(r, dot);  // < 16 entries: the scalar BLAS order (checked at analysis)
                        if (MODE & 2) r = __ddiv_rn(r, sv[(s.diag_at == 0 ? elo : ehi - 1) - S0]);
                        nat_publish(x + t, r);
                        done = true;
                        progress = true;
                    }
                }
                if (!__any_sync(full, !done)) break;
                if (!__any_sync(full, progress)) {
                    backoff = backoff ? min(backoff * 2, max_backoff) : min_backoff;
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



using NatKernel = void (*)(NatSrc, int, VecIn, const double *, double *, unsigned long long *, int, unsigned, unsigned,
                           Gate, double *, double *);

// (A pipelined static-schedule variant -- a warp owning slices w, w + W, ... and
// running three stages across them: pointers and right-hand side of s + 2W by
// plain loads, the span of s + W into a second shared-memory window by 4/8-byte
// cp.async, polls / chains / publish of s -- measured slower at every warp count:
// L1 0.92 / 0.54 / 0.42 / 0.36 ms at 8 / 16 / 24 / 32 warps per SM, U 0.69 at best
// against 0.35 / 0.54 for this kernel (profiles/r02b/trsv_sweep_nat_pipe.json).  With
// every load prefetched a slice still takes 5-7 us: what a slice waits for is its
// near dependencies -- 4.7 polling rounds of about a microsecond -- not its loads.)

// MINB resident blocks per SM the registers are budgeted for (4: 64 registers,
// 6: 40, 8: 32 with spills)
template <int MINB, bool STATIC>
NatKernel nat_kernel_b(int mode) {
    switch (mode & 3) {
        case 0: return k_trsv_nat<0, MINB, STATIC>;
        case 1: return k_trsv_nat<1, MINB, STATIC>;
        case 2: return k_trsv_nat<2, MINB, STATIC>;
        default: return k_trsv_nat<3, MINB, STATIC>;
    }
}
constexpr int kNatMinBlocks = 6;  // measured at n = 8e6: L1 0.351 / L1^T 0.294 / U 0.537 ms (4: 0.375 / 0.301 / 0.603)
constexpr bool kNatStatic = false;
NatKernel nat_kernel(int mode, int minb, bool st) {
    if (st) return minb <= 4 ? nat_kernel_b<4, true>(mode) : nat_kernel_b<6, true>(mode);
    if (minb >= 8) return nat_kernel_b<8, false>(mode);
    return minb <= 4 ? nat_kernel_b<4, false>(mode) : nat_kernel_b<6, false>(mode);
}

}  // namespace

size_t trsv_nat_smem(int mode, int cap) { return (size_t)kNatWarps * cap * nat_entry_bytes(mode); }

int launch_trsv_nat(rsb_ctx *ctx, const TriSched &T, const TriDev &v, VecIn a, const double *c, double *x, Gate g,
                    bool prefilled, double *fill_next, double *rhs_copy) {
    const char *em = getenv("RSB_NAT_MINB");  // experiments
    const int minb = em ? atoi(em) : kNatMinBlocks;
    const char *es = getenv("RSB_NAT_STATIC");
    const bool st = es ? atoi(es) != 0 : kNatStatic;
    const int mi = (minb <= 4 ? 0 : (minb >= 8 && !st ? 4 : 1)) + (st ? 2 : 0);
    NatKernel k = nat_kernel(T.mode, minb, st);
    const size_t smem = trsv_nat_smem(T.mode, T.nat_cap);
    static size_t granted[4][5] = {};  // grow-only opt-in above 48 KB
    if (smem > 48 * 1024 && smem > granted[T.mode & 3][mi]) {
        RSB_TRY_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        granted[T.mode & 3][mi] = smem;
    }
    int occ = 0, sms = 0;
    RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kNatBlock, smem));
    RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    occ = std::max(occ, 1);
    if (const char *eo = getenv("RSB_NAT_OCC")) occ = std::max(1, std::min(occ, atoi(eo)));  // experiments
    const char *eb = getenv("RSB_NAT_BACKOFF");
    const unsigned max_backoff = eb ? (unsigned)std::max(32, atoi(eb)) : kNatMaxBackoffNs;
    const char *emb = getenv("RSB_NAT_MINBACKOFF");
    const unsigned min_backoff = emb ? (unsigned)std::max(8, atoi(emb)) : kNatMinBackoffNs;
    const int64_t nsl = ((int64_t)T.n + 31) / 32;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, (nsl + kNatWarps - 1) / kNatWarps));
    if (!prefilled) RSB_TRY(launch_fill(ctx, x, T.n, kSentinel, g));
    if (st) {
        k_nat_gate_snap<<<1, 1, 0, ctx->stream>>>(g, v.ticket);
        RSB_TRY_CUDA(cudaGetLastError());
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kNatBlock);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // every warp resident: the round-robin schedule needs it
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        RSB_TRY_CUDA(cudaLaunchKernelEx(&cfg, k, T.nat, T.n, a, c, x, v.ticket, T.nat_cap, max_backoff, min_backoff, g,
                                        fill_next, rhs_copy));
        return RSB_OK;
    }
    k<<<grid, kNatBlock, smem, ctx->stream>>>(T.nat, T.n, a, c, x, v.ticket, T.nat_cap, max_backoff, min_backoff, g,
                                              fill_next, rhs_copy);
    return RSB_OK;
}

}  // namespace rsb
