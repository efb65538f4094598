// Dense-coupling preconditioner construction on the device:
//   build_y_explicit        pc.py:55-82    Y = L2 L1^{-1}, row i of Y solves
//                                          L1^T y = (row i of L2) by a sparse-RHS
//                                          solve in DFS reach order (sc.py:328-397)
//   _gram_plus_identity     pc.py:85-92    S = I + Y Y^T (lower triangle)
//   dense_cholesky_factorize sc.py:585-604 unblocked right-looking sweep
//
// Parity: Y is bit-identical to the reference (same reach order per row, the
// same multiply-then-subtract updates).  The Cholesky factor is bit-identical
// given the same S: a blocked right-looking sweep subtracts, per element, the
// products of columns j = 0, 1, ... in increasing order, exactly as the
// reference's rank-1 updates do.  S = I + Y Y^T is the one step whose
// reference order (numpy's `yd @ yd.T`, an OpenBLAS syrk/gemm) is not
// reproduced: it is a fixed-order FP64 product here (deterministic), within
// rounding of the reference (tests: <= 1e-13 relative).
//
// Layout: Y as CSR (rows ascending columns) and CSC, int32; dense panels of Y
// column-major (s x kc); S and its factor s x s column-major.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "device_common.cuh"
#include "rsb_internal.h"

struct rsb_dbuild {
    rsb_ctx *ctx = nullptr;
    int64_t s = 0, n = 0, nnz = 0;
    int32_t *y_rptr = nullptr, *y_ridx = nullptr;  // CSR of Y
    double *y_rval = nullptr;
    size_t y_cap = 0;
    int32_t *y_cptr = nullptr, *y_cidx = nullptr;  // CSC of Y
    double *y_cval = nullptr;
    double *S = nullptr;  // I + Y Y^T, symmetric (kept when asked)
    double *F = nullptr;  // lower Cholesky factor, upper zero
    double sec_y = 0, sec_gram = 0, sec_chol = 0;
};

namespace rsb {
namespace {

constexpr int kT = 256;
inline int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 32)); }
#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

struct Bufs {
    rsb_ctx *ctx;
    std::vector<std::pair<void *, size_t>> v;
    explicit Bufs(rsb_ctx *c) : ctx(c) {}
    template <class T>
    int get(T **p, size_t count) {
        const size_t b = std::max<size_t>(1, count) * sizeof(T);
        RSB_TRY(dev_alloc(ctx, (void **)p, b));
        v.emplace_back(*p, b);
        return RSB_OK;
    }
    ~Bufs() {
        cudaStreamSynchronize(ctx->stream);
        for (auto &b : v) dev_free(ctx, b.first, b.second);
    }
};

// ---- Y rows: one warp per row of L2 ------------------------------------------
// Scratch of one row slot (n entries each): DFS stack (node, cursor), the
// post-order, the dense work vector x and the row's output (column, value).
struct YSlot {
    uint32_t *gmark;  // global visit bitmap (when it does not fit shared memory), n bits per slot
    int32_t *sn, *sc, *topo, *ocol;
    double *x, *oval;
    int32_t *ocnt;
    int64_t words;  // bitmap words per slot
};

template <bool SMEM>
__global__ void __launch_bounds__(32) k_y_rows(const int32_t *__restrict__ lp, const int32_t *__restrict__ li,
                                               const double *__restrict__ lv, const int32_t *__restrict__ bp,
                                               const int32_t *__restrict__ bi, const double *__restrict__ bv,
                                               int64_t row0, int64_t nrows, int32_t n, YSlot w) {
    extern __shared__ uint32_t smark[];
    const int64_t slot = blockIdx.x;
    if (slot >= nrows) return;
    const int lane = threadIdx.x;
    const int64_t i = row0 + slot;
    uint32_t *mark = SMEM ? smark : w.gmark + slot * w.words;
    int32_t *sn = w.sn + slot * (int64_t)n, *sc = w.sc + slot * (int64_t)n, *topo = w.topo + slot * (int64_t)n;
    int32_t *ocol = w.ocol + slot * (int64_t)n;
    double *x = w.x + slot * (int64_t)n, *oval = w.oval + slot * (int64_t)n;
    for (int64_t q = lane; q < w.words; q += 32) mark[q] = 0u;
    __syncwarp();
    const int lo = bp[i], hi = bp[i + 1];
    // reach_pattern (sc.py:328-362): iterative DFS from the seeds in pattern
    // order, children in stored order, post-order appended; reversed later
    int T = 0;
    if (lane == 0) {
        for (int k = lo; k < hi; ++k) {
            const int sd = bi[k];
            if (mark[sd >> 5] & (1u << (sd & 31))) continue;
            mark[sd >> 5] |= 1u << (sd & 31);
            int depth = 0;
            sn[0] = sd;
            sc[0] = lp[sd];
            while (depth >= 0) {
                const int node = sn[depth];
                int cur = sc[depth];
                const int end = lp[node + 1];
                bool adv = false;
                while (cur < end) {
                    const int child = li[cur];
                    ++cur;
                    if (child != node && !(mark[child >> 5] & (1u << (child & 31)))) {
                        mark[child >> 5] |= 1u << (child & 31);
                        sc[depth] = cur;
                        ++depth;
                        sn[depth] = child;
                        sc[depth] = lp[child];
                        adv = true;
                        break;
                    }
                }
                if (!adv) {
                    topo[T++] = node;
                    --depth;
                }
            }
        }
    }
    T = __shfl_sync(0xffffffffu, T, 0);
    __syncwarp();
    // numeric solve (sc.py:377-397): x = 0 on the reach, x[pattern] = b, then
    // nodes in topological order (reversed post-order); unit diagonal
    for (int t = lane; t < T; t += 32) x[topo[t]] = 0.0;
    __syncwarp();
    for (int k = lo + lane; k < hi; k += 32) x[bi[k]] = bv[k];
    __syncwarp();
    for (int t = T - 1; t >= 0; --t) {
        const int node = topo[t];
        const double xv = x[node];
        if (xv != 0.0) {
            const int a = lp[node], b = lp[node + 1];
            for (int q = a + lane; q < b; q += 32) {
                const int c = li[q];
                if (c != node) x[c] = __dsub_rn(x[c], __dmul_rn(lv[q], xv));
            }
        }
        __syncwarp();
    }
    // pattern = sorted reach; zeros dropped (pc.py:70-71): scan the bitmap
    // in index order, 32 words (1024 indices) per pass
    int count = 0;
    for (int64_t q0 = 0; q0 < w.words; q0 += 32) {
        const int64_t q = q0 + lane;
        uint32_t bits = q < w.words ? mark[q] : 0u;
        uint32_t keep = 0u;
        for (uint32_t b = bits; b; b &= b - 1) {
            const int j = (int)(q * 32 + __ffs(b) - 1);
            if (x[j] != 0.0) keep |= b & (~b + 1);
        }
        const int c = __popc(keep);
        int pre = c;
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, pre, d);
            if (lane >= d) pre += v;
        }
        int pos = count + pre - c;
        for (uint32_t b = keep; b; b &= b - 1) {
            const int j = (int)(q * 32 + __ffs(b) - 1);
            ocol[pos] = j;
            oval[pos] = x[j];
            ++pos;
        }
        count += __shfl_sync(0xffffffffu, pre, 31);
    }
    if (lane == 0) w.ocnt[slot] = count;
}

__global__ void k_y_compact(const int32_t *ocnt, const int32_t *ooff, int64_t nrows, int64_t base, int32_t n,
                            const int32_t *ocol, const double *oval, int32_t *rptr_chunk, int32_t *ridx,
                            double *rval) {
    const int64_t slot = blockIdx.x;
    if (slot >= nrows) return;
    const int c = ocnt[slot];
    const int64_t dst = base + ooff[slot];
    if (threadIdx.x == 0) rptr_chunk[slot] = (int32_t)dst;
    for (int k = threadIdx.x; k < c; k += blockDim.x) {
        ridx[dst + k] = ocol[slot * (int64_t)n + k];
        rval[dst + k] = oval[slot * (int64_t)n + k];
    }
}

// CSR -> CSC (rows ascending inside a column: a stable sort by column)
__global__ void k_row_of(const int32_t *rptr, int64_t nrows, int32_t *row_of) {
    GRID_STRIDE(r, nrows) {
        for (int32_t k = rptr[r]; k < rptr[r + 1]; ++k) row_of[k] = (int32_t)r;
    }
}
__global__ void k_iota(int32_t *v, int64_t n) {
    GRID_STRIDE(i, n) v[i] = (int32_t)i;
}
__global__ void k_hist(const int32_t *keys, int64_t n, int32_t *cnt) {
    GRID_STRIDE(i, n) atomicAdd(cnt + keys[i], 1);
}
__global__ void k_gather_csc(const int32_t *perm, const int32_t *row_of, const double *rval, int64_t nnz,
                             int32_t *cidx, double *cval) {
    GRID_STRIDE(k, nnz) {
        const int32_t e = perm[k];
        cidx[k] = row_of[e];
        cval[k] = rval[e];
    }
}

// dense column panel [k0, k0 + kc) of Y, column-major s x kc
__global__ void k_densify(const int32_t *cptr, const int32_t *cidx, const double *cval, int64_t k0, int64_t kc,
                          int64_t s, double *P) {
    GRID_STRIDE(q, kc) {
        double *col = P + q * s;
        for (int32_t e = cptr[k0 + q]; e < cptr[k0 + q + 1]; ++e) col[cidx[e]] = cval[e];
    }
}

// ---- S = I + Y Y^T: lower 64 x 64 tiles, optional split over k ---------------
constexpr int kGT = 64;  // tile
constexpr int kGK = 16;  // k slab
__device__ __forceinline__ void tile_of(int64_t t, int64_t &bi, int64_t &bj) {
    // t -> (bi, bj), bi >= bj, row-major over the lower triangle of tiles
    int64_t r = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    bi = r;
    bj = t - r * (r + 1) / 2;
}

__global__ void __launch_bounds__(256) k_syrk(const double *__restrict__ P, int64_t s, int64_t kc, int64_t kper,
                                              double *__restrict__ part) {
    __shared__ double As[kGK][kGT + 1], Bs[kGK][kGT + 1];
    int64_t bi, bj;
    tile_of(blockIdx.x, bi, bj);
    const int64_t i0 = bi * kGT, j0 = bj * kGT;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t ka = blockIdx.y * kper, kb = min(kc, ka + kper);
    double acc[4][4] = {};
    for (int64_t k0 = ka; k0 < kb; k0 += kGK) {
        for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
            const int kk = e / kGT, r = e % kGT;
            const int64_t k = k0 + kk;
            As[kk][r] = (k < kb && i0 + r < s) ? P[k * s + i0 + r] : 0.0;
            Bs[kk][r] = (k < kb && j0 + r < s) ? P[k * s + j0 + r] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = As[kk][tx + 16 * r];
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = Bs[kk][ty + 16 * c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
    double *out = part + (int64_t)blockIdx.y * s * s;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t i = i0 + tx + 16 * r, j = j0 + ty + 16 * c;
            if (i < s && j < s && i >= j) out[j * s + i] = acc[r][c];
        }
}

// G(lower) += sum of the split partials in split order
__global__ void k_gram_acc(double *G, const double *part, int nsplit, int64_t s, int first) {
    GRID_STRIDE(e, s * s) {
        const int64_t i = e % s, j = e / s;
        if (i < j) continue;
        double v = first ? part[e] : G[e] + part[e];
        for (int z = 1; z < nsplit; ++z) v += part[(int64_t)z * s * s + e];
        G[e] = v;
    }
}

// S = tril(G) + tril(G, -1)^T, diagonal + 1 (pc.py:88-91)
__global__ void k_gram_finish(double *G, int64_t s) {
    GRID_STRIDE(e, s * s) {
        const int64_t i = e % s, j = e / s;
        if (i == j) G[e] = G[e] + 1.0;
        else if (i < j) G[e] = G[i * s + j];
    }
}

// ---- Cholesky: blocked right-looking, per-element subtraction order kept -----
constexpr int kCW = 32;  // panel width
__global__ void __launch_bounds__(1024) k_chol_panel(double *g, int64_t s, int64_t j0, int64_t j1, int64_t *bad) {
    __shared__ double dsh;
    __shared__ int stop;
    if (*bad >= 0) return;
    for (int64_t j = j0; j < j1; ++j) {
        if (threadIdx.x == 0) {
            double d = g[j + j * s];
            if (!(d > 0.0) || !isfinite(d)) {
                *bad = j;
                stop = 1;
            } else {
                d = __dsqrt_rn(d);
                g[j + j * s] = d;
                stop = 0;
            }
            dsh = d;
        }
        __syncthreads();
        if (stop) return;
        const double d = dsh;
        for (int64_t i = j + 1 + threadIdx.x; i < s; i += blockDim.x) g[i + j * s] = __ddiv_rn(g[i + j * s], d);
        __syncthreads();
        for (int64_t i = j + 1 + threadIdx.x; i < s; i += blockDim.x) {
            const double gi = g[i + j * s];
            for (int64_t k = j + 1; k < j1 && k <= i; ++k)
                g[i + k * s] = __dsub_rn(g[i + k * s], __dmul_rn(gi, g[k + j * s]));
        }
        __syncthreads();
    }
}

// trailing update of the lower triangle right of the panel [j0, j1):
// g[i,k] -= g[i,j] g[k,j] for j = j0 .. j1-1 in order (rows i >= k >= j1)
__global__ void __launch_bounds__(256) k_chol_trail(double *g, int64_t s, int64_t j0, int64_t j1,
                                                    const int64_t *bad) {
    __shared__ double Pi[kCW][kGT], Pk[kCW][kGT];
    if (*bad >= 0) return;
    int64_t bi, bk;
    tile_of(blockIdx.x, bi, bk);
    const int64_t i0 = j1 + bi * kGT, k0 = j1 + bk * kGT;
    const int W = (int)(j1 - j0);
    for (int e = threadIdx.x; e < W * kGT; e += 256) {
        const int jj = e / kGT, r = e % kGT;
        const int64_t col = (j0 + jj) * s;
        Pi[jj][r] = i0 + r < s ? g[col + i0 + r] : 0.0;
        Pk[jj][r] = k0 + r < s ? g[col + k0 + r] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int64_t k = k0 + ty + 16 * c;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i = i0 + tx + 16 * r;
            if (i >= s || k >= s || i < k) continue;
            double v = g[i + k * s];
            for (int jj = 0; jj < W; ++jj) v = __dsub_rn(v, __dmul_rn(Pi[jj][tx + 16 * r], Pk[jj][ty + 16 * c]));
            g[i + k * s] = v;
        }
    }
}

__global__ void k_tril(double *g, int64_t s) {
    GRID_STRIDE(e, s * s) {
        const int64_t i = e % s, j = e / s;
        if (i < j) g[e] = 0.0;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// In-place lower Cholesky of the s x s column-major g (device), bit-identical
// to dense_cholesky_factorize (sc.py:585-604); upper triangle zeroed.
int chol_factor_device(rsb_ctx *ctx, int64_t s, double *g) {
    if (s == 0) return RSB_OK;
    Bufs b(ctx);
    int64_t *bad = nullptr;
    RSB_TRY(b.get(&bad, 1));
    RSB_TRY_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(int64_t), ctx->stream));  // -1
    for (int64_t j0 = 0; j0 < s; j0 += kCW) {
        const int64_t j1 = std::min<int64_t>(s, j0 + kCW);
        k_chol_panel<<<1, 1024, 0, ctx->stream>>>(g, s, j0, j1, bad);
        ctx->launches += 1;
        const int64_t rest = s - j1;
        if (rest > 0) {
            const int64_t nt = (rest + kGT - 1) / kGT;
            k_chol_trail<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, ctx->stream>>>(g, s, j0, j1, bad);
            ctx->launches += 1;
        }
    }
    k_tril<<<blocks_for(s * s), kT, 0, ctx->stream>>>(g, s);
    ctx->launches += 1;
    RSB_TRY_CUDA(cudaGetLastError());
    int64_t h_bad = -1;
    RSB_TRY_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h_bad >= 0) {
        set_error("matrix is not positive definite (pivot %lld)", (long long)h_bad);
        return RSB_ESINGULAR;
    }
    return RSB_OK;
}

namespace {

size_t budget_bytes() {
    const char *e = getenv("RSB_DBUILD_BUDGET_MB");
    return (size_t)(e ? atoll(e) : 2048) << 20;
}

int build_y(rsb_dbuild *B, rsb_mat *L1, rsb_mat *L2) {
    rsb_ctx *ctx = B->ctx;
    const int64_t s = B->s, n = B->n;
    const int64_t words = (n + 31) / 32;
    const bool smem = words * 4 <= 200 * 1024;
    // slots: per row n * (4 sn + 4 sc + 4 topo + 4 ocol + 8 x + 8 oval) bytes (+ bitmap)
    const size_t per = (size_t)n * 32 + (smem ? 0 : (size_t)words * 4) + 16;
    const int64_t R = std::max<int64_t>(1, std::min<int64_t>(s, (int64_t)(budget_bytes() / per)));
    Bufs b(ctx);
    YSlot w{};
    w.words = words;
    RSB_TRY(b.get(&w.sn, (size_t)R * n));
    RSB_TRY(b.get(&w.sc, (size_t)R * n));
    RSB_TRY(b.get(&w.topo, (size_t)R * n));
    RSB_TRY(b.get(&w.ocol, (size_t)R * n));
    RSB_TRY(b.get(&w.x, (size_t)R * n));
    RSB_TRY(b.get(&w.oval, (size_t)R * n));
    RSB_TRY(b.get(&w.ocnt, (size_t)R));
    if (!smem) RSB_TRY(b.get(&w.gmark, (size_t)R * words));
    int32_t *ooff = nullptr;
    RSB_TRY(b.get(&ooff, (size_t)R));
    size_t scan_bytes = 0;
    RSB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, w.ocnt, ooff, (int)R, ctx->stream));
    char *scan_tmp = nullptr;
    RSB_TRY(b.get(&scan_tmp, scan_bytes));
    RSB_TRY(dev_alloc(ctx, (void **)&B->y_rptr, (size_t)(s + 1) * sizeof(int32_t)));
    B->y_cap = (size_t)std::max<int64_t>(1024, std::min<int64_t>(s * n, 1 << 20));
    RSB_TRY(dev_alloc(ctx, (void **)&B->y_ridx, B->y_cap * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&B->y_rval, B->y_cap * sizeof(double)));
    const int smem_bytes = smem ? (int)(words * 4) : 0;
    if (smem) RSB_TRY_CUDA(cudaFuncSetAttribute(k_y_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
    const rsb::Compressed l1 = L1->csr(), l2 = L2->csr();
    int64_t total = 0;
    for (int64_t r0 = 0; r0 < s; r0 += R) {
        const int64_t nr = std::min<int64_t>(R, s - r0);
        if (smem)
            k_y_rows<true><<<(unsigned)nr, 32, smem_bytes, ctx->stream>>>(l1.ptr, l1.idx, l1.val, l2.ptr, l2.idx, l2.val,
                                                                          r0, nr, (int32_t)n, w);
        else
            k_y_rows<false><<<(unsigned)nr, 32, 0, ctx->stream>>>(l1.ptr, l1.idx, l1.val, l2.ptr, l2.idx, l2.val, r0,
                                                                  nr, (int32_t)n, w);
        RSB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, w.ocnt, ooff, (int)nr, ctx->stream));
        int32_t last[2] = {0, 0};
        RSB_TRY_CUDA(cudaMemcpyAsync(&last[0], ooff + nr - 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
        RSB_TRY_CUDA(cudaMemcpyAsync(&last[1], w.ocnt + nr - 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
        RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
        const int64_t add = (int64_t)last[0] + last[1];
        if (total + add > INT32_MAX) {
            set_error("explicit Y has more than 2^31 entries");
            return RSB_EINVAL;
        }
        if ((size_t)(total + add) > B->y_cap) {
            size_t cap = B->y_cap;
            while (cap < (size_t)(total + add)) cap *= 2;
            int32_t *ni = nullptr;
            double *nv = nullptr;
            RSB_TRY(dev_alloc(ctx, (void **)&ni, cap * sizeof(int32_t)));
            RSB_TRY(dev_alloc(ctx, (void **)&nv, cap * sizeof(double)));
            if (total) {
                RSB_TRY_CUDA(cudaMemcpyAsync(ni, B->y_ridx, total * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
                RSB_TRY_CUDA(cudaMemcpyAsync(nv, B->y_rval, total * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
            }
            RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
            dev_free(ctx, B->y_ridx, B->y_cap * sizeof(int32_t));
            dev_free(ctx, B->y_rval, B->y_cap * sizeof(double));
            B->y_ridx = ni;
            B->y_rval = nv;
            B->y_cap = cap;
        }
        k_y_compact<<<(unsigned)nr, 128, 0, ctx->stream>>>(w.ocnt, ooff, nr, total, (int32_t)n, w.ocol, w.oval,
                                                            B->y_rptr + r0, B->y_ridx, B->y_rval);
        ctx->launches += 3;
        total += add;
    }
    const int32_t t32 = (int32_t)total;
    RSB_TRY_CUDA(cudaMemcpyAsync(B->y_rptr + s, &t32, 4, cudaMemcpyHostToDevice, ctx->stream));
    RSB_TRY_CUDA(cudaGetLastError());
    B->nnz = total;
    // CSC by a stable radix sort of the entries by column
    RSB_TRY(dev_alloc(ctx, (void **)&B->y_cptr, (size_t)(n + 1) * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&B->y_cidx, (size_t)std::max<int64_t>(1, total) * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&B->y_cval, (size_t)std::max<int64_t>(1, total) * sizeof(double)));
    int32_t *row_of, *perm_in, *perm, *keys_out, *cnt;
    RSB_TRY(b.get(&row_of, total));
    RSB_TRY(b.get(&perm_in, total));
    RSB_TRY(b.get(&perm, total));
    RSB_TRY(b.get(&keys_out, total));
    RSB_TRY(b.get(&cnt, n + 1));
    RSB_TRY_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int32_t), ctx->stream));
    if (total) {
        k_row_of<<<blocks_for(s), kT, 0, ctx->stream>>>(B->y_rptr, s, row_of);
        k_iota<<<blocks_for(total), kT, 0, ctx->stream>>>(perm_in, total);
        k_hist<<<blocks_for(total), kT, 0, ctx->stream>>>(B->y_ridx, total, cnt);
        ctx->launches += 3;
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) <= n) ++bits;
        size_t sb = 0;
        RSB_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sb, B->y_ridx, keys_out, perm_in, perm, (int)total, 0,
                                                     bits, ctx->stream));
        char *st = nullptr;
        RSB_TRY(b.get(&st, sb));
        RSB_TRY_CUDA(cub::DeviceRadixSort::SortPairs(st, sb, B->y_ridx, keys_out, perm_in, perm, (int)total, 0, bits,
                                                     ctx->stream));
        k_gather_csc<<<blocks_for(total), kT, 0, ctx->stream>>>(perm, row_of, B->y_rval, total, B->y_cidx, B->y_cval);
        ctx->launches += 1;
    }
    size_t cb = 0;
    RSB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, cb, cnt, B->y_cptr, (int)(n + 1), ctx->stream));
    char *ct = nullptr;
    RSB_TRY(b.get(&ct, cb));
    RSB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(ct, cb, cnt, B->y_cptr, (int)(n + 1), ctx->stream));
    RSB_TRY_CUDA(cudaGetLastError());
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    return RSB_OK;
}

int build_gram(rsb_dbuild *B, double *G) {
    rsb_ctx *ctx = B->ctx;
    const int64_t s = B->s, n = B->n;
    if (s == 0) return RSB_OK;
    Bufs b(ctx);
    const int64_t nt = (s + kGT - 1) / kGT, ntiles = nt * (nt + 1) / 2;
    int64_t kc = std::max<int64_t>(kGK, (int64_t)(budget_bytes() / 2 / (8 * (size_t)s)) / kGK * kGK);
    kc = std::min<int64_t>(kc, std::max<int64_t>(n, 1));
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(64, 296 / ntiles));
    nsplit = (int)std::min<int64_t>(nsplit, std::max<int64_t>(1, (kc + 255) / 256));
    double *P = nullptr, *part = nullptr;
    RSB_TRY(b.get(&P, (size_t)s * kc));
    RSB_TRY(b.get(&part, (size_t)nsplit * s * s));
    bool first = true;
    for (int64_t k0 = 0; k0 < n; k0 += kc) {
        const int64_t w = std::min<int64_t>(kc, n - k0);
        RSB_TRY_CUDA(cudaMemsetAsync(P, 0, (size_t)s * w * sizeof(double), ctx->stream));
        k_densify<<<blocks_for(w), kT, 0, ctx->stream>>>(B->y_cptr, B->y_cidx, B->y_cval, k0, w, s, P);
        const int64_t kper = ((w + nsplit - 1) / nsplit + kGK - 1) / kGK * kGK;
        const int ns = (int)((w + kper - 1) / kper);
        k_syrk<<<dim3((unsigned)ntiles, (unsigned)ns), 256, 0, ctx->stream>>>(P, s, w, kper, part);
        k_gram_acc<<<blocks_for(s * s), kT, 0, ctx->stream>>>(G, part, ns, s, first ? 1 : 0);
        ctx->launches += 3;
        first = false;
    }
    if (n == 0) RSB_TRY_CUDA(cudaMemsetAsync(G, 0, (size_t)s * s * sizeof(double), ctx->stream));
    k_gram_finish<<<blocks_for(s * s), kT, 0, ctx->stream>>>(G, s);
    ctx->launches += 1;
    RSB_TRY_CUDA(cudaGetLastError());
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    return RSB_OK;
}

void dbuild_free(rsb_dbuild *B) {
    rsb_ctx *ctx = B->ctx;
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    const size_t nz = (size_t)std::max<int64_t>(1, B->nnz), ss = (size_t)(B->s * B->s);
    if (B->y_rptr) dev_free(ctx, B->y_rptr, (B->s + 1) * sizeof(int32_t));
    if (B->y_ridx) dev_free(ctx, B->y_ridx, B->y_cap * sizeof(int32_t));
    if (B->y_rval) dev_free(ctx, B->y_rval, B->y_cap * sizeof(double));
    if (B->y_cptr) dev_free(ctx, B->y_cptr, (B->n + 1) * sizeof(int32_t));
    if (B->y_cidx) dev_free(ctx, B->y_cidx, nz * sizeof(int32_t));
    if (B->y_cval) dev_free(ctx, B->y_cval, nz * sizeof(double));
    if (B->S) dev_free(ctx, B->S, ss * sizeof(double));
    if (B->F) dev_free(ctx, B->F, ss * sizeof(double));
}

}  // namespace

// column_scale (sc.py:405-425) on the device: sq_j = reduceat(v * v) = p0 +
// pairwise(p1 ..) per column (numpy's order), norms = sqrt(sq), values /
// norms[column] -- IEEE multiply, add, sqrt and divide, so bit-identical to
// the reference and to the host version (rsb_column_scale).
namespace {
struct SqTerm {
    const double *v;
    __device__ double operator()(int64_t k) const { return __dmul_rn(v[k], v[k]); }
};
__global__ void k_colscale(int64_t ncols, const int64_t *ptr, const double *val, double *scaled, double *norms,
                           int *empty_min) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ncols; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = ptr[j], hi = ptr[j + 1];
        if (hi <= lo) {
            atomicMin(empty_min, (int)j);
            norms[j] = 0.0;
            continue;
        }
        const SqTerm t{val + lo};
        const int64_t m = hi - lo - 1;
        const double s2 = __dadd_rn(t(0), m <= 128 ? pw_leaf(t, 1, m) : Pairwise<25, SqTerm>::sum(t, 1, m));
        const double nj = __dsqrt_rn(s2);
        norms[j] = nj;
        for (int64_t k = lo; k < hi; ++k) scaled[k] = __ddiv_rn(val[k], nj);
    }
}
}  // namespace

}  // namespace rsb

using namespace rsb;

extern "C" {

int rsb_dense_build(rsb_mat *L1, rsb_mat *L2, int what, rsb_dbuild **out) {
    *out = nullptr;
    if (!L1 || !L2 || L1->ctx != L2->ctx) {
        set_error("L1 and L2 must be matrices of one context");
        return RSB_EINVAL;
    }
    if (L1->nrows != L1->ncols || L2->ncols != L1->ncols) {
        set_error("L1 must be n x n and L2 (m-n) x n");
        return RSB_EINVAL;
    }
    if (what < 0 || what > 2) {
        set_error("what must be 0 (Y), 1 (Y and the S factor) or 2 (also keep S)");
        return RSB_EINVAL;
    }
    rsb_ctx *ctx = L1->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    auto *B = new rsb_dbuild();
    B->ctx = ctx;
    B->s = L2->nrows;
    B->n = L1->ncols;
    double t0 = now_s();
    int rc = build_y(B, L1, L2);
    B->sec_y = now_s() - t0;
    if (rc == RSB_OK && what >= 1 && B->s > 0) {
        const size_t ss = (size_t)(B->s * B->s);
        rc = dev_alloc(ctx, (void **)&B->F, ss * sizeof(double));
        t0 = now_s();
        if (rc == RSB_OK) rc = build_gram(B, B->F);
        B->sec_gram = now_s() - t0;
        if (rc == RSB_OK && what == 2) {
            rc = dev_alloc(ctx, (void **)&B->S, ss * sizeof(double));
            if (rc == RSB_OK) {
                cudaError_t e = cudaMemcpyAsync(B->S, B->F, ss * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream);
                if (e != cudaSuccess) {
                    set_error("copy of S failed: %s", cudaGetErrorString(e));
                    rc = RSB_ECUDA;
                }
            }
        }
        t0 = now_s();
        if (rc == RSB_OK) rc = chol_factor_device(ctx, B->s, B->F);
        B->sec_chol = now_s() - t0;
    }
    if (rc != RSB_OK) {
        dbuild_free(B);
        delete B;
        return rc;
    }
    *out = B;
    return RSB_OK;
}

int rsb_dense_build_sizes(const rsb_dbuild *B, int64_t *s, int64_t *n, int64_t *nnz_y, double *seconds3) {
    *s = B->s;
    *n = B->n;
    *nnz_y = B->nnz;
    if (seconds3) {
        seconds3[0] = B->sec_y;
        seconds3[1] = B->sec_gram;
        seconds3[2] = B->sec_chol;
    }
    return RSB_OK;
}

int rsb_dense_build_copy(const rsb_dbuild *B, int64_t *y_ptr, int64_t *y_idx, double *y_val, double *S,
                         double *S_factor) {
    rsb_ctx *ctx = B->ctx;
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    const size_t ss = (size_t)(B->s * B->s);
    if ((S && !B->S) || (S_factor && !B->F && B->s > 0)) {
        set_error("S / S factor were not built (what = 2 / >= 1)");
        return RSB_ESTATE;
    }
    std::vector<int32_t> p32(B->n + 1), i32((size_t)std::max<int64_t>(1, B->nnz));
    RSB_TRY_CUDA(cudaMemcpyAsync(p32.data(), B->y_cptr, (B->n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    if (B->nnz) {
        RSB_TRY_CUDA(cudaMemcpyAsync(i32.data(), B->y_cidx, B->nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        if (y_val)
            RSB_TRY_CUDA(cudaMemcpyAsync(y_val, B->y_cval, B->nnz * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (S && ss) RSB_TRY_CUDA(cudaMemcpyAsync(S, B->S, ss * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (S_factor && ss)
        RSB_TRY_CUDA(cudaMemcpyAsync(S_factor, B->F, ss * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    if (y_ptr)
        for (int64_t j = 0; j <= B->n; ++j) y_ptr[j] = p32[j];
    if (y_idx)
        for (int64_t k = 0; k < B->nnz; ++k) y_idx[k] = i32[k];
    return RSB_OK;
}

int rsb_dense_build_destroy(rsb_dbuild *B) {
    if (!B) return RSB_OK;
    cudaSetDevice(B->ctx->device);
    dbuild_free(B);
    delete B;
    return RSB_OK;
}

int rsb_cholesky_factorize_device(rsb_ctx *ctx, int64_t s, double *g, int where) {
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    if (s < 0) {
        set_error("negative size");
        return RSB_EINVAL;
    }
    if (where != RSB_HOST) return chol_factor_device(ctx, s, g);
    const size_t ss = (size_t)(s * s);
    double *d = nullptr;
    RSB_TRY(dev_alloc(ctx, (void **)&d, std::max<size_t>(1, ss) * sizeof(double)));
    int rc = RSB_OK;
    cudaError_t e = cudaMemcpyAsync(d, g, ss * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) {
        set_error("upload failed: %s", cudaGetErrorString(e));
        rc = RSB_ECUDA;
    }
    if (rc == RSB_OK) rc = chol_factor_device(ctx, s, d);
    if (rc == RSB_OK) {
        e = cudaMemcpyAsync(g, d, ss * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            set_error("download failed: %s", cudaGetErrorString(e));
            rc = RSB_ECUDA;
        }
    }
    cudaStreamSynchronize(ctx->stream);
    dev_free(ctx, d, std::max<size_t>(1, ss) * sizeof(double));
    return rc;
}


int rsb_column_scale_device(rsb_ctx *ctx, int64_t ncols, const int64_t *col_ptr, const double *values,
                            double *scaled_values, double *norms) {
    RSB_TRY_CUDA(cudaSetDevice(ctx->device));
    if (ncols < 0) {
        set_error("negative size");
        return RSB_EINVAL;
    }
    if (ncols == 0) return RSB_OK;
    if (ncols > INT32_MAX) {
        set_error("too many columns");
        return RSB_EINVAL;
    }
    const int64_t nnz = col_ptr[ncols];
    int64_t *d_ptr = nullptr;
    double *d_val = nullptr, *d_out = nullptr, *d_norm = nullptr;
    int *d_empty = nullptr;
    int rc = RSB_OK;
    auto free_all = [&]() {
        cudaStreamSynchronize(ctx->stream);
        if (d_ptr) dev_free(ctx, d_ptr, (ncols + 1) * sizeof(int64_t));
        if (d_val) dev_free(ctx, d_val, std::max<int64_t>(1, nnz) * sizeof(double));
        if (d_out) dev_free(ctx, d_out, std::max<int64_t>(1, nnz) * sizeof(double));
        if (d_norm) dev_free(ctx, d_norm, ncols * sizeof(double));
        if (d_empty) dev_free(ctx, d_empty, sizeof(int));
    };
    if ((rc = dev_alloc(ctx, (void **)&d_ptr, (ncols + 1) * sizeof(int64_t))) != RSB_OK ||
        (rc = dev_alloc(ctx, (void **)&d_val, std::max<int64_t>(1, nnz) * sizeof(double))) != RSB_OK ||
        (rc = dev_alloc(ctx, (void **)&d_out, std::max<int64_t>(1, nnz) * sizeof(double))) != RSB_OK ||
        (rc = dev_alloc(ctx, (void **)&d_norm, ncols * sizeof(double))) != RSB_OK ||
        (rc = dev_alloc(ctx, (void **)&d_empty, sizeof(int))) != RSB_OK) {
        free_all();
        return rc;
    }
    const int big = INT32_MAX;
    int h_empty = big;
    cudaError_t e = cudaMemcpyAsync(d_ptr, col_ptr, (ncols + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess && nnz)
        e = cudaMemcpyAsync(d_val, values, nnz * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_empty, &big, sizeof(int), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        k_colscale<<<blocks_for(ncols), kT, 0, ctx->stream>>>(ncols, d_ptr, d_val, d_out, d_norm, d_empty);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_empty, d_empty, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e == cudaSuccess && h_empty != big) {
        set_error("cannot scale zero column %d", h_empty);
        free_all();
        return RSB_EINVAL;
    }
    if (e == cudaSuccess && nnz)
        e = cudaMemcpyAsync(scaled_values, d_out, nnz * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(norms, d_norm, ncols * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    free_all();
    if (e != cudaSuccess) {
        set_error("device column_scale failed: %s", cudaGetErrorString(e));
        return RSB_ECUDA;
    }
    return RSB_OK;
}

}  // extern "C"
