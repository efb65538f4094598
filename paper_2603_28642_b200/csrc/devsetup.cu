// Device-side setup of large matrices: the CSC upload
// with its CSR built on the device, and the level analysis of wide
// triangular solves.  At config 4's size (A: 96M entries; the factors 22M
// and 53M) the host versions (api.cu rsb_mat_create's CSR scatter,
// analysis.cpp) took 6 s for A and 13 s for the preconditioner; time to
// tolerance includes them.
//
// Everything here is integer bookkeeping; the floating-point values are
// only moved, so the schedules are identical to analysis.cpp's (the same
// per-task entry order, levels, task order inside a level and slice
// packing) and every solve stays bit-identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "rsb_internal.h"

namespace rsb {

namespace {

constexpr int kT = 256;

inline int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 64)); }

#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// scratch owned by one setup call
struct Scratch {
    rsb_ctx *ctx;
    std::vector<std::pair<void *, size_t>> bufs;
    explicit Scratch(rsb_ctx *c) : ctx(c) {}
    template <class T>
    int get(T **p, size_t count) {
        RSB_TRY(dev_alloc(ctx, (void **)p, std::max<size_t>(1, count) * sizeof(T)));
        bufs.emplace_back(*p, std::max<size_t>(1, count) * sizeof(T));
        return RSB_OK;
    }
    ~Scratch() {
        cudaStreamSynchronize(ctx->stream);
        for (auto &b : bufs) dev_free(ctx, b.first, b.second);
    }
};

// ---- CSC input checks (api.cu's host loops), int64 -> int32, column of each entry
__global__ void kd_check_csc(int64_t ncols, int64_t nrows, const int64_t *cp, const int64_t *ri, int64_t nnz,
                             int *bad, int32_t *cp32, int32_t *ci32, int32_t *col_of, int *maxc) {
    GRID_STRIDE(j, ncols) {
        const int64_t lo = cp[j], hi = cp[j + 1];
        if (hi < lo) atomicOr(bad, 1);
        cp32[j] = (int32_t)lo;
        if (j == ncols - 1) cp32[ncols] = (int32_t)hi;
        if (hi >= lo) atomicMax(maxc, (int)(hi - lo));
        for (int64_t k = max(lo, (int64_t)0); k < min(hi, nnz); ++k) col_of[k] = (int32_t)j;
    }
    GRID_STRIDE(k, nnz) {
        const int64_t r = ri[k];
        if (r < 0 || r >= nrows) atomicOr(bad, 2);
        ci32[k] = (int32_t)(r >= 0 && r < nrows ? r : 0);
    }
}

__global__ void kd_iota(int32_t *v, int64_t n) {
    GRID_STRIDE(i, n) v[i] = (int32_t)i;
}

__global__ void kd_hist(const int32_t *keys, int64_t n, int32_t *cnt) {
    GRID_STRIDE(i, n) atomicAdd(cnt + keys[i], 1);
}

__global__ void kd_max(const int32_t *v, int64_t n, int *out) {
    int m = 0;
    GRID_STRIDE(i, n) m = max(m, v[i]);
    atomicMax(out, m);
}

__global__ void kd_csr_fill(const int32_t *perm, const int32_t *col_of, const double *cval, int64_t nnz,
                            int32_t *r_idx, double *r_val) {
    GRID_STRIDE(k, nnz) {
        const int32_t e = perm[k];
        r_idx[k] = col_of[e];
        r_val[k] = cval[e];
    }
}

template <class T>
int scan_exclusive(rsb_ctx *ctx, Scratch &sc, const T *in, T *out, int64_t n) {
    size_t bytes = 0;
    RSB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, ctx->stream));
    char *tmp = nullptr;
    RSB_TRY(sc.get(&tmp, bytes));
    RSB_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, ctx->stream));
    return RSB_OK;
}

// stable sort of (key, value) pairs: CUB's radix sort keeps equal keys in input order
template <class K>
int sort_pairs(rsb_ctx *ctx, Scratch &sc, const K *kin, K *kout, const int32_t *vin, int32_t *vout, int64_t n,
               int end_bit) {
    size_t bytes = 0;
    RSB_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, ctx->stream));
    char *tmp = nullptr;
    RSB_TRY(sc.get(&tmp, bytes));
    RSB_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, ctx->stream));
    return RSB_OK;
}

int bits_for(int64_t v) {
    int b = 1;
    while (b < 32 && ((int64_t)1 << b) <= v) ++b;
    return b;
}

// ---- triangular analysis on the device ---------------------------------
// non-unit: every column (row) holds its diagonal, nonzero; the stored
// off-diagonal entries are strictly on the triangular side.  bad_diag /
// bad_tri get the smallest and largest failing line (the caller reports the
// first one in the reference's visiting order).
__global__ void kd_tri_check(TaskSrc s, int n, int lower_rows, int *diag_min, int *diag_max, int *tri_min,
                             int *tri_max) {
    GRID_STRIDE(t64, n) {
        const int t = (int)t64;
        const int lo = s.ptr[t], hi = s.ptr[t + 1];
        if (s.diag_at >= 0) {
            const int d = s.diag_at == 0 ? lo : hi - 1;
            if (hi == lo || s.idx[d] != t || s.val[d] == 0.0) {
                atomicMin(diag_min, t);
                atomicMax(diag_max, t);
            }
        }
        int64_t base;
        int len;
        s.task(t, base, len);
        for (int k = 0; k < len; ++k) {
            const int c = s.idx[base + (int64_t)s.step * k];
            if (lower_rows ? c >= t : c <= t) {
                atomicMin(tri_min, t);
                atomicMax(tri_max, t);
            }
        }
    }
}

// levels: lev[t] = 0 without dependencies, else 1 + max over them.  Tasks in
// dependency order (forward: t ascending, else descending) are taken in
// 32-wide slices from a ticket, so every dependency belongs to a slice held
// by a running warp: a lane waits on a dependency's level (-1: not yet).
__global__ void kd_levels(TaskSrc s, int n, int forward, int *lev, unsigned long long *ticket, int *maxlev) {
    const int lane = threadIdx.x & 31;
    const int nsl = (n + 31) / 32;
    int mx = 0;
    for (;;) {
        int w = 0;
        if (lane == 0) w = (int)atomicAdd(ticket, 1ull);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= nsl) break;
        const int p = w * 32 + lane;
        if (p < n) {
            const int t = forward ? p : n - 1 - p;
            int64_t base;
            int len;
            s.task(t, base, len);
            int L = 0;
            for (int k = 0; k < len; ++k) {
                const int c = s.idx[base + (int64_t)s.step * k];
                int lc;
                unsigned ns = 32;
                while ((lc = *(volatile const int *)(lev + c)) < 0) {
                    __nanosleep(ns);
                    ns = min(ns * 2, 512u);
                }
                L = max(L, lc + 1);
            }
            *(volatile int *)(lev + t) = L;
            mx = max(mx, L);
        }
    }
    if (mx) atomicMax(maxlev, mx);
}

struct TaskStats {
    int max_len, le4, le8, pad;
};

// sort key (level, longest first); task order inside equal keys stays
// ascending (stable sort of an ascending sequence), as analysis.cpp's
__global__ void kd_keys(TaskSrc s, int n, const int *lev, int len_bits, int sort_len, uint64_t *key, int32_t *cnt_lev,
                        TaskStats *st) {
    int mx = 0, le4 = 0, le8 = 0;
    GRID_STRIDE(t64, n) {
        const int t = (int)t64;
        int64_t base;
        int len;
        s.task(t, base, len);
        const uint64_t lmask = ((uint64_t)1 << len_bits) - 1;
        key[t] = ((uint64_t)lev[t] << len_bits) | (sort_len ? (lmask - (uint64_t)len) : 0);
        atomicAdd(cnt_lev + lev[t], 1);
        mx = max(mx, len);
        le4 += len <= 4;
        le8 += len <= 8;
    }
    atomicMax(&st->max_len, mx);
    atomicAdd(&st->le4, le4);
    atomicAdd(&st->le8, le8);
}

// the widest entry count of each 32-position slice, times 32
__global__ void kd_slice_width(TaskSrc s, int n, const int32_t *order, int64_t *w32) {
    const int64_t nsl = (n + 31) / 32;
    GRID_STRIDE(w, nsl) {
        int K = 0;
        for (int l = 0; l < 32; ++l) {
            const int64_t q = w * 32 + l;
            if (q >= n) break;
            int64_t base;
            int len;
            s.task(order[q], base, len);
            K = max(K, len);
        }
        w32[w] = 32 * (int64_t)K;
    }
}

// warp-interleaved packing: entry k of position q at soff[q/32] + 32k + q%32
__global__ void kd_pack(TaskSrc s, int n, const int32_t *order, const int64_t *soff, int32_t *ecol, double *eval,
                        double *tdiag) {
    GRID_STRIDE(q, n) {
        const int t = order[q];
        int64_t base;
        int len;
        s.task(t, base, len);
        const int64_t o = soff[q >> 5] + (q & 31);
        for (int k = 0; k < len; ++k) {
            const int64_t e = base + (int64_t)s.step * k;
            ecol[o + 32 * (int64_t)k] = s.idx[e];
            eval[o + 32 * (int64_t)k] = s.val[e];
        }
        if (tdiag) tdiag[q] = s.val[s.diag_at == 0 ? s.ptr[t] : s.ptr[t + 1] - 1];
    }
}

}  // namespace

// Upload of a CSC matrix given as host int64 / f64 arrays: checks, int32
// CSC and the CSR (rows in ascending column order -- np.add.at's scatter
// order, sc.py:220) built on the device by a stable radix sort of the
// entries by row.
int mat_upload_device(rsb_mat *A, const int64_t *col_ptr, const int64_t *row_idx, const double *values) {
    rsb_ctx *ctx = A->ctx;
    const int64_t m = A->nrows, n = A->ncols, nnz = A->nnz;
    Scratch sc(ctx);
    int64_t *d_cp = nullptr, *d_ri = nullptr;
    int32_t *col_of = nullptr, *perm_in = nullptr, *perm = nullptr, *rows_sorted = nullptr, *cnt = nullptr;
    int *flags = nullptr;  // [bad, maxc, maxr]
    RSB_TRY(sc.get(&d_cp, n + 1));
    RSB_TRY(sc.get(&d_ri, nnz));
    RSB_TRY(sc.get(&col_of, nnz));
    RSB_TRY(sc.get(&perm_in, nnz));
    RSB_TRY(sc.get(&perm, nnz));
    RSB_TRY(sc.get(&rows_sorted, nnz));
    RSB_TRY(sc.get(&cnt, m + 1));
    RSB_TRY(sc.get(&flags, 4));
    RSB_TRY(dev_alloc(ctx, (void **)&A->c_ptr, (n + 1) * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&A->c_idx, std::max<int64_t>(1, nnz) * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&A->c_val, std::max<int64_t>(1, nnz) * sizeof(double)));
    RSB_TRY(dev_alloc(ctx, (void **)&A->r_ptr, (m + 1) * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&A->r_idx, std::max<int64_t>(1, nnz) * sizeof(int32_t)));
    RSB_TRY(dev_alloc(ctx, (void **)&A->r_val, std::max<int64_t>(1, nnz) * sizeof(double)));
    cudaStream_t st = ctx->stream;
    RSB_TRY_CUDA(cudaMemcpyAsync(d_cp, col_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (nnz) {
        RSB_TRY_CUDA(cudaMemcpyAsync(d_ri, row_idx, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        RSB_TRY_CUDA(cudaMemcpyAsync(A->c_val, values, nnz * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    RSB_TRY_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(int), st));
    RSB_TRY_CUDA(cudaMemsetAsync(cnt, 0, (m + 1) * sizeof(int32_t), st));
    kd_check_csc<<<blocks_for(std::max(n, nnz)), kT, 0, st>>>(n, m, d_cp, d_ri, nnz, flags, A->c_ptr, A->c_idx, col_of,
                                                              flags + 1);
    RSB_TRY_CUDA(cudaGetLastError());
    int h_flags[4] = {0, 0, 0, 0};
    RSB_TRY_CUDA(cudaMemcpyAsync(h_flags, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    if (h_flags[0] & 1) {
        set_error("col_ptr not non-decreasing");
        return RSB_EINVAL;
    }
    if (h_flags[0] & 2) {
        set_error("row index out of range");
        return RSB_EINVAL;
    }
    A->max_col_len = h_flags[1];
    if (nnz) {
        kd_iota<<<blocks_for(nnz), kT, 0, st>>>(perm_in, nnz);
        RSB_TRY(sort_pairs(ctx, sc, A->c_idx, rows_sorted, perm_in, perm, nnz, bits_for(m)));
        kd_csr_fill<<<blocks_for(nnz), kT, 0, st>>>(perm, col_of, A->c_val, nnz, A->r_idx, A->r_val);
        kd_hist<<<blocks_for(nnz), kT, 0, st>>>(A->c_idx, nnz, cnt);
        RSB_TRY_CUDA(cudaGetLastError());
    }
    kd_max<<<blocks_for(m), kT, 0, st>>>(cnt, m, flags + 2);
    RSB_TRY(scan_exclusive<int32_t>(ctx, sc, cnt, A->r_ptr, m + 1));
    RSB_TRY_CUDA(cudaMemcpyAsync(h_flags + 2, flags + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    A->max_row_len = h_flags[2];
    return RSB_OK;
}

// ---- row bands ----------------------------------------------------------
__global__ void kd_band_count(const int32_t *cp, const int32_t *ci, int64_t ncols, int64_t rpb, int nb,
                              int32_t *cnt /* nb x (ncols + 1) */) {
    GRID_STRIDE(j, ncols) {
        int c[kMaxBands] = {};
        for (int k = cp[j]; k < cp[j + 1]; ++k) c[min((int64_t)nb - 1, ci[k] / rpb)]++;
        for (int b = 0; b < nb; ++b) cnt[(int64_t)b * (ncols + 1) + j] = c[b];
    }
}

__global__ void kd_band_fill(const int32_t *cp, const int32_t *ci, const double *cv, int64_t ncols, int64_t rpb,
                             int nb, const int32_t *bptr /* nb x (ncols + 1), absolute */, int32_t *bidx,
                             double *bval) {
    GRID_STRIDE(j, ncols) {
        int o[kMaxBands];
        for (int b = 0; b < nb; ++b) o[b] = bptr[(int64_t)b * (ncols + 1) + j];
        for (int k = cp[j]; k < cp[j + 1]; ++k) {
            const int b = (int)min((int64_t)nb - 1, ci[k] / rpb);
            bidx[o[b]] = ci[k];
            bval[o[b]] = cv[k];
            ++o[b];
        }
    }
}

__global__ void kd_add_const(int32_t *v, int64_t n, int32_t c) {
    GRID_STRIDE(i, n) v[i] += c;
}

int mat_build_bands(rsb_mat *A) {
    const int64_t m = A->nrows, n = A->ncols, nnz = A->nnz;
    if (A->bands.nbands || m * 8 <= kBandBytes || nnz == 0 || n == 0) return RSB_OK;
    // opt-in (RSB_BANDS=1): at config 4 it measured slower than the plain
    // tiled kernel (A^T y 2.17 vs 1.39 ms, L2^T w 1.14 vs 0.46 ms at n = 8e6:
    // the products' round trip through HBM and the per-column band segments
    // cost more than the L2 misses they avoid)
    const char *be = getenv("RSB_BANDS");
    if (!(be && atoi(be) != 0)) return RSB_OK;
    rsb_ctx *ctx = A->ctx;
    cudaStream_t st = ctx->stream;
    const int nb = (int)std::min<int64_t>(kMaxBands, (m * 8 + kBandBytes - 1) / kBandBytes);
    const int64_t rpb = (m + nb - 1) / nb;
    Scratch sc(ctx);
    int32_t *cnt = nullptr;
    RSB_TRY(sc.get(&cnt, (size_t)nb * (n + 1)));
    RSB_TRY_CUDA(cudaMemsetAsync(cnt, 0, (size_t)nb * (n + 1) * sizeof(int32_t), st));
    kd_band_count<<<blocks_for(n), kT, 0, st>>>(A->c_ptr, A->c_idx, n, rpb, nb, cnt);
    RSB_TRY_CUDA(cudaGetLastError());
    auto keep = [&](void *p, size_t bytes) { A->band_bufs.emplace_back(p, bytes); };
    int32_t *bp = nullptr, *bidx = nullptr;
    double *bval = nullptr, *prod = nullptr;
    RSB_TRY(dev_alloc(ctx, (void **)&bp, (size_t)nb * (n + 1) * sizeof(int32_t)));
    keep(bp, (size_t)nb * (n + 1) * sizeof(int32_t));
    // per band: exclusive scan of its column counts, offset by the earlier bands' totals
    int64_t base = 0;
    for (int b = 0; b < nb; ++b) {
        int32_t *pb = bp + (size_t)b * (n + 1);
        RSB_TRY(scan_exclusive<int32_t>(ctx, sc, cnt + (size_t)b * (n + 1), pb, n + 1));
        int32_t tot = 0;
        RSB_TRY_CUDA(cudaMemcpyAsync(&tot, pb + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        RSB_TRY_CUDA(cudaStreamSynchronize(st));
        if (base) kd_add_const<<<blocks_for(n + 1), kT, 0, st>>>(pb, n + 1, (int32_t)base);
        base += tot;
        A->bands.bptr[b] = pb;
    }
    RSB_TRY(dev_alloc(ctx, (void **)&bidx, (size_t)nnz * sizeof(int32_t)));
    keep(bidx, (size_t)nnz * sizeof(int32_t));
    RSB_TRY(dev_alloc(ctx, (void **)&bval, (size_t)nnz * sizeof(double)));
    keep(bval, (size_t)nnz * sizeof(double));
    RSB_TRY(dev_alloc(ctx, (void **)&prod, (size_t)nnz * sizeof(double)));
    keep(prod, (size_t)nnz * sizeof(double));
    kd_band_fill<<<blocks_for(n), kT, 0, st>>>(A->c_ptr, A->c_idx, A->c_val, n, rpb, nb, bp, bidx, bval);
    RSB_TRY_CUDA(cudaGetLastError());
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    A->bands.nbands = nb;
    A->bands.rows_per_band = rpb;
    A->bands.idx = bidx;
    A->bands.val = bval;
    A->bands.prod = prod;
    A->bands.owner = ctx;
    return RSB_OK;
}

// host copy of the CSC (for the host analysis of small or special schedules)
int mat_host_copy(rsb_mat *A) {
    if (!A->h_ptr.empty()) return RSB_OK;
    rsb_ctx *ctx = A->ctx;
    std::vector<int32_t> cp(A->ncols + 1), ci(A->nnz);
    A->h_val.resize(A->nnz);
    RSB_TRY_CUDA(cudaMemcpyAsync(cp.data(), A->c_ptr, cp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    if (A->nnz) {
        RSB_TRY_CUDA(cudaMemcpyAsync(ci.data(), A->c_idx, ci.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        RSB_TRY_CUDA(cudaMemcpyAsync(A->h_val.data(), A->c_val, A->nnz * sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    }
    RSB_TRY_CUDA(cudaStreamSynchronize(ctx->stream));
    A->h_ptr.assign(cp.begin(), cp.end());
    A->h_idx.assign(ci.begin(), ci.end());
    return RSB_OK;
}

// where the tasks of a solve kind live in the matrix's arrays
TaskSrc tri_task_src(const rsb_mat *T, int kind) {
    const bool unit = (kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_LOWER_T_UNIT);
    const bool is_dot = (kind == RSB_TRI_LOWER_T || kind == RSB_TRI_LOWER_T_UNIT || kind == RSB_TRI_UPPER_T);
    const bool lower = (kind == RSB_TRI_LOWER || kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_LOWER_T ||
                        kind == RSB_TRI_LOWER_T_UNIT);
    TaskSrc s{};
    s.forward = (kind == RSB_TRI_LOWER || kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_UPPER_T) ? 1 : 0;
    if (is_dot) {  // task j = column j, rows as stored; the diagonal first (lower) / last (upper)
        s.ptr = T->c_ptr;
        s.idx = T->c_idx;
        s.val = T->c_val;
        s.step = 1;
        s.first_off = (!unit && lower) ? 1 : 0;
        s.last_off = (!unit && !lower) ? 1 : 0;
        s.diag_at = unit ? -1 : (lower ? 0 : 1);
    } else {  // task i = row i, columns ascending (lower) / descending (upper); the diagonal last / first
        s.ptr = T->r_ptr;
        s.idx = T->r_idx;
        s.val = T->r_val;
        s.step = lower ? 1 : -1;
        s.first_off = (!unit && !lower) ? 1 : 0;  // upper rows: the diagonal comes first
        s.last_off = (!unit && lower) ? 1 : 0;    // lower rows: the diagonal comes last
        s.diag_at = unit ? -1 : (lower ? 1 : 0);
    }
    return s;
}

namespace {
// dependencies closer than `near` positions, and the longest line (diagonal included)
__global__ void kd_nat_stats(TaskSrc s, int n, int64_t near, unsigned long long *cnt, int *max_line) {
    unsigned long long c = 0;
    int ml = 0;
    GRID_STRIDE(t64, n) {
        const int t = (int)t64;
        int64_t base;
        int len;
        s.task(t, base, len);
        ml = max(ml, s.ptr[t + 1] - s.ptr[t]);
        for (int k = 0; k < len; ++k) {
            const int64_t d = (int64_t)s.idx[base + (int64_t)s.step * k] - t;
            c += (d < 0 ? -d : d) < near;
        }
    }
    if (c) atomicAdd(cnt, c);
    atomicMax(max_line, ml);
}
}  // namespace

// Decide whether a wide schedule runs the index-order kernel (trsv_nat.cu).
// A dependency closer than the tasks in flight (~kNatNear) may make its
// consumer wait; with fewer than one such dependency per task on average the
// waiting chains stay short (config 4 at n = 8e6: 0.4 - 0.8), while a banded
// matrix (every dependency near) would serialise, and keeps the level order.
int tri_setup_nat(rsb_mat *T, int kind, TriSched *S) {
    S->use_nat = false;
    if (!S->wide || S->n == 0) return RSB_OK;
    const char *oe = getenv("RSB_TRSV_ORDER");
    if (oe && std::strcmp(oe, "level") == 0) return RSB_OK;
    const bool force = oe && std::strcmp(oe, "natural") == 0;
    rsb_ctx *ctx = T->ctx;
    cudaStream_t st = ctx->stream;
    const TaskSrc s = tri_task_src(T, kind);
    Scratch sc(ctx);
    unsigned long long *cnt = nullptr;
    int *ml = nullptr;
    RSB_TRY(sc.get(&cnt, 1));
    RSB_TRY(sc.get(&ml, 1));
    RSB_TRY_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    RSB_TRY_CUDA(cudaMemsetAsync(ml, 0, sizeof(int), st));
    kd_nat_stats<<<blocks_for(S->n), kT, 0, st>>>(s, S->n, kNatNear, cnt, ml);
    RSB_TRY_CUDA(cudaGetLastError());
    unsigned long long h_cnt = 0;
    int h_ml = 0;
    RSB_TRY_CUDA(cudaMemcpyAsync(&h_cnt, cnt, sizeof h_cnt, cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaMemcpyAsync(&h_ml, ml, sizeof h_ml, cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    S->nat = s;
    S->nat_near = (int64_t)h_cnt;
    S->nat_max_line = h_ml;
    // window: 1.25 x the mean slice span + slack, at least the longest line
    const int64_t mean32 = 32 * T->nnz / std::max<int64_t>(1, S->n);
    int64_t cap = (mean32 * 5 / 4 + 48 + 31) / 32 * 32;
    cap = std::max<int64_t>(cap, ((int64_t)h_ml + 31) / 32 * 32);
    cap = std::max<int64_t>(cap, 96);
    if (const char *ce = getenv("RSB_NAT_CAP")) cap = std::max<int64_t>(((int64_t)h_ml + 31) / 32 * 32, atoi(ce));
    if (cap > kNatMaxCap) return RSB_OK;  // a line too long for the window: level order
    S->nat_cap = (int32_t)cap;
    S->use_nat = force || (int64_t)h_cnt < (int64_t)S->n;
    if (getenv("RSB_DEBUG_ANALYSIS"))
        fprintf(stderr, "[rsb] index-order solve kind=%d n=%d near=%lld max_line=%d cap=%d use=%d\n", kind, S->n,
                (long long)h_cnt, h_ml, (int)cap, (int)S->use_nat);
    return RSB_OK;
}

// Level analysis of a wide schedule on the device (n > kCtaTriMaxN: never
// single-CTA).  Produces analysis.cpp's grid schedule.
int tri_analyse_device(rsb_mat *T, int kind, TriSched **out) {
    rsb_ctx *ctx = T->ctx;
    cudaStream_t st = ctx->stream;
    const int n = (int)T->ncols;
    const bool unit = (kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_LOWER_T_UNIT);
    const bool is_dot = (kind == RSB_TRI_LOWER_T || kind == RSB_TRI_LOWER_T_UNIT || kind == RSB_TRI_UPPER_T);
    const bool lower = (kind == RSB_TRI_LOWER || kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_LOWER_T ||
                        kind == RSB_TRI_LOWER_T_UNIT);
    const bool forward = (kind == RSB_TRI_LOWER || kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_UPPER_T);
    const TaskSrc s = tri_task_src(T, kind);
    Scratch sc(ctx);
    int *chk = nullptr;
    RSB_TRY(sc.get(&chk, 4));
    const int init[4] = {INT32_MAX, -1, INT32_MAX, -1};
    RSB_TRY_CUDA(cudaMemcpyAsync(chk, init, sizeof init, cudaMemcpyHostToDevice, st));
    // the strictly-triangular side of the off-diagonal part: lower solves'
    // tasks depend on smaller indices in the row form, larger in the column form
    const int lower_rows = is_dot ? !lower : lower;
    kd_tri_check<<<blocks_for(n), kT, 0, st>>>(s, n, lower_rows, chk, chk + 1, chk + 2, chk + 3);
    RSB_TRY_CUDA(cudaGetLastError());
    int h_chk[4];
    RSB_TRY_CUDA(cudaMemcpyAsync(h_chk, chk, sizeof h_chk, cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    if (h_chk[1] >= 0) {
        // the reference visits columns ascending for L and U^T, descending otherwise
        const bool asc = (kind == RSB_TRI_LOWER || kind == RSB_TRI_UPPER_T);
        set_error("missing or zero diagonal in column %d", asc ? h_chk[0] : h_chk[1]);
        return RSB_ESINGULAR;
    }
    if (h_chk[3] >= 0) {
        set_error("matrix is not strictly %s triangular off the diagonal (line %d)", lower ? "lower" : "upper",
                  h_chk[2]);
        return RSB_EINVAL;
    }
    int *lev = nullptr, *maxlev = nullptr;
    unsigned long long *tick = nullptr;
    RSB_TRY(sc.get(&lev, n));
    RSB_TRY(sc.get(&maxlev, 1));
    RSB_TRY(sc.get(&tick, 1));
    RSB_TRY_CUDA(cudaMemsetAsync(lev, 0xFF, (size_t)n * sizeof(int), st));
    RSB_TRY_CUDA(cudaMemsetAsync(maxlev, 0, sizeof(int), st));
    RSB_TRY_CUDA(cudaMemsetAsync(tick, 0, sizeof(unsigned long long), st));
    {
        int occ = 0, sms = 0;
        RSB_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kd_levels, kT, 0));
        RSB_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int grid = (int)std::min<int64_t>((int64_t)sms * std::max(1, occ), ((int64_t)n + kT - 1) / kT);
        kd_levels<<<std::max(1, grid), kT, 0, st>>>(s, n, forward, lev, tick, maxlev);
        RSB_TRY_CUDA(cudaGetLastError());
    }
    int nlev = 0;
    RSB_TRY_CUDA(cudaMemcpyAsync(&nlev, maxlev, sizeof(int), cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    nlev += 1;
    // order: (level, longest task first), stable
    const char *sort_env = getenv("RSB_TRSV_SORT");
    const int sort_len = !(sort_env && std::strcmp(sort_env, "0") == 0);
    const int len_bits = bits_for(std::max<int64_t>(T->max_row_len, T->max_col_len) + 1);
    uint64_t *key = nullptr, *key_s = nullptr;
    int32_t *ids = nullptr, *cnt_lev = nullptr, *lptr = nullptr;
    TaskStats *tst = nullptr;
    RSB_TRY(sc.get(&key, n));
    RSB_TRY(sc.get(&key_s, n));
    RSB_TRY(sc.get(&ids, n));
    RSB_TRY(sc.get(&cnt_lev, nlev + 1));
    RSB_TRY(sc.get(&tst, 1));
    RSB_TRY_CUDA(cudaMemsetAsync(cnt_lev, 0, (nlev + 1) * sizeof(int32_t), st));
    RSB_TRY_CUDA(cudaMemsetAsync(tst, 0, sizeof(TaskStats), st));
    kd_keys<<<blocks_for(n), kT, 0, st>>>(s, n, lev, len_bits, sort_len, key, cnt_lev, tst);
    kd_iota<<<blocks_for(n), kT, 0, st>>>(ids, n);
    RSB_TRY_CUDA(cudaGetLastError());
    auto *S = new TriSched();
    int rc = RSB_OK;
    auto fail = [&](int code) {
        tri_free(ctx, S);
        return code;
    };
    S->kind = kind;
    S->n = n;
    S->nlevels = nlev;
    S->mode = (is_dot ? 1 : 0) | (unit ? 0 : 2);
    S->single_cta = false;
    S->padded_n = n;
    if ((rc = dev_alloc(ctx, (void **)&S->task_row, (size_t)n * sizeof(int32_t))) != RSB_OK) return fail(rc);
    if ((rc = sort_pairs(ctx, sc, key, key_s, ids, S->task_row, n, bits_for(nlev) + len_bits)) != RSB_OK) return fail(rc);
    if ((rc = dev_alloc(ctx, (void **)&S->level_ptr, (size_t)(nlev + 1) * sizeof(int32_t))) != RSB_OK) return fail(rc);
    if ((rc = scan_exclusive<int32_t>(ctx, sc, cnt_lev, S->level_ptr, nlev + 1)) != RSB_OK) return fail(rc);
    // slices
    const int64_t nsl = (n + 31) / 32;
    int64_t *w32 = nullptr;
    if ((rc = sc.get(&w32, nsl + 1)) != RSB_OK) return fail(rc);
    if ((rc = dev_alloc(ctx, (void **)&S->slice_off, (nsl + 1) * sizeof(int64_t))) != RSB_OK) return fail(rc);
    RSB_TRY_CUDA(cudaMemsetAsync(w32 + nsl, 0, sizeof(int64_t), st));
    kd_slice_width<<<blocks_for(nsl), kT, 0, st>>>(s, n, S->task_row, w32);
    RSB_TRY_CUDA(cudaGetLastError());
    if ((rc = scan_exclusive<int64_t>(ctx, sc, w32, S->slice_off, nsl + 1)) != RSB_OK) return fail(rc);
    int64_t slots = 0;
    TaskStats h_tst{};
    std::vector<int32_t> hl(nlev + 1);
    RSB_TRY_CUDA(cudaMemcpyAsync(&slots, S->slice_off + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaMemcpyAsync(&h_tst, tst, sizeof h_tst, cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaMemcpyAsync(hl.data(), S->level_ptr, hl.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RSB_TRY_CUDA(cudaStreamSynchronize(st));
    S->entries = slots;
    if ((rc = dev_alloc(ctx, (void **)&S->ecol, std::max<int64_t>(1, slots) * sizeof(int32_t))) != RSB_OK ||
        (rc = dev_alloc(ctx, (void **)&S->eval, std::max<int64_t>(1, slots) * sizeof(double))) != RSB_OK ||
        (!unit && (rc = dev_alloc(ctx, (void **)&S->diag, (size_t)n * sizeof(double))) != RSB_OK))
        return fail(rc);
    RSB_TRY_CUDA(cudaMemsetAsync(S->ecol, 0xFF, std::max<int64_t>(1, slots) * sizeof(int32_t), st));
    RSB_TRY_CUDA(cudaMemsetAsync(S->eval, 0, std::max<int64_t>(1, slots) * sizeof(double), st));
    kd_pack<<<blocks_for(n), kT, 0, st>>>(s, n, S->task_row, S->slice_off, S->ecol, S->eval, unit ? nullptr : S->diag);
    RSB_TRY_CUDA(cudaGetLastError());
    // the host-side fields analysis.cpp derives
    int64_t maxw = 0;
    for (int l = 0; l < nlev; ++l) maxw = std::max<int64_t>(maxw, hl[l + 1] - hl[l]);
    S->max_width = maxw;
    S->h_level_ptr = hl;
    const int ml = h_tst.max_len;
    S->max_task = ml;
    S->wide_n = (ml <= 4 || (int64_t)h_tst.le4 >= (int64_t)n * 94 / 100)
                    ? 4
                    : ((ml <= 8 || (int64_t)h_tst.le8 >= (int64_t)n * 94 / 100) ? 8 : 12);
    if (is_dot && ml >= S->wide_n) S->wide_n = 12;
    S->wide_static = (S->mode == 0) && (int64_t)h_tst.le4 >= (int64_t)n * 3 / 4;
    if (const char *wn = getenv("RSB_WIDE_N")) S->wide_n = std::max(4, std::min(12, atoi(wn))) <= 4 ? 4 : (atoi(wn) <= 8 ? 8 : 12);
    const char *wv = getenv("RSB_TRSV_WIDE");
    S->wide = !(is_dot && ml >= 16) && !(wv && std::strcmp(wv, "0") == 0);
    const char *gv = getenv("RSB_TRSV_GRID");
    S->level_launch = nlev <= kLevelLaunchMaxLevels || (gv && std::strcmp(gv, "levels") == 0);
    if (gv && std::strcmp(gv, "syncfree") == 0) S->level_launch = false;
    S->lsync = false;  // the item-list variant is built by the host analysis only
    S->level_sync = S->wide && !S->level_launch && gv && std::strcmp(gv, "levelsync") == 0;
    if ((rc = dev_alloc(ctx, (void **)&S->ticket, sizeof(unsigned long long))) != RSB_OK ||
        (S->wide && (rc = dev_alloc(ctx, (void **)&S->bpos, (size_t)n * sizeof(double))) != RSB_OK))
        return fail(rc);
    RSB_TRY_CUDA(cudaMemsetAsync(S->ticket, 0, sizeof(unsigned long long), st));
    if (getenv("RSB_TRSV_PROFILE") &&
        (rc = dev_alloc(ctx, (void **)&S->prof, (8 + 4096) * sizeof(long long))) != RSB_OK)
        return fail(rc);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_error("CUDA error %s in the device triangular analysis", cudaGetErrorString(e));
        return fail(RSB_ECUDA);
    }
    if (getenv("RSB_DEBUG_ANALYSIS"))
        fprintf(stderr, "[rsb] device analysis kind=%d n=%d levels=%d maxw=%lld max_task=%d wide_n=%d slots=%lld\n",
                kind, n, nlev, (long long)maxw, ml, S->wide_n, (long long)slots);
    *out = S;
    return RSB_OK;
}

}  // namespace rsb
