// Level analysis and device layout of the sparse triangular solves
// (host side, run once per (matrix, kind) and cached on the matrix).
//
// The reference solves column by column (sparse_core.py:243-313).  Each
// unknown's final value is a fixed sequence of operations on other
// unknowns; this file extracts that sequence per unknown ("task"), in the
// reference's order, computes the dependency level of every task, sorts the
// tasks by level and packs their entries in warp-interleaved slices (see
// TriDev in rsb_internal.h) so the device solve reads them coalesced.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <chrono>
#include <numeric>

#include "rsb_internal.h"

namespace rsb {

namespace {

struct Entry {
    int32_t col;
    double val;
};

}  // namespace

int tri_analyse(rsb_mat *T, int kind, TriSched **out) {
    if (T->nrows != T->ncols) {
        set_error("triangular solve needs a square matrix");
        return RSB_EINVAL;
    }
    if (T->h_ptr.empty()) {
        set_error("matrix has no host copy for triangular analysis");
        return RSB_ESTATE;
    }
    const int64_t n = T->ncols;
    const bool dbg = getenv("RSB_DEBUG_ANALYSIS") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto phase = [&](const char *what) {
        if (!dbg) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[rsb] analysis kind=%d %s %.3f s\n", kind, what,
                std::chrono::duration<double>(now - t_prev).count());
        t_prev = now;
    };
    const int64_t *ptr = T->h_ptr.data();
    const int64_t *idx = T->h_idx.data();
    const double *val = T->h_val.data();

    const bool unit = (kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_LOWER_T_UNIT);
    const bool is_dot = (kind == RSB_TRI_LOWER_T || kind == RSB_TRI_LOWER_T_UNIT || kind == RSB_TRI_UPPER_T);
    const bool lower = (kind == RSB_TRI_LOWER || kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_LOWER_T ||
                        kind == RSB_TRI_LOWER_T_UNIT);
    // forward: dependencies of task t are tasks < t
    const bool forward = (kind == RSB_TRI_LOWER || kind == RSB_TRI_LOWER_UNIT || kind == RSB_TRI_UPPER_T);

    // diagonal checks in the reference's column visiting order
    std::vector<double> diag;
    if (!unit) {
        diag.assign(n, 0.0);
        const bool diag_first = lower;
        const bool asc = (kind == RSB_TRI_LOWER || kind == RSB_TRI_UPPER_T);
        for (int64_t s = 0; s < n; ++s) {
            const int64_t j = asc ? s : n - 1 - s;
            const int64_t lo = ptr[j], hi = ptr[j + 1];
            const int64_t d = diag_first ? lo : hi - 1;
            if (hi == lo || idx[d] != j || val[d] == 0.0) {
                set_error("missing or zero diagonal in column %lld", (long long)j);
                return RSB_ESINGULAR;
            }
            diag[j] = val[d];
        }
    }
    // strict triangularity of the off-diagonal part
    for (int64_t j = 0; j < n; ++j) {
        int64_t lo = ptr[j], hi = ptr[j + 1];
        if (!unit) {
            if (lower) ++lo; else --hi;
        }
        for (int64_t k = lo; k < hi; ++k) {
            if (lower ? idx[k] <= j : idx[k] >= j) {
                set_error("matrix is not strictly %s triangular off the diagonal (entry %lld,%lld)",
                          lower ? "lower" : "upper", (long long)idx[k], (long long)j);
                return RSB_EINVAL;
            }
        }
    }

    phase("checks");
    // per-task entry lists in the reference's accumulation order
    std::vector<int64_t> tptr(n + 1, 0);
    std::vector<Entry> ent;
    if (is_dot) {
        // task j = column j: x_j -= vals @ x[rows] (rows ascending as stored)
        for (int64_t j = 0; j < n; ++j) {
            int64_t lo = ptr[j], hi = ptr[j + 1];
            if (!unit) {
                if (lower) ++lo; else --hi;
            }
            tptr[j + 1] = tptr[j] + (hi - lo);
        }
        ent.resize(tptr[n]);
        for (int64_t j = 0; j < n; ++j) {
            int64_t lo = ptr[j], hi = ptr[j + 1];
            if (!unit) {
                if (lower) ++lo; else --hi;
            }
            for (int64_t k = lo; k < hi; ++k) ent[tptr[j] + (k - lo)] = Entry{(int32_t)idx[k], val[k]};
        }
    } else {
        // task i = row i: contributions l_ij x_j in the order columns are visited
        // (ascending for the lower solve, descending for the upper solve)
        std::vector<int64_t> cnt(n + 1, 0);
        for (int64_t j = 0; j < n; ++j) {
            int64_t lo = ptr[j], hi = ptr[j + 1];
            if (!unit) {
                if (lower) ++lo; else --hi;
            }
            for (int64_t k = lo; k < hi; ++k) cnt[idx[k] + 1]++;
        }
        for (int64_t i = 0; i < n; ++i) tptr[i + 1] = tptr[i] + cnt[i + 1];
        ent.resize(tptr[n]);
        std::vector<int64_t> fill(tptr.begin(), tptr.end() - 1);
        for (int64_t s = 0; s < n; ++s) {
            const int64_t j = lower ? s : n - 1 - s;
            int64_t lo = ptr[j], hi = ptr[j + 1];
            if (!unit) {
                if (lower) ++lo; else --hi;
            }
            for (int64_t k = lo; k < hi; ++k) ent[fill[idx[k]]++] = Entry{(int32_t)j, val[k]};
        }
    }

    phase("entry lists");
    // dependency levels
    std::vector<int32_t> level(n, 0);
    if (forward) {
        for (int64_t t = 0; t < n; ++t) {
            int32_t L = 0;
            for (int64_t k = tptr[t]; k < tptr[t + 1]; ++k) L = std::max(L, level[ent[k].col] + 1);
            level[t] = L;
        }
    } else {
        for (int64_t t = n - 1; t >= 0; --t) {
            int32_t L = 0;
            for (int64_t k = tptr[t]; k < tptr[t + 1]; ++k) L = std::max(L, level[ent[k].col] + 1);
            level[t] = L;
        }
    }
    int32_t nlev = 0;
    for (int64_t t = 0; t < n; ++t) nlev = std::max(nlev, level[t] + 1);
    std::vector<int64_t> lstart(nlev + 1, 0);
    for (int64_t t = 0; t < n; ++t) lstart[level[t] + 1]++;
    int64_t maxw = 0;
    for (int32_t l = 0; l < nlev; ++l) maxw = std::max(maxw, lstart[l + 1]);
    for (int32_t l = 0; l < nlev; ++l) lstart[l + 1] += lstart[l];
    std::vector<int32_t> order(n);
    {
        std::vector<int64_t> pos(lstart.begin(), lstart.end() - 1);
        for (int64_t t = 0; t < n; ++t) order[pos[level[t]]++] = (int32_t)t;
    }
    // Wide DAGs (grid schedules): inside a level the order is free (its tasks
    // are independent), so put the longest tasks first.  Long tasks then share
    // slices -- a slice waits for its longest lane -- and start earliest.
    if (!(n <= kCtaTriMaxN && n / std::max<int64_t>(1, nlev) <= kCtaTriMaxMeanWidth) &&
        !(getenv("RSB_TRSV_SORT") && std::strcmp(getenv("RSB_TRSV_SORT"), "0") == 0)) {
        for (int32_t l = 0; l < nlev; ++l)
            std::stable_sort(order.begin() + lstart[l], order.begin() + lstart[l + 1], [&](int32_t a, int32_t b) {
                return tptr[a + 1] - tptr[a] > tptr[b + 1] - tptr[b];
            });
    }

    phase("levels + order");
    // warp-interleaved packing: slice widths
    const int64_t nslices = (n + 31) / 32;
    std::vector<int64_t> soff(nslices + 1, 0);
    for (int64_t w = 0; w < nslices; ++w) {
        int64_t K = 0;
        for (int64_t l = 0; l < 32 && w * 32 + l < n; ++l) {
            const int32_t t = order[w * 32 + l];
            K = std::max(K, tptr[t + 1] - tptr[t]);
        }
        soff[w + 1] = soff[w] + 32 * K;
    }
    const int64_t slots = soff[nslices];

    // variant: one CTA, level-synchronous, task data streamed into shared
    // memory, for narrow DAGs whose chunks fit the shared-memory budget
    const char *force = getenv("RSB_TRSV_VARIANT");  // "grid" | "cta" (experiments)
    bool single_cta = n <= kCtaTriMaxN && (n / std::max<int64_t>(1, nlev)) <= kCtaTriMaxMeanWidth;
    if (force && std::strcmp(force, "grid") == 0) single_cta = false;
    if (force && std::strcmp(force, "cta") == 0 && n <= kCtaTriMaxN) single_cta = true;
    // staged position space: every level padded to whole 32-task slices, so a
    // warp's 32 lanes are one slice of one level; records are lane-interleaved
    // per slice (entry q of lane l at slice_base + 32q + l, conflict-free
    // 16-byte shared loads) with the slice's longest task as its trip count
    std::vector<int64_t> sp;     // staged start of each level (multiple of 32)
    std::vector<int64_t> srb;    // record base of each staged slice (prefix sums of 32 * K)
    std::vector<int32_t> posof;  // staged position of each unknown
    int64_t ch = 0, emax = 0, ns = 0, maxw32 = 0, far = 0;
    int32_t lean_n = 0;
    if (single_cta) {
        sp.assign(nlev + 1, 0);
        for (int32_t l = 0; l < nlev; ++l) {
            const int64_t w = lstart[l + 1] - lstart[l];
            sp[l + 1] = sp[l] + (w + 31) / 32 * 32;
            maxw32 = std::max(maxw32, (w + 31) / 32 * 32);
        }
        ns = sp[nlev];
        posof.resize(n);
        for (int32_t l = 0; l < nlev; ++l)
            for (int64_t q = lstart[l]; q < lstart[l + 1]; ++q) posof[order[q]] = (int32_t)(sp[l] + (q - lstart[l]));
        // dependencies older than the ring, longest task
        int64_t maxlen = 0;
        for (int32_t l = 0; l < nlev; ++l)
            for (int64_t gq = lstart[l]; gq < lstart[l + 1]; ++gq) {
                const int32_t t = order[gq];
                const int64_t q = sp[l] + (gq - lstart[l]);
                maxlen = std::max(maxlen, tptr[t + 1] - tptr[t]);
                for (int64_t k = tptr[t]; k < tptr[t + 1]; ++k)
                    if (q - posof[ent[k].col] + maxw32 >= kRing) ++far;
            }
        // lean variant: one task per consumer thread and level, every task in
        // registers (dot tasks of >= 16 entries take the blocked BLAS order,
        // which the lean chain does not implement), no far dependencies
        const char *lean_env = getenv("RSB_TRSV_LEAN");
        if (!(lean_env && std::strcmp(lean_env, "0") == 0) && maxw32 <= kLeanMaxWidth && far == 0 &&
            maxlen <= (is_dot ? 15 : kLeanMaxN))
            lean_n = (int32_t)std::max<int64_t>(1, maxlen);
        if (lean_n && getenv("RSB_LEAN_N_MIN"))  // experiments: longer chains than needed
            lean_n = std::max<int32_t>(lean_n, std::min<int32_t>(is_dot ? 15 : 16, atoi(getenv("RSB_LEAN_N_MIN"))));
        const int64_t nsl = ns / 32;
        const int64_t ch_max = getenv("RSB_STAGE_CH_MAX") ? atoll(getenv("RSB_STAGE_CH_MAX")) : 1024;  // experiments
        // record layout and chunk size; a lean schedule whose chunks do not
        // fit falls back to the general staged layout
        for (int attempt = 0; attempt < 2 && ch == 0; ++attempt) {
            if (attempt == 1) {
                if (!lean_n) break;
                lean_n = 0;
            }
            srb.assign(nsl + 1, 0);
            for (int32_t l = 0; l < nlev; ++l)
                for (int64_t q0 = sp[l]; q0 < sp[l + 1]; q0 += 32) {
                    int64_t K = 0;
                    for (int64_t q = q0; q < q0 + 32; ++q) {
                        const int64_t src_q = lstart[l] + (q - sp[l]);
                        if (src_q < lstart[l + 1]) K = std::max(K, tptr[order[src_q] + 1] - tptr[order[src_q]]);
                    }
                    // lean: entry slots padded to whole quads (sources are read 4 at a time)
                    srb[q0 / 32 + 1] = 32 * (lean_n ? (K + 3) & ~3LL : K);
                }
            for (int64_t w = 0; w < nsl; ++w) srb[w + 1] += srb[w];
            for (int64_t cand : {1024, 512, 256, 128}) {
                if (cand > ch_max) continue;
                if (cand < maxw32) break;
                int64_t em = 0;
                for (int64_t c0 = 0; c0 < ns; c0 += cand)
                    em = std::max(em, srb[std::min(ns, c0 + cand) / 32] - srb[c0 / 32]);
                em = std::max<int64_t>(128, em);
                const int64_t lslots = (lean_n + 3) & ~3;  // lean: uniform entry slots per task
                if (lean_n) em = cand * lslots;
                const int64_t bytes = lean_n ? lean_dyn_smem_bytes(cand, lslots, !unit, nlev, (ns + cand - 1) / cand) +
                                                   kLeanRingBytes
                                             : stage_smem_bytes(cand, em, !unit, nlev, (ns + cand - 1) / cand);
                if (bytes <= kStageSmemBudget) {
                    ch = cand;
                    emax = em;
                    break;
                }
            }
        }
        if (ch == 0) {
            single_cta = false;
            lean_n = 0;
            far = 0;
        }
    }

    phase("slices + staged layout");
    std::vector<int32_t> ecol(slots, -1);
    std::vector<double> eval(slots, 0.0);
    const int64_t nchunks = single_cta ? (ns + ch - 1) / ch : 0;
    const int64_t padded = single_cta ? nchunks * ch : n;
    std::vector<double> tdiag;
    if (!unit) tdiag.assign(padded, 1.0);
    for (int64_t w = 0; w < nslices; ++w) {
        for (int64_t l = 0; l < 32 && w * 32 + l < n; ++l) {
            const int64_t q = w * 32 + l;  // task position
            const int32_t t = order[q];
            for (int64_t k = tptr[t]; k < tptr[t + 1]; ++k) {
                const int64_t e = soff[w] + (k - tptr[t]) * 32 + l;
                ecol[e] = ent[k].col;
                eval[e] = ent[k].val;
            }
            if (!unit) tdiag[q] = diag[t];
        }
    }
    // staged layout: per-position meta, {diag, 1/diag}, entry records whose
    // source is the ring byte offset of a live dependency or -(row + 2).
    // Records are lane-interleaved per slice (entry q of lane l at
    // slice_base + 32q + l), or, lean, values in lane pairs (entry q of lane l
    // at slice_base + 64(q/2) + 2l + q%2) and sources in lane quads (at
    // slice_base + 128(q/4) + 4l + q%4), zero past each task's length.
    std::vector<StageRec> recs;
    std::vector<double> rval;
    std::vector<int32_t> rsrc;
    std::vector<StageMeta> meta;
    std::vector<double> dd;
    std::vector<int64_t> croff;
    std::vector<int32_t> srows;
    const int64_t lslots = (lean_n + 3) & ~3;
    if (single_cta) {
        const int64_t nslots = std::max<int64_t>(128, srb[ns / 32]);
        if (lean_n) {
            // uniform slots: entry e of the task at position q at
            // (q - lane) * lslots + 64 (e / 2) + 2 lane + e % 2 (values) and
            // (q - lane) * lslots + 128 (e / 4) + 4 lane + e % 4 (sources);
            // empty slots read the ring's zero slot
            rval.assign(padded * lslots, 0.0);
            rsrc.assign(padded * lslots, (int32_t)(kRing * 8));
        } else {
            recs.assign(nslots, StageRec{0.0, 0, 0});
        }
        meta.assign(padded, StageMeta{-1, 0, 0, 0});
        srows.assign(padded, -1);
        croff.resize(nchunks + 1);
        for (int64_t c = 0; c <= nchunks; ++c) croff[c] = srb[std::min(ns, c * ch) / 32];
        dd.assign(2 * padded, 1.0);
        for (int32_t l = 0; l < nlev; ++l) {
            for (int64_t q = sp[l]; q < sp[l + 1]; ++q) {
                const int64_t sl = q / 32, lane = q & 31;
                int32_t K = 0;  // the slice's longest task
                for (int64_t q2 = sl * 32; q2 < sl * 32 + 32; ++q2) {
                    const int64_t g2 = lstart[l] + (q2 - sp[l]);
                    if (g2 < lstart[l + 1]) K = std::max<int32_t>(K, (int32_t)(tptr[order[g2] + 1] - tptr[order[g2]]));
                }
                // lean: the slice base in its chunk; else the lane's first record
                const int32_t roff = (int32_t)(srb[sl] - croff[q / ch] + (lean_n ? 0 : lane));
                const int64_t gq = lstart[l] + (q - sp[l]);
                if (gq >= lstart[l + 1]) {  // padding task
                    meta[q] = StageMeta{-1, 0, roff, K};
                    continue;
                }
                const int32_t t = order[gq];
                for (int64_t k = tptr[t]; k < tptr[t + 1]; ++k) {
                    const int32_t col = ent[k].col;
                    const int64_t p = posof[col];
                    const int32_t src = (q - p + maxw32 < kRing) ? (int32_t)((p & (kRing - 1)) * 8) : -(col + 2);
                    const int64_t e = k - tptr[t];
                    if (lean_n) {
                        const int64_t base = (q - lane) * lslots;
                        rval[base + (e >> 1) * 64 + lane * 2 + (e & 1)] = ent[k].val;
                        rsrc[base + (e >> 2) * 128 + lane * 4 + (e & 3)] = src;
                    } else {
                        recs[srb[sl] + e * 32 + lane] = StageRec{ent[k].val, src, 0};
                    }
                }
                meta[q] = StageMeta{t, (int32_t)(tptr[t + 1] - tptr[t]), roff, K};
                srows[q] = t;
                if (!unit) {
                    dd[2 * q] = diag[t];
                    const double y = 1.0 / diag[t];  // correctly rounded reciprocal
                    const double ad = std::fabs(diag[t]);
                    // lean: y = 0 marks a diagonal outside the exact-division range
                    dd[2 * q + 1] = (lean_n && !(ad > 0x1p-500 && ad < 0x1p500)) ? 0.0 : y;
                }
            }
        }
    }
    // lean producer events (k_trsv_lean): chunk c is issued once the level
    // barriers show that chunk c - kStageBufs is done with (levels below
    // lvl[j] are, after barrier j - 1), and awaited before barrier j when
    // iteration j + 1 prefetches from it (positions below lvl[j + 3]);
    // level -1 is the prologue, before the first barrier
    std::vector<int2> events;
    if (lean_n) {
        auto L = [&](int64_t i) { return (int64_t)(i <= nlev ? sp[i] : sp[nlev]); };
        std::vector<int64_t> iss(nchunks, -1), wt(nchunks, -1);
        for (int64_t c = 0, j = 0; c < nchunks; ++c) {
            if (c < kStageBufs) continue;
            while (j < nlev && L(j) / ch + kStageBufs - 1 < c) ++j;
            iss[c] = j;
        }
        for (int64_t c = 0, j = 0; c < nchunks; ++c) {
            if (c <= (std::max<int64_t>(L(2), 1) - 1) / ch) continue;
            while (j < nlev && (L(j + 3) - 1) / ch < c) ++j;
            wt[c] = j;
        }
        // both are non-decreasing in c: merge by level, issues first
        for (int64_t j = -1, ci = 0, cw = 0; j < nlev; ++j) {
            for (; ci < nchunks && iss[ci] == j; ++ci) events.push_back(make_int2((int)j, (int)ci));
            for (; cw < nchunks && wt[cw] == j; ++cw) events.push_back(make_int2((int)j, (int)(-cw - 1)));
        }
        events.push_back(make_int2((int)nlev + 1, 0));  // sentinel
    }
    phase("packing");
    if (getenv("RSB_DEBUG_ANALYSIS"))
        fprintf(stderr, "[rsb] tri kind=%d n=%lld levels=%d maxw=%lld single_cta=%d lean_n=%d far=%lld ch=%lld emax=%lld "
                "\n",
                kind, (long long)n, nlev, (long long)maxw, (int)single_cta, lean_n, (long long)far, (long long)ch,
                (long long)emax);
    std::vector<int32_t> rows(order.begin(), order.end());
    rows.resize(padded, 0);
    if (single_cta) rows = srows;  // the staged kernel's gather uses staged positions

    rsb_ctx *ctx = T->ctx;
    auto *S = new TriSched();
    S->kind = kind;
    S->n = (int32_t)n;
    S->nlevels = nlev;
    S->max_width = maxw;
    S->entries = slots;
    S->mode = (is_dot ? 1 : 0) | (unit ? 0 : 2);
    S->single_cta = single_cta;
    S->far_entries = far;
    S->has_far = far > 0;
    S->stage_ch = (int32_t)ch;
    S->stage_emax = (int32_t)emax;
    S->nchunks = (int32_t)nchunks;
    S->padded_n = padded;
    S->nrecs = (int64_t)(lean_n ? rval.size() : recs.size());
    if (lean_n) S->stage_emax = (int32_t)(ch * lslots);
    S->lean_nev = (int32_t)events.size();
    S->lean_n = lean_n;
    int rc = RSB_OK;
    if (S->single_cta &&
        (rc = lean_n ? prepare_trsv_lean(lean_dyn_smem_bytes(ch, lslots, !unit, nlev, nchunks))
                     : prepare_trsv_cta((int64_t)stage_smem_bytes(ch, emax, !unit, nlev, nchunks))) != RSB_OK) {
        delete S;
        return rc;
    }
    std::vector<int32_t> lptr(lstart.begin(), lstart.end());
    if (single_cta) lptr.assign(sp.begin(), sp.end());
    {
        int64_t ml = 0;
        for (int64_t t = 0; t < n; ++t) ml = std::max(ml, tptr[t + 1] - tptr[t]);
        S->max_task = (int32_t)ml;
        // the wide kernel's register entries: the smallest of 4 / 8 / 12 that
        // holds at least 94% of the tasks (the rest take the batched tail)
        {
            int64_t le4 = 0, le8 = 0;
            for (int64_t t = 0; t < n; ++t) {
                const int64_t len = tptr[t + 1] - tptr[t];
                le4 += len <= 4;
                le8 += len <= 8;
            }
            S->wide_n = (ml <= 4 || le4 >= n * 94 / 100) ? 4 : ((ml <= 8 || le8 >= n * 94 / 100) ? 8 : 12);
            S->wide_static = (S->mode == 0) && le4 >= n * 3 / 4;
            if (is_dot && ml >= S->wide_n) S->wide_n = 12;  // dot-order tasks: the tail keeps the scalar chain (< 16)
            const char *wn = getenv("RSB_WIDE_N");  // experiments
            if (wn) S->wide_n = std::max(4, std::min(12, atoi(wn))) <= 4 ? 4 : (atoi(wn) <= 8 ? 8 : 12);
        }
        const char *wv = getenv("RSB_TRSV_WIDE");  // "0": the previous grid kernel (experiments)
        S->wide = !single_cta && !(is_dot && ml >= 16) && !(wv && std::strcmp(wv, "0") == 0);
    }
    if (!single_cta) {
        // a grid launch per level is an option (RSB_TRSV_GRID=levels); on
        // config 4 at mu = 1 (23 / 66 levels) it measured 2x slower than the
        // sync-free kernel, so it is off by default
        const char *gv = getenv("RSB_TRSV_GRID");  // "levels" | "syncfree" (experiments)
        S->level_launch = nlev <= kLevelLaunchMaxLevels;
        if (gv && std::strcmp(gv, "levels") == 0) S->level_launch = true;
        if (gv && std::strcmp(gv, "syncfree") == 0) S->level_launch = false;
        S->h_level_ptr = lptr;
        // level-synchronous items (trsv_lsync.cu, RSB_TRSV_GRID=lsync) for wide
        // DAGs of at most kLsMaxLevels levels
        S->lsync = S->wide && nlev <= kLsMaxLevels && gv && std::strcmp(gv, "lsync") == 0;
        if (S->lsync) S->level_launch = false;
        // the level-synchronous cooperative kernel (RSB_TRSV_GRID=levelsync):
        // measured slower than the sync-free default on config 4 at n = 8e6
        // (U 1.13 vs 0.77 ms: every level waits for its longest rows;
        // profiles/trsv_sweep_r02.json)
        S->level_sync = S->wide && !S->lsync && !S->level_launch && gv && std::strcmp(gv, "levelsync") == 0;
    }
    std::vector<int32_t> ls_pos, ls_lev, ls_lit;
    if (S->lsync) {
        for (int32_t l = 0; l < nlev; ++l) {
            ls_lit.push_back((int32_t)ls_lev.size());
            // items end on slice boundaries (a warp's item is one slice's lanes)
            for (int64_t q = lptr[l]; q < lptr[l + 1]; q = (q / kLsItem + 1) * kLsItem) {
                ls_pos.push_back((int32_t)q);
                ls_lev.push_back(l);
            }
        }
        ls_lit.push_back((int32_t)ls_lev.size());
        ls_pos.push_back((int32_t)n);
        S->ls_nitems = (int32_t)ls_lev.size();
    }
    if ((rc = dev_upload(ctx, &S->level_ptr, lptr.data(), lptr.size())) != RSB_OK ||
        (rc = dev_upload(ctx, &S->task_row, rows.data(), rows.size())) != RSB_OK ||
        (rc = dev_upload(ctx, &S->slice_off, soff.data(), nslices + 1)) != RSB_OK ||
        (rc = dev_upload(ctx, &S->ecol, ecol.data(), slots)) != RSB_OK ||
        (rc = dev_upload(ctx, &S->eval, eval.data(), slots)) != RSB_OK ||
        (!unit && (rc = dev_upload(ctx, &S->diag, tdiag.data(), tdiag.size())) != RSB_OK) ||
        (single_cta && (rc = dev_upload(ctx, &S->chunk_roff, croff.data(), croff.size())) != RSB_OK) ||
        ((single_cta || S->wide) && (rc = dev_alloc(ctx, (void **)&S->bpos, padded * sizeof(double))) != RSB_OK) ||
        (single_cta && !lean_n && (rc = dev_upload(ctx, &S->recs, recs.data(), recs.size())) != RSB_OK) ||
        (lean_n && (rc = dev_upload(ctx, &S->rval, rval.data(), rval.size())) != RSB_OK) ||
        (lean_n && (rc = dev_upload(ctx, &S->rsrc, rsrc.data(), rsrc.size())) != RSB_OK) ||
        (lean_n && (rc = dev_upload(ctx, &S->lean_ev, events.data(), events.size())) != RSB_OK) ||
        (single_cta && (rc = dev_upload(ctx, &S->meta, meta.data(), meta.size())) != RSB_OK) ||
        (single_cta && !unit && (rc = dev_upload(ctx, &S->ddiag, dd.data(), dd.size())) != RSB_OK) ||
        (rc = dev_alloc(ctx, (void **)&S->ticket, sizeof(unsigned long long))) != RSB_OK ||
        (S->lsync && (rc = dev_upload(ctx, &S->ls_item_pos, ls_pos.data(), ls_pos.size())) != RSB_OK) ||
        (S->lsync && (rc = dev_upload(ctx, &S->ls_item_level, ls_lev.data(), ls_lev.size())) != RSB_OK) ||
        (S->lsync && (rc = dev_upload(ctx, &S->ls_level_items, ls_lit.data(), ls_lit.size())) != RSB_OK) ||
        (S->lsync && (rc = dev_alloc(ctx, (void **)&S->ls_cnt, kLsCounters * sizeof(unsigned))) != RSB_OK) ||
        (getenv("RSB_TRSV_PROFILE") && (rc = dev_alloc(ctx, (void **)&S->prof, (8 + 4096) * sizeof(long long))) != RSB_OK)) {
        tri_free(ctx, S);
        return rc;
    }
    cudaError_t e = cudaMemsetAsync(S->ticket, 0, sizeof(unsigned long long), ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // host vectors die here
    phase("upload");
    if (e != cudaSuccess) {
        set_error("CUDA error %s in triangular analysis upload", cudaGetErrorString(e));
        tri_free(ctx, S);
        return RSB_ECUDA;
    }
    *out = S;
    return RSB_OK;
}

void tri_free(rsb_ctx *ctx, TriSched *s) {
    if (!s) return;
    const int64_t n = s->n, nslices = (n + 31) / 32, padded = s->padded_n ? s->padded_n : n;
    dev_free(ctx, s->task_row, padded * sizeof(int32_t));
    dev_free(ctx, s->slice_off, (nslices + 1) * sizeof(int64_t));
    dev_free(ctx, s->ecol, s->entries * sizeof(int32_t));
    dev_free(ctx, s->eval, s->entries * sizeof(double));
    if (s->diag) dev_free(ctx, s->diag, padded * sizeof(double));
    dev_free(ctx, s->ticket, sizeof(unsigned long long));
    dev_free(ctx, s->level_ptr, (s->nlevels + 1) * sizeof(int32_t));
    if (s->ls_item_pos) dev_free(ctx, s->ls_item_pos, (s->ls_nitems + 1) * sizeof(int32_t));
    if (s->ls_item_level) dev_free(ctx, s->ls_item_level, s->ls_nitems * sizeof(int32_t));
    if (s->ls_level_items) dev_free(ctx, s->ls_level_items, (s->nlevels + 1) * sizeof(int32_t));
    if (s->ls_cnt) dev_free(ctx, s->ls_cnt, kLsCounters * sizeof(unsigned));
    if (s->chunk_roff) dev_free(ctx, s->chunk_roff, (s->nchunks + 1) * sizeof(int64_t));
    if (s->bpos) dev_free(ctx, s->bpos, padded * sizeof(double));
    if (s->recs) dev_free(ctx, s->recs, s->nrecs * sizeof(StageRec));
    if (s->rval) dev_free(ctx, s->rval, s->nrecs * sizeof(double));
    if (s->rsrc) dev_free(ctx, s->rsrc, s->nrecs * sizeof(int32_t));
    if (s->lean_ev) dev_free(ctx, s->lean_ev, s->lean_nev * sizeof(int2));
    if (s->meta) dev_free(ctx, s->meta, padded * sizeof(StageMeta));
    if (s->ddiag) dev_free(ctx, s->ddiag, 2 * padded * sizeof(double));
    if (s->prof) dev_free(ctx, s->prof, (8 + 4096) * sizeof(long long));
    delete s;
}

}  // namespace rsb
