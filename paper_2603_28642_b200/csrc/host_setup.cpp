// Host setup kept on the CPU (north star: "the serial ILUP threshold-pivoting
// factorization stays in the host setup, is timed separately, and produces
// factors the GPU path consumes unchanged").
//
// Native restatements, bit-identical to the reference package, of
//   ilup_factorize     pkg/src/rowsplit/ilup.py:211-368 (il.py)
//   build_y_explicit   pkg/src/rowsplit/precond.py:55-82 (with the
//                      sparse-RHS solve of sparse_core.py:328-397)
//   dense_cholesky_factorize  sparse_core.py:585-604
//   column_scale       sparse_core.py:405-425
// so the B200 path can be set up at the BASELINE sizes on a box that has no
// copy of the reference (the reference's Python ILUP needs ~1.5 h for config
// 4 at mu = 1 and months at mu = 0.1).  Every operation keeps
// the reference's order and rounding: numpy elementwise ops are one IEEE
// operation each, compiled here with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "../../include/rowsplit_b200.h"

namespace rsb {
void set_error(const char *fmt, ...);
}
using rsb::set_error;

struct rsb_ilup {
    int64_t m = 0, n = 0, nmod = 0;
    std::vector<int64_t> row_at, pos_of, rc;
    std::vector<int64_t> l1_ptr, l1_idx, l2_ptr, l2_idx, u_ptr, u_idx;
    std::vector<double> l1_val, l2_val, u_val;
};

namespace {

// numpy pairwise summation (same recipe as the device kernels)
double pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

// _dual_drop (il.py:159-167): keep |v| >= tau and v != 0; if more than p
// remain keep the p largest |v| (ties: smaller id first); return sorted by id.
// The same rule without sorting the whole column: the p survivors are kept
// in a small array ordered best-first by (|v| descending, id ascending) --
// np.lexsort((ids, -abs(vals))) -- while the entries stream past, then put
// in id order.  ids are unique, so the selection is the same set.
void dual_drop_fast(std::vector<int64_t> &ids, std::vector<double> &vals, int64_t p, double tau,
                    std::vector<int64_t> &sid, std::vector<double> &sv) {
    size_t k = 0;
    for (size_t i = 0; i < ids.size(); ++i)
        if (std::fabs(vals[i]) >= tau && vals[i] != 0.0) {
            ids[k] = ids[i];
            vals[k] = vals[i];
            ++k;
        }
    ids.resize(k);
    vals.resize(k);
    auto by_id = [&](std::vector<int64_t> &I, std::vector<double> &V) {
        for (size_t a = 1; a < I.size(); ++a) {
            const int64_t ki = I[a];
            const double kv = V[a];
            size_t b = a;
            for (; b > 0 && I[b - 1] > ki; --b) {
                I[b] = I[b - 1];
                V[b] = V[b - 1];
            }
            I[b] = ki;
            V[b] = kv;
        }
    };
    if ((int64_t)k <= p) {
        if (k > 64) {
            std::vector<size_t> ord(k);
            std::iota(ord.begin(), ord.end(), 0);
            std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return ids[a] < ids[b]; });
            sid.resize(k);
            sv.resize(k);
            for (size_t i = 0; i < k; ++i) {
                sid[i] = ids[ord[i]];
                sv[i] = vals[ord[i]];
            }
            ids.swap(sid);
            vals.swap(sv);
        } else {
            by_id(ids, vals);
        }
        return;
    }
    // key order: larger |v| first; NaN magnitudes last (numpy sorts NaN to
    // the end); ties by smaller id
    auto better = [](double ma, int64_t ia, double mb, int64_t ib) {
        const bool na = std::isnan(ma), nb = std::isnan(mb);
        if (na || nb) return na == nb ? ia < ib : nb;
        if (ma != mb) return ma > mb;
        return ia < ib;
    };
    sid.clear();
    sv.clear();
    thread_local std::vector<double> smag;
    smag.clear();
    for (size_t i = 0; i < k; ++i) {
        const double mi = std::fabs(vals[i]);
        const int64_t ii = ids[i];
        if ((int64_t)sid.size() == p && !better(mi, ii, smag.back(), sid.back())) continue;
        if ((int64_t)sid.size() < p) {
            sid.push_back(ii);
            sv.push_back(vals[i]);
            smag.push_back(mi);
        } else {
            sid.back() = ii;
            sv.back() = vals[i];
            smag.back() = mi;
        }
        for (size_t b = sid.size() - 1; b > 0 && better(smag[b], sid[b], smag[b - 1], sid[b - 1]); --b) {
            std::swap(sid[b], sid[b - 1]);
            std::swap(sv[b], sv[b - 1]);
            std::swap(smag[b], smag[b - 1]);
        }
    }
    ids.assign(sid.begin(), sid.end());
    vals.assign(sv.begin(), sv.end());
    by_id(ids, vals);
}

// CscMatrix.from_coo for entries without duplicates or zeros (the factor
// assembly of il.py:349-359): sort rows inside every column.
void coo_to_csc(int64_t ncols, const std::vector<int64_t> &rows, const std::vector<int64_t> &cols,
                const std::vector<double> &vals, std::vector<int64_t> &ptr, std::vector<int64_t> &idx,
                std::vector<double> &val) {
    const size_t nnz = rows.size();
    ptr.assign(ncols + 1, 0);
    for (size_t k = 0; k < nnz; ++k) ptr[cols[k] + 1]++;
    for (int64_t j = 0; j < ncols; ++j) ptr[j + 1] += ptr[j];
    idx.resize(nnz);
    val.resize(nnz);
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (size_t k = 0; k < nnz; ++k) {
        const int64_t d = fill[cols[k]]++;
        idx[d] = rows[k];
        val[d] = vals[k];
    }
    std::vector<std::pair<int64_t, double>> tmp;
    for (int64_t j = 0; j < ncols; ++j) {
        const int64_t lo = ptr[j], hi = ptr[j + 1];
        bool sorted = true;
        for (int64_t k = lo + 1; k < hi; ++k)
            if (idx[k] < idx[k - 1]) {
                sorted = false;
                break;
            }
        if (sorted) continue;
        tmp.clear();
        for (int64_t k = lo; k < hi; ++k) tmp.emplace_back(idx[k], val[k]);
        std::sort(tmp.begin(), tmp.end(), [](const auto &a, const auto &b) { return a.first < b.first; });
        for (int64_t k = lo; k < hi; ++k) {
            idx[k] = tmp[k - lo].first;
            val[k] = tmp[k - lo].second;
        }
    }
}

}  // namespace

extern "C" {

int rsb_ilup_factorize(int64_t m, int64_t n, const int64_t *ptr, const int64_t *ridx, const double *avals,
                       int64_t p, double tau, double mu, double small, rsb_ilup **out) {
    *out = nullptr;
    if (p < 1 || tau < 0.0 || !(mu > 0.0 && mu <= 1.0) || !(small > 0.0)) {
        set_error("invalid IlupParams");
        return RSB_EINVAL;
    }
    if (n < 1 || m < 1) {
        set_error("empty matrix");
        return RSB_EINVAL;
    }
    if (m < n) {
        set_error("need nrows >= ncols, got %lld x %lld", (long long)m, (long long)n);
        return RSB_EINVAL;
    }
    auto F = new rsb_ilup();
    F->m = m;
    F->n = n;
    if (m >= (int64_t)1 << 31) {
        set_error("ilup_factorize: %lld rows exceed the int32 row index", (long long)m);
        delete F;
        return RSB_EINVAL;
    }
    // Per-row working state in one 16-byte record, so that touching a row of
    // the column's pattern (mark, position, value, remaining count) costs one
    // cache line: at config-4 size (m = 1.6e7) every pattern row is a miss.
    // rcm = 2 * remaining_row_count + mark; a pivotal row also carries its
    // L column (loff, llen), so the reach DFS goes row record -> L rows ->
    // child records with no detour through a per-position pointer array.
    struct alignas(32) RowSt {
        double x;
        int32_t pos;
        int32_t rcm;
        int64_t loff;
        int32_t llen;
        int32_t pad;
    };
    std::vector<RowSt> R(m);
    std::vector<int32_t> row_at(m);
    for (int64_t i = 0; i < m; ++i) {
        R[i].x = 0.0;
        R[i].pos = (int32_t)i;
        R[i].rcm = 0;
        R[i].loff = 0;
        R[i].llen = 0;
        row_at[i] = (int32_t)i;
    }
    for (int64_t k = 0; k < ptr[n]; ++k) R[ridx[k]].rcm += 2;  // remaining_row_counts (il.py:153-156)
    std::vector<double> col_inf(n, 0.0);  // np.maximum.reduceat(|A|) (il.py:235-238)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k) col_inf[j] = std::max(col_inf[j], std::fabs(avals[k]));

    // L columns (original row ids, as kept) and U columns (pivot positions,
    // diagonal last), both appended column by column
    std::vector<int64_t> l_ptr(1, 0), u_ptr(1, 0);
    std::vector<int32_t> l_rows, u_rows;
    std::vector<double> l_vals, u_vals;
    l_ptr.reserve(n + 1);
    u_ptr.reserve(n + 1);
    l_rows.reserve((size_t)n * std::min<int64_t>(p, 12));
    l_vals.reserve((size_t)n * std::min<int64_t>(p, 12));
    u_rows.reserve((size_t)n * std::min<int64_t>(p + 1, 12));
    u_vals.reserve((size_t)n * std::min<int64_t>(p + 1, 12));

    std::vector<int32_t> pattern, post, stack_node, stack_cur;
    std::vector<int64_t> u_pos, cand_pos;
    std::vector<int32_t> cand;
    std::vector<double> u_val, cval;
    std::vector<int64_t> sel_id;
    std::vector<double> sel_v;
    int64_t nmod = 0;
    auto mark_of = [&](int32_t r) { return R[r].rcm & 1; };
    auto set_mark = [&](int32_t r) { R[r].rcm |= 1; };
    // the children of a node about to be expanded are checked one after the
    // other; start all their record loads at once
    auto prefetch_children = [&](int32_t node) {
        const int64_t lo = R[node].loff, hi = lo + R[node].llen;
        for (int64_t e = lo; e < hi; ++e) __builtin_prefetch(&R[l_rows[e]]);
    };

    for (int64_t j = 0; j < n; ++j) {
        const int64_t alo = ptr[j], ahi = ptr[j + 1], alen = ahi - alo;
        for (int64_t k = alo; k < ahi; ++k) R[ridx[k]].x = avals[k];
        pattern.clear();
        u_pos.clear();
        u_val.clear();
        if (j == 0 || alen == 0) {
            for (int64_t k = alo; k < ahi; ++k) {
                set_mark((int32_t)ridx[k]);
                pattern.push_back((int32_t)ridx[k]);
            }
        } else if (alen >= std::max<int64_t>(8, j / 8)) {
            // dense-ish column: sweep pivot positions in order (il.py:258-279)
            for (int64_t k = alo; k < ahi; ++k) {
                set_mark((int32_t)ridx[k]);
                pattern.push_back((int32_t)ridx[k]);
            }
            for (int64_t q = 0; q < j; ++q) {
                const int32_t u = row_at[q];
                const double xu = R[u].x;
                if (xu == 0.0) continue;
                u_pos.push_back(q);
                u_val.push_back(xu);
                for (int64_t e = l_ptr[q]; e < l_ptr[q + 1]; ++e) {
                    RowSt &rr = R[l_rows[e]];
                    const double c = l_vals[e] * xu;
                    rr.x = rr.x - c;
                }
                for (int64_t e = l_ptr[q]; e < l_ptr[q + 1]; ++e) {
                    const int32_t r = l_rows[e];
                    if (!mark_of(r)) {
                        set_mark(r);
                        pattern.push_back(r);
                    }
                }
            }
        } else {
            // sparse column: DFS reach over the partial factor (il.py:170-208)
            post.clear();
            for (int64_t k = alo; k < ahi; ++k) {
                const int32_t s = (int32_t)ridx[k];
                if (mark_of(s)) continue;
                set_mark(s);
                pattern.push_back(s);
                if (R[s].pos >= j) continue;
                stack_node.assign(1, s);
                stack_cur.assign(1, 0);
                prefetch_children(s);
                while (!stack_node.empty()) {
                    const int32_t node = stack_node.back();
                    int32_t cursor = stack_cur.back();
                    const int64_t clo = R[node].loff;
                    const int32_t clen = R[node].llen;
                    bool advanced = false;
                    while (cursor < clen) {
                        const int32_t child = l_rows[clo + cursor];
                        ++cursor;
                        if (!mark_of(child)) {
                            set_mark(child);
                            pattern.push_back(child);
                            if (R[child].pos < j) {
                                stack_cur.back() = cursor;
                                stack_node.push_back(child);
                                stack_cur.push_back(0);
                                prefetch_children(child);
                                advanced = true;
                                break;
                            }
                        }
                    }
                    if (!advanced) {
                        stack_node.pop_back();
                        stack_cur.pop_back();
                        post.push_back(node);
                    }
                }
            }
            // eliminate reached pivots in topological order (reversed post-order)
            for (auto it = post.rbegin(); it != post.rend(); ++it) {
                const int32_t u = *it;
                const double xu = R[u].x;
                if (xu == 0.0) continue;
                const int64_t q = R[u].pos;
                u_pos.push_back(q);
                u_val.push_back(xu);
                for (int64_t e = R[u].loff, ee = e + R[u].llen; e < ee; ++e) {
                    RowSt &rr = R[l_rows[e]];
                    const double c = l_vals[e] * xu;
                    rr.x = rr.x - c;
                }
            }
        }

        dual_drop_fast(u_pos, u_val, p, tau, sel_id, sel_v);  // il.py:300

        // active part: reached rows not yet pivotal, nonzero (il.py:303-307)
        cand.clear();
        cval.clear();
        for (int32_t r : pattern) {
            const RowSt &rr = R[r];
            if (rr.pos >= j && rr.x != 0.0) {
                cand.push_back(r);
                cval.push_back(rr.x);
            }
        }

        int32_t pivot_orig;
        double pivot_val;
        // modify_pivot (il.py:142-150)
        auto modified = [&]() {
            const double beta = std::pow(10.0, -2.0 * (1.0 - (double)(j + 1) / (double)n));
            return std::max(beta * col_inf[j], small);
        };
        if (cand.empty()) {
            pivot_orig = row_at[j];
            pivot_val = modified();
            ++nmod;
        } else {
            // choose_pivot (il.py:122-139): |v| >= mu * max|v|, then fewest
            // remaining row entries, then smallest position
            double mx = std::fabs(cval[0]);
            bool has_nan = std::isnan(mx);
            for (size_t i = 1; i < cval.size(); ++i) {
                const double a = std::fabs(cval[i]);
                if (std::isnan(a)) has_nan = true;
                mx = std::max(mx, a);
            }
            if (has_nan) {
                set_error("non-finite value in column %lld of the factorization", (long long)j);
                delete F;
                return RSB_ESINGULAR;
            }
            const double thr = mu * mx;
            int64_t best = -1;
            int32_t best_rc = 0, best_pos = 0;
            for (size_t i = 0; i < cand.size(); ++i) {
                if (!(std::fabs(cval[i]) >= thr)) continue;
                const RowSt &rr = R[cand[i]];
                const int32_t rc = rr.rcm >> 1;
                if (best < 0 || rc < best_rc || (rc == best_rc && rr.pos < best_pos)) {
                    best = (int64_t)i;
                    best_rc = rc;
                    best_pos = rr.pos;
                }
            }
            pivot_orig = cand[best];
            pivot_val = R[pivot_orig].x;
            if (std::fabs(pivot_val) < small) {
                pivot_val = modified();
                ++nmod;
            }
            size_t k = 0;
            for (size_t i = 0; i < cand.size(); ++i)
                if (cand[i] != pivot_orig) {
                    cand[k] = cand[i];
                    cval[k] = cval[i];
                    ++k;
                }
            cand.resize(k);
            cval.resize(k);
        }

        // interchange (il.py:324-328)
        const int32_t q = R[pivot_orig].pos;
        if (q != j) {
            const int32_t other = row_at[j];
            row_at[j] = pivot_orig;
            row_at[q] = other;
            R[pivot_orig].pos = (int32_t)j;
            R[other].pos = q;
        }

        // scale, then drop in the L column by current position (il.py:331-339)
        cand_pos.clear();
        for (size_t i = 0; i < cand.size(); ++i) {
            cand_pos.push_back(R[cand[i]].pos);
            cval[i] = cval[i] / pivot_val;
        }
        dual_drop_fast(cand_pos, cval, p, tau, sel_id, sel_v);
        for (size_t i = 0; i < cand_pos.size(); ++i) {
            l_rows.push_back(row_at[cand_pos[i]]);
            l_vals.push_back(cval[i]);
        }
        R[pivot_orig].loff = l_ptr.back();
        R[pivot_orig].llen = (int32_t)(l_rows.size() - l_ptr.back());
        l_ptr.push_back((int64_t)l_rows.size());

        for (size_t i = 0; i < u_pos.size(); ++i) {
            u_rows.push_back((int32_t)u_pos[i]);
            u_vals.push_back(u_val[i]);
        }
        u_rows.push_back((int32_t)j);
        u_vals.push_back(pivot_val);
        u_ptr.push_back((int64_t)u_rows.size());

        for (int64_t k = alo; k < ahi; ++k) R[ridx[k]].rcm -= 2;
        for (int32_t r : pattern) {
            R[r].x = 0.0;
            R[r].rcm &= ~1;
        }
    }
    F->nmod = nmod;
    F->row_at.assign(row_at.begin(), row_at.end());
    F->pos_of.resize(m);
    F->rc.resize(m);
    for (int64_t i = 0; i < m; ++i) {
        F->pos_of[i] = R[i].pos;
        F->rc[i] = R[i].rcm >> 1;
    }
    std::vector<RowSt>().swap(R);

    // assemble in final pivot coordinates (il.py:349-359).  U: the rows of
    // column j are positions < j (fixed once pivotal), ascending, then j --
    // already CscMatrix.from_coo's sorted order.
    F->u_ptr = u_ptr;
    F->u_idx.assign(u_rows.begin(), u_rows.end());
    F->u_val = u_vals;
    {
        // L: final positions, split at n, rows sorted inside each column
        F->l1_ptr.assign(n + 1, 0);
        F->l2_ptr.assign(n + 1, 0);
        for (int64_t j = 0; j < n; ++j) {
            int64_t c1 = 0, c2 = 0;
            for (int64_t e = l_ptr[j]; e < l_ptr[j + 1]; ++e) (F->pos_of[l_rows[e]] < n ? c1 : c2)++;
            F->l1_ptr[j + 1] = F->l1_ptr[j] + c1;
            F->l2_ptr[j + 1] = F->l2_ptr[j] + c2;
        }
        F->l1_idx.resize(F->l1_ptr[n]);
        F->l1_val.resize(F->l1_ptr[n]);
        F->l2_idx.resize(F->l2_ptr[n]);
        F->l2_val.resize(F->l2_ptr[n]);
        std::vector<std::pair<int64_t, double>> tmp;
        for (int64_t j = 0; j < n; ++j) {
            int64_t d1 = F->l1_ptr[j], d2 = F->l2_ptr[j];
            tmp.clear();
            for (int64_t e = l_ptr[j]; e < l_ptr[j + 1]; ++e) tmp.emplace_back(F->pos_of[l_rows[e]], l_vals[e]);
            std::sort(tmp.begin(), tmp.end(), [](const auto &a, const auto &b) { return a.first < b.first; });
            for (const auto &t : tmp) {
                if (t.first < n) {
                    F->l1_idx[d1] = t.first;
                    F->l1_val[d1++] = t.second;
                } else {
                    F->l2_idx[d2] = t.first - n;
                    F->l2_val[d2++] = t.second;
                }
            }
        }
    }
    *out = F;
    return RSB_OK;
}
int rsb_ilup_sizes(const rsb_ilup *F, int64_t *nnz_l1, int64_t *nnz_l2, int64_t *nnz_u, int64_t *nmod) {
    *nnz_l1 = (int64_t)F->l1_idx.size();
    *nnz_l2 = (int64_t)F->l2_idx.size();
    *nnz_u = (int64_t)F->u_idx.size();
    *nmod = F->nmod;
    return RSB_OK;
}

int rsb_ilup_copy(const rsb_ilup *F, int64_t *perm, int64_t *l1_ptr, int64_t *l1_idx, double *l1_val,
                  int64_t *l2_ptr, int64_t *l2_idx, double *l2_val, int64_t *u_ptr, int64_t *u_idx,
                  double *u_val, int64_t *row_counts) {
    auto cp = [](auto *dst, const auto &src) {
        if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
    };
    cp(perm, F->row_at);
    cp(l1_ptr, F->l1_ptr);
    cp(l1_idx, F->l1_idx);
    cp(l1_val, F->l1_val);
    cp(l2_ptr, F->l2_ptr);
    cp(l2_idx, F->l2_idx);
    cp(l2_val, F->l2_val);
    cp(u_ptr, F->u_ptr);
    cp(u_idx, F->u_idx);
    cp(u_val, F->u_val);
    cp(row_counts, F->rc);
    return RSB_OK;
}

int rsb_ilup_destroy(rsb_ilup *F) {
    delete F;
    return RSB_OK;
}

// build_y_explicit (pc.py:55-82): row i of Y solves L1^T y = (row i of L2)
// by a sparse-RHS solve (sc.py:365-397) whose DFS order (sc.py:328-362)
// fixes the floating-point order; exact zeros from cancellation are dropped
// (pc.py:70-71).
int rsb_build_y_explicit(int64_t s, int64_t n, const int64_t *l1_ptr, const int64_t *l1_idx,
                         const double *l1_val, const int64_t *l2_ptr, const int64_t *l2_idx,
                         const double *l2_val, int64_t *nnz_y, int64_t *y_ptr, int64_t *y_idx, double *y_val) {
    // T = L1^T and L2^T as CSC (CscMatrix.transpose -> from_coo: rows sorted)
    std::vector<int64_t> tp(n + 1, 0), ti;
    std::vector<double> tv;
    {
        const int64_t nnz = l1_ptr[n];
        for (int64_t k = 0; k < nnz; ++k) tp[l1_idx[k] + 1]++;
        for (int64_t i = 0; i < n; ++i) tp[i + 1] += tp[i];
        ti.resize(nnz);
        tv.resize(nnz);
        std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
        for (int64_t j = 0; j < n; ++j)
            for (int64_t k = l1_ptr[j]; k < l1_ptr[j + 1]; ++k) {
                const int64_t d = fill[l1_idx[k]]++;
                ti[d] = j;
                tv[d] = l1_val[k];
            }
    }
    std::vector<int64_t> bp(s + 1, 0), bi;
    std::vector<double> bv;
    {
        const int64_t nnz = l2_ptr[n];
        for (int64_t k = 0; k < nnz; ++k) bp[l2_idx[k] + 1]++;
        for (int64_t i = 0; i < s; ++i) bp[i + 1] += bp[i];
        bi.resize(nnz);
        bv.resize(nnz);
        std::vector<int64_t> fill(bp.begin(), bp.end() - 1);
        for (int64_t j = 0; j < n; ++j)
            for (int64_t k = l2_ptr[j]; k < l2_ptr[j + 1]; ++k) {
                const int64_t d = fill[l2_idx[k]]++;
                bi[d] = j;
                bv[d] = l2_val[k];
            }
    }
    std::vector<int64_t> yr, yc;
    std::vector<double> yv;
    std::vector<double> x(n, 0.0);
    std::vector<char> marked(n, 0);
    std::vector<int64_t> topo, sn, sc;
    for (int64_t i = 0; i < s; ++i) {
        const int64_t lo = bp[i], hi = bp[i + 1];
        if (hi == lo) continue;
        // reach_pattern (sc.py:328-362): iterative DFS, reversed post-order
        topo.clear();
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t sd = bi[k];
            if (marked[sd]) continue;
            marked[sd] = 1;
            sn.assign(1, sd);
            sc.assign(1, tp[sd]);
            while (!sn.empty()) {
                const int64_t node = sn.back();
                int64_t cursor = sc.back();
                bool adv = false;
                while (cursor < tp[node + 1]) {
                    const int64_t child = ti[cursor];
                    ++cursor;
                    if (child != node && !marked[child]) {
                        marked[child] = 1;
                        sc.back() = cursor;
                        sn.push_back(child);
                        sc.push_back(tp[child]);
                        adv = true;
                        break;
                    }
                }
                if (!adv) {
                    sn.pop_back();
                    sc.pop_back();
                    topo.push_back(node);
                }
            }
        }
        std::reverse(topo.begin(), topo.end());
        for (int64_t k = lo; k < hi; ++k) x[bi[k]] = bv[k];
        for (int64_t node : topo) {  // unit diagonal: no division
            const double xv = x[node];
            if (xv != 0.0)
                for (int64_t t = tp[node]; t < tp[node + 1]; ++t) {
                    const int64_t r = ti[t];
                    if (r != node) {
                        const double c = tv[t] * xv;
                        x[r] = x[r] - c;
                    }
                }
        }
        std::vector<int64_t> pat(topo);
        std::sort(pat.begin(), pat.end());
        for (int64_t c : pat) {
            if (x[c] != 0.0) {
                yr.push_back(i);
                yc.push_back(c);
                yv.push_back(x[c]);
            }
            x[c] = 0.0;
            marked[c] = 0;
        }
    }
    const int64_t nnz = (int64_t)yr.size();
    if (!y_idx) {
        *nnz_y = nnz;
        return RSB_OK;
    }
    if (*nnz_y < nnz) {
        set_error("Y buffer too small");
        return RSB_EINVAL;
    }
    std::vector<int64_t> p, idx;
    std::vector<double> val;
    coo_to_csc(n, yr, yc, yv, p, idx, val);
    std::memcpy(y_ptr, p.data(), (n + 1) * sizeof(int64_t));
    if (nnz) {
        std::memcpy(y_idx, idx.data(), nnz * sizeof(int64_t));
        std::memcpy(y_val, val.data(), nnz * sizeof(double));
    }
    *nnz_y = nnz;
    return RSB_OK;
}

// dense_cholesky_factorize (sc.py:585-604), lower factor in place
int rsb_cholesky_factorize(int64_t s, double *g) {
    for (int64_t j = 0; j < s; ++j) {
        double d = g[j + j * s];
        if (d <= 0.0 || !std::isfinite(d)) {
            set_error("matrix is not positive definite (pivot %lld)", (long long)j);
            return RSB_ESINGULAR;
        }
        d = std::sqrt(d);
        g[j + j * s] = d;
        for (int64_t i = j + 1; i < s; ++i) g[i + j * s] /= d;
        for (int64_t k = j + 1; k < s; ++k) {
            const double gk = g[k + j * s];
            for (int64_t i = j + 1; i < s; ++i) {
                const double c = g[i + j * s] * gk;
                g[i + k * s] = g[i + k * s] - c;
            }
        }
    }
    for (int64_t k = 1; k < s; ++k)
        for (int64_t i = 0; i < k; ++i) g[i + k * s] = 0.0;
    return RSB_OK;
}

// column_scale (sc.py:405-425): sq_j = reduceat(v*v) = p0 + pairwise(rest)
int rsb_column_scale(int64_t ncols, const int64_t *ptr, const double *values, double *scaled, double *norms) {
    std::vector<double> sq;
    for (int64_t j = 0; j < ncols; ++j) {
        const int64_t lo = ptr[j], hi = ptr[j + 1];
        if (hi == lo) {
            set_error("cannot scale zero column %lld", (long long)j);
            return RSB_EINVAL;
        }
        sq.resize(hi - lo);
        for (int64_t k = lo; k < hi; ++k) sq[k - lo] = values[k] * values[k];
        const double s2 = sq[0] + pairwise(sq.data() + 1, hi - lo - 1);
        norms[j] = std::sqrt(s2);
    }
    for (int64_t j = 0; j < ncols; ++j)
        for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k) scaled[k] = values[k] / norms[j];
    return RSB_OK;
}

}  // extern "C"
