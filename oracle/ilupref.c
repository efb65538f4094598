/*
 * oracle/ilupref.c -- CPU restatement of the reference's ILUP factorization.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/rsref.c).  It lets bench.py's
 * reference arm set up the BASELINE configurations without loading the
 * product library: the reference's own ilup_factorize is pure Python and
 * does not exist on the GPU box.
 *
 * Restates pkg/src/rowsplit/ilup.py (il.py below):
 *   ilup_factorize    il.py:211-368  left-looking column ILU with threshold
 *                                    partial pivoting over the rectangular A
 *   _reach_factor     il.py:170-208  iterative DFS reach, reversed post-order
 *   _dual_drop        il.py:159-167  |v| >= tau and v != 0, then the p
 *                                    largest |v| (ties: smaller id), by id
 *   choose_pivot      il.py:122-139  |v| >= mu max|v|, fewest remaining row
 *                                    entries, then smallest position
 *   modify_pivot      il.py:142-150
 * Every arithmetic operation is the one numpy performs elementwise, so the
 * factors are bit-identical (pinned by tests/test_oracle_pin.py against the
 * reference's factors and tests/golden/cfg4_factor_hashes.json).
 *
 * Output: the factors as three CSC matrices in final pivot coordinates,
 * assembled like CscMatrix.from_coo (rows sorted inside each column), the
 * row permutation, nmod and the final remaining-row counts.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ESINGULAR 2
#define ORC_ENOMEM 4

typedef struct {
    double x;     /* working column value */
    int64_t pos;  /* current pivot position of the row */
    int64_t rc;   /* entries of the row in columns not yet processed */
    int64_t lo;   /* L column of the row once pivotal: l_rows[lo .. lo+len) */
    int32_t len;
    int32_t mark;
} orc_row;

/* growable arrays */
typedef struct { int64_t *a; int64_t n, cap; } ivec;
typedef struct { double *a; int64_t n, cap; } dvec;

static int ipush(ivec *v, int64_t x)
{
    if (v->n == v->cap) {
        int64_t c = v->cap ? 2 * v->cap : 256;
        int64_t *p = realloc(v->a, (size_t)c * sizeof(int64_t));
        if (!p) return 0;
        v->a = p;
        v->cap = c;
    }
    v->a[v->n++] = x;
    return 1;
}

static int dpush(dvec *v, double x)
{
    if (v->n == v->cap) {
        int64_t c = v->cap ? 2 * v->cap : 256;
        double *p = realloc(v->a, (size_t)c * sizeof(double));
        if (!p) return 0;
        v->a = p;
        v->cap = c;
    }
    v->a[v->n++] = x;
    return 1;
}

/* numpy's lexsort((ids, -abs(vals))) ascending: -|v| first (NaN last), id second */
static int ahead(double va, int64_t ia, double vb, int64_t ib)
{
    double ka = -fabs(va), kb = -fabs(vb);
    int na = isnan(ka), nb = isnan(kb);
    if (na || nb) return na == nb ? ia < ib : nb;
    if (ka != kb) return ka < kb;
    return ia < ib;
}

/* _dual_drop in place on (ids, vals)[0..*k); survivors sorted by id */
static void dual_drop(int64_t *ids, double *vals, int64_t *k, int64_t p, double tau)
{
    int64_t w = 0;
    for (int64_t i = 0; i < *k; i++)
        if (fabs(vals[i]) >= tau && vals[i] != 0.0) {
            ids[w] = ids[i];
            vals[w] = vals[i];
            w++;
        }
    if (w > p) {
        /* selection: move the p entries that lexsort puts first to the front */
        for (int64_t s = 0; s < p; s++) {
            int64_t b = s;
            for (int64_t i = s + 1; i < w; i++)
                if (ahead(vals[i], ids[i], vals[b], ids[b])) b = i;
            int64_t ti = ids[s]; ids[s] = ids[b]; ids[b] = ti;
            double tv = vals[s]; vals[s] = vals[b]; vals[b] = tv;
        }
        w = p;
    }
    /* np.argsort(ids): ids are distinct */
    for (int64_t a = 1; a < w; a++) {
        int64_t ki = ids[a];
        double kv = vals[a];
        int64_t b = a;
        while (b > 0 && ids[b - 1] > ki) {
            ids[b] = ids[b - 1];
            vals[b] = vals[b - 1];
            b--;
        }
        ids[b] = ki;
        vals[b] = kv;
    }
    *k = w;
}

typedef struct {
    int64_t m, n, nmod;
    int64_t *perm, *row_counts;
    int64_t *l1_ptr, *l1_idx, *l2_ptr, *l2_idx, *u_ptr, *u_idx;
    double *l1_val, *l2_val, *u_val;
} orc_factors;

void orc_ilup_free(orc_factors *F)
{
    if (!F) return;
    free(F->perm); free(F->row_counts);
    free(F->l1_ptr); free(F->l1_idx); free(F->l1_val);
    free(F->l2_ptr); free(F->l2_idx); free(F->l2_val);
    free(F->u_ptr); free(F->u_idx); free(F->u_val);
    free(F);
}

static int cmp_pair(const void *a, const void *b)
{
    int64_t x = ((const int64_t *)a)[0], y = ((const int64_t *)b)[0];
    return (x > y) - (x < y);
}

/* returns ORC_OK and *out, or an error code (column in *err_col) */
int orc_ilup_factorize(int64_t m, int64_t n, const int64_t *ptr, const int64_t *ridx, const double *avals,
                       int64_t p, double tau, double mu, double small, orc_factors **out, int64_t *err_col)
{
    *out = NULL;
    *err_col = -1;
    if (p < 1 || tau < 0.0 || !(mu > 0.0 && mu <= 1.0) || !(small > 0.0) || n < 1 || m < 1 || m < n)
        return ORC_EINVAL;
    int rc = ORC_ENOMEM;
    orc_row *R = malloc((size_t)m * sizeof(orc_row));
    int64_t *row_at = malloc((size_t)m * sizeof(int64_t));
    double *col_inf = calloc((size_t)n, sizeof(double));
    int64_t *l_ptr = malloc((size_t)(n + 1) * sizeof(int64_t));
    int64_t *u_ptr = malloc((size_t)(n + 1) * sizeof(int64_t));
    ivec l_rows = {0}, u_rows = {0}, pattern = {0}, post = {0}, st_node = {0}, st_cur = {0};
    ivec ids = {0}, cand = {0};
    dvec l_vals = {0}, u_vals = {0}, vals = {0};
    orc_factors *F = calloc(1, sizeof(orc_factors));
    if (!R || !row_at || !col_inf || !l_ptr || !u_ptr || !F) goto done;
    for (int64_t i = 0; i < m; i++) {
        R[i].x = 0.0;
        R[i].pos = i;
        R[i].rc = 0;
        R[i].lo = 0;
        R[i].len = 0;
        R[i].mark = 0;
        row_at[i] = i;
    }
    for (int64_t k = 0; k < ptr[n]; k++) R[ridx[k]].rc++;            /* il.py:153-156 */
    for (int64_t j = 0; j < n; j++)                                    /* il.py:235-238 */
        for (int64_t k = ptr[j]; k < ptr[j + 1]; k++)
            if (fabs(avals[k]) > col_inf[j]) col_inf[j] = fabs(avals[k]);
    l_ptr[0] = 0;
    u_ptr[0] = 0;
    int64_t nmod = 0;

    for (int64_t j = 0; j < n; j++) {
        const int64_t alo = ptr[j], ahi = ptr[j + 1], alen = ahi - alo;
        for (int64_t k = alo; k < ahi; k++) R[ridx[k]].x = avals[k];
        pattern.n = 0;
        ids.n = 0;
        vals.n = 0;
        if (j == 0 || alen == 0) {
            for (int64_t k = alo; k < ahi; k++) {
                R[ridx[k]].mark = 1;
                if (!ipush(&pattern, ridx[k])) goto done;
            }
        } else if (alen >= (j / 8 > 8 ? j / 8 : 8)) {
            /* dense-ish column: pivot positions in order (il.py:258-279) */
            for (int64_t k = alo; k < ahi; k++) {
                R[ridx[k]].mark = 1;
                if (!ipush(&pattern, ridx[k])) goto done;
            }
            for (int64_t q = 0; q < j; q++) {
                const int64_t u = row_at[q];
                const double xu = R[u].x;
                if (xu == 0.0) continue;
                if (!ipush(&ids, q) || !dpush(&vals, xu)) goto done;
                for (int64_t e = l_ptr[q]; e < l_ptr[q + 1]; e++) {
                    double c = l_vals.a[e] * xu;
                    R[l_rows.a[e]].x = R[l_rows.a[e]].x - c;
                }
                for (int64_t e = l_ptr[q]; e < l_ptr[q + 1]; e++) {
                    const int64_t r = l_rows.a[e];
                    if (!R[r].mark) {
                        R[r].mark = 1;
                        if (!ipush(&pattern, r)) goto done;
                    }
                }
            }
        } else {
            /* sparse column: _reach_factor (il.py:170-208), then eliminate
             * the reached pivots in reversed post-order (il.py:281-297) */
            post.n = 0;
            for (int64_t k = alo; k < ahi; k++) {
                const int64_t s = ridx[k];
                if (R[s].mark) continue;
                R[s].mark = 1;
                if (!ipush(&pattern, s)) goto done;
                if (R[s].pos >= j) continue;
                st_node.n = 0;
                st_cur.n = 0;
                if (!ipush(&st_node, s) || !ipush(&st_cur, 0)) goto done;
                while (st_node.n) {
                    const int64_t node = st_node.a[st_node.n - 1];
                    int64_t cur = st_cur.a[st_cur.n - 1];
                    const int64_t clo = R[node].lo, clen = R[node].len;
                    int adv = 0;
                    while (cur < clen) {
                        const int64_t child = l_rows.a[clo + cur];
                        cur++;
                        if (!R[child].mark) {
                            R[child].mark = 1;
                            if (!ipush(&pattern, child)) goto done;
                            if (R[child].pos < j) {
                                st_cur.a[st_cur.n - 1] = cur;
                                if (!ipush(&st_node, child) || !ipush(&st_cur, 0)) goto done;
                                adv = 1;
                                break;
                            }
                        }
                    }
                    if (!adv) {
                        st_node.n--;
                        st_cur.n--;
                        if (!ipush(&post, node)) goto done;
                    }
                }
            }
            for (int64_t t = post.n - 1; t >= 0; t--) {
                const int64_t u = post.a[t];
                const double xu = R[u].x;
                if (xu == 0.0) continue;
                if (!ipush(&ids, R[u].pos) || !dpush(&vals, xu)) goto done;
                for (int64_t e = R[u].lo; e < R[u].lo + R[u].len; e++) {
                    double c = l_vals.a[e] * xu;
                    R[l_rows.a[e]].x = R[l_rows.a[e]].x - c;
                }
            }
        }
        /* U column: dual drop (il.py:300), then the diagonal */
        int64_t nu = ids.n;
        dual_drop(ids.a, vals.a, &nu, p, tau);
        for (int64_t i = 0; i < nu; i++)
            if (!ipush(&u_rows, ids.a[i]) || !dpush(&u_vals, vals.a[i])) goto done;

        /* active part (il.py:303-307) */
        cand.n = 0;
        vals.n = 0;
        for (int64_t t = 0; t < pattern.n; t++) {
            const int64_t r = pattern.a[t];
            if (R[r].pos >= j && R[r].x != 0.0)
                if (!ipush(&cand, r) || !dpush(&vals, R[r].x)) goto done;
        }
        int64_t pivot;
        double pval;
        const double beta = pow(10.0, -2.0 * (1.0 - (double)(j + 1) / (double)n)); /* il.py:142-150 */
        double modified = beta * col_inf[j];
        if (modified < small) modified = small;
        if (cand.n == 0) {
            pivot = row_at[j];
            pval = modified;
            nmod++;
        } else {
            double mx = -1.0;
            for (int64_t i = 0; i < cand.n; i++) {
                double a = fabs(vals.a[i]);
                if (isnan(a)) {
                    *err_col = j;
                    rc = ORC_ESINGULAR;
                    goto done;
                }
                if (a > mx) mx = a;
            }
            const double thr = mu * mx;
            int64_t best = -1;
            for (int64_t i = 0; i < cand.n; i++) {
                if (!(fabs(vals.a[i]) >= thr)) continue;
                const int64_t r = cand.a[i];
                if (best < 0) { best = i; continue; }
                const int64_t b = cand.a[best];
                if (R[r].rc < R[b].rc || (R[r].rc == R[b].rc && R[r].pos < R[b].pos)) best = i;
            }
            pivot = cand.a[best];
            pval = R[pivot].x;
            if (fabs(pval) < small) {
                pval = modified;
                nmod++;
            }
            int64_t w = 0;
            for (int64_t i = 0; i < cand.n; i++)
                if (cand.a[i] != pivot) {
                    cand.a[w] = cand.a[i];
                    vals.a[w] = vals.a[i];
                    w++;
                }
            cand.n = w;
            vals.n = w;
        }
        /* interchange (il.py:324-328) */
        const int64_t q = R[pivot].pos;
        if (q != j) {
            const int64_t other = row_at[j];
            row_at[j] = pivot;
            row_at[q] = other;
            R[pivot].pos = j;
            R[other].pos = q;
        }
        /* L column: scale, drop by current position (il.py:331-339) */
        ids.n = 0;
        for (int64_t i = 0; i < cand.n; i++) {
            if (!ipush(&ids, R[cand.a[i]].pos)) goto done;
            vals.a[i] = vals.a[i] / pval;
        }
        int64_t nl = cand.n;
        dual_drop(ids.a, vals.a, &nl, p, tau);
        R[pivot].lo = l_rows.n;
        R[pivot].len = (int32_t)nl;
        for (int64_t i = 0; i < nl; i++)
            if (!ipush(&l_rows, row_at[ids.a[i]]) || !dpush(&l_vals, vals.a[i])) goto done;
        l_ptr[j + 1] = l_rows.n;
        if (!ipush(&u_rows, j) || !dpush(&u_vals, pval)) goto done;
        u_ptr[j + 1] = u_rows.n;

        for (int64_t k = alo; k < ahi; k++) R[ridx[k]].rc--;
        for (int64_t t = 0; t < pattern.n; t++) {
            R[pattern.a[t]].x = 0.0;
            R[pattern.a[t]].mark = 0;
        }
    }

    /* assembly in final pivot coordinates (il.py:342-359) */
    F->m = m;
    F->n = n;
    F->nmod = nmod;
    F->perm = malloc((size_t)m * sizeof(int64_t));
    F->row_counts = malloc((size_t)m * sizeof(int64_t));
    F->u_ptr = u_ptr;
    u_ptr = NULL;
    F->u_idx = u_rows.a;
    F->u_val = u_vals.a;
    u_rows.a = NULL;
    u_vals.a = NULL;
    F->l1_ptr = calloc((size_t)(n + 1), sizeof(int64_t));
    F->l2_ptr = calloc((size_t)(n + 1), sizeof(int64_t));
    if (!F->perm || !F->row_counts || !F->l1_ptr || !F->l2_ptr) goto done;
    memcpy(F->perm, row_at, (size_t)m * sizeof(int64_t));
    for (int64_t i = 0; i < m; i++) F->row_counts[i] = R[i].rc;
    for (int64_t j = 0; j < n; j++) {
        int64_t c1 = 0, c2 = 0;
        for (int64_t e = l_ptr[j]; e < l_ptr[j + 1]; e++) {
            if (R[l_rows.a[e]].pos < n) c1++;
            else c2++;
        }
        F->l1_ptr[j + 1] = F->l1_ptr[j] + c1;
        F->l2_ptr[j + 1] = F->l2_ptr[j] + c2;
    }
    F->l1_idx = malloc((size_t)(F->l1_ptr[n] + 1) * sizeof(int64_t));
    F->l1_val = malloc((size_t)(F->l1_ptr[n] + 1) * sizeof(double));
    F->l2_idx = malloc((size_t)(F->l2_ptr[n] + 1) * sizeof(int64_t));
    F->l2_val = malloc((size_t)(F->l2_ptr[n] + 1) * sizeof(double));
    if (!F->l1_idx || !F->l1_val || !F->l2_idx || !F->l2_val) goto done;
    {
        int64_t tmp[2 * 4096];
        for (int64_t j = 0; j < n; j++) {
            const int64_t lo = l_ptr[j], len = l_ptr[j + 1] - lo;
            int64_t *buf = len <= 4096 ? tmp : malloc((size_t)(2 * len) * sizeof(int64_t));
            if (!buf) goto done;
            for (int64_t e = 0; e < len; e++) {
                buf[2 * e] = R[l_rows.a[lo + e]].pos;
                buf[2 * e + 1] = lo + e;
            }
            qsort(buf, (size_t)len, 2 * sizeof(int64_t), cmp_pair);
            int64_t d1 = F->l1_ptr[j], d2 = F->l2_ptr[j];
            for (int64_t e = 0; e < len; e++) {
                const int64_t pos = buf[2 * e];
                const double v = l_vals.a[buf[2 * e + 1]];
                if (pos < n) {
                    F->l1_idx[d1] = pos;
                    F->l1_val[d1++] = v;
                } else {
                    F->l2_idx[d2] = pos - n;
                    F->l2_val[d2++] = v;
                }
            }
            if (buf != tmp) free(buf);
        }
    }
    *out = F;
    F = NULL;
    rc = ORC_OK;
done:
    free(R);
    free(row_at);
    free(col_inf);
    free(l_ptr);
    free(u_ptr);
    free(l_rows.a); free(u_rows.a); free(pattern.a); free(post.a); free(st_node.a); free(st_cur.a);
    free(ids.a); free(cand.a); free(l_vals.a); free(u_vals.a); free(vals.a);
    orc_ilup_free(F);
    return rc;
}

/* sizes for the caller's buffers */
void orc_ilup_sizes(const orc_factors *F, int64_t *nnz_l1, int64_t *nnz_l2, int64_t *nnz_u, int64_t *nmod)
{
    *nnz_l1 = F->l1_ptr[F->n];
    *nnz_l2 = F->l2_ptr[F->n];
    *nnz_u = F->u_ptr[F->n];
    *nmod = F->nmod;
}

void orc_ilup_copy(const orc_factors *F, int64_t *perm, int64_t *row_counts, int64_t *l1_ptr, int64_t *l1_idx,
                   double *l1_val, int64_t *l2_ptr, int64_t *l2_idx, double *l2_val, int64_t *u_ptr,
                   int64_t *u_idx, double *u_val)
{
    const int64_t n = F->n, m = F->m;
    memcpy(perm, F->perm, (size_t)m * sizeof(int64_t));
    memcpy(row_counts, F->row_counts, (size_t)m * sizeof(int64_t));
    memcpy(l1_ptr, F->l1_ptr, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(l2_ptr, F->l2_ptr, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(u_ptr, F->u_ptr, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(l1_idx, F->l1_idx, (size_t)F->l1_ptr[n] * sizeof(int64_t));
    memcpy(l1_val, F->l1_val, (size_t)F->l1_ptr[n] * sizeof(double));
    memcpy(l2_idx, F->l2_idx, (size_t)F->l2_ptr[n] * sizeof(int64_t));
    memcpy(l2_val, F->l2_val, (size_t)F->l2_ptr[n] * sizeof(double));
    memcpy(u_idx, F->u_idx, (size_t)F->u_ptr[n] * sizeof(int64_t));
    memcpy(u_val, F->u_val, (size_t)F->u_ptr[n] * sizeof(double));
}
