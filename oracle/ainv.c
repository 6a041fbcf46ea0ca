/* ainv.c -- oracle: AINV(A, tau), the approximate inverse A^-1 ~ Z D^-1 Z^T.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Built with -ffp-contract=off.
 *
 * The paper's "P_B1": "obtained by means of the A-orthogonalization
 * method ... posing a (fixed) drop tolerance and by ignoring the elements below the
 * fixed tolerance"; AINV itself is cited at PAPER.md:26 and PAPER.md:224.  The
 * orthogonalisation, drop rule and pivot are the readings R11-R13 of DESIGN.md
 * (SURVEY §8(c.2)), followed here step by step:
 *
 *   1. s_p = 1/sqrt(A_pp);  a^_pq = A_pq * fl(s_p * s_q)     (Jacobi pre-scaling)
 *   2. for j = 0..n-1:  z = e_j;  for candidates i < j in increasing order:
 *        pi = sum_k a^_ik z_k  (row i of A^, ascending k);  skip if pi == 0;
 *        c = pi / p_i;  z_k <- z_k - c * zhat_i[k] for the entries of zhat_i (ascending k);
 *        drop every touched k != j with |z_k| < tau.
 *      p_j = sum_k a^_jk z_k;  NOT_SPD(j) if p_j <= 1e-12 or not finite;  zhat_j = z.
 *   3. Z = S Zhat, z_kj = fl(s_k * zhat_kj);  A^-1 ~ Z Dhat^-1 Z^T.
 *
 * Two formulations are provided and cross-checked by the tests: the
 * sparse left-looking one (candidates from a heap) and a dense right-looking O(n^3)
 * loop "for i, for j > i".  They perform the same operations on every column in the
 * same order, so they must agree bitwise.
 */
#include "oracle_internal.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PIVOT_MIN 1e-12

/* A local symmetric matrix (a principal submatrix of A^) in CSR, columns ascending. */
typedef struct {
    int64_t n;
    const int64_t* rowptr;
    const int64_t* col;
    const double* a;
} lcsr;

/* growable column store for Zhat (CSC) */
typedef struct {
    int64_t n, nnz, cap;
    int64_t *colptr, *row;
    double* val;
} cstore;

static void cs_init(cstore* c, int64_t n) {
    c->n = n; c->nnz = 0; c->cap = 4 * (n ? n : 1);
    c->colptr = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    c->row = (int64_t*)malloc(sizeof(int64_t) * c->cap);
    c->val = (double*)malloc(sizeof(double) * c->cap);
    c->colptr[0] = 0;
}
static void cs_push(cstore* c, int64_t r, double v) {
    if (c->nnz == c->cap) {
        c->cap *= 2;
        c->row = (int64_t*)realloc(c->row, sizeof(int64_t) * c->cap);
        c->val = (double*)realloc(c->val, sizeof(double) * c->cap);
    }
    c->row[c->nnz] = r; c->val[c->nnz] = v; c->nnz++;
}
static void cs_free(cstore* c) { free(c->colptr); free(c->row); free(c->val); }

/* binary min-heap of candidate indices */
typedef struct { int64_t* h; int64_t n, cap; } heap;
static void hp_push(heap* H, int64_t v) {
    if (H->n == H->cap) { H->cap = H->cap ? 2 * H->cap : 64; H->h = (int64_t*)realloc(H->h, sizeof(int64_t) * H->cap); }
    int64_t k = H->n++;
    H->h[k] = v;
    while (k > 0) {
        int64_t par = (k - 1) / 2;
        if (H->h[par] <= H->h[k]) break;
        int64_t t = H->h[par]; H->h[par] = H->h[k]; H->h[k] = t; k = par;
    }
}
static int64_t hp_pop(heap* H) {
    int64_t top = H->h[0];
    H->h[0] = H->h[--H->n];
    int64_t k = 0;
    for (;;) {
        int64_t l = 2 * k + 1, r = l + 1, m = k;
        if (l < H->n && H->h[l] < H->h[m]) m = l;
        if (r < H->n && H->h[r] < H->h[m]) m = r;
        if (m == k) break;
        int64_t t = H->h[m]; H->h[m] = H->h[k]; H->h[k] = t; k = m;
    }
    return top;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Sparse left-looking AINV on a local matrix.  Output: CSC Zhat (rows ascending), pivots.
 * Returns -1 on success or the failing column. */
/* P_B2 count rule ("predetermined the number of non-zeros elements on each its
 * row"; reading R26): after each update (and the tau drop), keep the
 * diagonal and the fill-1 largest-magnitude off-diagonal entries of the column, ties to the
 * smaller row index; fill = 0 means no limit (P_B1). */
static const double* g_keep_w;
static int cmp_keep(const void* x, const void* y) {
    const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    const double fa = fabs(g_keep_w[a]), fb = fabs(g_keep_w[b]);
    if (fa > fb) return -1;
    if (fa < fb) return 1;
    return a < b ? -1 : (a > b);
}
/* cand[0..cnt) = present off-diagonal rows; returns how many to drop (they end the sorted list) */
static int64_t keep_largest(int64_t* cand, int64_t cnt, const double* w, int32_t fill) {
    if (fill <= 0 || cnt <= (int64_t)fill - 1) return 0;
    g_keep_w = w;
    qsort(cand, (size_t)cnt, sizeof(int64_t), cmp_keep);
    return cnt - ((int64_t)fill - 1);
}

static int64_t ainv_sparse(const lcsr* A, double tau, int32_t fill, cstore* Z, double* p) {
    int64_t n = A->n;
    double* w = (double*)calloc(n ? n : 1, sizeof(double));
    char* inz = (char*)calloc(n ? n : 1, 1);
    int64_t* inlist = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));   /* stamp: in zlist for column j */
    int64_t* pushed = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));   /* stamp: pushed for column j */
    for (int64_t k = 0; k < n; ++k) { inlist[k] = -1; pushed[k] = -1; }
    int64_t zcap = 64, nz;
    int64_t* zlist = (int64_t*)malloc(sizeof(int64_t) * zcap);
    int64_t tcap = 64, nt;
    int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * tcap);
    heap H = {0, 0, 0};
    int64_t fail = -1;
    cs_init(Z, n);
    for (int64_t j = 0; j < n && fail < 0; ++j) {
        nz = 0;
        zlist[nz++] = j; inlist[j] = j; inz[j] = 1; w[j] = 1.0;
        H.n = 0;
        for (int64_t e = A->rowptr[j]; e < A->rowptr[j + 1]; ++e) {
            int64_t i = A->col[e];
            if (i < j && pushed[i] != j) { pushed[i] = j; hp_push(&H, i); }
        }
        while (H.n) {
            int64_t i = hp_pop(&H);
            double pi = 0.0;
            for (int64_t e = A->rowptr[i]; e < A->rowptr[i + 1]; ++e) {
                int64_t k = A->col[e];
                if (inz[k]) pi = pi + A->a[e] * w[k];
            }
            if (pi == 0.0) continue;                       /* no explicit zeros */
            double c = pi / p[i];
            nt = 0;
            for (int64_t e = Z->colptr[i]; e < Z->colptr[i + 1]; ++e) {
                int64_t k = Z->row[e];
                double v = Z->val[e];
                if (!inz[k]) {
                    inz[k] = 1; w[k] = 0.0;
                    if (inlist[k] != j) {
                        inlist[k] = j;
                        if (nz == zcap) { zcap *= 2; zlist = (int64_t*)realloc(zlist, sizeof(int64_t) * zcap); }
                        zlist[nz++] = k;
                    }
                    for (int64_t e2 = A->rowptr[k]; e2 < A->rowptr[k + 1]; ++e2) {
                        int64_t i2 = A->col[e2];
                        if (i2 > i && i2 < j && pushed[i2] != j) { pushed[i2] = j; hp_push(&H, i2); }
                    }
                }
                w[k] = w[k] - c * v;
                if (nt == tcap) { tcap *= 2; touched = (int64_t*)realloc(touched, sizeof(int64_t) * tcap); }
                touched[nt++] = k;
            }
            for (int64_t t = 0; t < nt; ++t) {
                int64_t k = touched[t];
                if (k != j && fabs(w[k]) < tau) { inz[k] = 0; w[k] = 0.0; }
            }
            if (fill > 0) {
                int64_t cnt = 0;
                if (nz > tcap) { tcap = nz; touched = (int64_t*)realloc(touched, sizeof(int64_t) * tcap); }
                for (int64_t t = 0; t < nz; ++t)
                    if (zlist[t] != j && inz[zlist[t]]) touched[cnt++] = zlist[t];
                const int64_t ndrop = keep_largest(touched, cnt, w, fill);
                for (int64_t t = cnt - ndrop; t < cnt; ++t) { inz[touched[t]] = 0; w[touched[t]] = 0.0; }
            }
        }
        double pj = 0.0;
        for (int64_t e = A->rowptr[j]; e < A->rowptr[j + 1]; ++e) {
            int64_t k = A->col[e];
            if (inz[k]) pj = pj + A->a[e] * w[k];
        }
        if (!(pj > PIVOT_MIN) || !isfinite(pj)) { fail = j; }
        p[j] = pj;
        qsort(zlist, nz, sizeof(int64_t), cmp_i64);
        for (int64_t t = 0; t < nz; ++t) {
            int64_t k = zlist[t];
            if (inz[k]) cs_push(Z, k, w[k]);
            inz[k] = 0; w[k] = 0.0;
        }
        Z->colptr[j + 1] = Z->nnz;
    }
    free(w); free(inz); free(inlist); free(pushed); free(zlist); free(touched); free(H.h);
    return fail;
}

/* The dense formulation's own P_B2 selection (independent of keep_largest's sort, so the two
 * formulations cross-check the rule, not just the update sequence): fill-1 rounds, each picking
 * the present off-diagonal entry of largest |z| by an ascending scan with a strict '>' (ties go
 * to the smaller row index, R26); every present off-diagonal entry not picked is dropped. */
static void dense_keep(char* pres, double* z, int64_t j, int64_t n, int32_t fill, int64_t* mark) {
    int64_t cnt = 0;
    for (int64_t k = 0; k < n; ++k) {
        mark[k] = 0;
        if (k != j && pres[k]) ++cnt;
    }
    if (cnt <= (int64_t)fill - 1) return;
    for (int32_t r = 0; r < fill - 1; ++r) {
        int64_t best = -1;
        for (int64_t k = 0; k < n; ++k)
            if (k != j && pres[k] && !mark[k] && (best < 0 || fabs(z[k]) > fabs(z[best]))) best = k;
        mark[best] = 1;
    }
    for (int64_t k = 0; k < n; ++k)
        if (k != j && pres[k] && !mark[k]) { pres[k] = 0; z[k] = 0.0; }
}

/* Dense right-looking AINV (cross-check; n small): for i = 0..n-1: p_i = a^_i^T z_i;
 * for j > i: pi = a^_i^T z_j; skip if 0; z_j -= (pi/p_i) z_i; drop touched entries. */
static int64_t ainv_dense(const lcsr* A, double tau, int32_t fill, cstore* Z, double* p) {
    int64_t n = A->n;
    double* Zc = (double*)calloc((size_t)n * n, sizeof(double));     /* column-major */
    char* pres = (char*)calloc((size_t)n * n, 1);
    int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t fail = -1;
    for (int64_t j = 0; j < n; ++j) { Zc[j * n + j] = 1.0; pres[j * n + j] = 1; }
    for (int64_t i = 0; i < n && fail < 0; ++i) {
        const double* zi = Zc + i * n;
        const char* pi_ = pres + i * n;
        double piv = 0.0;
        for (int64_t e = A->rowptr[i]; e < A->rowptr[i + 1]; ++e) {
            int64_t k = A->col[e];
            if (pi_[k]) piv = piv + A->a[e] * zi[k];
        }
        if (!(piv > PIVOT_MIN) || !isfinite(piv)) { fail = i; p[i] = piv; break; }
        p[i] = piv;
        for (int64_t j = i + 1; j < n; ++j) {
            double* zj = Zc + j * n;
            char* pj_ = pres + j * n;
            double pi = 0.0;
            for (int64_t e = A->rowptr[i]; e < A->rowptr[i + 1]; ++e) {
                int64_t k = A->col[e];
                if (pj_[k]) pi = pi + A->a[e] * zj[k];
            }
            if (pi == 0.0) continue;
            double c = pi / piv;
            int64_t nt = 0;
            for (int64_t k = 0; k <= i; ++k) {
                if (!pi_[k]) continue;
                if (!pj_[k]) { pj_[k] = 1; zj[k] = 0.0; }
                zj[k] = zj[k] - c * zi[k];
                touched[nt++] = k;
            }
            for (int64_t t = 0; t < nt; ++t) {
                int64_t k = touched[t];
                if (k != j && fabs(zj[k]) < tau) { pj_[k] = 0; zj[k] = 0.0; }
            }
            if (fill > 0) dense_keep(pj_, zj, j, n, fill, touched);
        }
    }
    cs_init(Z, n);
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t k = 0; k <= j; ++k)
            if (pres[j * n + k]) cs_push(Z, k, Zc[j * n + k]);
        Z->colptr[j + 1] = Z->nnz;
    }
    free(Zc); free(pres); free(touched);
    return fail;
}

int orc_ainv_build(const orc_problem* P, double tau, int32_t method, int32_t parts, int32_t halo,
             orc_ainv** out, int64_t* failed_col) {
    return orc_ainv_build_fill(P, tau, 0, method, parts, halo, out, failed_col);
}

int orc_ainv_build_fill(const orc_problem* P, double tau, int32_t keep, int32_t method, int32_t parts, int32_t halo,
             orc_ainv** out, int64_t* failed_col) {
    *out = NULL;
    if (failed_col) *failed_col = -1;
    if (!(tau >= 0.0) || parts < 1 || halo < 0 || parts > P->nj || keep < 0) return ORC_ERR_ARG;
    int64_t n = P->n;
    if (method == 1 && n > 4000) return ORC_ERR_ARG;
    for (int64_t q = 0; q < n; ++q)
        if (!(P->diag[q] > 0.0)) { if (failed_col) *failed_col = q; return ORC_ERR_NOT_SPD; }
    /* step 1: Jacobi pre-scaling, s_p = 1/sqrt(A_pp) (IEEE sqrt, then divide) */
    double* s = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (int64_t q = 0; q < n; ++q) s[q] = 1.0 / sqrt(P->diag[q]);
    double* ah = (double*)malloc(sizeof(double) * (P->nnz ? P->nnz : 1));
    for (int64_t q = 0; q < n; ++q)
        for (int64_t e = P->rowptr[q]; e < P->rowptr[q + 1]; ++e)
            ah[e] = P->val[e] * (s[q] * s[P->col[e]]);

    orc_ainv* R = (orc_ainv*)calloc(1, sizeof(orc_ainv));
    R->n = n; R->s = s;
    R->p = (double*)malloc(sizeof(double) * (n ? n : 1));
    cstore G; cs_init(&G, n);
    int rc = ORC_OK;

    int32_t* rb = (int32_t*)malloc(sizeof(int32_t) * (parts + 1));
    if (parts == 1) { rb[0] = 0; rb[1] = P->nj; }
    else orc_partition(P->nj, P->ni, P->mask, parts, rb);

    for (int32_t part = 0; part < parts && rc == ORC_OK; ++part) {
        /* index set: unknowns in grid rows [max(0, rb-halo), re) (halo = 0 when parts == 1) */
        int32_t jb = rb[part], je = rb[part + 1];
        int32_t jl = parts == 1 ? 0 : (jb - halo < 0 ? 0 : jb - halo);
        int64_t lo = -1, hi = -1, own = -1;        /* unknown range [lo, hi), owned from own */
        for (int64_t q = 0; q < n; ++q) {
            int32_t jq = (int32_t)(P->grid_of[q] / P->ni);
            if (jq >= jl && lo < 0) lo = q;
            if (jq >= jb && own < 0) own = q;
            if (jq >= je && hi < 0) hi = q;
        }
        if (lo < 0) lo = n;
        if (own < 0) own = n;
        if (hi < 0) hi = n;
        int64_t m = hi - lo;
        /* principal submatrix of A^ over [lo, hi) (natural order is monotone in rows) */
        int64_t* lrp = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
        int64_t* lc = (int64_t*)malloc(sizeof(int64_t) * (5 * m + 1));
        double* la = (double*)malloc(sizeof(double) * (5 * m + 1));
        int64_t nn = 0;
        for (int64_t q = lo; q < hi; ++q) {
            lrp[q - lo] = nn;
            for (int64_t e = P->rowptr[q]; e < P->rowptr[q + 1]; ++e) {
                int64_t c = P->col[e];
                if (c >= lo && c < hi) { lc[nn] = c - lo; la[nn] = ah[e]; ++nn; }
            }
        }
        lrp[m] = nn;
        lcsr L = {m, lrp, lc, la};
        cstore Zl;
        double* pl = (double*)malloc(sizeof(double) * (m ? m : 1));
        int64_t f = method == 1 ? ainv_dense(&L, tau, keep, &Zl, pl) : ainv_sparse(&L, tau, keep, &Zl, pl);
        if (f >= 0) {
            rc = ORC_ERR_NOT_SPD;
            if (failed_col) *failed_col = f + lo;
        } else {
            /* keep the owned columns [own, hi) */
            for (int64_t q = own; q < hi; ++q) {
                int64_t jl_ = q - lo;
                for (int64_t e = Zl.colptr[jl_]; e < Zl.colptr[jl_ + 1]; ++e) cs_push(&G, Zl.row[e] + lo, Zl.val[e]);
                G.colptr[q + 1] = G.nnz;
                R->p[q] = pl[jl_];
            }
        }
        cs_free(&Zl); free(pl); free(lrp); free(lc); free(la);
    }
    free(rb); free(ah);
    if (rc != ORC_OK) { cs_free(&G); free(R->p); free(R->s); free(R); return rc; }

    R->nnz = G.nnz; R->colptr = G.colptr; R->row = G.row; R->zhat = G.val;
    /* step 3: z_kj = fl(s_k * zhat_kj) */
    R->z = (double*)malloc(sizeof(double) * (R->nnz ? R->nnz : 1));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t e = R->colptr[j]; e < R->colptr[j + 1]; ++e) R->z[e] = s[R->row[e]] * R->zhat[e];
    /* row-wise copy of Z for s = Z t (columns ascending within a row) */
    R->rptr = (int64_t*)calloc(n + 1, sizeof(int64_t));
    R->rcol = (int64_t*)malloc(sizeof(int64_t) * (R->nnz ? R->nnz : 1));
    R->rval = (double*)malloc(sizeof(double) * (R->nnz ? R->nnz : 1));
    for (int64_t e = 0; e < R->nnz; ++e) R->rptr[R->row[e] + 1]++;
    for (int64_t q = 0; q < n; ++q) R->rptr[q + 1] += R->rptr[q];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t q = 0; q < n; ++q) fill[q] = R->rptr[q];
    for (int64_t j = 0; j < n; ++j)                      /* columns visited ascending -> rows sorted */
        for (int64_t e = R->colptr[j]; e < R->colptr[j + 1]; ++e) {
            int64_t r = R->row[e];
            R->rcol[fill[r]] = j; R->rval[fill[r]] = R->z[e]; fill[r]++;
        }
    free(fill);
    *out = R;
    return ORC_OK;
}

void orc_ainv_free(orc_ainv* R) {
    if (!R) return;
    free(R->colptr); free(R->row); free(R->zhat); free(R->z); free(R->p); free(R->s);
    free(R->rptr); free(R->rcol); free(R->rval); free(R);
}

int64_t orc_ainv_nnz(const orc_ainv* R) { return R->nnz; }

void orc_ainv_export(const orc_ainv* R, int64_t* colptr, int64_t* row, double* zhat, double* z,
                     double* pivots, double* scale) {
    if (colptr) memcpy(colptr, R->colptr, sizeof(int64_t) * (R->n + 1));
    if (row) memcpy(row, R->row, sizeof(int64_t) * R->nnz);
    if (zhat) memcpy(zhat, R->zhat, sizeof(double) * R->nnz);
    if (z) memcpy(z, R->z, sizeof(double) * R->nnz);
    if (pivots) memcpy(pivots, R->p, sizeof(double) * R->n);
    if (scale) memcpy(scale, R->s, sizeof(double) * R->n);
}

/* s = Z Dhat^-1 Z^T r (plain order): t_j = (sum_k z_kj r_k) / p_j ; s_i = sum_j z_ij t_j.
 * The two sparse products of Alg. 1 line 7 and of PAPER.md:399-402. */
void orc_ainv_apply(const orc_ainv* R, const double* r, double* s) {
    int64_t n = R->n;
    double* t = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (int64_t j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int64_t e = R->colptr[j]; e < R->colptr[j + 1]; ++e) acc = acc + R->z[e] * r[R->row[e]];
        t[j] = acc / R->p[j];
    }
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t e = R->rptr[i]; e < R->rptr[i + 1]; ++e) acc = acc + R->rval[e] * t[R->rcol[e]];
        s[i] = acc;
    }
    free(t);
}
