/* assemble.c -- oracle: five-point operator A, anchor check, partition.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Built with -ffp-contract=off.
 *
 * PAPER.md:131-143 (Eq. 10): row (i,j) couples to its four neighbours; diagonal =
 * sum of the four couplings; "symmetric", "positive-definite"; natural ordering
 * "from west to east and from south to north".  We assemble the NEGATION of Eq. 10
 * as printed so that A is SPD (reading R1), treat land as "not an unknown"
 * with land faces kept on the diagonal (Dirichlet, reading R3) and wrap E-W
 * periodically (north star; reading R3).
 */
#include "oracle_internal.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

int orc_assemble(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                 const double* sigma, const uint8_t* mask, orc_problem** out) {
    *out = NULL;
    if (ni < 3 || nj < 3 || !cE || !cN || !mask) return ORC_ERR_ARG;
    int64_t ng = (int64_t)ni * nj;
    for (int64_t g = 0; g < ng; ++g) {
        if (!(cE[g] >= 0.0) || !isfinite(cE[g])) return ORC_ERR_ARG;
        if (!(cN[g] >= 0.0) || !isfinite(cN[g])) return ORC_ERR_ARG;
        if (sigma && (!(sigma[g] >= 0.0) || !isfinite(sigma[g]))) return ORC_ERR_ARG;
        if (mask[g] > 1) return ORC_ERR_ARG;
    }
    orc_problem* P = (orc_problem*)calloc(1, sizeof(orc_problem));
    P->ni = ni; P->nj = nj; P->periodic = periodic ? 1 : 0;
    P->cE = (double*)malloc(sizeof(double) * ng);
    P->cN = (double*)malloc(sizeof(double) * ng);
    P->mask = (uint8_t*)malloc(ng);
    memcpy(P->cE, cE, sizeof(double) * ng);
    memcpy(P->cN, cN, sizeof(double) * ng);
    memcpy(P->mask, mask, ng);
    P->unk_of = (int64_t*)malloc(sizeof(int64_t) * ng);
    int64_t n = 0;
    for (int64_t g = 0; g < ng; ++g) P->unk_of[g] = mask[g] ? n++ : -1;   /* natural order */
    P->n = n;
    P->grid_of = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    P->sigma = (double*)calloc(n ? n : 1, sizeof(double));
    for (int64_t g = 0; g < ng; ++g)
        if (mask[g]) {
            P->grid_of[P->unk_of[g]] = g;
            if (sigma) P->sigma[P->unk_of[g]] = sigma[g];
        }
    P->rowptr = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    P->col = (int64_t*)malloc(sizeof(int64_t) * 5 * (n ? n : 1));
    P->val = (double*)malloc(sizeof(double) * 5 * (n ? n : 1));
    P->diag = (double*)malloc(sizeof(double) * (n ? n : 1));
    int64_t nnz = 0;
    for (int64_t p = 0; p < n; ++p) {
        int64_t g = P->grid_of[p];
        int32_t i = (int32_t)(g % ni), j = (int32_t)(g / ni);
        struct face f[4];
        orc_faces(P, i, j, f);
        /* A_pp = ((c_E + c_W) + c_N) + c_S (+ sigma_p), absent faces contribute 0
         * (Eq. 10's diagonal). */
        double dE = f[FACE_E].present ? f[FACE_E].c : 0.0;
        double dW = f[FACE_W].present ? f[FACE_W].c : 0.0;
        double dN = f[FACE_N].present ? f[FACE_N].c : 0.0;
        double dS = f[FACE_S].present ? f[FACE_S].c : 0.0;
        double d = ((dE + dW) + dN) + dS;
        if (sigma) d = d + P->sigma[p];
        P->diag[p] = d;
        /* entries: diagonal + A_pq = -c for faces whose neighbour q is ocean and c > 0 */
        int64_t cols[5]; double vals[5]; int m = 0;
        cols[m] = p; vals[m] = d; ++m;
        for (int k = 0; k < 4; ++k) {
            if (!f[k].present || f[k].q < 0 || !(f[k].c > 0.0)) continue;
            cols[m] = f[k].q; vals[m] = -f[k].c; ++m;
        }
        /* sort columns ascending (insertion sort, m <= 5) */
        for (int a = 1; a < m; ++a)
            for (int b = a; b > 0 && cols[b - 1] > cols[b]; --b) {
                int64_t tc = cols[b]; cols[b] = cols[b - 1]; cols[b - 1] = tc;
                double tv = vals[b]; vals[b] = vals[b - 1]; vals[b - 1] = tv;
            }
        P->rowptr[p] = nnz;
        for (int a = 0; a < m; ++a) { P->col[nnz] = cols[a]; P->val[nnz] = vals[a]; ++nnz; }
    }
    P->rowptr[n] = nnz;
    P->nnz = nnz;
    *out = P;
    (void)cmp_i64;
    return ORC_OK;
}

/* Faces of grid cell (i,j):
 *   E: (i+1 mod ni, j), c = cE[j][i];      W: (i-1 mod ni, j), c = cE[j][i-1 mod ni];
 *   N: (i, j+1), c = cN[j][i] if j+1 < nj; S: (i, j-1), c = cN[j-1][i] if j >= 1.
 * Without periodicity the W face at i = 0 and the E face at i = ni-1 are absent.
 * q = unknown index of the neighbour, -1 if land. */
void orc_faces(const orc_problem* P, int32_t i, int32_t j, struct face f[4]) {
    int32_t ni = P->ni, nj = P->nj;
    for (int k = 0; k < 4; ++k) { f[k].present = 0; f[k].q = -1; f[k].c = 0.0; f[k].g = -1; }
    if (i + 1 < ni || P->periodic) {
        int32_t ie = (i + 1) % ni;
        f[FACE_E].present = 1; f[FACE_E].c = P->cE[(int64_t)j * ni + i];
        f[FACE_E].g = (int64_t)j * ni + ie;
    }
    if (i >= 1 || P->periodic) {
        int32_t iw = (i - 1 + ni) % ni;
        f[FACE_W].present = 1; f[FACE_W].c = P->cE[(int64_t)j * ni + iw];
        f[FACE_W].g = (int64_t)j * ni + iw;
    }
    if (j + 1 < nj) {
        f[FACE_N].present = 1; f[FACE_N].c = P->cN[(int64_t)j * ni + i];
        f[FACE_N].g = (int64_t)(j + 1) * ni + i;
    }
    if (j >= 1) {
        f[FACE_S].present = 1; f[FACE_S].c = P->cN[(int64_t)(j - 1) * ni + i];
        f[FACE_S].g = (int64_t)(j - 1) * ni + i;
    }
    for (int k = 0; k < 4; ++k)
        if (f[k].present) f[k].q = P->unk_of[f[k].g];
}

void orc_problem_free(orc_problem* P) {
    if (!P) return;
    free(P->cE); free(P->cN); free(P->mask); free(P->unk_of); free(P->grid_of);
    free(P->sigma); free(P->rowptr); free(P->col); free(P->val); free(P->diag);
    free(P);
}

int64_t orc_n(const orc_problem* P) { return P->n; }
int64_t orc_nnz(const orc_problem* P) { return P->nnz; }

void orc_csr(const orc_problem* P, int64_t* rowptr, int64_t* col, double* val) {
    memcpy(rowptr, P->rowptr, sizeof(int64_t) * (P->n + 1));
    memcpy(col, P->col, sizeof(int64_t) * P->nnz);
    memcpy(val, P->val, sizeof(double) * P->nnz);
}

void orc_grid_index(const orc_problem* P, int64_t* g) { memcpy(g, P->grid_of, sizeof(int64_t) * P->n); }
void orc_diag(const orc_problem* P, double* d) { memcpy(d, P->diag, sizeof(double) * P->n); }

/* y = A x: each row summed left to right in column order. */
void orc_apply(const orc_problem* P, const double* x, double* y) {
    for (int64_t p = 0; p < P->n; ++p) {
        double acc = 0.0;
        for (int64_t e = P->rowptr[p]; e < P->rowptr[p + 1]; ++e) acc = acc + P->val[e] * x[P->col[e]];
        y[p] = acc;
    }
}

/* Anchor check (reading R22): 4-connected components of
 * ocean points linked by faces with c > 0 (E-W wrap included).  A component is anchored
 * if it contains a point with a positive face to a LAND cell or sigma_p > 0; otherwise
 * A restricted to it has zero row sums and is singular. */
int64_t orc_anchor_check(const orc_problem* P) {
    int64_t n = P->n;
    int64_t* comp = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t p = 0; p < n; ++p) comp[p] = -1;
    int64_t bad = -1;
    for (int64_t root = 0; root < n && bad < 0; ++root) {
        if (comp[root] >= 0) continue;
        int anchored = 0;
        int64_t sp = 0;
        stack[sp++] = root; comp[root] = root;
        while (sp) {
            int64_t p = stack[--sp];
            int64_t g = P->grid_of[p];
            struct face f[4];
            orc_faces(P, (int32_t)(g % P->ni), (int32_t)(g / P->ni), f);
            if (P->sigma[p] > 0.0) anchored = 1;
            for (int k = 0; k < 4; ++k) {
                if (!f[k].present || !(f[k].c > 0.0)) continue;
                if (f[k].q < 0) { anchored = 1; continue; }
                if (comp[f[k].q] < 0) { comp[f[k].q] = root; stack[sp++] = f[k].q; }
            }
        }
        if (!anchored) bad = root;
    }
    free(comp); free(stack);
    return bad;
}

/* Row-block partition balanced by ocean count:
 *   cum[j] = ocean points in rows 0..j-1,  N = cum[nj];
 *   row_begin[p] = min{ j : cum[j] * parts >= p * N }  for p = 1..parts-1,
 *   then forced strictly increasing (every part owns >= 1 row) and row_begin[parts] = nj. */
void orc_partition(int32_t nj, int32_t ni, const uint8_t* mask, int32_t parts, int32_t* rb) {
    int64_t* cum = (int64_t*)malloc(sizeof(int64_t) * (nj + 1));
    cum[0] = 0;
    for (int32_t j = 0; j < nj; ++j) {
        int64_t c = 0;
        for (int32_t i = 0; i < ni; ++i) c += mask[(int64_t)j * ni + i] ? 1 : 0;
        cum[j + 1] = cum[j] + c;
    }
    int64_t N = cum[nj];
    rb[0] = 0;
    for (int32_t p = 1; p < parts; ++p) {
        int32_t j = 0;
        while (j < nj && cum[j] * parts < (int64_t)p * N) ++j;
        if (j <= rb[p - 1]) j = rb[p - 1] + 1;
        int32_t maxj = nj - (parts - p);          /* leave >= 1 row for each later part */
        if (j > maxj) j = maxj;
        rb[p] = j;
    }
    rb[parts] = nj;
    free(cum);
}
