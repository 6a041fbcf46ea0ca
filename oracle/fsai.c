/* fsai.c -- the paper's own preconditioner P = Z~ Z~^t (NEXT-1), plain C.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Written from PAPER.md only:
 *   - T = band(A, 1): the entries a_ij of A with |j - i| <= 1 in the unknown numbering
 *     (scheme step 1);
 *   - T = U^t U, U upper bidiagonal, diagonally dominant (Prop. 3.2);
 *   - Z = U^-1 column by column by backward substitution, Eq. 19:
 *       z_{k-i,k} = (-1)^i / u_kk * prod_{r=1..i} u_{k-r,k-r+1} / u_{k-r,k-r};
 *   - banded truncation z~_ij = 0 for j > i + q (scheme steps 4-5).
 * Stored as the unit-diagonal factor zhat = u_kk * z (so zhat_{k-i,k} = prod_{r=1..i} rho_{k-r},
 * rho_m = -u_{m,m+1} / u_mm) with pivots p_k = u_kk^2: P = Zhat diag(p)^-1 Zhat^t = Z~ Z~^t
 * (reading R25).  The Jacobi scale of the AINV object is 1 (z = zhat).
 */
#include <math.h>
#include <stdlib.h>

#include "oracle.h"
#include "oracle_internal.h"

int orc_fsai_build(const orc_problem* P, int32_t q, orc_ainv** out, int64_t* failed_col) {
    *out = NULL;
    if (failed_col) *failed_col = -1;
    if (q < 0) return ORC_ERR_ARG;
    const int64_t n = P->n;
    double* t = (double*)malloc(sizeof(double) * (n ? n : 1));     /* T's diagonal */
    double* o = (double*)calloc(n ? n : 1, sizeof(double));         /* T's superdiagonal t_{k,k+1} */
    double* u = (double*)malloc(sizeof(double) * (n ? n : 1));      /* u_kk */
    double* rho = (double*)calloc(n ? n : 1, sizeof(double));       /* -u_{k,k+1} / u_kk */
    for (int64_t k = 0; k < n; ++k) {
        t[k] = P->diag[k];
        for (int64_t e = P->rowptr[k]; e < P->rowptr[k + 1]; ++e)
            if (P->col[e] == k + 1) o[k] = P->val[e];
    }
    /* tridiagonal Cholesky: u_00 = sqrt(t_0); u_{k,k+1} = t_{k,k+1} / u_kk;
     * u_{k+1,k+1} = sqrt(t_{k+1} - u_{k,k+1}^2) */
    int rc = ORC_OK;
    for (int64_t k = 0; k < n && rc == ORC_OK; ++k) {
        double rad = t[k];
        if (k > 0) {
            const double v = o[k - 1] / u[k - 1];
            rad = t[k] - v * v;
        }
        if (!(rad > 0.0) || !isfinite(rad)) {
            rc = ORC_ERR_NOT_SPD;
            if (failed_col) *failed_col = k;
            break;
        }
        u[k] = sqrt(rad);
        if (k > 0) rho[k - 1] = -((o[k - 1] / u[k - 1]) / u[k - 1]);
    }
    if (rc != ORC_OK) { free(t); free(o); free(u); free(rho); return rc; }

    orc_ainv* R = (orc_ainv*)calloc(1, sizeof(orc_ainv));
    R->n = n;
    R->colptr = (int64_t*)calloc(n + 1, sizeof(int64_t));
    /* column k: zhat_{k-i,k} = zhat_{k-i+1,k} * rho_{k-i}, i = 1..q, until the chain breaks */
    int64_t cap = n * (int64_t)(q + 1) + 1, nnz = 0;
    R->row = (int64_t*)malloc(sizeof(int64_t) * cap);
    R->zhat = (double*)malloc(sizeof(double) * cap);
    double* col = (double*)malloc(sizeof(double) * (q + 1));
    for (int64_t k = 0; k < n; ++k) {
        int32_t m = 0;                       /* off-diagonal entries of column k */
        double prod = 1.0;
        for (int32_t i = 1; i <= q && k - i >= 0; ++i) {
            prod = prod * rho[k - i];
            if (prod == 0.0) break;
            col[m++] = prod;                 /* row k - i */
        }
        for (int32_t e = m - 1; e >= 0; --e) {   /* rows ascending: k-m .. k-1, then k */
            R->row[nnz] = k - (e + 1);
            R->zhat[nnz] = col[e];
            ++nnz;
        }
        R->row[nnz] = k;
        R->zhat[nnz] = 1.0;
        ++nnz;
        R->colptr[k + 1] = nnz;
    }
    free(col);
    R->nnz = nnz;
    R->p = (double*)malloc(sizeof(double) * (n ? n : 1));
    R->s = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (int64_t k = 0; k < n; ++k) {
        R->p[k] = u[k] * u[k];
        R->s[k] = 1.0;
    }
    R->z = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
    for (int64_t e = 0; e < nnz; ++e) R->z[e] = R->zhat[e];
    /* row-wise copy (columns ascending within a row) for s = Z t */
    R->rptr = (int64_t*)calloc(n + 1, sizeof(int64_t));
    R->rcol = (int64_t*)malloc(sizeof(int64_t) * (nnz ? nnz : 1));
    R->rval = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
    for (int64_t e = 0; e < nnz; ++e) R->rptr[R->row[e] + 1]++;
    for (int64_t r = 0; r < n; ++r) R->rptr[r + 1] += R->rptr[r];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t r = 0; r < n; ++r) fill[r] = R->rptr[r];
    for (int64_t j = 0; j < n; ++j)
        for (int64_t e = R->colptr[j]; e < R->colptr[j + 1]; ++e) {
            const int64_t r = R->row[e];
            R->rcol[fill[r]] = j;
            R->rval[fill[r]] = R->z[e];
            fill[r]++;
        }
    free(fill);
    free(t); free(o); free(u); free(rho);
    *out = R;
    return ORC_OK;
}
