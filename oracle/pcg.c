/* pcg.c -- oracle: preconditioned conjugate gradient, Alg. 1 of the paper.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Built with -ffp-contract=off.
 *
 * Alg. 1 "FSAI-PCG solver", with the line-8 typo fixed
 * (d_{k+1} = s_{k+1} + beta_k d_k, reading R6), the loop bound "k <= n"
 * read as k < maxit (reading R7) and the stopping test on the recurrence residual
 * ||r_k||/||b|| <= tol (reading R8):
 *
 *   x = x0;  r = b - A x;  s = P r;  d = s;  rho = (s, r);  nb = ||b||
 *   if nb == 0: return x = 0, k = 0
 *   h_0 = ||r||/nb;  k = 0
 *   while h_k > tol and k < maxit:
 *       q = A d;  gamma = (d, q);  BREAKDOWN unless gamma > 0 and finite
 *       alpha = rho/gamma;  x += alpha d;  r -= alpha q                    (lines 6-7)
 *       s = P r;  rho' = (s, r);  beta = rho'/rho;  d = s + beta d;  rho = rho'   (7-8)
 *       k += 1;  h_k = ||r||/nb
 *   report x, k, h_0..h_k, converged = (h_k <= tol), true ||b - A x||/||b||.
 *
 * Two arithmetic orders:
 *   PLAIN      -- every dot product and every sparse row summed sequentially, left to
 *                 right in natural order, separate multiply and add.
 *   CANONICAL  -- the GPU path's documented order, re-implemented here
 *                 from that document: fma updates, the fixed W,E,S,N stencil order,
 *                 fma row sums, and the block-tree dot products over the pitched grid.
 */
#include "oracle_internal.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * CANONICAL reduction order.  One rank owns grid rows [jb, je) (nloc
 * rows); each row is cut into nbx = ceil(pitch/B) segments of B columns.  The partial of
 * (local row jl, segment bx) is the block sum of the B values fl(a_e * b_e) of its columns
 * i = bx*B + t (0 at land and for i >= ni), stored at index m = jl*nbx + bx.  tree32 is the
 * warp shuffle-down tree (offsets 16, 8, 4, 2, 1; lane 0 result); a block sum is tree32 of
 * the per-warp tree32 results (zero-padded to 32).  Final: thread t of a B-thread block sums
 * partials t, t+B, t+2B, ... left to right from 0.0, then the block sum of those B values.
 * Several ranks: tree32 of the rank sums in rank order.
 * ------------------------------------------------------------------------------------ */
static double tree32(double u[32]) {
    for (int off = 16; off >= 1; off >>= 1)
        for (int l = 0; l + off < 32; ++l) u[l] = u[l] + u[l + off];
    return u[0];
}

static double block_sum(const double* v, int B) {
    double w[32] = {0};
    for (int k = 0; k < B / 32; ++k) {
        double u[32];
        memcpy(u, v + 32 * k, sizeof u);
        w[k] = tree32(u);
    }
    return tree32(w);
}

typedef struct {
    const orc_problem* P;
    int32_t pitch, B, parts;
    int32_t* rb;        /* parts+1 row bounds */
    double* vals;       /* scratch B */
    double* partial;    /* scratch, max blocks */
} canon;

static double canon_dot(canon* C, const double* a, const double* b) {
    const orc_problem* P = C->P;
    double ranks[32] = {0};
    for (int r = 0; r < C->parts; ++r) {
        int64_t jb = C->rb[r], je = C->rb[r + 1], nloc = je - jb;
        int64_t nbx = (C->pitch + C->B - 1) / C->B;
        int64_t G = nbx * nloc;
        for (int64_t blk = 0; blk < G; ++blk) {
            int64_t bx = blk % nbx, jl = blk / nbx;
            for (int t = 0; t < C->B; ++t) {
                int64_t i = bx * C->B + t;
                double v = 0.0;
                if (i < P->ni) {
                    int64_t u = P->unk_of[(jb + jl) * P->ni + i];
                    if (u >= 0) v = a[u] * b[u];
                }
                C->vals[t] = v;
            }
            C->partial[blk] = block_sum(C->vals, C->B);
        }
        for (int t = 0; t < C->B; ++t) {
            double acc = 0.0;
            for (int64_t m = t; m < G; m += C->B) acc = acc + C->partial[m];
            C->vals[t] = acc;
        }
        ranks[r] = block_sum(C->vals, C->B);
    }
    if (C->parts == 1) return ranks[0];
    return tree32(ranks);
}

/* canonical stencil y = A x: acc = A_pp x_p, then
 * acc = fma(-c, x_nb, acc) for the W, E, S, N faces in that order. */
static void canon_apply(const orc_problem* P, const double* x, double* y) {
    for (int64_t p = 0; p < P->n; ++p) {
        int64_t g = P->grid_of[p];
        struct face f[4];
        orc_faces(P, (int32_t)(g % P->ni), (int32_t)(g / P->ni), f);
        double acc = P->diag[p] * x[p];
        for (int k = 0; k < 4; ++k)           /* FACE_W, FACE_E, FACE_S, FACE_N */
            if (f[k].present && f[k].q >= 0) acc = fma(-f[k].c, x[f[k].q], acc);
        y[p] = acc;
    }
}

/* canonical AINV apply: t_j = (fma-sum over column j of Z, rows
 * ascending) / p_j ;  s_i = fma-sum over row i of Z, columns ascending. */
static void canon_ainv_apply(const orc_ainv* R, const double* r, double* s, double* t) {
    for (int64_t j = 0; j < R->n; ++j) {
        double acc = 0.0;
        for (int64_t e = R->colptr[j]; e < R->colptr[j + 1]; ++e) acc = fma(R->z[e], r[R->row[e]], acc);
        t[j] = acc / R->p[j];
    }
    for (int64_t i = 0; i < R->n; ++i) {
        double acc = 0.0;
        for (int64_t e = R->rptr[i]; e < R->rptr[i + 1]; ++e) acc = fma(R->rval[e], t[R->rcol[e]], acc);
        s[i] = acc;
    }
}

void orc_apply_canonical(const orc_problem* P, const double* x, double* y) { canon_apply(P, x, y); }

void orc_ainv_apply_canonical(const orc_ainv* R, const double* r, double* s) {
    double* t = (double*)malloc(sizeof(double) * (R->n ? R->n : 1));
    canon_ainv_apply(R, r, s, t);
    free(t);
}

double orc_dot_canonical(const orc_problem* P, const orc_pcg_opts* o, const double* a, const double* b) {
    canon C = {0};
    C.P = P; C.pitch = o->pitch; C.B = o->block; C.parts = o->parts;
    C.rb = (int32_t*)malloc(sizeof(int32_t) * (o->parts + 1));
    if (o->parts == 1) { C.rb[0] = 0; C.rb[1] = P->nj; }
    else orc_partition(P->nj, P->ni, P->mask, o->parts, C.rb);
    C.vals = (double*)malloc(sizeof(double) * o->block);
    C.partial = (double*)malloc(sizeof(double) * (((int64_t)P->nj + 1) * (o->pitch / o->block + 2)));
    double r = canon_dot(&C, a, b);
    free(C.rb); free(C.vals); free(C.partial);
    return r;
}

static double plain_dot(int64_t n, const double* a, const double* b) {
    double acc = 0.0;
    for (int64_t k = 0; k < n; ++k) acc = acc + a[k] * b[k];
    return acc;
}

/* CHUNKED dot: chunk partials (4096 consecutive unknowns, left to right), then the partials
 * left to right; independent of the thread count */
#define ORC_CHUNK 4096
static double chunked_dot(int64_t n, const double* a, const double* b, double* part) {
    const int64_t nc = (n + ORC_CHUNK - 1) / ORC_CHUNK;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t k1 = (c + 1) * ORC_CHUNK < n ? (c + 1) * ORC_CHUNK : n;
        double acc = 0.0;
        for (int64_t k = c * ORC_CHUNK; k < k1; ++k) acc = acc + a[k] * b[k];
        part[c] = acc;
    }
    double acc = 0.0;
    for (int64_t c = 0; c < nc; ++c) acc = acc + part[c];
    return acc;
}

/* the PLAIN row operations on all cores (each row's arithmetic unchanged) */
static void par_apply(const orc_problem* P, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P->n; ++p) {
        double acc = 0.0;
        for (int64_t e = P->rowptr[p]; e < P->rowptr[p + 1]; ++e) acc = acc + P->val[e] * x[P->col[e]];
        y[p] = acc;
    }
}
static void par_ainv_apply(const orc_ainv* R, const double* r, double* s, double* t) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < R->n; ++j) {
        double acc = 0.0;
        for (int64_t e = R->colptr[j]; e < R->colptr[j + 1]; ++e) acc = acc + R->z[e] * r[R->row[e]];
        t[j] = acc / R->p[j];
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < R->n; ++i) {
        double acc = 0.0;
        for (int64_t e = R->rptr[i]; e < R->rptr[i + 1]; ++e) acc = acc + R->rval[e] * t[R->rcol[e]];
        s[i] = acc;
    }
}

int orc_pcg(const orc_problem* P, const orc_ainv* R, const orc_pcg_opts* o, const double* b,
            const double* x0, double tol, int32_t maxit, double* x, double* hist, orc_pcg_report* rep) {
    memset(rep, 0, sizeof *rep);
    rep->failed_index = -1;
    int64_t n = P->n;
    if (!(tol >= 0.0) || maxit < 0) return rep->status = ORC_ERR_ARG;
    if (o->precond == ORC_PRECOND_AINV && !R) return rep->status = ORC_ERR_ARG;
    int canonical = o->mode == ORC_MODE_CANONICAL;
    const int chunked = o->mode == ORC_MODE_CHUNKED;
    double* cpart = chunked ? (double*)malloc(sizeof(double) * ((n + ORC_CHUNK - 1) / ORC_CHUNK + 1)) : NULL;
    canon C = {0};
    if (canonical) {
        if (o->pitch < P->ni || o->block < 32 || o->block > 1024 || (o->block & (o->block - 1)) ||
            o->parts < 1 || o->parts > 32 || o->parts > P->nj)
            return rep->status = ORC_ERR_ARG;
        C.P = P; C.pitch = o->pitch; C.B = o->block; C.parts = o->parts;
        C.rb = (int32_t*)malloc(sizeof(int32_t) * (o->parts + 1));
        if (o->parts == 1) { C.rb[0] = 0; C.rb[1] = P->nj; }
        else orc_partition(P->nj, P->ni, P->mask, o->parts, C.rb);
        C.vals = (double*)malloc(sizeof(double) * o->block);
        int64_t maxrows = 0;
        for (int r = 0; r < o->parts; ++r) if (C.rb[r + 1] - C.rb[r] > maxrows) maxrows = C.rb[r + 1] - C.rb[r];
        C.partial = (double*)malloc(sizeof(double) * ((maxrows + 1) * (o->pitch / o->block + 2)));
    }
#define DOT(a, b) (canonical ? canon_dot(&C, (a), (b)) : chunked ? chunked_dot(n, (a), (b), cpart) : plain_dot(n, (a), (b)))
#define APPLY_A(in, out) (canonical ? canon_apply(P, (in), (out)) : chunked ? par_apply(P, (in), (out)) : orc_apply(P, (in), (out)))
    size_t sz = sizeof(double) * (n ? n : 1);
    double *r = malloc(sz), *s = malloc(sz), *d = malloc(sz), *q = malloc(sz), *t = malloc(sz);

    /* preconditioner apply s = P r */
#define PRECOND(rin, sout)                                                        \
    do {                                                                          \
        if (o->precond == ORC_PRECOND_AINV) {                                     \
            if (canonical) canon_ainv_apply(R, (rin), (sout), t);                 \
            else if (chunked) par_ainv_apply(R, (rin), (sout), t);                \
            else orc_ainv_apply(R, (rin), (sout));                                \
        } else if (o->precond == ORC_PRECOND_JACOBI) {                            \
            for (int64_t k_ = 0; k_ < n; ++k_) (sout)[k_] = (rin)[k_] / P->diag[k_]; \
        } else {                                                                  \
            memcpy((sout), (rin), sz);                                            \
        }                                                                         \
    } while (0)

    /* lines 1-4 */
    for (int64_t k = 0; k < n; ++k) x[k] = x0 ? x0[k] : 0.0;
    double nb = sqrt(DOT(b, b));
    if (nb == 0.0) {
        for (int64_t k = 0; k < n; ++k) x[k] = 0.0;
        hist[0] = 0.0;
        rep->iterations = 0; rep->converged = 1;
        rep->status = ORC_OK;
        goto done;
    }
    APPLY_A(x, q);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - q[k];
    PRECOND(r, s);
    memcpy(d, s, sz);
    double rho = DOT(s, r);
    double h = sqrt(DOT(r, r)) / nb;
    hist[0] = h;
    int32_t it = 0;
    rep->status = ORC_OK;
    /* line 5 */
    while (h > tol && it < maxit) {
        /* line 6 */
        APPLY_A(d, q);
        double gamma = DOT(d, q);
        if (!(gamma > 0.0) || !isfinite(gamma)) { rep->status = ORC_ERR_BREAKDOWN; break; }
        double alpha = rho / gamma;
        if (canonical) {
            for (int64_t k = 0; k < n; ++k) x[k] = fma(alpha, d[k], x[k]);
            for (int64_t k = 0; k < n; ++k) r[k] = fma(-alpha, q[k], r[k]);
        } else {
#pragma omp parallel for schedule(static) if (chunked)
            for (int64_t k = 0; k < n; ++k) x[k] = x[k] + alpha * d[k];
#pragma omp parallel for schedule(static) if (chunked)
            for (int64_t k = 0; k < n; ++k) r[k] = r[k] - alpha * q[k];
        }
        /* line 7 */
        PRECOND(r, s);
        double rr = DOT(r, r);
        double rho_new = DOT(s, r);
        if (!isfinite(rho_new) || !isfinite(rr)) { rep->status = ORC_ERR_BREAKDOWN; it++; hist[it] = NAN; break; }
        double beta = rho_new / rho;
        /* line 8 (with s, not r: reading R6) */
        if (canonical) for (int64_t k = 0; k < n; ++k) d[k] = fma(beta, d[k], s[k]);
        else {
#pragma omp parallel for schedule(static) if (chunked)
            for (int64_t k = 0; k < n; ++k) d[k] = s[k] + beta * d[k];
        }
        rho = rho_new;
        it++;
        h = sqrt(rr) / nb;
        hist[it] = h;
    }
    rep->iterations = it;
    rep->rel_residual = hist[it];
    rep->converged = rep->status == ORC_OK && hist[it] <= tol;
    /* true residual, recomputed explicitly */
    APPLY_A(x, q);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - q[k];
    rep->true_rel_residual = sqrt(DOT(r, r)) / nb;
done:
    free(r); free(s); free(d); free(q); free(t); free(cpart);
    if (canonical) { free(C.rb); free(C.vals); free(C.partial); }
    return rep->status;
#undef DOT
#undef APPLY_A
#undef PRECOND
}

/* Chronopoulos-Gear PCG (Alg. 1 of PAPER.md:318-334 rearranged so that its two
 * inner products share one reduction point).  With s_k = A p_k, w_k = A u_k and u_k = P r_k:
 *   p_k = u_k + beta_k p_{k-1};  s_k = w_k + beta_k s_{k-1};  x += alpha_k p_k;  r -= alpha_k s_k;
 *   u = P r;  gamma' = (u, r);  rr = (r, r);  w = A u;  delta = (w, u);
 *   beta' = gamma'/gamma;  alpha' = gamma' / (delta - beta' gamma' / alpha)
 * (alpha_0 = gamma_0/delta_0, beta_0 = 0).  In exact arithmetic the iterates are Alg. 1's. */
int orc_pcg_cg(const orc_problem* P, const orc_ainv* R, const orc_pcg_opts* o, const double* b,
               const double* x0, double tol, int32_t maxit, double* x, double* hist, orc_pcg_report* rep) {
    memset(rep, 0, sizeof *rep);
    rep->failed_index = -1;
    int64_t n = P->n;
    if (!(tol >= 0.0) || maxit < 0) return rep->status = ORC_ERR_ARG;
    if (o->precond == ORC_PRECOND_AINV && !R) return rep->status = ORC_ERR_ARG;
    int canonical = o->mode == ORC_MODE_CANONICAL;
    canon C = {0};
    if (canonical) {                 /* as orc_pcg: parts > 1 = the rank-ordered tree over row blocks */
        if (o->pitch < P->ni || o->block < 32 || o->block > 1024 || (o->block & (o->block - 1)) ||
            o->parts < 1 || o->parts > 32 || o->parts > P->nj)
            return rep->status = ORC_ERR_ARG;
        C.P = P; C.pitch = o->pitch; C.B = o->block; C.parts = o->parts;
        C.rb = (int32_t*)malloc(sizeof(int32_t) * (o->parts + 1));
        if (o->parts == 1) { C.rb[0] = 0; C.rb[1] = P->nj; }
        else orc_partition(P->nj, P->ni, P->mask, o->parts, C.rb);
        C.vals = (double*)malloc(sizeof(double) * o->block);
        int64_t maxrows = 0;
        for (int r = 0; r < o->parts; ++r) if (C.rb[r + 1] - C.rb[r] > maxrows) maxrows = C.rb[r + 1] - C.rb[r];
        C.partial = (double*)malloc(sizeof(double) * ((maxrows + 1) * (o->pitch / o->block + 2)));
    }
#define DOT(a, b) (canonical ? canon_dot(&C, (a), (b)) : plain_dot(n, (a), (b)))
#define APPLY_A(in, out) (canonical ? canon_apply(P, (in), (out)) : orc_apply(P, (in), (out)))
    size_t sz = sizeof(double) * (n ? n : 1);
    double *r = malloc(sz), *u = malloc(sz), *w = malloc(sz), *p = malloc(sz), *sv = malloc(sz), *t = malloc(sz);
#define PRECOND(rin, sout)                                                        \
    do {                                                                          \
        if (o->precond == ORC_PRECOND_AINV) {                                     \
            if (canonical) canon_ainv_apply(R, (rin), (sout), t);                 \
            else orc_ainv_apply(R, (rin), (sout));                                \
        } else if (o->precond == ORC_PRECOND_JACOBI) {                            \
            for (int64_t k_ = 0; k_ < n; ++k_) (sout)[k_] = (rin)[k_] / P->diag[k_]; \
        } else {                                                                  \
            memcpy((sout), (rin), sz);                                            \
        }                                                                         \
    } while (0)
    for (int64_t k = 0; k < n; ++k) x[k] = x0 ? x0[k] : 0.0;
    double nb = sqrt(DOT(b, b));
    if (nb == 0.0) {
        for (int64_t k = 0; k < n; ++k) x[k] = 0.0;
        hist[0] = 0.0;
        rep->iterations = 0; rep->converged = 1;
        rep->status = ORC_OK;
        goto done;
    }
    APPLY_A(x, w);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - w[k];
    PRECOND(r, u);
    double gamma = DOT(u, r);
    double h = sqrt(DOT(r, r)) / nb;
    hist[0] = h;
    int32_t it = 0;
    rep->status = ORC_OK;
    if (!isfinite(h)) { rep->status = ORC_ERR_BREAKDOWN; goto fin; }
    double alpha = 0.0, beta = 0.0;
    if (h > tol && maxit > 0) {
        APPLY_A(u, w);
        double delta = DOT(w, u);
        if (!(delta > 0.0) || !isfinite(delta)) { rep->status = ORC_ERR_BREAKDOWN; goto fin; }
        alpha = gamma / delta;
    }
    for (int64_t k = 0; k < n; ++k) { p[k] = 0.0; sv[k] = 0.0; }
    while (h > tol && it < maxit) {
        if (canonical) {
            for (int64_t k = 0; k < n; ++k) {
                p[k] = fma(beta, p[k], u[k]);
                sv[k] = fma(beta, sv[k], w[k]);
                x[k] = fma(alpha, p[k], x[k]);
                r[k] = fma(-alpha, sv[k], r[k]);
            }
        } else {
            for (int64_t k = 0; k < n; ++k) {
                p[k] = u[k] + beta * p[k];
                sv[k] = w[k] + beta * sv[k];
                x[k] = x[k] + alpha * p[k];
                r[k] = r[k] - alpha * sv[k];
            }
        }
        PRECOND(r, u);
        double rr = DOT(r, r);
        double gamma_new = DOT(u, r);
        it++;
        if (!isfinite(gamma_new) || !isfinite(rr)) { rep->status = ORC_ERR_BREAKDOWN; hist[it] = NAN; break; }
        h = sqrt(rr) / nb;
        hist[it] = h;
        if (!(h > tol && it < maxit)) break;
        APPLY_A(u, w);
        double delta = DOT(w, u);
        beta = gamma_new / gamma;
        double den = delta - (beta * gamma_new) / alpha;
        if (!(den > 0.0) || !isfinite(den)) { rep->status = ORC_ERR_BREAKDOWN; break; }
        alpha = gamma_new / den;
        gamma = gamma_new;
    }
fin:
    rep->iterations = it;
    rep->rel_residual = hist[it];
    rep->converged = rep->status == ORC_OK && hist[it] <= tol;
    APPLY_A(x, w);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - w[k];
    rep->true_rel_residual = sqrt(DOT(r, r)) / nb;
done:
    free(r); free(u); free(w); free(p); free(sv); free(t);
    if (canonical) { free(C.rb); free(C.vals); free(C.partial); }
    return rep->status;
#undef DOT
#undef APPLY_A
#undef PRECOND
}

/* Pipelined PCG (Ghysels & Vanroose, "Hiding global synchronization latency
 * in the preconditioned conjugate gradient algorithm", Alg. 4 -- Alg. 1 of PAPER.md:318-334
 * rearranged once more so that the single reduction point of each iteration can overlap the
 * next preconditioner and matrix product).  Extra recurrences carry the products that
 * orc_pcg_cg recomputes: with u = P r, w = A u, m = P w, n = A m,
 *   k = 0:  beta = 0, alpha = gamma/delta;
 *   k > 0:  beta = gamma/gamma_prev, alpha = gamma / (delta - beta gamma / alpha_prev);
 *   z = n + beta z;  q = m + beta q;  s = w + beta s;  p = u + beta p;
 *   x += alpha p;  r -= alpha s;  u -= alpha q;  w -= alpha z;
 *   gamma = (r, u);  delta = (w, u);  rr = (r, r);  k += 1;  h_k = sqrt(rr)/||b||.
 * In exact arithmetic z = A q, q = P s, s = A p, so the iterates are Alg. 1's (the pins in
 * tests/test_oracle_pins.py check that against orc_pcg).  Breakdown: alpha's denominator
 * not > 0, gamma not > 0, or a non-finite value.  Same interface and modes as orc_pcg. */
int orc_pcg_pipe(const orc_problem* P, const orc_ainv* R, const orc_pcg_opts* o, const double* b,
                 const double* x0, double tol, int32_t maxit, double* x, double* hist, orc_pcg_report* rep) {
    memset(rep, 0, sizeof *rep);
    rep->failed_index = -1;
    int64_t n = P->n;
    if (!(tol >= 0.0) || maxit < 0) return rep->status = ORC_ERR_ARG;
    if (o->precond == ORC_PRECOND_AINV && !R) return rep->status = ORC_ERR_ARG;
    int canonical = o->mode == ORC_MODE_CANONICAL;
    canon C = {0};
    if (canonical) {
        if (o->pitch < P->ni || o->block < 32 || o->block > 1024 || (o->block & (o->block - 1)) ||
            o->parts < 1 || o->parts > 32 || o->parts > P->nj)
            return rep->status = ORC_ERR_ARG;
        C.P = P; C.pitch = o->pitch; C.B = o->block; C.parts = o->parts;
        C.rb = (int32_t*)malloc(sizeof(int32_t) * (o->parts + 1));
        if (o->parts == 1) { C.rb[0] = 0; C.rb[1] = P->nj; }
        else orc_partition(P->nj, P->ni, P->mask, o->parts, C.rb);
        C.vals = (double*)malloc(sizeof(double) * o->block);
        int64_t maxrows = 0;
        for (int r = 0; r < o->parts; ++r) if (C.rb[r + 1] - C.rb[r] > maxrows) maxrows = C.rb[r + 1] - C.rb[r];
        C.partial = (double*)malloc(sizeof(double) * ((maxrows + 1) * (o->pitch / o->block + 2)));
    }
#define DOT(a, b) (canonical ? canon_dot(&C, (a), (b)) : plain_dot(n, (a), (b)))
#define APPLY_A(in, out) (canonical ? canon_apply(P, (in), (out)) : orc_apply(P, (in), (out)))
    size_t sz = sizeof(double) * (n ? n : 1);
    double *r = malloc(sz), *u = malloc(sz), *w = malloc(sz), *m = malloc(sz), *nv = malloc(sz);
    double *z = malloc(sz), *q = malloc(sz), *sv = malloc(sz), *p = malloc(sz), *t = malloc(sz);
#define PRECOND(rin, sout)                                                        \
    do {                                                                          \
        if (o->precond == ORC_PRECOND_AINV) {                                     \
            if (canonical) canon_ainv_apply(R, (rin), (sout), t);                 \
            else orc_ainv_apply(R, (rin), (sout));                                \
        } else if (o->precond == ORC_PRECOND_JACOBI) {                            \
            for (int64_t k_ = 0; k_ < n; ++k_) (sout)[k_] = (rin)[k_] / P->diag[k_]; \
        } else {                                                                  \
            memcpy((sout), (rin), sz);                                            \
        }                                                                         \
    } while (0)
    for (int64_t k = 0; k < n; ++k) x[k] = x0 ? x0[k] : 0.0;
    double nb = sqrt(DOT(b, b));
    if (nb == 0.0) {
        for (int64_t k = 0; k < n; ++k) x[k] = 0.0;
        hist[0] = 0.0;
        rep->iterations = 0; rep->converged = 1;
        rep->status = ORC_OK;
        goto done;
    }
    APPLY_A(x, w);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - w[k];
    PRECOND(r, u);
    APPLY_A(u, w);
    double gamma = DOT(r, u), delta = DOT(w, u), rr = DOT(r, r);
    double h = sqrt(rr) / nb;
    hist[0] = h;
    int32_t it = 0;
    rep->status = ORC_OK;
    if (!isfinite(h) || !isfinite(gamma) || !isfinite(delta)) { rep->status = ORC_ERR_BREAKDOWN; goto fin; }
    for (int64_t k = 0; k < n; ++k) { z[k] = 0.0; q[k] = 0.0; sv[k] = 0.0; p[k] = 0.0; }
    double gamma_prev = 0.0, alpha_prev = 0.0;
    while (h > tol && it < maxit) {
        PRECOND(w, m);
        APPLY_A(m, nv);
        double beta, den;
        if (it == 0) { beta = 0.0; den = delta; }
        else { beta = gamma / gamma_prev; den = delta - (beta * gamma) / alpha_prev; }
        if (!(den > 0.0) || !isfinite(den) || !(gamma > 0.0)) { rep->status = ORC_ERR_BREAKDOWN; break; }
        double alpha = gamma / den;
        if (canonical) {
            for (int64_t k = 0; k < n; ++k) {
                z[k] = fma(beta, z[k], nv[k]);
                q[k] = fma(beta, q[k], m[k]);
                sv[k] = fma(beta, sv[k], w[k]);
                p[k] = fma(beta, p[k], u[k]);
                x[k] = fma(alpha, p[k], x[k]);
                r[k] = fma(-alpha, sv[k], r[k]);
                u[k] = fma(-alpha, q[k], u[k]);
                w[k] = fma(-alpha, z[k], w[k]);
            }
        } else {
            for (int64_t k = 0; k < n; ++k) {
                z[k] = nv[k] + beta * z[k];
                q[k] = m[k] + beta * q[k];
                sv[k] = w[k] + beta * sv[k];
                p[k] = u[k] + beta * p[k];
                x[k] = x[k] + alpha * p[k];
                r[k] = r[k] - alpha * sv[k];
                u[k] = u[k] - alpha * q[k];
                w[k] = w[k] - alpha * z[k];
            }
        }
        gamma_prev = gamma;
        alpha_prev = alpha;
        gamma = DOT(r, u);
        delta = DOT(w, u);
        rr = DOT(r, r);
        it++;
        if (!isfinite(gamma) || !isfinite(delta) || !isfinite(rr)) {
            rep->status = ORC_ERR_BREAKDOWN; hist[it] = NAN; break;
        }
        h = sqrt(rr) / nb;
        hist[it] = h;
    }
fin:
    rep->iterations = it;
    rep->rel_residual = hist[it];
    rep->converged = rep->status == ORC_OK && hist[it] <= tol;
    APPLY_A(x, w);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - w[k];
    rep->true_rel_residual = sqrt(DOT(r, r)) / nb;
done:
    free(r); free(u); free(w); free(m); free(nv); free(z); free(q); free(sv); free(p); free(t);
    if (canonical) { free(C.rb); free(C.vals); free(C.partial); }
    return rep->status;
#undef DOT
#undef APPLY_A
#undef PRECOND
}
