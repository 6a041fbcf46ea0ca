/* oracle.h -- plain CPU oracle for arXiv 1210.1878's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  It shares no code,
 * header, table or helper with the CUDA path (paper_1210_1878_b200/csrc) and neither
 * side includes the other.
 *
 * What it computes (all fp64, built with -ffp-contract=off so every a*b+c is two
 * rounded operations unless std fma() is called explicitly):
 *   - assembly of the SPD five-point operator A on the masked, E-W periodic grid
 *     (Eq. 9-10; reading R1-R5 in DESIGN.md);
 *   - the anchor (non-singularity) check (reading R22);
 *   - AINV(A, tau): A-orthogonalisation with a drop tolerance, the paper's
 *     "Bridson P_B1", in two independent
 *     formulations (sparse left-looking and dense right-looking);
 *   - the partitioned ("per partition, halo w") AINV (reading R15);
 *   - the paper's own preconditioner, the banded FSAI of T = band(A, 1) (PAPER.md:226-309,
 *     Eq. 19; NEXT-1, reading R25), as an AINV-form factor;
 *   - PCG, Alg. 1 with the line-8 fix d = s + beta d (reading R6),
 *     in "plain" order (sequential sums) and in "canonical" order (the GPU's documented
 *     arithmetic order, re-implemented here from DESIGN.md §5, not from GPU code).
 *
 * Unknowns are the ocean points in natural order: j outer (south->north), i inner
 * (west->east).  Vectors passed in/out are unknown-indexed unless a
 * function says "grid".
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_NOT_SPD = 2, ORC_ERR_BREAKDOWN = 3, ORC_ERR_NOMEM = 6 };
enum { ORC_PRECOND_AINV = 0, ORC_PRECOND_JACOBI = 1, ORC_PRECOND_NONE = 2 };
enum { ORC_MODE_PLAIN = 0, ORC_MODE_CANONICAL = 1, ORC_MODE_CHUNKED = 2 };
/* CHUNKED: PLAIN arithmetic for every row (A x, Z^T r, Z t, updates), dot products as
 * partials of fixed 4096-element chunks of the natural order (each summed left to right), the
 * partials then summed left to right in chunk order.  Rows and chunks run on all host cores
 * (OpenMP); the result does not depend on the thread count.  Used for the all-cores CPU baseline
 * (SURVEY §8(d)). */

typedef struct orc_problem orc_problem;
typedef struct orc_ainv orc_ainv;

/* ---- assembly (Eq. 9-10) ---- */
int  orc_assemble(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                  const double* sigma /*nullable*/, const uint8_t* mask, orc_problem** out);
void orc_problem_free(orc_problem*);
int64_t orc_n(const orc_problem*);
int64_t orc_nnz(const orc_problem*);
void orc_csr(const orc_problem*, int64_t* rowptr, int64_t* col, double* val);
void orc_grid_index(const orc_problem*, int64_t* grid_of_unknown);   /* j*ni + i */
void orc_diag(const orc_problem*, double* d);
/* y = A x, CSR rows summed left to right (column ascending), separate mul/add. */
void orc_apply(const orc_problem*, const double* x, double* y);
/* Returns -1 if every ocean component is anchored, else the smallest unknown index of
 * the first (natural order) unanchored component. */
int64_t orc_anchor_check(const orc_problem*);

/* ---- partition (row blocks balanced by ocean count) ---- */
void orc_partition(int32_t nj, int32_t ni, const uint8_t* mask, int32_t parts, int32_t* row_begin /*parts+1*/);

/* ---- AINV ---- */
/* method 0 = sparse left-looking, 1 = dense right-looking (n <= 4000).
 * parts >= 1 row blocks, halo w >= 0 southern rows (parts == 1: global AINV). */
int  orc_ainv_build(const orc_problem*, double tau, int32_t method, int32_t parts, int32_t halo,
              orc_ainv** out, int64_t* failed_col);
/* P_B2 (reading R26): as orc_ainv_build, and after every update keep
 * only the diagonal plus the fill-1 largest-magnitude entries of the column (ties: smaller row);
 * fill = 0 = no limit (orc_ainv_build).  Use tau = 0 for the pure fixed-fill preconditioner. */
int  orc_ainv_build_fill(const orc_problem*, double tau, int32_t fill, int32_t method, int32_t parts,
                         int32_t halo, orc_ainv** out, int64_t* failed_col);
void orc_ainv_free(orc_ainv*);
int64_t orc_ainv_nnz(const orc_ainv*);          /* nnz of Zhat incl. unit diagonal */
/* Zhat as CSC (columns j, rows k ascending), pivots p (=Dhat), scale s = 1/sqrt(A_pp),
 * and the apply-ready values z_kj = fl(s_k * zhat_kj). */
void orc_ainv_export(const orc_ainv*, int64_t* colptr, int64_t* row, double* zhat, double* z,
                     double* pivots, double* scale);
/* s = Z D^-1 Z^T r, plain order: t_j = (sum_k z_kj r_k)/p_j, s_i = sum_j z_ij t_j. */
void orc_ainv_apply(const orc_ainv*, const double* r, double* s);

/* ---- the paper's banded FSAI of T (NEXT-1; Eq. 19) ---- */
/* T = band(A, 1) in the unknown numbering; T = U^t U; zhat_{k-i,k} = prod_{r=1..i} rho_{k-r},
 * rho_m = -u_{m,m+1}/u_mm, truncated at bandwidth q (and where the chain breaks); pivots
 * p_k = u_kk^2; scale 1.  Returned as an orc_ainv: every apply / PCG routine takes it. */
int  orc_fsai_build(const orc_problem*, int32_t q, orc_ainv** out, int64_t* failed_col);

/* ---- PCG (Alg. 1, with d = s + beta d) ---- */
typedef struct {
    int32_t precond;      /* ORC_PRECOND_* */
    int32_t mode;         /* ORC_MODE_* */
    int32_t pitch;        /* canonical mode: row pitch of the grid layout (>= ni) */
    int32_t block;        /* canonical mode: threads per block (power of two, >= 32) */
    int32_t parts;        /* canonical mode: number of rank row blocks (>=1) */
    int32_t rows;         /* unused (kept for ABI stability of the test binding) */
} orc_pcg_opts;

typedef struct {
    int32_t iterations, converged, status;
    double rel_residual, true_rel_residual;
    int64_t failed_index;
} orc_pcg_report;

/* The canonical-order pieces on their own: y = A x with the W,E,S,N fma
 * stencil; s = Z D^-1 Z^T r with fma row sums; the block-tree dot product. */
void   orc_apply_canonical(const orc_problem*, const double* x, double* y);
void   orc_ainv_apply_canonical(const orc_ainv*, const double* r, double* s);
double orc_dot_canonical(const orc_problem*, const orc_pcg_opts*, const double* a, const double* b);

/* x, hist are outputs (hist length >= maxit+1).  x0 may be NULL (= 0).  tol = 0 runs
 * exactly maxit iterations. */
int orc_pcg(const orc_problem*, const orc_ainv* /*nullable unless AINV*/, const orc_pcg_opts*,
            const double* b, const double* x0, double tol, int32_t maxit,
            double* x, double* hist, orc_pcg_report* rep);

/* Chronopoulos-Gear PCG: Alg. 1's iterates with ONE reduction point per
 * iteration -- (r, u), (w, u) and (r, r) are formed together after w = A u -- using the
 * recurrences p = u + beta p, s = w + beta s (s = A p), x += alpha p, r -= alpha s, u = P r,
 * w = A u, beta = gamma'/gamma, alpha = gamma' / (delta - beta gamma'/alpha).  Same interface
 * and modes as orc_pcg (canonical = the GPU's documented order). */
int orc_pcg_cg(const orc_problem*, const orc_ainv* /*nullable unless AINV*/, const orc_pcg_opts*,
               const double* b, const double* x0, double tol, int32_t maxit,
               double* x, double* hist, orc_pcg_report* rep);

/* Pipelined PCG (Ghysels-Vanroose Alg. 4): Alg. 1 with the recurrences
 * z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p (m = P w, n = A m) so that the
 * three inner products (r,u), (w,u), (r,r) form one reduction point per iteration that does not
 * wait on P or A.  Same interface and modes as orc_pcg. */
int orc_pcg_pipe(const orc_problem*, const orc_ainv* /*nullable unless AINV*/, const orc_pcg_opts*,
                 const double* b, const double* x0, double tol, int32_t maxit,
                 double* x, double* hist, orc_pcg_report* rep);

#ifdef __cplusplus
}
#endif
#endif
