/* libpcg.h -- C ABI of libpcg: B200-native fp64 PCG with an AINV approximate-inverse
 * preconditioner for the elliptic sea-surface equation of NEMO-OPA (arXiv 1210.1878).
 *
 * The three calls of the north star:
 *   pcg_setup  -- assemble the SPD five-point operator A on an (ni, nj) ORCA-style grid
 *                 with land mask and periodic east-west wrap (Eq. 9-10),
 *                 then build AINV factors Z, D with a drop tolerance (the paper's "P_B1",
 *                 PAPER.md:459; AINV cited at PAPER.md:26, 224).
 *   pcg_solve  -- Alg. 1 of the paper (d = s + beta d: DESIGN.md R6):
 *                 per iteration q = A d (stencil), s = Z D^-1 Z^T r (two SELL products, no
 *                 triangular solves), fused dot products and axpys; returns x, the
 *                 iteration count and the residual history.
 *   pcg_free   -- release everything.
 *
 * CONVENTIONS
 *   Grid arrays are row-major [nj][ni]: i = east-west (fastest, periodic), j = south-north
 *   (reading R2).  cE[j][i] is the coupling of cell (i,j) with (i+1 mod ni, j)
 *   (paper C^EW on the east face); cN[j][i] couples (i,j) with (i,j+1) (paper C^NS on
 *   the north face); row nj-1 of cN is ignored.  mask: 1 = ocean unknown, 0 = land (not an
 *   unknown, x = 0 there, b ignored).  A is the NEGATION of Eq. 10 as printed, so it is
 *   SPD (reading R1): A_pp = ((c_E + c_W) + c_N) + c_S (+ sigma_p) over the existing faces
 *   of ocean point p (faces to land included: Dirichlet anchor, reading R3), A_pq = -c for
 *   each face to an ocean neighbour q.
 *   All arithmetic is IEEE fp64.  The GPU arithmetic order is documented in DESIGN.md §5
 *   (the oracle's "canonical" mode reproduces it bit for bit).
 *
 * MULTI-GPU
 *   One process per GPU.  Rank p owns grid rows [j_begin, j_end) (use pcg_partition for
 *   the documented split); rows are ordered south -> north by rank.  With nranks > 1 the
 *   calls pcg_setup, pcg_solve, pcg_solve_host, pcg_apply_operator and pcg_free are
 *   COLLECTIVE: every rank calls them with equal scalar arguments.  The NCCL communicator
 *   is borrowed (create one with pcg_comm_init_rank).
 *
 * ERRORS
 *   Every call returns pcg_status.  Non-convergence within maxit is PCG_OK with
 *   report.converged = 0.  pcg_last_error(ctx) (or pcg_last_error(NULL) after
 *   a failed pcg_setup) returns a message naming the offending argument or grid point.
 *   Library state is unchanged by a failed call except where stated.
 */
#ifndef LIBPCG_H
#define LIBPCG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LIBPCG_ABI_VERSION 1

typedef struct pcg_ctx pcg_ctx;     /* opaque, owned by the library */
typedef struct pcg_plan pcg_plan;   /* opaque host-only setup product (no GPU needed) */

typedef enum {
    PCG_OK = 0,
    PCG_ERR_ARG = 1,        /* bad dimension, pointer, NaN/negative coefficient, tol < 0 ... */
    PCG_ERR_NOT_SPD = 2,    /* non-positive diagonal, failed anchor check, AINV pivot <= 1e-12 */
    PCG_ERR_BREAKDOWN = 3,  /* (d, q) <= 0 or a non-finite reduction during the solve */
    PCG_ERR_CUDA = 4,       /* CUDA runtime error (message from cudaGetErrorString) */
    PCG_ERR_COMM = 5,       /* NCCL error */
    PCG_ERR_NOMEM = 6       /* host or device allocation failed */
} pcg_status;

typedef enum {
    PCG_PRECOND_AINV = 0,   /* s = Z D^-1 Z^T r  (north star) */
    PCG_PRECOND_JACOBI = 1, /* s = r / A_pp: NEMO's diagonal preconditioner (Eq. 15) */
    PCG_PRECOND_NONE = 2,   /* s = r: plain CG */
    PCG_PRECOND_FSAI = 3    /* the paper's own P = Z~ Z~^t: banded FSAI of T = band(A, 1), bandwidth
                               fsai_q (Eq. 19; R25).
                               One rank only (nranks > 1 -> PCG_ERR_ARG). */
} pcg_precond;

/* flags */
#define PCG_FLAG_HOST_LOOP   1  /* drive iterations from the host instead of one CUDA graph
                                   with a device-side WHILE node (results are identical) */
#define PCG_FLAG_COMM_PATH   2  /* use the multi-rank code path (NCCL) even when nranks == 1 */
#define PCG_FLAG_LOCAL_RANKS 4  /* this context is one rank of an in-process, one-GPU emulation of a
                                   multi-rank run (no NCCL); solve with pcg_solve_local_ranks */
#define PCG_FLAG_SINGLE_REDUCTION 8  /* Chronopoulos-Gear PCG: the iteration's
                                        two inner products share one reduction point (kernels KA,
                                        K3, KC).  One rank, factored preconditioners (AINV, P_B2,
                                        FSAI through the ELL form); otherwise PCG_ERR_ARG. */
#define PCG_FLAG_PIPELINED 16  /* pipelined PCG (Ghysels & Vanroose Alg. 4, the
                                  oracle's orc_pcg_pipe): the reduction of (r,u), (w,u), (r,r) is
                                  consumed one phase later, so it overlaps the next application of
                                  the preconditioner (kernels KPA, KPB, KPC); across ranks the rank
                                  sums ride in the halo exchange of m = P w.  Factored
                                  preconditioners only, block-local AINV across ranks, not with
                                  PCG_FLAG_SINGLE_REDUCTION; otherwise PCG_ERR_ARG.  The stop test
                                  and breakdown are Alg. 1's (reading R29). */
#define PCG_FLAG_DEVICE_COMM 32  /* multi-rank NCCL path: every reduction's rank sums are gathered
                                    inside the reducing kernel -- its last block stores them into
                                    every rank's symmetric NCCL window over NVLink (ncclMemAlloc +
                                    ncclCommWindowRegister, peer pointers from ncclGetPeerPointer)
                                    and runs the scalar step (rank tree, alpha / beta, stop test)
                                    inline -- instead of a host-enqueued ncclAllGather and a
                                    scalar kernel (bitwise the same results).  With
                                    PCG_DC_HALO=1 (opt-in), for Alg. 1 with block-local AINV
                                    (ainv_halo = 0), the s array also lives in the window and K3
                                    stores its first / last owned row into the neighbours' halo
                                    rows itself: no NCCL call per iteration.  Needs
                                    nccl_comm with every rank load/store reachable (one NVLink
                                    domain, else PCG_ERR_COMM); not with PCG_FLAG_LOCAL_RANKS
                                    (PCG_ERR_ARG).  pcg_setup is then collective over the
                                    communicator (window registration). */

/* "grid": geometry of this rank's part of the problem. */
typedef struct {
    int32_t ni, nj;          /* global grid, ni >= 3, nj >= 3 */
    int32_t periodic_ew;     /* 1 = east-west periodic (ORCA), 0 = W/E faces at the ends absent */
    int32_t j_begin, j_end;  /* owned rows [j_begin, j_end); [0, nj) on one GPU */
    int32_t rank, nranks;    /* row blocks in rank order (rank 0 is southernmost) */
    void*   nccl_comm;       /* borrowed ncclComm_t; NULL when nranks == 1 */
    int32_t device;          /* CUDA device ordinal of this rank */
    void*   stream;          /* borrowed cudaStream_t (NULL = legacy default stream) */
} pcg_grid;

/* "coefficients, mask": HOST pointers to the GLOBAL [nj][ni] arrays (every rank passes the
 * full arrays; only the rows it needs are read).  Copied by pcg_setup; the caller may free
 * them on return. */
typedef struct {
    const double*  cE;     /* >= 0, finite.  Eq. 9 C^EW on east faces */
    const double*  cN;     /* >= 0, finite.  Eq. 9 C^NS on north faces; row nj-1 ignored      */
    const double*  sigma;  /* optional diagonal shift >= 0 (identity term of Eq. 2, reading R5); NULL = 0 */
    const uint8_t* mask;   /* 0/1 */
} pcg_coeffs;

typedef struct {
    pcg_precond precond;
    double  drop_tol;      /* AINV drop tolerance tau >= 0 (+inf: Jacobi-equivalent AINV) */
    int32_t flags;         /* PCG_FLAG_* */
    int32_t ainv_parts;    /* 0/1: AINV over this rank's rows; P > 1 (one GPU only): build the
                              preconditioner as P row blocks, exactly as P ranks would */
    int32_t ainv_halo;     /* halo-AINV width w (grid rows south of each block); 0 = block-local.
                              With ainv_parts > 1 (one GPU) or nranks > 1: each block starts w
                              rows below its first row, giving one global triangular Z (SURVEY
                              §8e, R15 and §6).  Across ranks every rank but the last
                              needs >= 16 owned rows (else PCG_ERR_ARG); the solve then exchanges
                              the rows of q and r the owned columns reach (<= w) after K1 and the
                              needed rows of t after K2.  w >= nj: every block starts at row 0, so
                              each rank holds its columns of the GLOBAL Z (the
                              preconditioner is bitwise independent of the rank count; the setup
                              of rank p costs the AINV of rows [0, j_end)). */
    int32_t setup_threads; /* host threads for the AINV build (0 = automatic) */
    int32_t fsai_q;        /* PCG_PRECOND_FSAI: upper bandwidth q >= 0 of Z~ (entries z_ij with
                              j > i + q dropped); ignored otherwise */
    int32_t ainv_fill;     /* PCG_PRECOND_AINV: 0 = drop tolerance only (P_B1); m > 0 = also keep at
                              most m entries per column of Zhat (the diagonal and the m-1 largest
                              |z|, ties to the smaller row) after every update: the paper's P_B2
                              (R26); use drop_tol = 0 for pure
                              P_B2 */
} pcg_opts;

typedef struct {
    int32_t iterations;        /* PCG iterations performed */
    int32_t converged;         /* final recurrence residual <= tol */
    double  rel_residual;      /* ||r_k|| / ||b|| from the recurrence */
    double  true_rel_residual; /* ||b - A x|| / ||b|| recomputed at exit */
    double  setup_s;           /* host wall seconds spent in pcg_setup */
    double  solve_s;           /* device seconds of the solve (CUDA events) */
    double  bytes_per_iter;    /* algorithmic HBM bytes per iteration */
    int64_t n_ocean;           /* ocean unknowns owned by this rank */
    int64_t nnz_z;             /* off-diagonal nonzeros of this rank's Z columns */
    int64_t failed_index;      /* global unknown index for NOT_SPD, else -1 */
    int32_t driver;            /* how the iterations ran (PCG_DRIVER_*): one rank -- the resident-strip
                                  loop kernel, the WHILE-node graph, the cooperative loop kernel or the
                                  host loop; several ranks -- the NCCL graph, or the NCCL host loop
                                  when the graph could not be captured (PCG_DRIVER_NCCL_FALLBACK: the
                                  capture failure is reported here, not hidden) */
    int32_t kernels_per_iter;  /* this library's kernel launches per iteration of the driver used
                                  (graph / host loop: the iteration's kernels incl. scalar steps;
                                  resident strips and the cooperative loop: 0 -- one kernel per solve) */
} pcg_report;

enum { PCG_DRIVER_GRAPH = 0, PCG_DRIVER_LOOP = 1, PCG_DRIVER_RESIDENT = 2, PCG_DRIVER_HOST_LOOP = 3,
       PCG_DRIVER_NCCL_GRAPH = 4, PCG_DRIVER_NCCL_FALLBACK = 5, PCG_DRIVER_NCCL_HOST_LOOP = 6,
       PCG_DRIVER_LOCAL_RANKS = 7 };

/* ---------------------------------------------------------------- the three calls */

/* Validate, partition, assemble A, run the anchor check, build AINV(A_pp, tau) on the host,
 * pack Z and Z^T as SELL-32, upload to the device and (unless PCG_FLAG_HOST_LOOP) capture
 * the solve graph.  *out receives the context on PCG_OK, NULL otherwise.
 * Errors: PCG_ERR_ARG (NULL pointers, ni/nj < 3, bad row range, coefficient < 0 or not
 * finite, mask not 0/1, tau < 0 or NaN), PCG_ERR_NOT_SPD (ocean point with A_pp <= 0, an
 * ocean component with no positive land face and sigma = 0, or an AINV pivot <= 1e-12;
 * report via pcg_last_error(NULL)), PCG_ERR_CUDA, PCG_ERR_COMM, PCG_ERR_NOMEM. */
pcg_status pcg_setup(const pcg_coeffs* coeffs, const pcg_grid* grid, const pcg_opts* opts,
                     pcg_ctx** out);

/* Solve A x = b on this rank's rows.
 *   b, x0, x : DEVICE pointers to [j_end - j_begin][ni] row-major fp64 arrays (owned rows,
 *              no padding).  x0 == NULL means x0 = 0.  x may alias x0.
 *   tol      : stop when ||r_k||/||b|| <= tol (Alg. 1 line 5); tol = 0 runs
 *              exactly maxit iterations.  tol < 0 -> PCG_ERR_ARG.
 *   maxit    : iteration cap (reading R7); < 0 -> PCG_ERR_ARG.
 *   iterations (host out, may be NULL); res_hist (host out, may be NULL): res_hist[k] =
 *   ||r_k||/||b|| for k = 0..min(iterations, hist_cap-1); report (host out, may be NULL).
 * b = 0 gives x = 0 and 0 iterations.  Breakdown ((d,q) <= 0 or non-finite, or
 * a non-finite ||b|| or ||r_0|| -- NaN / Inf in b or x0) returns PCG_ERR_BREAKDOWN with the
 * iterations done so far and x from the last valid iterate.  Synchronises the context's stream
 * before returning. */
pcg_status pcg_solve(pcg_ctx* ctx, const double* b, const double* x0, double tol, int32_t maxit,
                     double* x, int32_t* iterations, double* res_hist, int32_t hist_cap,
                     pcg_report* report);

/* As pcg_solve, but b, x0 and x are HOST pointers (pinned or pageable); the host<->device
 * copies run inside the call on the context's stream. */
pcg_status pcg_solve_host(pcg_ctx* ctx, const double* b, const double* x0, double tol,
                          int32_t maxit, double* x, int32_t* iterations, double* res_hist,
                          int32_t hist_cap, pcg_report* report);

/* One-GPU emulation of an n-rank run (testing the multi-rank device path without n GPUs):
 * ctxs[r] was set up as rank r of n (pcg_partition rows) with PCG_FLAG_LOCAL_RANKS on the same
 * device.  The host steps all ranks phase by phase on one stream; the allgather of rank sums and
 * the halo rows are device-to-device copies between the contexts (no kernel waits on another
 * rank).  Same arithmetic as the NCCL path.  b, x0 (NULL = 0), x: DEVICE pointers to the GLOBAL
 * [nj][ni] arrays; the other arguments as pcg_solve (report sums n_ocean / nnz_z over ranks). */
pcg_status pcg_solve_local_ranks(pcg_ctx* const* ctxs, int32_t n, const double* b, const double* x0, double tol,
                                 int32_t maxit, double* x, int32_t* iterations, double* res_hist,
                                 int32_t hist_cap, pcg_report* report);

/* NULL-safe.  Frees device memory and graphs; does not free the borrowed comm/stream. */
void pcg_free(pcg_ctx* ctx);

/* Message for the last non-OK status of ctx, or of the calling thread if ctx == NULL. */
const char* pcg_last_error(const pcg_ctx* ctx);

/* ---------------------------------------------------------------- utilities */

/* y = A x on this rank's rows (Eq. 10 negated; same stencil kernel and order as the solve).
 * x, y: DEVICE [rows][ni] pointers.  Collective with nranks > 1 (halo exchange). */
pcg_status pcg_apply_operator(pcg_ctx* ctx, const double* x, double* y);

/* s = P r with the context's preconditioner (AINV: Z D^-1 Z^T r).  DEVICE [rows][ni].
 * Single rank only (PCG_ERR_ARG otherwise). */
pcg_status pcg_apply_preconditioner(pcg_ctx* ctx, const double* r, double* s);

/* NEMO's first guess for the next time step's solve (Alg. 1 l.1 "x0 = 2D^{t-1}",
 * read as the extrapolation 2 D^t - D^{t-1} of NEMO's solver, R27):
 * x0[e] = 2 x_t[e] - x_tm1[e] (2 x_t is exact, one IEEE subtraction) on this rank's rows.
 * x_t, x_tm1, x0: DEVICE [rows][ni]; x0 may alias either input.  Ordered after the context's
 * user stream, returns when done.  Used by the time-stepping driver. */
pcg_status pcg_extrapolate(pcg_ctx* ctx, const double* x_t, const double* x_tm1, double* x0);

/* Documented row-block split: with cum[j] = ocean points in rows < j and
 * N = cum[nj], row_begin[p] = min{ j : cum[j]*parts >= p*N } (forced strictly increasing),
 * row_begin[0] = 0, row_begin[parts] = nj.  row_begin has parts+1 entries (host).
 * PCG_ERR_ARG if parts < 1 or parts > nj. */
pcg_status pcg_partition(int32_t ni, int32_t nj, const uint8_t* mask, int32_t parts,
                         int32_t* row_begin);

/* Device layout that fixes the canonical arithmetic order: row pitch
 * (elements, multiple of 32), threads per block (= grid columns per tile) and grid rows per
 * tile.  Any output pointer may be NULL. */
pcg_status pcg_layout(const pcg_ctx* ctx, int32_t* pitch, int32_t* block, int32_t* rows);

/* Device time (ms) of each per-iteration kernel over n_iter iterations run on the
 * context's stream with CUDA events around every launch, on the state left by the last
 * solve (a profiling aid for bench.py).  ms_out[0..3] = median per-launch time of K1
 * (stencil), K2 (r update + Z^T gather), K3 (Z gather), and of the whole iteration; bytes_out[0..2] = algorithmic bytes per
 * launch of K1..K3.  With the kfin reduction kernels (large grids) K1's and
 * K3's times include their kfin launch, as they otherwise include their last-block tails.
 * Single rank only. */
pcg_status pcg_kernel_times(pcg_ctx* ctx, int32_t n_iter, double* ms_out, double* bytes_out);

/* Device bytes allocated by the context. */
int64_t pcg_device_bytes(const pcg_ctx* ctx);

/* Device time (ms, CUDA events on the context's stream) of the resident-strip loop kernel of the
 * last pcg_solve -- one persistent cooperative launch that runs every PCG iteration (DESIGN.md
 * §7.4) -- and the iterations it ran.  *ms = -1 when the last solve did not use that driver
 * (several ranks, the host loop, the graph or cooperative-loop drivers).  Host pointers; iterations
 * may be NULL.  PCG_ERR_ARG on a NULL ctx or ms. */
pcg_status pcg_loop_time(const pcg_ctx* ctx, double* ms, int32_t* iterations);

/* ---------------------------------------------------------------- host-only setup
 * The host half of pcg_setup (validation, partition, anchor check, AINV, SELL packing),
 * usable without a GPU; tests compare it bit for bit with the oracle. */
pcg_status pcg_plan_build(const pcg_coeffs* coeffs, const pcg_grid* grid, const pcg_opts* opts,
                          pcg_plan** out);
void       pcg_plan_free(pcg_plan* plan);
/* counts: [0] n_ocean owned, [1] nnz of owned Zhat columns incl. diagonal, [2] pitch,
 * [3] SELL entries (with padding) of Z rows, [4] SELL entries of Z^T rows,
 * [5] first global unknown index owned by this rank. */
pcg_status pcg_plan_counts(const pcg_plan* plan, int64_t* counts6);
/* Owned columns of Zhat in CSC with GLOBAL unknown row indices (natural order), the
 * pivots Dhat and the scale s = 1/sqrt(A_pp) of the owned unknowns.  Arrays sized from
 * pcg_plan_counts (colptr: n_ocean+1, row/zhat: nnz). */
pcg_status pcg_plan_export_zhat(const pcg_plan* plan, int64_t* colptr, int64_t* row,
                                double* zhat, double* pivots, double* scale);

/* ---------------------------------------------------------------- NCCL plumbing */
/* 128-byte ncclUniqueId into out[128] (rank 0 creates it; broadcast it with torch.distributed). */
pcg_status pcg_comm_unique_id(char* out128);
/* ncclCommInitRank on `device`; *comm receives an ncclComm_t to pass in pcg_grid.nccl_comm. */
pcg_status pcg_comm_init_rank(const char* id128, int32_t nranks, int32_t rank, int32_t device,
                              void** comm);
pcg_status pcg_comm_destroy(void* comm);

/* Diagnostics: the device-comm protocol of PCG_FLAG_DEVICE_COMM (dc_publish / dc_collect, DESIGN.md
 * §6.3) run by nranks virtual ranks -- the blocks of one cooperative launch on the current device,
 * windows carved from one buffer -- for `rounds` reductions.  In round k rank r contributes the four
 * values v(k, r, q) of a fixed hash of (seed, k, r, q) (odd rounds through the split publish /
 * collect form); out[(k * nranks + r) * 4 + q] (host, rounds * nranks * 4 doubles) receives rank
 * r's canonical rank tree of slot q.  Every rank must obtain the same sums, equal
 * to the host's tree over the same values.  1 <= nranks <= 32, rounds >= 1, else PCG_ERR_ARG. */
pcg_status pcg_devcomm_selftest(int32_t nranks, int32_t rounds, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
