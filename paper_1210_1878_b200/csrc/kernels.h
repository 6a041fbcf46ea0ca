// kernels.h -- device state and kernel launchers of libpcg (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace pcg {

enum : int32_t { kStOk = 0, kStBreakdown = 3 };
constexpr int kMaxRowsK1 = 16;     // rows per K1 block (register march), <= kMaxRowsK1

// Device-resident scalars of one solve.  Written only by the last block of a
// reduction kernel (one rank) or by the 1-thread scalar kernels after an NCCL allgather.
struct DevScalars {
    double alpha, beta, rho, nb, tol, true_rel;
    double hpre;          // sqrt((r,r)) / nb of the current iteration, formed early by K3's block 0
    double hlast;         // the last history value written (report.rel_residual; the history buffer may be shorter)
    double rho_prev;      // rho of the previous iteration: K1 forms beta = rho / rho_prev itself
    double red[4];        // global reductions: [0] (d,q)  [1] (s,r)  [2] (r,r)  [3] (b,b) / true (r,r)
    double loc[4];        // this rank's block-tree sums (multi-rank path)
    int32_t k, maxit, active, status, bzero, xpend, guard;
    int32_t pstage;       // pipelined PCG: 0 = the pending reduction is the prologue's, 1 = an iteration's
    double rhop[2];       // redundant-sum mode: rho of the iterations of parity 0 / 1 (rhop[1] = inf before the first)
    uint32_t counter[4];  // last-block detection, reset by the last block
    unsigned long long ticket[4];   // dynamic unit assignment, reset by the last block
};

// Device view of an ELL(kEll) + overflow-SELL matrix (see internal.h).
struct EllDev {
    const double* val;          // kEll * n
    const int32_t* col;         // kEll * n, packed (di, dj)
    const int64_t* ooff;        // overflow slice offsets (nslices + 1)
    const double* oval;
    const int32_t* ocol;
    int64_t n;
    const int16_t* col16 = nullptr;   // kEll * n slot offsets from the element's own array index
};


// Resident-strip driver (rs.cu): one persistent cooperative block of 512 or 768 threads
// per SM runs the whole PCG loop.  Block b owns a contiguous range of units (row segments, in
// row-major order) per phase -- ub1 for the K1 phase (stencil), ub2 for the K2/K3 phase
// (preconditioner) -- and keeps the vector that phase gathers from (d, r_new, t) for its range
// plus the halo its stencil / Z rows reach in shared memory, so every gather is a shared-memory
// load.  Two grid barriers per iteration (the two dot products of Alg. 1) and one neighbour flag
// (t rows of the blocks to the north).
constexpr int kRsThreadsSmall = 512, kRsThreadsLarge = 768;   // the two rs_loop_kernel block sizes
struct RsDev {
    int32_t on;                   // eligible and enabled
    int32_t nblk;                 // blocks (= SMs, one resident block each)
    int32_t nt;                   // threads per block (kRsThreadsSmall or kRsThreadsLarge)
    int32_t cap;                  // shared-memory buffer (doubles)
    int32_t maxu1, maxu2;         // most units of one block per phase
    int32_t maxnx;                // most 32-element chunks any pass of one block touches
    size_t smem;                  // dynamic shared memory per block (bytes)
    const int32_t* ub1;     // [nblk + 1] K1-phase unit bounds
    const int32_t* ub2;     // [nblk + 1] K2/K3-phase unit bounds
    const int64_t* lo2;     // [nblk] first array index of the r_new buffer (Z^T reach)
    const int64_t* hi2;     // [nblk] end of the t buffer (Z reach)
    const int32_t* wait2;   // [nblk] last block whose t this block gathers
    uint32_t* sync;         // [0] grid-barrier counter, [1 + b] t-ready stamp of block b
    const int64_t* pf;      // [nblk][4] SELL overflow entry range of each block (Z^T first, count, Z first, count)
};

struct KArgs {
    int32_t ni, pitch, nloc, nranks;
    int32_t halo;                     // halo grid rows on each side (owned row j at array row j + halo)
    int64_t hoff;                     // halo * pitch: array index of owned element 0
    int32_t nbx, rpb;                 // column segments of kBlock per row; rows per K1 strip
    int32_t g_k1, g_k2, g_k3, g_kd, g_row;   // persistent grid sizes (configure_kernels)
    int32_t dynamic, dynamic_k1;      // units from an atomic ticket instead of a block stride
    int32_t g_loop;                   // cooperative grid of the fused loop kernel
    int32_t k1flat, g_k1f;            // K1 in row-segment form (one element per thread)
    int32_t pdl;                      // programmatic dependent launch of the iteration kernels
    const int32_t* sched2;            // K2 scheduled static walk: unit list (NULL = dynamic tickets)
    const int32_t* soff2;             // [g_k2 + 1] offsets of each block's list
    const int32_t* sched3;            // same for K3
    const int32_t* soff3;
    int32_t sched_max;                // longest list (shared memory per block)
    int64_t sched_u0;                 // units [sched_u0, U) come from the dynamic ticket
    int32_t landskip;
    int32_t dia_q;                    // FSAI DIA form: diagonals per factor (0 = ELL path)
    const double* dia;                // [dia_q][nel] chain coefficients (see internal.h Plan::dia)                 // K2/K3 (dynamic): land / padding lanes issue no memory traffic
    const uint32_t* ocean;            // [nloc][nbx][kWarps] ocean bit masks (bit l: column 32w + l)
    int32_t precond;                  // pcg_precond
    int64_t nel;                      // owned elements nloc * pitch
    const double *cE, *cN, *sigma, *diag, *piv;
    EllDev zt, z;                     // rows of Z^T (K2) and of Z (K3)
    int64_t nel_all;                  // elements of every per-point array, halo rows included
    int32_t periodic;
    double *x, *b, *q, *t, *s;
    double *r[2], *d[2];
    double* partial[3];
    double* gath;                     // nranks * 4 gathered rank sums (multi-rank)
    DevScalars* sc;
    double* hist;
    int32_t hist_cap;
    int32_t multi;                    // 1: reductions end at rank sums (NCCL path)
    int32_t use_cond;
    cudaGraphConditionalHandle cond;
    // Redundant-sum mode (one rank, K1 / K2 / K3 launches): no last-block tails; every block of the
    // consumer kernel forms the canonical final sum it needs (K1: (s, r) -> beta, K2: (d, q) ->
    // alpha) and K3's block 0 does the history / stop test from K2's (r, r) at its start.
    int32_t redundant;
    int32_t red_gamma;                // Jacobi / none (one rank): K1 without a last block, K2's blocks form (d, q)
    int32_t cgcg;                     // Chronopoulos-Gear single-reduction PCG (NEXT-2; KA, K3, KC)
    double* p;                        // its search direction p (s = A p lives in d[0] / d[1], w in q, u in s)
    // Pipelined PCG (NEXT-2, Ghysels-Vanroose Alg. 4; KPA / KPB / KPC): u in s, w in q, r in r[0],
    // p in p, s = A p in d[0]; z = A q, q = P s and m = P w in their own arrays (n = A m is formed
    // in KPC's registers and never stored)
    int32_t pipe;
    double *pz, *pq, *pm;
    void* l2_base;                    // persisting L2 access-policy window of the iteration kernels
    size_t l2_bytes;                  // (0: none)
    float l2_ratio;
    RsDev rs;                         // resident-strip driver (rs.on = 0: not used)
    // device comm (PCG_FLAG_DEVICE_COMM, dev_comm.cuh): the last block of each reduction gathers
    // the rank sums through the NCCL window itself and runs the scalar step inline
    char* const* dc_peer;             // [nranks] window base of every rank (device pointers)
    uint32_t* dc_seq;                 // this rank's reduction counter (persists across solves)
    int32_t dc;
    int32_t rank;                     // this rank (multi-rank path)
    int32_t dch;                      // device comm with halo stores: K3 / k2_diag write s's first / last
    double* dch_south;                //   owned row into rank-1's northern / rank+1's southern halo row
    double* dch_north;                //   (peer pointers into the window; null at the ends)
    // K1 bulk-copy form (k1_tma_kernel; one rank): strips of kK1W columns x chunks of k1t_rows rows
    int32_t k1tma, k1t_strips, k1t_rows, g_k1t;
    int32_t kfin;                     // one rank, large grids: reduction tails in kfin_kernel (no last blocks)
};

int64_t grid_blocks(const KArgs& A);

#ifdef __CUDACC__
// history entry k (kept only while k < hist_cap) and the last value (always)
template <class KA>
__device__ __forceinline__ void put_hist(const KA& A, int k, double h) {
    if (k < A.hist_cap) A.hist[k] = h;
    A.sc->hlast = h;
}
#endif

// per-iteration kernels (par = iteration parity; init = the a3 pass with alpha = 0)
void launch_k1(const KArgs& A, int par, cudaStream_t st);
void launch_k2_ainv(const KArgs& A, int par, int init, cudaStream_t st);
void launch_k3_ainv(const KArgs& A, int par, int init, cudaStream_t st);
void launch_k2_diag(const KArgs& A, int par, int init, int none, cudaStream_t st);
void launch_kc(const KArgs& A, int par, int init, cudaStream_t st);   // CG-CG: w = A u, (w, u), alpha / beta
// pipelined PCG: KPA t = Dhat^-1 Z^T w (+ the pending reduction's scalars, one rank); KPB m = Z t;
// KPC n = A m, the eight vector updates, (r,u) (w,u) (r,r)  (init: w = A u and the three dots)
void launch_kpa(const KArgs& A, cudaStream_t st);
void launch_kfin(const KArgs& A, int which, cudaStream_t st);   // 0: (d, q) -> red[0]; 1: (s, r) -> fin_iter
void launch_kpb(const KArgs& A, cudaStream_t st);
void launch_kpc(const KArgs& A, int init, cudaStream_t st);
// solve prologue / epilogue
void launch_prep(const KArgs& A, cudaStream_t st);
void launch_init_residual(const KArgs& A, cudaStream_t st);       // r0 = b - A x0 -> r[1], (b,b)
void launch_fin(const KArgs& A, cudaStream_t st);                 // pending x update / b = 0
void launch_true_residual(const KArgs& A, cudaStream_t st);       // ||b - A x|| / ||b||
void launch_apply(const KArgs& A, const double* x_arr, double* y_arr, cudaStream_t st);   // y = A x
// multi-rank scalar steps (one thread) after an allgather of DevScalars::loc
enum ScalarStep : int32_t { kSsBB = 0, kSsGamma = 1, kSsInit = 2, kSsIter = 3, kSsTrue = 4,
                            kSsCgInit = 5, kSsCgIter = 6,     // Chronopoulos-Gear: (delta, gamma, rr) at once
                            kSsPipe = 7 };                    // pipelined: (gamma, delta, rr) -> alpha, beta
void launch_scalar(const KArgs& A, int step, cudaStream_t st);
void launch_set_cond(cudaGraphConditionalHandle h, cudaStream_t st);
void launch_extrapolate(const double* xt, const double* xm, double* x0, int64_t n, cudaStream_t st);
void configure_kernels(KArgs& A, int sms);
cudaError_t launch_loop(const KArgs& A, cudaStream_t st);   // whole PCG loop, cooperative (1 rank)
cudaError_t launch_rs(const KArgs& A, cudaStream_t st);     // whole PCG loop, resident strips (rs.cu)
const void* rs_kernel_fn(const KArgs& A);                  // the rs kernel a launch_rs call uses
int rs_timeline(unsigned long long* out, int nblk);       // -DRS_TIMELINE builds: pass durations
size_t rs_smem_bytes(int32_t cap, int32_t maxu1, int32_t maxu2, int32_t maxnx);   // dynamic smem of rs_loop_kernel

}  // namespace pcg
