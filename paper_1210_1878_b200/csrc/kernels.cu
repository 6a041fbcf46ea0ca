// kernels.cu -- the per-iteration CUDA kernels of libpcg for sm_100a (fp64, no tensor cores:
// the path is HBM-bound, ~0.17 flop/byte).
//
// One PCG iteration (Alg. 1, with d = s + beta d, R6) is three
// launches, each streaming its arrays once and ending in a deterministic reduction:
//   K1  d = s + beta d_old ; x += alpha_prev d_old ; q = A d ; partial (d, q)          Alg.1 l.6, l.8
//   K2  alpha = rho/(d,q) ; r = r - alpha q ; t = Dhat^-1 Z^T r ; partial (r, r)      l.6-7
//   K3  s = Z t ; partial (s, r) ; beta, history, convergence flag                      l.7
// (Jacobi / no preconditioner: K2 also forms s = r/A_pp or s = r and K3 is skipped.)
//
// ARITHMETIC ORDER (DESIGN.md §5 -- reproduced bit for bit by the oracle's canonical mode):
//   * every expression uses __fma_rn/__dmul_rn/__dadd_rn/__ddiv_rn/__dsqrt_rn, so nvcc's
//     contraction cannot change it;
//   * stencil: A_pp = ((c_E + c_W) + c_N) + c_S (+ sigma); acc = A_pp x_p, then
//     acc = fma(-c, x_nb, acc) for W, E, S, N;
//   * Z / Z^T rows: acc = 0, fma over the stored entries in ascending column order (ELL slots,
//     then overflow); K2 then divides by Dhat;
//   * updates: x = fma(alpha, d, x); r = fma(-alpha, q, r); d = fma(beta, d_old, s);
//   * dot products: one partial per (grid row, 256-column segment) = block tree of the 256
//     values fl(a*b) (shuffle-down tree 16,8,4,2,1 per warp, then the same tree over the 8 warp
//     sums), stored at row*nbx + segment; the last block to finish sums partials t, t+256, ...
//     left to right per thread and applies the block tree.  This order does not depend on
//     how kernels map blocks to rows.
//
// EXECUTION SHAPE: every reduction kernel is persistent -- gridDim = SMs x resident blocks --
// and walks its units (row segments; K1: strips of rpb rows) north to south with a block
// stride, keeping each unit's 8 warp sums in shared memory.  A block publishes its partials and
// takes its ticket on the completion counter once, at the end: a per-unit fence + atomic would
// stall every short-lived block (measured: ~15 us per kernel at ORCA025, profiles/r01).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "internal.h"
#include "kernels.h"
#include "dev_common.cuh"
#include "dev_comm.cuh"

namespace pcg {

namespace {

// After thread 0 wrote this block's partials: count the block, report whether it is last.
__device__ __forceinline__ bool count_block(uint32_t* counter) {
    __shared__ bool am_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        // acq_rel at gpu scope: releases this block's partials (written by thread 0) and, in the
        // last block, acquires every other block's; one L2 round trip instead of fence + atomic
        uint32_t t;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(counter) : "memory");
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return am_last;
}

#ifndef PCG_RED_NB
#define PCG_RED_NB 12                // partial loads in flight per thread in the redundant sums
                                     // (8: 81.0, 12: 80.5, 16: 84.7 us/iteration at cfg4 -- spills)
#endif
// final_sum in every thread of the block (redundant-sum mode: each block of the consumer kernel
// forms the same canonical sum, bitwise)
template <int NB>
__device__ __forceinline__ double final_sum_all(const double* partial, int64_t G) {
    __shared__ double bc;
    const double v = final_sum<NB>(partial, G);
    if (threadIdx.x == 0) bc = v;
    __syncthreads();
    const double r = bc;
    __syncthreads();
    return r;
}

// tree over the per-rank sums in rank order, zero padded to 32
// (u[l] += u[l + off] for off = 16, 8, 4, 2, 1, as warp_tree).  Evaluated depth first: leaf t of
// the in-order walk is rank bitrev5(t), and after leaf t the stack merges (left + right) once per
// trailing one bit of t -- the same additions with the same operands, in 6 live registers instead
// of 32, so the reduction kernels that run it in their last block keep their register budget.
__device__ __forceinline__ double rank_tree(const double* gath, int nranks, int slot) {
    double st[6];
    int sp = 0;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
        const int l = (int)(__brev((unsigned)t) >> 27);
        double v = l < nranks ? gath[l * 4 + slot] : 0.0;
#pragma unroll
        for (int c = t; c & 1; c >>= 1) v = __dadd_rn(st[--sp], v);
        st[sp++] = v;
    }
    return st[0];
}

template <class KA>
__device__ __forceinline__ void set_cond(const KA& A, int v) {
    if (A.use_cond) cudaGraphSetConditional(A.cond, (unsigned)v);
}

template <class KA>
__device__ __forceinline__ void stop(const KA& A, int status) {
    DevScalars* sc = A.sc;
    sc->status = status;
    sc->active = 0;
    set_cond(A, 0);
}

// Programmatic dependent launch (PDL): an iteration kernel is launched while its predecessor
// drains; griddepcontrol.wait blocks until the predecessor has completed and its writes are
// visible (a no-op for a normal launch), launch_dependents lets the successor's blocks start as
// soon as every block of this kernel has finished its units.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Diagnostic build only (-DPCG_TIMELINE): per-block globaltimer stamps of the last launch of K1/K2/K3
// (slot 0 entry, 1 after griddepcontrol.wait, 2 before the block count, 3 last block done).
#ifdef PCG_TIMELINE
__device__ unsigned long long g_timeline[3][2048][8];
__device__ unsigned g_units[2048];
__device__ unsigned long long g_tail[3][4];
#define TT(kk, slot) \
    if (threadIdx.x == 0) g_tail[kk][slot] = gtimer()
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TL(kk, slot) \
    if (threadIdx.x == 0 && blockIdx.x < 2048) g_timeline[kk][blockIdx.x][slot] = gtimer()
#else
#define TL(kk, slot) ((void)0)
#define TT(kk, slot) ((void)0)
#endif

// The flag only changes between launches (or in the last block of a reduction, after every
// other block has read it), so a cached read is exact.
__device__ __forceinline__ bool is_active(const KArgs& A) { return __ldg(&A.sc->active) != 0; }

// multi-rank scalar step after the rank sums are gathered (scalar_kernel; inline with device comm)
template <class KA>
__device__ void scalar_step(const KA& A, int step);
// The fields of KArgs the scalar steps use.  The device-comm tails below run in the last block of
// a reduction kernel; as out-of-line calls on this small view they cost the kernels' main loops
// no registers (inlined, or called with the whole KArgs, they made K1 / K2 / K3 spill).
struct SArgs {
    DevScalars* sc;
    double* gath;
    double* hist;
    char* const* dc_peer;
    uint32_t* dc_seq;
    int32_t hist_cap, nranks, rank, use_cond;
    cudaGraphConditionalHandle cond;
};
__device__ __forceinline__ SArgs sargs(const KArgs& A) {
    return SArgs{A.sc, A.gath, A.hist, A.dc_peer, A.dc_seq, A.hist_cap, A.nranks, A.rank, A.use_cond, A.cond};
}
// device comm: gather this rank's DevScalars::loc from every rank into gath, then the scalar step
__device__ __noinline__ void dc_reduce(const SArgs S, int step) {
    dc_allgather(S.dc_peer, S.nranks, S.rank, S.dc_seq, S.sc->loc, S.gath);
    scalar_step(S, step);
}
__device__ __noinline__ void dc_publish_loc(const SArgs S) { dc_publish(S.dc_peer, S.nranks, S.rank, S.dc_seq, S.sc->loc); }
__device__ __noinline__ void dc_collect_step(const SArgs S, int step) {
    dc_collect(S.dc_peer, S.nranks, S.rank, S.dc_seq, S.gath);
    scalar_step(S, step);
}


// ---- scalar updates (one thread) --------------------------------------------------------
template <class KA>
__device__ void fin_bb(const KA& A, double bb) {
    DevScalars* sc = A.sc;
    sc->nb = __dsqrt_rn(bb);
    sc->bzero = sc->nb == 0.0;
    sc->alpha = 0.0; sc->beta = 0.0; sc->k = 0; sc->status = kStOk; sc->xpend = 0;
    sc->pstage = 0;
    sc->active = 1;                       // provisional: decided after s0 (fin_init)
}

template <class KA>
__device__ void fin_init(const KA& A, double rho0, double rr0) {
    DevScalars* sc = A.sc;
    if (sc->bzero) {
        put_hist(A, 0, 0.0);
        sc->active = 0;
        set_cond(A, 0);
        return;
    }
    sc->rho = rho0;
    sc->beta = 0.0;
    sc->rho_prev = INFINITY;                 // beta of the first iteration = rho / inf = +0 (d_old = 0)
    const double h = __ddiv_rn(__dsqrt_rn(rr0), sc->nb);
    put_hist(A, 0, h);
    if (!isfinite(h)) {                      // NaN / Inf in b or x0: breakdown before the first iteration
        stop(A, kStBreakdown);
        return;
    }
    const int act = (h > sc->tol) && (sc->maxit > 0);
    sc->active = act;
    set_cond(A, act);
}

// Scalars fin_iter reads, loaded by the last block's thread 0 before its final sum so the loads
// overlap the partial walk instead of following it.
struct FinPre {
    double rr, rho, nb, tol, h;
    int32_t k, maxit;
};

template <class KA>
__device__ __forceinline__ FinPre fin_prefetch(const KA& A) {
    const DevScalars* sc = A.sc;
    FinPre f;
    f.rr = sc->red[2];
    f.h = sc->hpre;
    f.rho = sc->rho;
    f.nb = sc->nb;
    f.tol = sc->tol;
    f.k = sc->k;
    f.maxit = sc->maxit;
    return f;
}

template <class KA>
__device__ void fin_iter(const KA& A, double rho_new, const FinPre& f) {
    DevScalars* sc = A.sc;
    const int k = f.k + 1;
    sc->k = k;
    if (!isfinite(rho_new) || !isfinite(f.rr)) {
        put_hist(A, k, NAN);
        stop(A, kStBreakdown);
        return;
    }
    sc->rho_prev = f.rho;                    // beta = rho_new / rho is formed by K1 (same IEEE division)
    sc->rho = rho_new;
    const double h = f.h;
    put_hist(A, k, h);
    const int act = (h > f.tol) && (k < f.maxit);
    sc->active = act;
    TT(2, 2);
    set_cond(A, act);
    TT(2, 3);
}

template <class KA>
__device__ void fin_iter(const KA& A, double rho_new, double rr) {
    FinPre f = fin_prefetch(A);
    f.rr = rr;
    f.h = __ddiv_rn(__dsqrt_rn(rr), f.nb);
    fin_iter(A, rho_new, f);
}

// alpha of the current iteration from the global (d, q); false on breakdown
__device__ __forceinline__ bool get_alpha(const KArgs& A, int init, double& alpha) {
    if (init) { alpha = 0.0; return true; }
    const double gamma = A.sc->red[0];
    if (!(gamma > 0.0) || !isfinite(gamma)) return false;
    alpha = __ddiv_rn(A.sc->rho, gamma);
    return true;
}

// ---- units -----------------------------------------------------------------------------------
// A unit is one 256-column segment bx of one owned row j; unit u runs from the north
// (j = nloc-1 - u/nbx) so the long Z rows near the pole start first.  Its partial index is
// m = j*nbx + bx whatever block computes it.
struct Unit {
    int32_t i, j, bx;
    bool valid, inrow;     // i < ni ; i < pitch
    bool live;             // the thread computes this point (inrow; ocean only with A.landskip)
    int64_t a;             // array index of (i, j)
};

__device__ __forceinline__ int64_t n_units(const KArgs& A) { return (int64_t)A.nloc * A.nbx; }

__device__ __forceinline__ Unit unit_of(const KArgs& A, int64_t u) {
    Unit W;
    W.bx = (int32_t)(u % A.nbx);
    W.j = A.nloc - 1 - (int32_t)(u / A.nbx);
    W.i = W.bx * kBlock + (int32_t)threadIdx.x;
    W.valid = W.i < A.ni;
    W.inrow = W.i < A.pitch;
    W.live = W.inrow;
    W.a = (int64_t)(W.j + A.halo) * A.pitch + W.i;
    return W;
}

// device comm with halo stores: a point of the first / last owned row also goes to the
// neighbour's halo row (NVLink store into its window); before the block's completion count, a
// system-scope fence orders the block's stores before the count -> the last block's stamp ->
// the neighbour's acquire of it, so the neighbour's next K1 reads them
__device__ __forceinline__ void dc_halo_store(const KArgs& A, const Unit& W, double v) {
    if (!A.dch) return;
    if (W.j == 0 && A.dch_south) A.dch_south[W.i] = v;
    if (W.j == A.nloc - 1 && A.dch_north) A.dch_north[W.i] = v;
}
__device__ __forceinline__ void dc_halo_fence(const KArgs& A) {
    if (!A.dch) return;
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

// warp sum of v for local slot k (shared memory ws[k][warp])
__device__ __forceinline__ void put_warp_sum(double* ws, int k, double v) {
    v = warp_tree(v);
    if ((threadIdx.x & 31) == 0) ws[k * kWarps + (threadIdx.x >> 5)] = v;
}

// End of a persistent row kernel: warp 0 turns the stored warp sums of every unit this block
// processed into the unit partials (second level of the block tree), then the block takes its
// completion ticket.  NV = number of dot products (slots k*NV + n).
template <int NV>
__device__ __forceinline__ bool finish_units(const KArgs& A, const double* ws, double* p0, double* p1,
                                             uint32_t* counter) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int64_t U = n_units(A);
        int k = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k) {
            const int64_t m = (int64_t)(A.nloc - 1 - (int32_t)(u / A.nbx)) * A.nbx + (u % A.nbx);
#pragma unroll
            for (int n = 0; n < NV; ++n) {
                double w = lane < kWarps ? ws[(k * NV + n) * kWarps + lane] : 0.0;
                w = warp_tree(w);
                if (lane == 0) (n == 0 ? p0 : p1)[m] = w;
            }
        }
    }
    if (!counter) {                                        // partials only, no last block
        __syncthreads();
        return false;
    }
    return count_block(counter);
}

// Scheduled static variant (A.sched2/3): units [0, sched_u0) -- the northern rows, with the long
// pole rows -- are assigned at setup by longest-processing-time on a cost model (overflow rounds
// of the unit's slowest warp), heaviest first; block b walks sched[soff[b] .. soff[b+1]) with no
// ticket and no barrier per unit (each warp leaves its warp sum in shared memory and moves on; the
// block trees run once at the end, finish_sched).  The remaining units [sched_u0, U) are then
// taken from the dynamic ticket, which absorbs the cost model's error.
template <class Body>
__device__ __forceinline__ int sched_units(const KArgs& A, const int32_t* sched, const int32_t* soff, double* ws, Body body) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t k0 = soff[blockIdx.x], k1 = soff[blockIdx.x + 1];
#ifdef PCG_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 2048) g_timeline[sched == A.sched2 ? 1 : 2][blockIdx.x][7] = (unsigned long long)(k1 - k0);
#endif
    for (int32_t k = k0; k < k1; ++k) {
        Unit W = unit_of(A, sched[k]);
        if (A.landskip) W.live = W.inrow && ((__ldg(A.ocean + ((int64_t)W.j * A.nbx + W.bx) * kWarps + warp) >> lane) & 1u);
        double v = warp_tree(body(W));
        if (lane == 0) ws[(k - k0) * kWarps + warp] = v;
    }
    return k1 - k0;
}

__device__ __forceinline__ void finish_sched(const KArgs& A, const int32_t* sched, const int32_t* soff, const double* ws,
                                             double* partial) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int32_t k0 = soff[blockIdx.x], k1 = soff[blockIdx.x + 1];
        for (int32_t k = k0; k < k1; ++k) {
            const int64_t u = sched[k];
            const int64_t m = (int64_t)(A.nloc - 1 - (int32_t)(u / A.nbx)) * A.nbx + (u % A.nbx);
            double w = lane < kWarps ? ws[(k - k0) * kWarps + lane] : 0.0;
            w = warp_tree(w);
            if (lane == 0) partial[m] = w;
        }
    }
}

// Dynamic variant: units are handed out by an atomic ticket, so blocks that get slower memory do
// fewer units; each unit's partial is completed and stored right away (block tree over its 8 warp
// sums).  Same partials, same canonical order.  The ticket for the next unit is drawn when a unit
// starts and published to the block when it ends, so no warp waits on the atomic.  (Drawing two
// ahead was measured 25 % slower at ORCA025: consecutive tickets are neighbouring segments of the
// same long pole row, and one block then holds two of the slowest units.)
// With A.landskip each warp first loads the ocean bit mask of its 32 columns of the unit; lanes on
// land or padding then issue no memory traffic (their vector entries are zero and stay zero, so
// the partials are bitwise unchanged).
template <class Body>
__device__ __forceinline__ void dynamic_units(const KArgs& A, unsigned long long* ticket, double* partial, Body body,
                                              int64_t u0 = 0) {
    __shared__ long long s_next;
    __shared__ double wsd[kWarps];
    const int64_t U = n_units(A);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(ticket, 1ull) + u0;
    __syncthreads();
    int64_t u = s_next;
#ifdef PCG_TIMELINE
    unsigned long long dyn_count = 0;
#endif
    while (u < U) {
        __syncthreads();                                   // everyone has read s_next
        unsigned long long tk = 0;
        if (threadIdx.x == 0) tk = atomicAdd(ticket, 1ull) + (unsigned long long)u0;
        Unit W = unit_of(A, u);
        if (A.landskip) W.live = W.inrow && ((__ldg(A.ocean + ((int64_t)W.j * A.nbx + W.bx) * kWarps + warp) >> lane) & 1u);
        double v = body(W);
        v = warp_tree(v);
        if (lane == 0) wsd[warp] = v;
        if (threadIdx.x == 0) s_next = (long long)tk;
        __syncthreads();
        if (warp == 0) {
            double w = lane < kWarps ? wsd[lane] : 0.0;
            w = warp_tree(w);
            if (lane == 0) partial[(int64_t)W.j * A.nbx + W.bx] = w;
        }
        u = s_next;
#ifdef PCG_TIMELINE
        if (threadIdx.x == 0 && blockIdx.x < 2048) { g_units[blockIdx.x] += 1; dyn_count += 1; }
#endif
    }
#ifdef PCG_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 2048) g_timeline[ticket == &A.sc->ticket[1] ? 1 : (ticket == &A.sc->ticket[2] ? 2 : 0)][blockIdx.x][6] = dyn_count;
#endif
}

// ---- K1: d = s + beta d_old ; x += alpha_prev d_old ; q = A d ; (d, q) --------------------
// Units are strips of rpb rows.  Each thread marches up its column: d at (i, j-1), (i, j),
// (i, j+1) stay in registers, E/W neighbours come from the adjacent lanes by shuffle (lanes at a
// warp edge and the two ends of a periodic row load them), and the loads of the next row are
// issued before the current row computes.  Per point: s, d_old, x, cE, cN read once; d, x, q
// written.
// One K1 strip (segment bx, rows [j0, j1)): leaves the per-row warp sums in wout[row][warp].
template <bool SIGMA>
__device__ __forceinline__ void k1_strip(const KArgs& A, int par, int64_t st, double beta, double alpha, double* wout) {
    const double* __restrict__ dold = A.d[par];
    double* __restrict__ dnew = A.d[par ^ 1];
    const double* __restrict__ s = A.s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t P = A.pitch, ni = A.ni;
    const int32_t nby = (A.nloc + A.rpb - 1) / A.rpb;
    const int32_t bx = (int32_t)(st % A.nbx), by = nby - 1 - (int32_t)(st / A.nbx);
    const int32_t i = bx * kBlock + (int32_t)threadIdx.x;
    const int32_t j0 = by * A.rpb, j1 = min(j0 + A.rpb, A.nloc);
    const bool valid = i < ni;
    const int32_t iw = i == 0 ? ni - 1 : i - 1, ie = i == ni - 1 ? 0 : i + 1;
    const bool ldw = valid && (lane == 0 || i == 0);
    const bool lde = valid && (lane == 31 || i == ni - 1);
    int64_t a = (int64_t)(j0 + A.halo) * P + i;
    double dS = 0.0, dC = 0.0, doC = 0.0, cNs = 0.0;
    double pdo = 0.0, ps = 0.0, pcE = 0.0, pcN = 0.0, px = 0.0;   // next row's loads
    if (valid) {
        dS = __fma_rn(beta, dold[a - P], s[a - P]);
        doC = dold[a];
        dC = __fma_rn(beta, doC, s[a]);
        cNs = fabs(A.cN[a - P]);
        if (j0 == 0) dnew[a - P] = dS;             // southern halo row (multi-rank)
        pdo = dold[a + P]; ps = s[a + P];
        pcE = A.cE[a]; pcN = A.cN[a]; px = A.x[a];
    }
    for (int32_t j = j0; j < j1; ++j, a += P) {
        const double doN = pdo, cEp = pcE, cNr = pcN, xv = px;
        const double dN = __fma_rn(beta, doN, ps);
        if (valid && j + 1 < j1) {
            pdo = dold[a + 2 * P]; ps = s[a + 2 * P];
            pcE = A.cE[a + P]; pcN = A.cN[a + P]; px = A.x[a + P];
        }
        double dW = __shfl_up_sync(kFull, dC, 1);
        double dE = __shfl_down_sync(kFull, dC, 1);
        double cEw = __shfl_up_sync(kFull, cEp, 1);
        if (ldw) {
            const int64_t aw = a - i + iw;
            dW = __fma_rn(beta, dold[aw], s[aw]);
            cEw = A.cE[aw];
        }
        if (lde) {
            const int64_t ae = a - i + ie;
            dE = __fma_rn(beta, dold[ae], s[ae]);
        }
        double v = 0.0;
        if (valid) {
            const bool land = signbit(cNr);
            const double cNp = fabs(cNr);
            double app = __dadd_rn(__dadd_rn(__dadd_rn(cEp, cEw), cNp), cNs);
            if (SIGMA) app = __dadd_rn(app, A.sigma[a]);
            double acc = __dmul_rn(app, dC);
            acc = __fma_rn(-cEw, dW, acc);
            acc = __fma_rn(-cEp, dE, acc);
            acc = __fma_rn(-cNs, dS, acc);
            acc = __fma_rn(-cNp, dN, acc);
            const double qv = land ? 0.0 : acc;
            dnew[a] = dC;
            A.q[a] = qv;
            A.x[a] = __fma_rn(alpha, doC, xv);
            v = __dmul_rn(dC, qv);
            cNs = cNp;
        }
        v = warp_tree(v);
        if (lane == 0) wout[(j - j0) * kWarps + warp] = v;
        dS = dC;
        dC = dN;
        doC = doN;
    }
    if (valid && j1 == A.nloc) dnew[a] = dC;       // northern halo row (multi-rank)
}

// beta of K1 (both K1 forms).  Redundant-sum mode: rho = (s, r) of K3's partials formed by every
// block, beta = rho / rho of the last iteration, block 0 keeps the books; false = breakdown (stop).
__device__ __forceinline__ bool k1_beta(const KArgs& A, int par, double& beta) {
    if (!A.redundant) {
        beta = __ddiv_rn(A.sc->rho, A.sc->rho_prev);
        return true;
    }
    const double rho = final_sum_all<PCG_RED_NB>(A.partial[2], n_units(A));
    if (!isfinite(rho)) {                                // fin_iter's breakdown on (s, r)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const int k = A.sc->k;
            put_hist(A, k, NAN);
            stop(A, kStBreakdown);
        }
        return false;
    }
    beta = __ddiv_rn(rho, A.sc->rhop[par ^ 1]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.sc->rhop[par] = rho;
        A.sc->rho = rho;
        A.sc->xpend = 0;                                   // this kernel does x += alpha_prev d_old
        A.sc->ticket[1] = 0;                               // K2's / K3's tickets (both finished)
        A.sc->ticket[2] = 0;
    }
    return true;
}

// End of every K1 form, after its partials are stored: who sums (d, q).  Redundant-sum mode: K2's
// blocks; Jacobi / none: k2_diag's blocks; otherwise the last block (rank sum on the NCCL path).
template <bool DC>
__device__ __forceinline__ void k1_tail(const KArgs& A) {
    if (A.redundant || A.kfin) return;                 // (d, q) is summed by K2's blocks / by kfin
    if (A.red_gamma) {                                 // Jacobi / none: k2_diag's blocks sum (d, q)
        if (blockIdx.x == 0 && threadIdx.x == 0) A.sc->xpend = 0;   // x += alpha_prev d_old done
        return;
    }
    if (count_block(&A.sc->counter[0])) {
        const double tot = final_sum(A.partial[0], n_units(A));
        if (threadIdx.x == 0) {
            if (A.multi) {
                A.sc->loc[0] = tot;
                if constexpr (DC) dc_reduce(sargs(A), kSsGamma);
            } else {
                A.sc->red[0] = tot;
            }
            A.sc->xpend = 0;
            A.sc->counter[0] = 0;
            A.sc->ticket[0] = 0;
        }
        TL(0, 3);
    }
}

#ifndef PCG_MINB_K1
#define PCG_MINB_K1 4
#endif
// DC (device comm, multi-rank only): the last block gathers the rank sums itself (dev_comm.cuh);
// a separate instantiation, so the one-rank kernels carry none of its code or registers
template <bool SIGMA, bool DC = false>
__global__ void __launch_bounds__(kBlock, PCG_MINB_K1) k1_kernel(const KArgs A, const int par) {
    TL(0, 0);
    pdl_wait();
    TL(0, 1);
    if (!is_active(A)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // safety net: the WHILE node ends even if a reduction never clears the flag
        if (++A.sc->guard > A.sc->maxit + 2) {
            A.sc->active = 0;
            A.sc->status = kStBreakdown;
            set_cond(A, 0);
        }
    }
    extern __shared__ double ws[];
    __shared__ double wrow[kMaxRowsK1][kWarps];
    __shared__ long long s_next;
    double beta;
    if (!k1_beta(A, par, beta)) return;
    const double alpha = A.sc->alpha;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t nby = (A.nloc + A.rpb - 1) / A.rpb;
    const int64_t S = (int64_t)nby * A.nbx;
    // strips come from an atomic ticket (A.dynamic_k1) or a block stride
    const bool dyn = A.dynamic_k1 != 0;
    int64_t st;
    if (dyn) {
        if (threadIdx.x == 0) s_next = (long long)atomicAdd(&A.sc->ticket[0], 1ull);
        __syncthreads();
        st = s_next;
    } else {
        st = blockIdx.x;
    }
    int kslot = 0;
    while (st < S) {
        if (dyn) {
            __syncthreads();                               // everyone has read s_next
            if (threadIdx.x == 0) s_next = (long long)atomicAdd(&A.sc->ticket[0], 1ull);
        }
        k1_strip<SIGMA>(A, par, st, beta, alpha, dyn ? &wrow[0][0] : &ws[kslot * kWarps]);
        const int32_t bx = (int32_t)(st % A.nbx), by = nby - 1 - (int32_t)(st / A.nbx);
        const int32_t j0 = by * A.rpb, j1 = min(j0 + A.rpb, A.nloc);
        if (dyn) {
            __syncthreads();
            if (warp == 0)                                 // row partials of this strip
                for (int32_t j = j0; j < j1; ++j) {
                    double w = lane < kWarps ? wrow[j - j0][lane] : 0.0;
                    w = warp_tree(w);
                    if (lane == 0) A.partial[0][(int64_t)j * A.nbx + bx] = w;
                }
            st = s_next;
        } else {
            st += gridDim.x;
            kslot += A.rpb;
        }
    }
    if (!dyn) {
        __syncthreads();
        if (threadIdx.x < 32) {
            kslot = 0;
            for (int64_t t2 = blockIdx.x; t2 < S; t2 += gridDim.x, kslot += A.rpb) {
                const int32_t bx = (int32_t)(t2 % A.nbx), by = nby - 1 - (int32_t)(t2 / A.nbx);
                const int32_t j0 = by * A.rpb, j1 = min(j0 + A.rpb, A.nloc);
                for (int32_t j = j0; j < j1; ++j) {
                    double w = lane < kWarps ? ws[(kslot + j - j0) * kWarps + lane] : 0.0;
                    w = warp_tree(w);
                    if (lane == 0) A.partial[0][(int64_t)j * A.nbx + bx] = w;
                }
            }
        }
    }
    pdl_trigger();
    TL(0, 2);
    k1_tail<DC>(A);
}

// ---- K1, bulk-copy (TMA) form: the HBM-bound grids (cfg5) --------------------------------------
// Each block owns one strip of kK1W columns of a chunk of rows and marches north through it.  One
// thread issues 1-D bulk copies (cp.async.bulk, SASS UBLKCP) of the next rows' segments of s,
// d_old, x, cE, cN (+ sigma) -- kK1W columns plus two halo columns each side, and for the strips
// that hold the periodic seam the row's element at the other end -- into a ring of kK1S stages
// signalled by mbarriers, so kK1S - 3 rows per block are in flight whatever the register budget.
// Geometry measured at cfg5 (K1 us per launch): 256 columns x 4 stages x 4 blocks per SM 154;
// 512 x 4 x 2 158; 512 x 5 x 2 158; 512 x 8 x 1 (256 threads) 229, (512 threads) 193; the
// 4-row strip kernel 205.  Row j is computed from stages j-1, j, j+1 entirely out of shared memory: d at
// the point and its four neighbours recomputed as fma(beta, d_old, s) (bitwise k1_strip's values),
// the canonical stencil, x += alpha d_old, and d, q, x stored with coalesced
// 256-byte warp stores.  The (row, 256-column segment) partials of (d, q) are the canonical block
// trees, as in every K1 form.
#ifndef PCG_K1T_W
#define PCG_K1T_W 256
#endif
#ifndef PCG_K1T_STAGES
#define PCG_K1T_STAGES 4
#endif
#ifndef PCG_K1T_THREADS
#define PCG_K1T_THREADS 256
#endif
#ifndef PCG_K1T_MINB
#define PCG_K1T_MINB 4
#endif
constexpr int kK1W = PCG_K1T_W;                    // strip width, a multiple of kBlock
constexpr int kK1S = PCG_K1T_STAGES;               // ring stages (>= 4)
constexpr int kK1T = PCG_K1T_THREADS;              // threads per block
constexpr int kK1Row = kK1W + 4;                   // staged doubles per row segment: halo 2 + 2
constexpr int kK1Seg = kK1W / kBlock;              // canonical segments per strip
static_assert(kK1W % kBlock == 0 && kK1S >= 4 && kK1W % kK1T == 0 && kK1T % 32 == 0, "K1 bulk-copy geometry");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}

template <int NA>
struct K1tSmem {
    double row[kK1S][NA][kK1Row];                  // staged row segments (element col0 - 2 + o at o)
    double seamW[kK1S][3][4];                      // west seam: s, d_old, cE of the 32-byte block holding ni-1
    double seamE[kK1S][2][4];                      // east seam: s, d_old of elements 0..3
    uint64_t full[kK1S];
    double wsum[2][kK1Seg][kWarps];
};
template <bool SIGMA>
size_t k1t_smem_bytes() { return sizeof(K1tSmem<SIGMA ? 6 : 5>); }

// stage t of a block: grid row r (owned numbering; -1 and nloc are the halo rows) of its strip
template <int NA>
__device__ __forceinline__ void k1t_fill(K1tSmem<NA>& S, int slot, const KArgs& A, int par, int32_t r, int32_t col0,
                                         int32_t lo, int32_t hi, int32_t seamW, int32_t seamE) {
    const int64_t base = (int64_t)(r + A.halo) * A.pitch;
    const unsigned nb = (unsigned)(hi - lo) * 8u;
    const unsigned seam_bytes = (seamW >= 0 ? 3u * 32u : 0u) + (seamE >= 0 ? 2u * 32u : 0u);
    mbar_expect_tx(&S.full[slot], (unsigned)NA * nb + seam_bytes);
    const double* src[6] = {A.s, A.d[par], A.x, A.cE, A.cN, A.sigma};
    const int off = lo - (col0 - 2);
#pragma unroll
    for (int v = 0; v < NA; ++v) bulk_g2s(&S.row[slot][v][off], src[v] + base + lo, nb, &S.full[slot]);
    if (seamW >= 0) {                              // 4 doubles (32-byte aligned) holding element ni-1
        bulk_g2s(S.seamW[slot][0], A.s + base + seamW, 32u, &S.full[slot]);
        bulk_g2s(S.seamW[slot][1], A.d[par] + base + seamW, 32u, &S.full[slot]);
        bulk_g2s(S.seamW[slot][2], A.cE + base + seamW, 32u, &S.full[slot]);
    }
    if (seamE >= 0) {                              // elements 0..3 (element 0 is the east neighbour of ni-1)
        bulk_g2s(S.seamE[slot][0], A.s + base, 32u, &S.full[slot]);
        bulk_g2s(S.seamE[slot][1], A.d[par] + base, 32u, &S.full[slot]);
    }
}

template <bool SIGMA>
__global__ void __launch_bounds__(kK1T, PCG_K1T_MINB) k1_tma_kernel(const KArgs A, const int par) {
    constexpr int NA = SIGMA ? 6 : 5;
    pdl_wait();
    if (!is_active(A)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (++A.sc->guard > A.sc->maxit + 2) {             // the WHILE node's safety net (k1_kernel)
            A.sc->active = 0;
            A.sc->status = kStBreakdown;
            set_cond(A, 0);
        }
    }
    extern __shared__ __align__(128) unsigned char k1t_raw[];
    K1tSmem<NA>& S = *reinterpret_cast<K1tSmem<NA>*>(k1t_raw);
    double beta;
    if (!k1_beta(A, par, beta)) return;
    const double alpha = A.sc->alpha;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t P = A.pitch, ni = A.ni;
    const int32_t c = blockIdx.x % A.k1t_strips, chunk = blockIdx.x / A.k1t_strips;
    const int32_t j0 = chunk * A.k1t_rows, j1 = min(j0 + A.k1t_rows, A.nloc);
    const int32_t col0 = c * kK1W, width = min(kK1W, P - col0);
    const int32_t lo = c == 0 ? col0 : col0 - 2;                    // staged columns [lo, hi)
    const int32_t hi = col0 + width == P ? P : col0 + width + 2;
    const int32_t seamW = (c == 0) ? ((ni - 1) & ~3) : -1;          // 32-byte block holding ni - 1
    const int32_t seamE = (ni - 1 >= col0 && ni - 1 < col0 + width) ? 0 : -1;
    const int32_t R = j1 - j0 + 2;                                  // staged rows j0-1 .. j1
    double* __restrict__ dnew = A.d[par ^ 1];
    if (j0 < j1) {
        if (tid == 0) {
            for (int s = 0; s < kK1S; ++s) mbar_init(&S.full[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int t = 0; t < min(kK1S, R); ++t) k1t_fill<NA>(S, t, A, par, j0 - 1 + t, col0, lo, hi, seamW, seamE);
        }
        __syncthreads();
        mbar_wait(&S.full[0], 0);
        mbar_wait(&S.full[1], 0);
        for (int32_t j = j0; j < j1; ++j) {
            const int t = j - j0;                                    // stages t (row j-1), t+1 (j), t+2 (j+1)
            const int sS = t % kK1S, sC = (t + 1) % kK1S, sN = (t + 2) % kK1S;
            mbar_wait(&S.full[sN], (unsigned)((t + 2) / kK1S) & 1u);
            const int64_t arow = (int64_t)(j + A.halo) * P;
#pragma unroll
            for (int k = 0; k < kK1W / kK1T; ++k) {
                const int32_t ic = k * kK1T + tid;                   // column within the strip
                const int32_t i = col0 + ic;
                double v = 0.0;
                if (ic < width && i < ni) {
                    const int o = ic + 2;
                    const double doC = S.row[sC][1][o];
                    const double dC = __fma_rn(beta, doC, S.row[sC][0][o]);
                    const double dS = __fma_rn(beta, S.row[sS][1][o], S.row[sS][0][o]);
                    const double dN = __fma_rn(beta, S.row[sN][1][o], S.row[sN][0][o]);
                    double dW, dE, cEw;
                    if (i == 0) {
                        const int q = (ni - 1) & 3;
                        dW = __fma_rn(beta, S.seamW[sC][1][q], S.seamW[sC][0][q]);
                        cEw = S.seamW[sC][2][q];
                    } else {
                        dW = __fma_rn(beta, S.row[sC][1][o - 1], S.row[sC][0][o - 1]);
                        cEw = S.row[sC][3][o - 1];
                    }
                    if (i == ni - 1) dE = __fma_rn(beta, S.seamE[sC][1][0], S.seamE[sC][0][0]);
                    else dE = __fma_rn(beta, S.row[sC][1][o + 1], S.row[sC][0][o + 1]);
                    const double cEp = S.row[sC][3][o];
                    const double cNr = S.row[sC][4][o];
                    const double cNs = fabs(S.row[sS][4][o]);
                    const bool land = signbit(cNr);
                    const double cNp = fabs(cNr);
                    double app = __dadd_rn(__dadd_rn(__dadd_rn(cEp, cEw), cNp), cNs);
                    if constexpr (SIGMA) app = __dadd_rn(app, S.row[sC][5][o]);
                    double acc = __dmul_rn(app, dC);
                    acc = __fma_rn(-cEw, dW, acc);
                    acc = __fma_rn(-cEp, dE, acc);
                    acc = __fma_rn(-cNs, dS, acc);
                    acc = __fma_rn(-cNp, dN, acc);
                    const double qv = land ? 0.0 : acc;
                    const int64_t a = arow + i;
                    dnew[a] = dC;
                    A.q[a] = qv;
                    A.x[a] = __fma_rn(alpha, doC, S.row[sC][2][o]);
                    v = __dmul_rn(dC, qv);
                }
                v = warp_tree(v);
                if (lane == 0) S.wsum[j & 1][ic >> 8][(ic & (kBlock - 1)) >> 5] = v;   // canonical (segment, warp)
            }
            __syncthreads();                                         // stage t is free; warp sums of row j
            if (tid == 0 && t + kK1S < R) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                k1t_fill<NA>(S, sS, A, par, j0 - 1 + t + kK1S, col0, lo, hi, seamW, seamE);
            }
            if (warp == 0) {
#pragma unroll
                for (int k = 0; k < kK1Seg; ++k) {
                    const int32_t seg = c * kK1Seg + k;
                    double w = lane < kWarps ? S.wsum[j & 1][k][lane] : 0.0;
                    w = warp_tree(w);
                    if (lane == 0 && seg < A.nbx) A.partial[0][(int64_t)j * A.nbx + seg] = w;
                }
            }
        }
    }
    pdl_trigger();
    k1_tail<false>(A);                                     // one rank only (no halo-row stores)
}

#ifndef PCG_MINB_K1F
#define PCG_MINB_K1F 4           // 64 registers: no spills (6 blocks/SM spilled and ran slower)
#endif
// ---- K1, row-segment form: one element per thread, units from the dynamic ticket ----------------
// Same arithmetic as k1_strip (bitwise): d at the point and at its S/N neighbours recomputed from
// s and d_old, E/W neighbours by shuffle (warp-edge lanes and the periodic seam load them).
// loads of one K1 point (row-segment form), issued before any of its arithmetic
struct K1Ld {
    double doC, sC, dSo, sS, dNo, sN, cEp, cNr, cNs, xv;
};
__device__ __forceinline__ void k1_load(const KArgs& A, const Unit& W, int par, K1Ld& L) {
    const double* __restrict__ dold = A.d[par];
    const double* __restrict__ s = A.s;
    const int64_t a = W.a, P = A.pitch;
    if (W.valid) {
        L.doC = dold[a]; L.sC = s[a];
        L.dSo = dold[a - P]; L.sS = s[a - P]; L.dNo = dold[a + P]; L.sN = s[a + P];
        L.cEp = A.cE[a]; L.cNr = A.cN[a]; L.cNs = A.cN[a - P]; L.xv = A.x[a];
    } else {
        L.doC = L.sC = L.dSo = L.sS = L.dNo = L.sN = L.cEp = L.cNr = L.cNs = L.xv = 0.0;
    }
}

// arithmetic and stores of one K1 point from its loads
template <bool SIGMA>
__device__ __forceinline__ double k1_compute(const KArgs& A, const Unit& W, int par, double beta, double alpha, const K1Ld& L) {
    const double* __restrict__ dold = A.d[par];
    double* __restrict__ dnew = A.d[par ^ 1];
    const double* __restrict__ s = A.s;
    const int lane = threadIdx.x & 31;
    const int32_t P = A.pitch, ni = A.ni, i = W.i;
    const bool valid = W.valid;
    const int64_t a = W.a;
    double dC = 0.0, dS = 0.0, dN = 0.0, doC = 0.0, cEp = 0.0, cNr = 0.0, cNs = 0.0, xv = 0.0;
    if (valid) {
        doC = L.doC;
        cEp = L.cEp; cNr = L.cNr; cNs = fabs(L.cNs); xv = L.xv;
        dC = __fma_rn(beta, doC, L.sC);
        dS = __fma_rn(beta, L.dSo, L.sS);
        dN = __fma_rn(beta, L.dNo, L.sN);
    }
    double dW = __shfl_up_sync(kFull, dC, 1);
    double dE = __shfl_down_sync(kFull, dC, 1);
    double cEw = __shfl_up_sync(kFull, cEp, 1);
    if (valid && (lane == 0 || i == 0)) {
        const int64_t aw = a - i + (i == 0 ? ni - 1 : i - 1);
        dW = __fma_rn(beta, dold[aw], s[aw]);
        cEw = A.cE[aw];
    }
    if (valid && (lane == 31 || i == ni - 1)) {
        const int64_t ae = a - i + (i == ni - 1 ? 0 : i + 1);
        dE = __fma_rn(beta, dold[ae], s[ae]);
    }
    if (!valid) return 0.0;
    const bool land = signbit(cNr);
    const double cNp = fabs(cNr);
    double app = __dadd_rn(__dadd_rn(__dadd_rn(cEp, cEw), cNp), cNs);
    if (SIGMA) app = __dadd_rn(app, A.sigma[a]);
    double acc = __dmul_rn(app, dC);
    acc = __fma_rn(-cEw, dW, acc);
    acc = __fma_rn(-cEp, dE, acc);
    acc = __fma_rn(-cNs, dS, acc);
    acc = __fma_rn(-cNp, dN, acc);
    const double qv = land ? 0.0 : acc;
    dnew[a] = dC;
    A.q[a] = qv;
    A.x[a] = __fma_rn(alpha, doC, xv);
    if (W.j == 0) dnew[a - P] = dS;                     // halo rows (multi-rank)
    if (W.j == A.nloc - 1) dnew[a + P] = dN;
    return __dmul_rn(dC, qv);
}

// K1, row-segment form: one element per thread, units from the dynamic ticket or a block stride.
// Same arithmetic as k1_strip (bitwise): d at the point and at its S/N neighbours recomputed from
// s and d_old, E/W neighbours by shuffle (warp-edge lanes and the periodic seam load them).
template <bool SIGMA>
__device__ __forceinline__ double k1_point(const KArgs& A, const Unit& W, int par, double beta, double alpha) {
    K1Ld L;
    k1_load(A, W, par, L);
    return k1_compute<SIGMA>(A, W, par, beta, alpha, L);
}

template <bool SIGMA, bool DC = false>
__global__ void __launch_bounds__(kBlock, PCG_MINB_K1F) k1_flat_kernel(const KArgs A, const int par) {
    pdl_wait();
    if (!is_active(A)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (++A.sc->guard > A.sc->maxit + 2) {          // safety net for the WHILE node
            A.sc->active = 0;
            A.sc->status = kStBreakdown;
            set_cond(A, 0);
        }
    }
    double beta;
    const double alpha = A.sc->alpha;
    if (!k1_beta(A, par, beta)) return;
    if (A.red_gamma && !A.redundant && blockIdx.x == 0 && threadIdx.x == 0)
        A.sc->xpend = 0;                                   // this kernel does x += alpha_prev d_old
    bool last;
    if (A.redundant || A.red_gamma) {                      // (d, q) is formed by K2's blocks
        extern __shared__ double ws[];
        const int64_t U = n_units(A);
        int k = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k)
            put_warp_sum(ws, k, k1_point<SIGMA>(A, unit_of(A, u), par, beta, alpha));
        pdl_trigger();
        finish_units<1>(A, ws, A.partial[0], nullptr, nullptr);
        return;
    } else if (A.k1flat == 2) {
        // static block stride, no barrier per unit: warp sums in shared memory, trees at the end
        extern __shared__ double ws[];
        const int64_t U = n_units(A);
        int k = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k)
            put_warp_sum(ws, k, k1_point<SIGMA>(A, unit_of(A, u), par, beta, alpha));
        pdl_trigger();
        last = finish_units<1>(A, ws, A.partial[0], nullptr, A.kfin ? nullptr : &A.sc->counter[0]);
    } else {
        dynamic_units(A, &A.sc->ticket[0], A.partial[0], [&](const Unit& W) { return k1_point<SIGMA>(A, W, par, beta, alpha); });
        pdl_trigger();
        last = A.kfin ? false : count_block(&A.sc->counter[0]);
    }
    if (last) {
        const double tot = final_sum(A.partial[0], n_units(A));
        if (threadIdx.x == 0) {
            if (A.multi) {
                A.sc->loc[0] = tot;
                if constexpr (DC) dc_reduce(sargs(A), kSsGamma);
            } else {
                A.sc->red[0] = tot;
            }
            A.sc->xpend = 0;
            A.sc->counter[0] = 0;
            A.sc->ticket[0] = 0;
        }
    }
}

// ---- ELL(4) + overflow row sums ---------------------------------------------
// The first kEll entries of a row sit at fixed slots (no offset load) and store the gathered
// point's array index, so all column/value loads issue together with the thread's other loads
// and a gather is one address add.  Entries beyond kEll come from the overflow SELL (empty for
// ~80% of slices), one at a time.  Accumulation: acc = fma(z, x, acc) over the ELL slots then the
// overflow entries -- ascending column order; padding (value 0, own index) contributes 0.
static_assert(kEll == 4, "ell_row loads the 4 ELL slots as one int4 and one 256-bit double vector");

// Overflow entries of a long row (near the pole: up to ~80 at ORCA025), continuing the fma chain.
// Four entries per round, the next round's column/value loads issued before this round's
// gathers, so a long row costs about one L2 round trip per 4 entries -- a plain loop is two
// dependent memory latencies per entry, and those pole warps set the kernel time.
template <class Gather>
__device__ __forceinline__ double overflow_sum(const EllDev& E, int64_t e, double acc, Gather gat) {
#ifdef PCG_DIAG_NOOVF
    return acc;
#endif
    const int64_t sl = e >> 5;
    const int64_t o0 = __ldg(E.ooff + sl);
    const int L = (int)((__ldg(E.ooff + sl + 1) - o0) >> 5);
    if (L == 0) return acc;
    const int32_t* cp = E.ocol + o0 + (e & 31);
    const double* vp = E.oval + o0 + (e & 31);
    int32_t cn[4];
    double zn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t m = (int64_t)min(u, L - 1) << 5;
        cn[u] = __ldg(cp + m);
        zn[u] = __ldg(vp + m);
    }
    for (int m0 = 0; m0 < L; m0 += 4) {
        int32_t c[4];
        double z[4], x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { c[u] = cn[u]; z[u] = zn[u]; }
        if (m0 + 4 < L) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t m = (int64_t)min(m0 + 4 + u, L - 1) << 5;
                cn[u] = __ldg(cp + m);
                zn[u] = __ldg(vp + m);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = gat(c[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = __fma_rn(m0 + u < L ? z[u] : 0.0, x[u], acc);
    }
    return acc;
}

template <class Gather>
__device__ __forceinline__ double ell_row(const EllDev& E, int64_t e, Gather gat) {
    double z[kEll], x[kEll];
    const int4 cv = __ldg(reinterpret_cast<const int4*>(E.col) + e);
    ld_nc_f64x4(E.val + e * kEll, z);
#ifdef PCG_DIAG_NOGATHER
    const int32_t c[kEll] = {(int32_t)(e + 32), (int32_t)(e + 32), (int32_t)(e + 32), (int32_t)(e + 32)};
#else
    const int32_t c[kEll] = {cv.x, cv.y, cv.z, cv.w};
#endif
#pragma unroll
    for (int m = 0; m < kEll; ++m) x[m] = gat(c[m]);
    // schedule pin (emits nothing): the fma chain may only start once all four gathers have
    // returned, so ptxas issues them back to back instead of one gather per fma.
    asm volatile("" : "+d"(x[0]), "+d"(x[1]), "+d"(x[2]), "+d"(x[3]));
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < kEll; ++m) acc = __fma_rn(z[m], x[m], acc);
    return overflow_sum(E, e, acc, gat);
}

// ---- FSAI in DIA form (NEXT-1, A.dia_q > 0): the factor's entries are chains
// along grid rows, dia[m-1][e] = zhat between owned elements e - m and e.  Same entries, same
// ascending-column fma order as the ELL row (zero slots are skipped, exactly like absent
// entries).  Q >= dia_q is the compile-time width: all coefficient loads, then all gathers,
// then the fma chain, so a row costs one load latency and one gather latency.
// Z^T row of element e (for K2): columns e-M .. e-1, then the unit diagonal.
template <int Q, class Gather>
__device__ __forceinline__ double dia_zt_row(const KArgs& A, const Unit& W, double xself, Gather gat) {
    const int64_t e = W.a - A.hoff;
    double z[Q], x[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m)
        z[m] = (m < A.dia_q && W.i > m) ? __ldg(A.dia + (int64_t)m * A.nel + e) : 0.0;
#pragma unroll
    for (int m = 0; m < Q; ++m) x[m] = z[m] != 0.0 ? gat(W.a - (m + 1)) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int m = Q - 1; m >= 0; --m)
        if (z[m] != 0.0) acc = __fma_rn(z[m], x[m], acc);
    return __fma_rn(1.0, xself, acc);
}
// Z row of element e (for K3): the unit diagonal, then columns e+1 .. e+M (chain order).
template <int Q>
__device__ __forceinline__ double dia_z_row(const KArgs& A, const Unit& W, const double* __restrict__ t) {
    const int64_t e = W.a - A.hoff;
    double z[Q], x[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m)
        z[m] = (m < A.dia_q && W.i + m + 1 < A.ni) ? __ldg(A.dia + (int64_t)m * A.nel + e + m + 1) : 0.0;
    const double xs = __ldg(t + W.a);
#pragma unroll
    for (int m = 0; m < Q; ++m) x[m] = z[m] != 0.0 ? __ldg(t + W.a + m + 1) : 0.0;
    double acc = __fma_rn(1.0, xs, 0.0);
#pragma unroll
    for (int m = 0; m < Q; ++m)
        if (z[m] != 0.0) acc = __fma_rn(z[m], x[m], acc);
    return acc;
}

// ELL row with int16 slot offsets (DQ = -1 kernels): one 8-byte column load per element instead
// of 16; the gathered array index is the element's own index plus the offset.  Same entries and
// order as ell_row.
template <class Gather>
__device__ __forceinline__ double ell_row16(const EllDev& E, int64_t e, int64_t self, Gather gat) {
    double z[kEll], x[kEll];
    const uint2 cw = __ldg(reinterpret_cast<const uint2*>(E.col16) + e);
    ld_nc_f64x4(E.val + e * kEll, z);
    const int32_t s = (int32_t)self;
    const int32_t c[kEll] = {s + (int32_t)(int16_t)(cw.x & 0xffffu), s + (int32_t)(int16_t)(cw.x >> 16),
                             s + (int32_t)(int16_t)(cw.y & 0xffffu), s + (int32_t)(int16_t)(cw.y >> 16)};
#pragma unroll
    for (int m = 0; m < kEll; ++m) x[m] = gat(c[m]);
    asm volatile("" : "+d"(x[0]), "+d"(x[1]), "+d"(x[2]), "+d"(x[3]));
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < kEll; ++m) acc = __fma_rn(z[m], x[m], acc);
    return overflow_sum(E, e, acc, gat);
}

#ifndef PCG_MINB_K2
#define PCG_MINB_K2 4            // register budgets: resident 256-thread blocks per SM ptxas targets
#endif
#ifndef PCG_MINB_K3
#define PCG_MINB_K3 5
#endif

#ifndef PCG_FINAL_NB_K3
#define PCG_FINAL_NB_K3 8            // measured: 93.4 -> 92.0 us/iteration vs 32 (fewer spills in K3)
#endif
// K2 has no last block: its (r, r) is first needed by the convergence test at the end of K3.
// K3's block 0 forms that final sum as soon as K2 has completed (K2's partials are still in L2),
// while the other blocks stream; k3_finish (K3's last block) then forms K3's own (s, r), does
// K2's bookkeeping (alpha for the pending x update, ticket / counter reset) and fin_init /
// fin_iter.  Block 0's store of (r, r) precedes its release in count_block, so the last block
// (which acquires there) reads it.
__device__ __forceinline__ void k3_sum_rr(const KArgs& A, int init) {
    if (blockIdx.x != 0) return;
    const double rr = final_sum<PCG_FINAL_NB_K3>(A.partial[1], n_units(A));
    if (A.redundant) {
        // redundant-sum mode: the history value and the stop test need only (r, r), so block 0
        // does fin_init / fin_iter's bookkeeping here; the (s, r) breakdown test moves to K1
        if (threadIdx.x == 0) {
            DevScalars* sc = A.sc;
            sc->red[2] = rr;
            const double h = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
            sc->hpre = h;
            if (init) {
                sc->rhop[1] = INFINITY;                  // beta of the first iteration = rho / inf = +0
                sc->rho_prev = INFINITY;
                if (sc->bzero) {
                    put_hist(A, 0, 0.0);
                    sc->active = 0;
                    set_cond(A, 0);
                } else if (!isfinite(h)) {                 // NaN / Inf in b or x0
                    put_hist(A, 0, h);
                    stop(A, kStBreakdown);
                } else {
                    put_hist(A, 0, h);
                    const int act = (h > sc->tol) && (sc->maxit > 0);
                    sc->active = act;
                    set_cond(A, act);
                }
            } else {
                const int k = sc->k + 1;
                sc->k = k;
                if (!isfinite(rr)) {
                    put_hist(A, k, NAN);
                    stop(A, kStBreakdown);
                } else {
                    put_hist(A, k, h);
                    const int act = (h > sc->tol) && (k < sc->maxit);
                    sc->active = act;
                    set_cond(A, act);
                }
            }
        }
        return;
    }
    if (threadIdx.x == 0) {
        DevScalars* sc = A.sc;
        if (A.multi) {
            sc->loc[2] = rr;
        } else {
            // everything of fin that does not depend on K3's own sum, off the last block's path:
            // the history value h and K2's alpha (same IEEE operations as in fin_iter / get_alpha)
            sc->red[2] = rr;
            sc->hpre = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
        }
        if (!A.cgcg) {                                   // CG-CG: alpha / beta come from KC, x is updated in KA
            sc->alpha = init ? 0.0 : __ddiv_rn(sc->rho, sc->red[0]);   // K2 checked gamma > 0
            sc->xpend = init ? 0 : 1;
        }
    }
}

template <bool DC>
__device__ __forceinline__ void k3_finish(const KArgs& A, int init) {
    TT(2, 0);
    FinPre pre{};
    if (threadIdx.x == 0) pre = fin_prefetch(A);       // independent of the walk: overlaps it
    const double rs = final_sum<PCG_FINAL_NB_K3>(A.partial[2], n_units(A));
    TT(2, 1);
    if (threadIdx.x == 0) {
        DevScalars* sc = A.sc;
        sc->counter[1] = 0;
        sc->ticket[1] = 0;
        sc->counter[2] = 0;
        sc->ticket[2] = 0;
        if (A.multi) {
            sc->loc[1] = rs;
            if constexpr (DC) {
                if (!A.cgcg) dc_reduce(sargs(A), init ? kSsInit : kSsIter);   // CG-CG: gathered after KC
            }
        } else if (init) {
            fin_init(A, rs, pre.rr);
        } else {
            fin_iter(A, rs, pre);
        }
    }
}

// ---- K2 (AINV): r -= alpha q ; t = Dhat^-1 Z^T r ; (r, r) --------------------------------
// r_new at a gathered point c is recomputed as fma(-alpha, q_c, r_old_c) (bitwise the value
// its own thread stores), so no grid-wide barrier is needed between the update and the gather.
template <int DQ>
__global__ void __launch_bounds__(kBlock, PCG_MINB_K2) k2_ainv_kernel(const KArgs A, const int par, const int init) {
    TL(1, 0);
    pdl_wait();
    TL(1, 1);
    if (!is_active(A)) return;
    double alpha;
    if (A.redundant) {
        // alpha = rho / (d, q), (d, q) from K1's partials formed by every block
        alpha = 0.0;
        if (!init) {
            const double gamma = final_sum_all<PCG_RED_NB>(A.partial[0], n_units(A));
            if (!(gamma > 0.0) || !isfinite(gamma)) {
                if (blockIdx.x == 0 && threadIdx.x == 0) stop(A, kStBreakdown);
                return;
            }
            alpha = __ddiv_rn(A.sc->rhop[par], gamma);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            A.sc->alpha = alpha;                           // the pending x update of the next K1 / fin
            A.sc->xpend = init ? 0 : 1;
        }
    } else if (!get_alpha(A, init, alpha)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) stop(A, kStBreakdown);
        return;
    }
    extern __shared__ double ws[];
    const double* __restrict__ ro = A.r[par];
    double* __restrict__ rn = A.r[par ^ 1];
    const double* __restrict__ q = A.q;
    auto body = [&](const Unit& W) {
        double v = 0.0;
        if (W.live) {
            const double rnew = __fma_rn(-alpha, q[W.a], ro[W.a]);
            const double pv = A.piv[W.a];
            auto gat = [&](int64_t g) { return __fma_rn(-alpha, __ldg(q + g), __ldg(ro + g)); };
            double acc;
            if constexpr (DQ > 0) acc = dia_zt_row<DQ>(A, W, rnew, gat);
            else if constexpr (DQ < 0) acc = ell_row16(A.zt, W.a - A.hoff, W.a, gat);
            else acc = ell_row(A.zt, W.a - A.hoff, gat);
            A.t[W.a] = __ddiv_rn(acc, pv);
            rn[W.a] = rnew;
            v = __dmul_rn(rnew, rnew);
        }
        return v;
    };
    if (A.sched2) {
        sched_units(A, A.sched2, A.soff2, ws, body);
        TL(1, 4);
        finish_sched(A, A.sched2, A.soff2, ws, A.partial[1]);
        TL(1, 5);
        dynamic_units(A, &A.sc->ticket[1], A.partial[1], body, A.sched_u0);
        pdl_trigger();
        TL(1, 2);
    } else if (A.dynamic) {
        dynamic_units(A, &A.sc->ticket[1], A.partial[1], body);
        pdl_trigger();
        TL(1, 2);
    } else {
        const int64_t U = n_units(A);
        int k = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k) put_warp_sum(ws, k, body(unit_of(A, u)));
        finish_units<1>(A, ws, A.partial[1], nullptr, nullptr);
        pdl_trigger();
    }
}

// ---- KA (Chronopoulos-Gear, NEXT-2): p = u + beta p ; s = w + beta s ; x += alpha p ;
// r -= alpha s ; t = Dhat^-1 Z^T r ; (r, r).  u lives in A.s, w in A.q, s = A p in d[par] (old) /
// d[par^1] (new).  r_new at a gathered point is recomputed as fma(-alpha, fma(beta, s_old, w),
// r_old) -- bitwise what its own thread stores -- so no barrier separates the update and the
// gather.  alpha, beta are KC's.  Same units, walks and partials as K2.
__global__ void __launch_bounds__(kBlock, PCG_MINB_K2) ka_cg_kernel(const KArgs A, const int par) {
    pdl_wait();
    if (!is_active(A)) return;
    const double alpha = A.sc->alpha, beta = A.sc->beta;
    extern __shared__ double ws[];
    const double* __restrict__ ro = A.r[par];
    double* __restrict__ rn = A.r[par ^ 1];
    const double* __restrict__ so = A.d[par];
    double* __restrict__ sn = A.d[par ^ 1];
    const double* __restrict__ w = A.q;
    auto body = [&](const Unit& W) {
        double v = 0.0;
        if (W.live) {
            const int64_t a = W.a;
            const double pn = __fma_rn(beta, A.p[a], A.s[a]);
            const double svn = __fma_rn(beta, so[a], w[a]);
            A.x[a] = __fma_rn(alpha, pn, A.x[a]);
            const double rnew = __fma_rn(-alpha, svn, ro[a]);
            A.p[a] = pn;
            sn[a] = svn;
            auto gat = [&](int64_t g) { return __fma_rn(-alpha, __fma_rn(beta, __ldg(so + g), __ldg(w + g)), __ldg(ro + g)); };
            const double acc = A.zt.col16 ? ell_row16(A.zt, a - A.hoff, a, gat) : ell_row(A.zt, a - A.hoff, gat);
            A.t[a] = __ddiv_rn(acc, A.piv[a]);
            rn[a] = rnew;
            v = __dmul_rn(rnew, rnew);
        }
        return v;
    };
    if (A.sched2) {
        sched_units(A, A.sched2, A.soff2, ws, body);
        finish_sched(A, A.sched2, A.soff2, ws, A.partial[1]);
        dynamic_units(A, &A.sc->ticket[1], A.partial[1], body, A.sched_u0);
    } else {
        dynamic_units(A, &A.sc->ticket[1], A.partial[1], body);
    }
    pdl_trigger();
}

// ---- K3 (AINV): s = Z t ; (s, r) ; beta / history / flag -----------------------------------
template <int DQ, bool DC = false>
__global__ void __launch_bounds__(kBlock, PCG_MINB_K3) k3_ainv_kernel(const KArgs A, const int par, const int init) {
    TL(2, 0);
    pdl_wait();
    TL(2, 1);
    if (!is_active(A)) return;
    k3_sum_rr(A, init);
    extern __shared__ double ws[];
    const double* __restrict__ rn = A.r[par ^ 1];
    const double* __restrict__ t = A.t;
    auto body = [&](const Unit& W) {
        double v = 0.0;
        if (W.live) {
            const double rv = rn[W.a];
            double acc;
            if constexpr (DQ > 0) acc = dia_z_row<DQ>(A, W, t);
            else if constexpr (DQ < 0) acc = ell_row16(A.z, W.a - A.hoff, W.a, [&](int32_t g) { return __ldg(t + g); });
            else acc = ell_row(A.z, W.a - A.hoff, [&](int32_t g) { return __ldg(t + g); });
            A.s[W.a] = acc;
            if constexpr (DC) dc_halo_store(A, W, acc);
            v = __dmul_rn(acc, rv);
        }
        return v;
    };
    bool last;
    if (A.sched3) {
        sched_units(A, A.sched3, A.soff3, ws, body);
        TL(2, 4);
        finish_sched(A, A.sched3, A.soff3, ws, A.partial[2]);
        TL(2, 5);
        dynamic_units(A, &A.sc->ticket[2], A.partial[2], body, A.sched_u0);
        pdl_trigger();
        TL(2, 2);
        if (A.redundant || (A.kfin && !init)) return;    // (s, r) is summed by the next K1's blocks / kfin
        if constexpr (DC) dc_halo_fence(A);
        last = count_block(&A.sc->counter[2]);
    } else if (A.dynamic) {
        dynamic_units(A, &A.sc->ticket[2], A.partial[2], body);
        pdl_trigger();
        TL(2, 2);
        if (A.redundant || (A.kfin && !init)) return;
        if constexpr (DC) dc_halo_fence(A);
        last = count_block(&A.sc->counter[2]);
    } else {
        const int64_t U = n_units(A);
        int k = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k) put_warp_sum(ws, k, body(unit_of(A, u)));
        if constexpr (DC) dc_halo_fence(A);
        last = finish_units<1>(A, ws, A.partial[2], nullptr, (A.redundant || (A.kfin && !init)) ? nullptr : &A.sc->counter[2]);
    }
    if (last) {
        k3_finish<DC>(A, init);
        TL(2, 3);
    }
}

// ---- kfin: the reduction tails of the large grids (cfg5, one rank, PCG_KFIN) ----------------------
// At cfg5 a reduction has 52 k partials; the last block of K1 / K3 walks them with 256 threads
// and few loads in flight (~15 us per reduction), and the redundant-sum mode makes every block of
// the consumer read all of them (L2-bound).  kfin is one block of 1024 threads between the
// kernels: all threads load a window of partials into shared memory (24 loads each in flight),
// then threads t < 256 add their chains t, t + 256, ... from shared memory in order -- the
// canonical final sum of DESIGN.md §5.2, bitwise -- and thread 0 does the last block's scalars.
#ifndef PCG_KFIN_WIN
#define PCG_KFIN_WIN 24576                           // doubles per window (192 KB), a multiple of 256
#endif
constexpr int kKfinT = 1024;
constexpr int kKfinWin = PCG_KFIN_WIN;
static_assert(kKfinWin % kBlock == 0 && kKfinWin % kKfinT == 0, "kfin window");

__device__ __forceinline__ double kfin_sum(const double* partial, int64_t G, double* win) {
    double acc = 0.0;
    for (int64_t w0 = 0; w0 < G; w0 += kKfinWin) {
        const int n = (int)((G - w0) < kKfinWin ? (G - w0) : kKfinWin);
        double v[kKfinWin / kKfinT];
#pragma unroll
        for (int u = 0; u < kKfinWin / kKfinT; ++u) {
            const int k = threadIdx.x + u * kKfinT;
            v[u] = k < n ? __ldcg(partial + w0 + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kKfinWin / kKfinT; ++u) {
            const int k = threadIdx.x + u * kKfinT;
            if (k < n) win[k] = v[u];
        }
        __syncthreads();
        if (threadIdx.x < kBlock)
            for (int m = threadIdx.x; m < n; m += kBlock) acc = __dadd_rn(acc, win[m]);
        __syncthreads();
    }
    return block_tree(acc);                                  // threads >= 256 add nothing
}

// which = 0: (d, q) after K1 -> red[0] (K2 forms alpha); which = 1: (s, r) after K3 -> fin_iter
__global__ void __launch_bounds__(kKfinT, 1) kfin_kernel(const KArgs A, const int which) {
    pdl_wait();
    if (!is_active(A)) return;
    extern __shared__ double kfin_win[];
    DevScalars* sc = A.sc;
    if (which == 0) {
        const double tot = kfin_sum(A.partial[0], n_units(A), kfin_win);
        if (threadIdx.x == 0) {
            sc->red[0] = tot;
            sc->xpend = 0;                                   // K1 did x += alpha_prev d_old
            sc->counter[0] = 0;
            sc->ticket[0] = 0;
        }
    } else {
        FinPre pre{};
        if (threadIdx.x == 0) pre = fin_prefetch(A);
        const double rs = kfin_sum(A.partial[2], n_units(A), kfin_win);
        if (threadIdx.x == 0) {
            sc->counter[1] = 0;
            sc->ticket[1] = 0;
            sc->counter[2] = 0;
            sc->ticket[2] = 0;
            fin_iter(A, rs, pre);
        }
    }
    pdl_trigger();
}

// final_sum over two partial arrays in one walk (each sum in final_sum's order: bitwise the same)
template <int NB>
__device__ __forceinline__ void final_sum_pair(const double* pa, const double* pb, int64_t G, double& ra, double& rb) {
    double aa = 0.0, ab = 0.0;
    int64_t m = threadIdx.x < kBlock ? (int64_t)threadIdx.x : G;
    for (; m < G; m += NB * kBlock) {
        double p[NB], q[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const bool in = m + u * kBlock < G;
            p[u] = in ? __ldcg(pa + m + u * kBlock) : 0.0;
            q[u] = in ? __ldcg(pb + m + u * kBlock) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NB; ++u)
            if (m + u * kBlock < G) { aa = __dadd_rn(aa, p[u]); ab = __dadd_rn(ab, q[u]); }
    }
    ra = block_tree(aa);
    rb = block_tree(ab);
}

// ---- the whole PCG loop as one cooperative persistent kernel (single rank) ---------------------
// Phases K1 | K2 | K3 of each iteration are separated by grid barriers; every block then forms
// the global sums itself (same canonical final sum, so every block holds bitwise the same α, β,
// ρ, h and takes the same branch).  No launches, no WHILE node and no last-block tails per
// iteration.  Block 0 records the history and, at exit, the scalars the epilogue reads.
__device__ __forceinline__ double block_final(const double* partial, int64_t G) {
    __shared__ double bcast;
    const double v = final_sum(partial, G);
    if (threadIdx.x == 0) bcast = v;
    __syncthreads();
    const double r = bcast;
    __syncthreads();
    return r;
}

// dynamic units with two dot products per unit (Jacobi / none)
template <class Body>
__device__ __forceinline__ void dynamic_units2(const KArgs& A, unsigned long long* ticket, double* p1, double* p2,
                                               Body body) {
    __shared__ long long s_next2;
    __shared__ double w1[kWarps], w2[kWarps];
    const int64_t U = n_units(A);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_next2 = (long long)atomicAdd(ticket, 1ull);
    __syncthreads();
    int64_t u = s_next2;
    while (u < U) {
        __syncthreads();
        if (threadIdx.x == 0) s_next2 = (long long)atomicAdd(ticket, 1ull);
        const Unit W = unit_of(A, u);
        double v1, v2;
        body(W, v1, v2);
        v1 = warp_tree(v1);
        v2 = warp_tree(v2);
        if (lane == 0) { w1[warp] = v1; w2[warp] = v2; }
        __syncthreads();
        if (warp == 0) {
            double a = lane < kWarps ? w1[lane] : 0.0, b = lane < kWarps ? w2[lane] : 0.0;
            a = warp_tree(a);
            b = warp_tree(b);
            if (lane == 0) { p1[(int64_t)W.j * A.nbx + W.bx] = a; p2[(int64_t)W.j * A.nbx + W.bx] = b; }
        }
        u = s_next2;
    }
}

// Units of a phase: block b takes unit b when there are no more units than blocks (no ticket
// round trips -- the small-grid, latency-bound case), otherwise dynamic tickets.
template <class Body>
__device__ __forceinline__ void phase_units(const KArgs& A, unsigned long long* ticket, double* partial, Body body) {
    const int64_t U = n_units(A);
    if (U <= (int64_t)gridDim.x) {
        __shared__ double wst[kWarps];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if ((int64_t)blockIdx.x < U) {
            const Unit W = unit_of(A, blockIdx.x);
            double v = warp_tree(body(W));
            if (lane == 0) wst[warp] = v;
            __syncthreads();
            if (warp == 0) {
                double w = lane < kWarps ? wst[lane] : 0.0;
                w = warp_tree(w);
                if (lane == 0) partial[(int64_t)W.j * A.nbx + W.bx] = w;
            }
        }
    } else {
        dynamic_units(A, ticket, partial, body);
    }
}

template <class Body>
__device__ __forceinline__ void phase_units2(const KArgs& A, unsigned long long* ticket, double* p1, double* p2,
                                             Body body) {
    const int64_t U = n_units(A);
    if (U <= (int64_t)gridDim.x) {
        __shared__ double wa[kWarps], wb[kWarps];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if ((int64_t)blockIdx.x < U) {
            const Unit W = unit_of(A, blockIdx.x);
            double v1, v2;
            body(W, v1, v2);
            v1 = warp_tree(v1);
            v2 = warp_tree(v2);
            if (lane == 0) { wa[warp] = v1; wb[warp] = v2; }
            __syncthreads();
            if (warp == 0) {
                double a = lane < kWarps ? wa[lane] : 0.0, b = lane < kWarps ? wb[lane] : 0.0;
                a = warp_tree(a);
                b = warp_tree(b);
                if (lane == 0) { p1[(int64_t)W.j * A.nbx + W.bx] = a; p2[(int64_t)W.j * A.nbx + W.bx] = b; }
            }
        }
    } else {
        dynamic_units2(A, ticket, p1, p2, body);
    }
}

__device__ __forceinline__ double k2_unit(const KArgs& A, const Unit& W, int par, double alpha) {
    if (!W.inrow) return 0.0;
    const double* __restrict__ ro = A.r[par];
    const double* __restrict__ q = A.q;
    const double rnew = __fma_rn(-alpha, q[W.a], ro[W.a]);
    const double pv = A.piv[W.a];
    auto gat = [&](int64_t g) { return __fma_rn(-alpha, __ldg(q + g), __ldg(ro + g)); };
    const double acc = A.dia_q > 8 ? dia_zt_row<16>(A, W, rnew, gat) : A.dia_q > 0 ? dia_zt_row<8>(A, W, rnew, gat)
                                                                                   : ell_row(A.zt, W.a - A.hoff, gat);
    A.t[W.a] = __ddiv_rn(acc, pv);
    A.r[par ^ 1][W.a] = rnew;
    return __dmul_rn(rnew, rnew);
}

__device__ __forceinline__ double k3_unit(const KArgs& A, const Unit& W, int par) {
    if (!W.inrow) return 0.0;
    const double* __restrict__ t = A.t;
    const double rv = A.r[par ^ 1][W.a];
    const double acc = A.dia_q > 8 ? dia_z_row<16>(A, W, t) : A.dia_q > 0 ? dia_z_row<8>(A, W, t)
                                   : ell_row(A.z, W.a - A.hoff, [&](int32_t g) { return __ldg(t + g); });
    A.s[W.a] = acc;
    return __dmul_rn(acc, rv);
}

#ifndef PCG_MINB_LOOP
#define PCG_MINB_LOOP 4
#endif

template <bool SIGMA>
__global__ void __launch_bounds__(kBlock, PCG_MINB_LOOP) loop_kernel(const KArgs A) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double wrow[kMaxRowsK1][kWarps];
    __shared__ long long s_next;
    DevScalars* sc = A.sc;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    double rho = sc->rho, beta = sc->beta, alpha = sc->alpha;
    const double nb = sc->nb, tol = sc->tol;
    int k = sc->k, status = sc->status, xpend = 0;
    const int maxit = sc->maxit;
    bool active = sc->active != 0;
    const int64_t U = n_units(A);
    const int32_t nby = (A.nloc + A.rpb - 1) / A.rpb;
    const int64_t S = (int64_t)nby * A.nbx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int par = 0;
    while (active) {
        // ---- K1: strips from ticket[0] (block b takes strip b when S <= gridDim)
        const bool st_static = S <= (int64_t)gridDim.x;
        int64_t st;
        if (st_static) {
            st = blockIdx.x;
        } else {
            if (threadIdx.x == 0) s_next = (long long)atomicAdd(&sc->ticket[0], 1ull);
            __syncthreads();
            st = s_next;
        }
        while (st < S) {
            if (!st_static) {
                __syncthreads();
                if (threadIdx.x == 0) s_next = (long long)atomicAdd(&sc->ticket[0], 1ull);
            }
            k1_strip<SIGMA>(A, par, st, beta, alpha, &wrow[0][0]);
            __syncthreads();
            if (warp == 0) {
                const int32_t bx = (int32_t)(st % A.nbx), by = nby - 1 - (int32_t)(st / A.nbx);
                const int32_t j0 = by * A.rpb, j1 = min(j0 + A.rpb, A.nloc);
                for (int32_t j = j0; j < j1; ++j) {
                    double w = lane < kWarps ? wrow[j - j0][lane] : 0.0;
                    w = warp_tree(w);
                    if (lane == 0) A.partial[0][(int64_t)j * A.nbx + bx] = w;
                }
            }
            st = st_static ? S : s_next;
        }
        xpend = 0;                                         // x += alpha_prev d_old done
        grid.sync();
        if (lead) sc->ticket[0] = 0;
        const double gamma = block_final(A.partial[0], U);
        if (!(gamma > 0.0) || !isfinite(gamma)) { status = kStBreakdown; break; }
        alpha = __ddiv_rn(rho, gamma);
        // ---- K2 (+ K3)
        if (A.precond == 0) {
            phase_units(A, &sc->ticket[1], A.partial[1], [&](const Unit& W) { return k2_unit(A, W, par, alpha); });
            grid.sync();
            if (lead) sc->ticket[1] = 0;
            phase_units(A, &sc->ticket[2], A.partial[2], [&](const Unit& W) { return k3_unit(A, W, par); });
            grid.sync();
            if (lead) sc->ticket[2] = 0;
        } else {
            const bool none = A.precond == 2;
            phase_units2(A, &sc->ticket[1], A.partial[1], A.partial[2], [&](const Unit& W, double& v1, double& v2) {
                v1 = 0.0;
                v2 = 0.0;
                if (!W.inrow) return;
                const double rnew = __fma_rn(-alpha, A.q[W.a], A.r[par][W.a]);
                const double sv = none ? rnew : __ddiv_rn(rnew, A.diag[W.a]);
                A.s[W.a] = sv;
                A.r[par ^ 1][W.a] = rnew;
                v1 = __dmul_rn(rnew, rnew);
                v2 = __dmul_rn(sv, rnew);
            });
            grid.sync();
            if (lead) sc->ticket[1] = 0;
        }
        const double rr = block_final(A.partial[1], U);
        const double rho_new = block_final(A.partial[2], U);
        k += 1;
        xpend = 1;
        if (!isfinite(rho_new) || !isfinite(rr)) {
            if (lead) put_hist(A, k, NAN);
            status = kStBreakdown;
            break;
        }
        beta = __ddiv_rn(rho_new, rho);
        rho = rho_new;
        const double h = __ddiv_rn(__dsqrt_rn(rr), nb);
        if (lead) put_hist(A, k, h);
        active = (h > tol) && (k < maxit);
        par ^= 1;
    }
    if (lead) {
        sc->k = k; sc->alpha = alpha; sc->beta = beta; sc->rho = rho;
        sc->xpend = xpend; sc->status = status; sc->active = 0;
    }
}

// ---- K2 (Jacobi / none): r -= alpha q ; s = r / A_pp (or r) ; (r, r), (s, r) ---------------
#ifndef KD2_UNROLL
#define KD2_UNROLL 2                 // measured at cfg4 (Jacobi): 1 / 2 / 4 / 8 -> 47.5 / 45.7 / 48.3 / 51.1 us/iteration
#endif
template <bool DC = false>
__global__ void __launch_bounds__(kBlock) k2_diag_kernel(const KArgs A, const int par, const int init,
                                                         const int none) {
    pdl_wait();
    if (!is_active(A)) return;
    double alpha;
    if (A.red_gamma && !init) {
        // (d, q) of K1's partials formed by every block (K1 has no last block); same IEEE alpha
        const double gamma = final_sum_all<PCG_RED_NB>(A.partial[0], n_units(A));
        if (!(gamma > 0.0) || !isfinite(gamma)) {
            if (blockIdx.x == 0 && threadIdx.x == 0) stop(A, kStBreakdown);
            return;
        }
        alpha = __ddiv_rn(A.sc->rho, gamma);
        if (blockIdx.x == 0 && threadIdx.x == 0) A.sc->red[0] = gamma;
    } else if (!get_alpha(A, init, alpha)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) stop(A, kStBreakdown);
        return;
    }
    extern __shared__ double ws[];
    const double* __restrict__ ro = A.r[par];
    double* __restrict__ rn = A.r[par ^ 1];
    const int64_t U = n_units(A), G = gridDim.x;
    // KD2_UNROLL units of the block stride at once: every unit's three loads are issued before
    // any unit computes (the body is too short to hide a memory latency per unit otherwise)
    constexpr int NU = KD2_UNROLL;
    int k = 0;
    for (int64_t u0 = blockIdx.x; u0 < U; u0 += NU * G, k += NU) {
        Unit W[NU];
        double qv[NU], rv[NU], dv[NU];
#pragma unroll
        for (int m = 0; m < NU; ++m) {
            const int64_t u = u0 + m * G;
            W[m] = unit_of(A, u < U ? u : u0);
            const bool ld = u < U && W[m].inrow;
            qv[m] = ld ? A.q[W[m].a] : 0.0;
            rv[m] = ld ? ro[W[m].a] : 0.0;
            dv[m] = (ld && !none) ? A.diag[W[m].a] : 1.0;
        }
#pragma unroll
        for (int m = 0; m < NU; ++m) {
            if (u0 + m * G >= U) break;
            double v1 = 0.0, v2 = 0.0;
            if (W[m].inrow) {
                const double rnew = __fma_rn(-alpha, qv[m], rv[m]);
                const double sv = none ? rnew : __ddiv_rn(rnew, dv[m]);
                A.s[W[m].a] = sv;
                if constexpr (DC) dc_halo_store(A, W[m], sv);
                rn[W[m].a] = rnew;
                v1 = __dmul_rn(rnew, rnew);
                v2 = __dmul_rn(sv, rnew);
            }
            put_warp_sum(ws, 2 * (k + m), v1);
            put_warp_sum(ws, 2 * (k + m) + 1, v2);
        }
    }
    pdl_trigger();
    if constexpr (DC) dc_halo_fence(A);
    if (finish_units<2>(A, ws, A.partial[1], A.partial[2], &A.sc->counter[1])) {
        double rr, rs;                                     // both walks in one pass (same sums)
        final_sum_pair<PCG_FINAL_NB_K3>(A.partial[1], A.partial[2], n_units(A), rr, rs);
        if (threadIdx.x == 0) {
            A.sc->counter[1] = 0;
            A.sc->alpha = alpha;
            A.sc->xpend = init ? 0 : 1;
            if (A.multi) {
                A.sc->loc[2] = rr; A.sc->loc[1] = rs;
                if constexpr (DC) dc_reduce(sargs(A), init ? kSsInit : kSsIter);
            }
            else if (init) fin_init(A, rs, rr);
            else fin_iter(A, rs, rr);
        }
    }
}

// ---- canonical stencil on a vector x (array layout): acc = A_pp x_p, fma(-c, x_nb) W,E,S,N ----
__device__ __forceinline__ double stencil(const KArgs& A, const double* __restrict__ x, int64_t a, int32_t i,
                                          bool& land) {
    const int64_t aw = i == 0 ? a + (A.ni - 1) : a - 1;
    const int64_t ae = i == A.ni - 1 ? a - (A.ni - 1) : a + 1;
    const int64_t as = a - A.pitch, an = a + A.pitch;
    const double cep = A.cE[a], cew = A.cE[aw];
    const double cnr = A.cN[a];
    land = signbit(cnr);
    const double cnp = fabs(cnr), cns = fabs(A.cN[as]);
    double app = __dadd_rn(__dadd_rn(__dadd_rn(cep, cew), cnp), cns);
    if (A.sigma) app = __dadd_rn(app, A.sigma[a]);
    double acc = __dmul_rn(app, x[a]);
    acc = __fma_rn(-cew, x[aw], acc);
    acc = __fma_rn(-cep, x[ae], acc);
    acc = __fma_rn(-cns, x[as], acc);
    acc = __fma_rn(-cnp, x[an], acc);
    return acc;
}

// alpha, beta of Chronopoulos-Gear from delta = (w, u) and gamma' = rho (one thread; fin_init /
// fin_iter has set rho, rho_prev and decided the stop test)
template <class KA>
__device__ void cg_alpha_beta(const KA& A, double delta, int init) {
    DevScalars* sc = A.sc;
    sc->red[0] = delta;
    const double gamma = sc->rho;
    double beta, den;
    if (init) {
        beta = 0.0;
        den = delta;
    } else {
        beta = __ddiv_rn(gamma, sc->rho_prev);
        den = __dadd_rn(delta, -__ddiv_rn(__dmul_rn(beta, gamma), sc->alpha));
    }
    if (!(den > 0.0) || !isfinite(den)) {
        stop(A, kStBreakdown);
        return;
    }
    sc->alpha = __ddiv_rn(gamma, den);
    sc->beta = beta;
}

// ---- KC (Chronopoulos-Gear, NEXT-2): w = A u ; (w, u) ; then alpha, beta -------------------
// The one reduction point of the iteration: K3 has formed gamma' = (u, r) (as rho, fin_iter)
// and (r, r); the last block here forms delta = (w, u) and beta = gamma'/gamma,
// alpha = gamma' / (delta - beta gamma' / alpha) (init: alpha = gamma/delta, beta = 0), with the
// breakdown test on the denominator.  Stencil in the canonical order of §5.3.
__global__ void __launch_bounds__(kBlock) kc_cg_kernel(const KArgs A, const int init) {
    pdl_wait();
    if (!is_active(A)) return;
    extern __shared__ double ws[];
    const int64_t U = n_units(A);
    int k = 0;
    for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k) {
        const Unit W = unit_of(A, u);
        double v = 0.0;
        if (W.valid) {
            bool land;
            const double ax = stencil(A, A.s, W.a, W.i, land);
            const double wv = land ? 0.0 : ax;
            A.q[W.a] = wv;
            v = __dmul_rn(wv, A.s[W.a]);
        }
        put_warp_sum(ws, k, v);
    }
    pdl_trigger();
    if (!finish_units<1>(A, ws, A.partial[0], nullptr, &A.sc->counter[0])) return;
    const double delta = final_sum(A.partial[0], U);
    if (threadIdx.x == 0) {
        A.sc->counter[0] = 0;
        if (A.multi) {                                   // rank sum: the allgather + kSsCg* follow
            A.sc->loc[0] = delta;
            if (A.dc) dc_reduce(sargs(A), init ? kSsCgInit : kSsCgIter);
        } else {
            cg_alpha_beta(A, delta, init);
        }
    }
}

// ---- pipelined PCG (NEXT-2; Ghysels-Vanroose Alg. 4, oracle orc_pcg_pipe) -------------------
// Per iteration: KPA t = Dhat^-1 Z^T w, KPB m = Z t (m = P w), KPC n = A m and
//   z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p,
//   x += alpha p, r -= alpha s, u -= alpha q, w -= alpha z, (r,u) (w,u) (r,r).
// The reduction KPC starts is not needed until the next KPC: one rank, KPA's block 0 forms the
// three canonical final sums and the scalars (history, stop test, alpha, beta) while the other
// blocks stream t; several ranks, the rank sums ride in the allgather fused with the m halo
// exchange after KPB.  Scalars: rho = gamma of the previous iteration, alpha = alpha_prev.
template <class KA>
__device__ void pipe_fin(const KA& A, double gamma, double delta, double rr) {
    DevScalars* sc = A.sc;
    const bool init = sc->pstage == 0;
    int k = 0;
    if (!init) {
        k = sc->k + 1;
        sc->k = k;
    }
    if (!isfinite(gamma) || !isfinite(delta) || !isfinite(rr)) {
        put_hist(A, k, init ? __ddiv_rn(__dsqrt_rn(rr), sc->nb) : NAN);
        stop(A, kStBreakdown);
        return;
    }
    const double h = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
    put_hist(A, k, h);
    if (!((h > sc->tol) && (k < sc->maxit))) {
        sc->active = 0;
        set_cond(A, 0);
        return;
    }
    double beta, den;
    if (init) {
        beta = 0.0;
        den = delta;
    } else {
        beta = __ddiv_rn(gamma, sc->rho);
        den = __dadd_rn(delta, -__ddiv_rn(__dmul_rn(beta, gamma), sc->alpha));
    }
    if (!(den > 0.0) || !isfinite(den) || !(gamma > 0.0)) {
        stop(A, kStBreakdown);
        return;
    }
    sc->alpha = __ddiv_rn(gamma, den);
    sc->beta = beta;
    sc->rho = gamma;
    sc->pstage = 1;
}

// units from the dynamic ticket, no reduction (the ticket is reset by the next KPC)
template <class Body>
__device__ __forceinline__ void ticket_units(const KArgs& A, unsigned long long* ticket, Body body) {
    __shared__ long long s_next;
    const int64_t U = n_units(A);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(ticket, 1ull);
    __syncthreads();
    int64_t u = s_next;
    while (u < U) {
        __syncthreads();                                   // everyone has read s_next
        unsigned long long tk = 0;
        if (threadIdx.x == 0) tk = atomicAdd(ticket, 1ull);
        Unit W = unit_of(A, u);
        if (A.landskip) W.live = W.inrow && ((__ldg(A.ocean + ((int64_t)W.j * A.nbx + W.bx) * kWarps + warp) >> lane) & 1u);
        body(W);
        if (threadIdx.x == 0) s_next = (long long)tk;
        __syncthreads();
        u = s_next;
    }
}

__global__ void __launch_bounds__(kBlock, PCG_MINB_K2) kpa_kernel(const KArgs A) {
    pdl_wait();
    if (!is_active(A)) return;
    if (A.multi && A.dc && blockIdx.x == 0) {          // device comm: the previous KPC's rank sums
        if (threadIdx.x == 0) {
            dc_collect_step(sargs(A), kSsPipe);
        }
        __syncthreads();
    }
    if (!A.multi && blockIdx.x == 0) {
        const int64_t U = n_units(A);
        const double g = final_sum<PCG_FINAL_NB_K3>(A.partial[0], U);
        const double dl = final_sum<PCG_FINAL_NB_K3>(A.partial[1], U);
        const double rr = final_sum<PCG_FINAL_NB_K3>(A.partial[2], U);
        if (threadIdx.x == 0) pipe_fin(A, g, dl, rr);
        __syncthreads();
    }
    const double* __restrict__ w = A.q;
    ticket_units(A, &A.sc->ticket[1], [&](const Unit& W) {
        if (W.live) {
            auto gat = [&](int32_t g) { return __ldg(w + g); };
            const double acc = A.zt.col16 ? ell_row16(A.zt, W.a - A.hoff, W.a, gat) : ell_row(A.zt, W.a - A.hoff, gat);
            A.t[W.a] = __ddiv_rn(acc, A.piv[W.a]);
        }
    });
    pdl_trigger();
}

__global__ void __launch_bounds__(kBlock, PCG_MINB_K3) kpb_kernel(const KArgs A) {
    pdl_wait();
    if (!is_active(A)) return;
    const double* __restrict__ t = A.t;
    ticket_units(A, &A.sc->ticket[2], [&](const Unit& W) {
        if (W.live) {
            auto gat = [&](int32_t g) { return __ldg(t + g); };
            A.pm[W.a] = A.z.col16 ? ell_row16(A.z, W.a - A.hoff, W.a, gat) : ell_row(A.z, W.a - A.hoff, gat);
        }
    });
    pdl_trigger();
}

// init: w = A u and the three dots of the prologue; otherwise the iteration's updates
__global__ void __launch_bounds__(kBlock) kpc_kernel(const KArgs A, const int init) {
    pdl_wait();
    if (!is_active(A)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {          // KPA / KPB have completed
        A.sc->ticket[1] = 0;
        A.sc->ticket[2] = 0;
    }
    extern __shared__ double ws[];
    const double alpha = A.sc->alpha, beta = A.sc->beta;
    double* __restrict__ r = A.r[0];
    double* __restrict__ u = A.s;
    double* __restrict__ w = A.q;
    const int64_t U = n_units(A);
    int k = 0;
    for (int64_t un = blockIdx.x; un < U; un += gridDim.x, ++k) {
        const Unit W = unit_of(A, un);
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        if (W.valid) {
            const int64_t a = W.a;
            bool land;
            if (init) {
                const double ax = stencil(A, u, a, W.i, land);
                const double wv = land ? 0.0 : ax;
                w[a] = wv;
                const double rv = r[a], uv = u[a];
                v0 = __dmul_rn(rv, uv);
                v1 = __dmul_rn(wv, uv);
                v2 = __dmul_rn(rv, rv);
            } else {
                const double nv = stencil(A, A.pm, a, W.i, land);
                if (!land) {
                    const double zn = __fma_rn(beta, A.pz[a], nv);
                    const double qn = __fma_rn(beta, A.pq[a], A.pm[a]);
                    const double sn = __fma_rn(beta, A.d[0][a], w[a]);
                    const double pn = __fma_rn(beta, A.p[a], u[a]);
                    A.x[a] = __fma_rn(alpha, pn, A.x[a]);
                    const double rv = __fma_rn(-alpha, sn, r[a]);
                    const double uv = __fma_rn(-alpha, qn, u[a]);
                    const double wv = __fma_rn(-alpha, zn, w[a]);
                    A.pz[a] = zn;
                    A.pq[a] = qn;
                    A.d[0][a] = sn;
                    A.p[a] = pn;
                    r[a] = rv;
                    u[a] = uv;
                    w[a] = wv;
                    v0 = __dmul_rn(rv, uv);
                    v1 = __dmul_rn(wv, uv);
                    v2 = __dmul_rn(rv, rv);
                }
            }
        }
        v0 = warp_tree(v0);
        v1 = warp_tree(v1);
        v2 = warp_tree(v2);
        if ((threadIdx.x & 31) == 0) {
            ws[(k * 3 + 0) * kWarps + (threadIdx.x >> 5)] = v0;
            ws[(k * 3 + 1) * kWarps + (threadIdx.x >> 5)] = v1;
            ws[(k * 3 + 2) * kWarps + (threadIdx.x >> 5)] = v2;
        }
    }
    pdl_trigger();
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        k = 0;
        for (int64_t un = blockIdx.x; un < U; un += gridDim.x, ++k) {
            const int64_t m = (int64_t)(A.nloc - 1 - (int32_t)(un / A.nbx)) * A.nbx + (un % A.nbx);
#pragma unroll
            for (int n = 0; n < 3; ++n) {
                double v = lane < kWarps ? ws[(k * 3 + n) * kWarps + lane] : 0.0;
                v = warp_tree(v);
                if (lane == 0) A.partial[n][m] = v;
            }
        }
    }
    if (!A.multi) return;                                // one rank: the next KPA's block 0 sums
    if (!count_block(&A.sc->counter[0])) return;
    const double g = final_sum(A.partial[0], U);
    const double dl = final_sum(A.partial[1], U);
    const double rr = final_sum(A.partial[2], U);
    if (threadIdx.x == 0) {
        A.sc->counter[0] = 0;
        A.sc->loc[0] = g;
        A.sc->loc[1] = dl;
        A.sc->loc[2] = rr;
        if (A.dc) dc_publish_loc(sargs(A));             // collected by the next KPA
    }
}

// prep: zero land entries of x and b (land is not an unknown, reading R20), zero d[0] everywhere
__global__ void __launch_bounds__(kBlock) prep_kernel(const KArgs A) {
    const int64_t n = (int64_t)(A.nloc + 2 * A.halo) * A.pitch;
    for (int64_t a = (int64_t)blockIdx.x * kBlock + threadIdx.x; a < n; a += (int64_t)gridDim.x * kBlock) {
        A.d[0][a] = 0.0;
        if (A.p) A.p[a] = 0.0;                               // CG-CG / pipelined search direction
        if (A.pipe) { A.pz[a] = 0.0; A.pq[a] = 0.0; A.pm[a] = 0.0; }
        const int64_t row = a / A.pitch;
        if (row >= A.halo && row < A.halo + A.nloc) {
            if (signbit(A.cN[a])) { A.x[a] = 0.0; A.b[a] = 0.0; }
        }
    }
}

// a3: r0 = b - A x0 into r[1]; (b, b)
__global__ void __launch_bounds__(kBlock) init_residual_kernel(const KArgs A) {
    extern __shared__ double ws[];
    const int64_t U = n_units(A);
    int k = 0;
    for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k) {
        const Unit W = unit_of(A, u);
        double v = 0.0;
        if (W.valid) {
            bool land;
            const double ax = stencil(A, A.x, W.a, W.i, land);
            const double bv = A.b[W.a];
            A.r[1][W.a] = land ? 0.0 : __dadd_rn(bv, -ax);
            v = __dmul_rn(bv, bv);
        }
        put_warp_sum(ws, k, v);
    }
    if (finish_units<1>(A, ws, A.partial[0], nullptr, &A.sc->counter[3])) {
        const double tot = final_sum(A.partial[0], n_units(A));
        if (threadIdx.x == 0) {
            A.sc->counter[3] = 0;
            if (A.multi) {
                A.sc->loc[3] = tot;
                if (A.dc) dc_reduce(sargs(A), kSsBB);
            } else {
                fin_bb(A, tot);
            }
        }
    }
}

// a9: ||b - A x|| / ||b||
__global__ void __launch_bounds__(kBlock) true_residual_kernel(const KArgs A) {
    extern __shared__ double ws[];
    const int64_t U = n_units(A);
    int k = 0;
    for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++k) {
        const Unit W = unit_of(A, u);
        double v = 0.0;
        if (W.valid) {
            bool land;
            const double ax = stencil(A, A.x, W.a, W.i, land);
            const double r = land ? 0.0 : __dadd_rn(A.b[W.a], -ax);
            v = __dmul_rn(r, r);
        }
        put_warp_sum(ws, k, v);
    }
    if (finish_units<1>(A, ws, A.partial[0], nullptr, &A.sc->counter[3])) {
        const double tot = final_sum(A.partial[0], n_units(A));
        if (threadIdx.x == 0) {
            A.sc->counter[3] = 0;
            if (A.multi) {
                A.sc->loc[3] = tot;
                if (A.dc) dc_reduce(sargs(A), kSsTrue);
            } else A.sc->true_rel = A.sc->bzero ? 0.0 : __ddiv_rn(__dsqrt_rn(tot), A.sc->nb);
        }
    }
}

// a9: pending x update (or x = 0 when b = 0)
__global__ void __launch_bounds__(kBlock) fin_kernel(const KArgs A) {
    const DevScalars* sc = A.sc;
    const Unit W = unit_of(A, blockIdx.x);
    if (!W.valid) return;
    if (sc->bzero) A.x[W.a] = 0.0;
    else if (sc->xpend) A.x[W.a] = __fma_rn(sc->alpha, A.d[sc->k & 1][W.a], A.x[W.a]);
}

__global__ void __launch_bounds__(kBlock) apply_kernel(const KArgs A, const double* __restrict__ x,
                                                       double* __restrict__ y) {
    const Unit W = unit_of(A, blockIdx.x);
    if (!W.valid) return;
    bool land;
    const double ax = stencil(A, x, W.a, W.i, land);
    y[W.a] = land ? 0.0 : ax;
}

// x0 = 2 x_t - x_tm1 on n contiguous elements (pcg_extrapolate; 2 x_t is exact)
__global__ void __launch_bounds__(kBlock) extrapolate_kernel(const double* __restrict__ xt, const double* __restrict__ xm,
                                                             double* __restrict__ x0, int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x; e < n; e += (int64_t)gridDim.x * kBlock)
        x0[e] = __dadd_rn(__dmul_rn(2.0, xt[e]), -xm[e]);
}

template <class KA>
__device__ void scalar_step(const KA& A, int step) {
    DevScalars* sc = A.sc;
    const int P = A.nranks;
    switch (step) {
        case kSsBB: fin_bb(A, rank_tree(A.gath, P, 3)); break;
        case kSsGamma: sc->red[0] = rank_tree(A.gath, P, 0); break;
        case kSsInit: if (sc->active) fin_init(A, rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2)); break;
        case kSsIter: if (sc->active) fin_iter(A, rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2)); break;
        case kSsCgInit:
            if (sc->active) {
                fin_init(A, rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2));
                if (sc->active) cg_alpha_beta(A, rank_tree(A.gath, P, 0), 1);
            }
            break;
        case kSsCgIter:
            if (sc->active) {
                fin_iter(A, rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2));
                if (sc->active) cg_alpha_beta(A, rank_tree(A.gath, P, 0), 0);
            }
            break;
        case kSsPipe:
            if (sc->active) pipe_fin(A, rank_tree(A.gath, P, 0), rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2));
            break;
        case kSsTrue: {
            const double tot = rank_tree(A.gath, P, 3);
            sc->true_rel = sc->bzero ? 0.0 : __ddiv_rn(__dsqrt_rn(tot), sc->nb);
        } break;
    }
}

__global__ void scalar_kernel(const KArgs A, const int step) { scalar_step(A, step); }

__global__ void set_cond_kernel(cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1u); }

// shared memory of a persistent row kernel: NV warp-sum slots per unit it may process
size_t row_smem(const KArgs& A, int grid, int NV) {
    const int64_t U = (int64_t)A.nloc * A.nbx;
    const int64_t per = std::max<int64_t>((U + grid - 1) / grid, A.sched_max);
    return (size_t)std::max<int64_t>(per, 1) * NV * kWarps * sizeof(double);
}

size_t k1_smem(const KArgs& A, int grid) {
    const int64_t S = (int64_t)A.nbx * ((A.nloc + A.rpb - 1) / A.rpb);
    const int64_t per = (S + grid - 1) / grid;
    return (size_t)std::max<int64_t>(per, 1) * A.rpb * kWarps * sizeof(double);
}

// persistent grid: resident blocks per SM (occupancy API) x SMs, capped by the units
template <class K>
int persistent_grid(K kernel, int64_t units, int sms, size_t smem_guess, int block = kBlock) {
    if (const char* e = getenv("PCG_PERSIST"))          // tuning: 0 = one unit per block
        if (atoi(e) == 0) return (int)units;
    if (const char* e = getenv("PCG_BLOCKS_PER_SM"))    // tuning: fixed resident blocks per SM
        return (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)atoi(e) * sms));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem_guess);
    per_sm = std::max(per_sm, 1);
    return (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)per_sm * sms));
}

template <class K>
void allow_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

// Grid sizes and shared memory of the persistent kernels.
void configure_kernels(KArgs& A, int sms) {
    A.dynamic = 1;                                     // K2/K3: measured -21 % per iteration at ORCA025
    if (const char* e = getenv("PCG_DYNAMIC")) A.dynamic = atoi(e) != 0;
    A.dynamic_k1 = 0;                                  // K1 (4-row strips): static stride measured faster
    if (const char* e = getenv("PCG_DYNAMIC_K1")) A.dynamic_k1 = atoi(e) != 0;
    const int64_t U = (int64_t)A.nloc * A.nbx;
    const int64_t S = (int64_t)A.nbx * ((A.nloc + A.rpb - 1) / A.rpb);
    A.g_k1 = persistent_grid(k1_kernel<false>, S, sms, 4096);
    // PCG_K1_EVEN: the same number of strips for every block (measured no faster at ORCA025)
    if (!A.dynamic_k1 && getenv("PCG_K1_EVEN")) {
        const int64_t per = (S + A.g_k1 - 1) / A.g_k1;
        A.g_k1 = (int)((S + per - 1) / per);
    }
    A.g_k2 = persistent_grid(k2_ainv_kernel<0>, U, sms, 2048);
    A.g_k3 = persistent_grid(k3_ainv_kernel<0>, U, sms, 2048);
    A.g_kd = persistent_grid(k2_diag_kernel<false>, U, sms, 4096);
    A.g_row = persistent_grid(init_residual_kernel, U, sms, 2048);
    // K1 form: 2 = row-segment units, static block stride, no barrier per unit (default: 94.7 ->
    // 91.9 us/iteration at ORCA025 against the 4-row strips, 0); 1 = same units, dynamic tickets
    A.k1flat = 2;
    if (const char* e = getenv("PCG_K1FLAT")) A.k1flat = atoi(e);
    A.pdl = 1;
    if (const char* e = getenv("PCG_PDL")) A.pdl = atoi(e) != 0;
    A.landskip = A.ocean != nullptr;
    if (const char* e = getenv("PCG_LANDSKIP")) A.landskip = A.landskip && atoi(e) != 0;
    A.g_k1f = persistent_grid(k1_flat_kernel<false>, U, sms, 0);
    {
        int bl = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bl, A.sigma ? (const void*)loop_kernel<true> : (const void*)loop_kernel<false>,
                                                      kBlock, 0);
        // cooperative (every block co-resident), no more blocks than the largest phase has units
        const int64_t work = std::max<int64_t>(U, S);
        A.g_loop = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(bl, 1) * sms, work));
    }
    allow_smem(k1_kernel<false>, k1_smem(A, A.g_k1));
    allow_smem(k1_kernel<true>, k1_smem(A, A.g_k1));
    allow_smem(k2_ainv_kernel<0>, row_smem(A, A.g_k2, 1));
    allow_smem(k3_ainv_kernel<0>, row_smem(A, A.g_k3, 1));
    allow_smem(k2_ainv_kernel<-1>, row_smem(A, A.g_k2, 1));
    allow_smem(k3_ainv_kernel<-1>, row_smem(A, A.g_k3, 1));
    allow_smem(k2_ainv_kernel<4>, row_smem(A, A.g_k2, 1));
    allow_smem(k3_ainv_kernel<4>, row_smem(A, A.g_k3, 1));
    allow_smem(k2_ainv_kernel<8>, row_smem(A, A.g_k2, 1));
    allow_smem(k3_ainv_kernel<8>, row_smem(A, A.g_k3, 1));
    allow_smem(k2_ainv_kernel<16>, row_smem(A, A.g_k2, 1));
    allow_smem(k3_ainv_kernel<16>, row_smem(A, A.g_k3, 1));
    // K1 bulk-copy form: strips of kK1W columns x row chunks, one block per SM
    A.k1t_strips = (A.pitch + kK1W - 1) / kK1W;
    {
        const int nch = std::max(1, sms * PCG_K1T_MINB / A.k1t_strips);
        A.k1t_rows = (A.nloc + nch - 1) / nch;
        A.g_k1t = A.k1t_strips * ((A.nloc + A.k1t_rows - 1) / A.k1t_rows);
    }
    allow_smem(k1_tma_kernel<false>, k1t_smem_bytes<false>());
    allow_smem(k1_tma_kernel<true>, k1t_smem_bytes<true>());
    allow_smem(k2_diag_kernel<false>, row_smem(A, A.g_kd, 2));
    allow_smem(k2_diag_kernel<true>, row_smem(A, A.g_kd, 2));
    allow_smem(k1_kernel<false, true>, k1_smem(A, A.g_k1));
    allow_smem(k1_kernel<true, true>, k1_smem(A, A.g_k1));
    allow_smem(k3_ainv_kernel<0, true>, row_smem(A, A.g_k3, 1));
    allow_smem(k3_ainv_kernel<-1, true>, row_smem(A, A.g_k3, 1));
    allow_smem(ka_cg_kernel, row_smem(A, A.g_k2, 1));
    allow_smem(kc_cg_kernel, row_smem(A, A.g_row, 1));
    allow_smem(kpc_kernel, row_smem(A, A.g_row, 3));
    allow_smem(kfin_kernel, (size_t)kKfinWin * sizeof(double));
    allow_smem(init_residual_kernel, row_smem(A, A.g_row, 1));
    allow_smem(true_residual_kernel, row_smem(A, A.g_row, 1));
}

int64_t grid_blocks(const KArgs& A) { return (int64_t)A.nbx * A.nloc; }

// Launch an iteration kernel, with the programmatic-stream-serialization attribute when A.pdl.
template <class... P, class... Args>
static void launch_pdl(const KArgs& A, void (*kern)(P...), int grid, int block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned n = 0;
    if (A.pdl) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (A.l2_bytes) {
        at[n].id = cudaLaunchAttributeAccessPolicyWindow;
        at[n].val.accessPolicyWindow.base_ptr = A.l2_base;
        at[n].val.accessPolicyWindow.num_bytes = A.l2_bytes;
        at[n].val.accessPolicyWindow.hitRatio = A.l2_ratio;
        at[n].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[n].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

void launch_k1(const KArgs& A, int par, cudaStream_t st) {
    if (A.k1tma) {
        if (A.sigma) launch_pdl(A, k1_tma_kernel<true>, A.g_k1t, kK1T, k1t_smem_bytes<true>(), st, A, par);
        else launch_pdl(A, k1_tma_kernel<false>, A.g_k1t, kK1T, k1t_smem_bytes<false>(), st, A, par);
        return;
    }
    if (A.k1flat) {
        const size_t sm = A.k1flat == 2 ? row_smem(A, A.g_k1f, 1) : 0;
        if (A.dc) {
            if (A.sigma) launch_pdl(A, k1_flat_kernel<true, true>, A.g_k1f, kBlock, sm, st, A, par);
            else launch_pdl(A, k1_flat_kernel<false, true>, A.g_k1f, kBlock, sm, st, A, par);
        } else if (A.sigma) launch_pdl(A, k1_flat_kernel<true>, A.g_k1f, kBlock, sm, st, A, par);
        else launch_pdl(A, k1_flat_kernel<false>, A.g_k1f, kBlock, sm, st, A, par);
    } else {
        if (A.dc) {
            if (A.sigma) launch_pdl(A, k1_kernel<true, true>, A.g_k1, kBlock, k1_smem(A, A.g_k1), st, A, par);
            else launch_pdl(A, k1_kernel<false, true>, A.g_k1, kBlock, k1_smem(A, A.g_k1), st, A, par);
        } else if (A.sigma) launch_pdl(A, k1_kernel<true>, A.g_k1, kBlock, k1_smem(A, A.g_k1), st, A, par);
        else launch_pdl(A, k1_kernel<false>, A.g_k1, kBlock, k1_smem(A, A.g_k1), st, A, par);
    }
}
void launch_kc(const KArgs& A, int par, int init, cudaStream_t st) {
    (void)par;
    launch_pdl(A, kc_cg_kernel, A.g_row, kBlock, row_smem(A, A.g_row, 1), st, A, init);
}
void launch_kfin(const KArgs& A, int which, cudaStream_t st) {
    launch_pdl(A, kfin_kernel, 1, kKfinT, (size_t)kKfinWin * sizeof(double), st, A, which);
}
void launch_kpa(const KArgs& A, cudaStream_t st) { launch_pdl(A, kpa_kernel, A.g_k2, kBlock, 0, st, A); }
void launch_kpb(const KArgs& A, cudaStream_t st) { launch_pdl(A, kpb_kernel, A.g_k3, kBlock, 0, st, A); }
void launch_kpc(const KArgs& A, int init, cudaStream_t st) {
    launch_pdl(A, kpc_kernel, A.g_row, kBlock, row_smem(A, A.g_row, 3), st, A, init);
}
void launch_k2_ainv(const KArgs& A, int par, int init, cudaStream_t st) {
    if (A.cgcg && !init) {
        launch_pdl(A, ka_cg_kernel, A.g_k2, kBlock, row_smem(A, A.g_k2, 1), st, A, par);
        return;
    }
    if (A.dia_q > 8) launch_pdl(A, k2_ainv_kernel<16>, A.g_k2, kBlock, row_smem(A, A.g_k2, 1), st, A, par, init);
    else if (A.dia_q > 4) launch_pdl(A, k2_ainv_kernel<8>, A.g_k2, kBlock, row_smem(A, A.g_k2, 1), st, A, par, init);
    else if (A.dia_q > 0) launch_pdl(A, k2_ainv_kernel<4>, A.g_k2, kBlock, row_smem(A, A.g_k2, 1), st, A, par, init);
    else if (A.zt.col16) launch_pdl(A, k2_ainv_kernel<-1>, A.g_k2, kBlock, row_smem(A, A.g_k2, 1), st, A, par, init);
    else launch_pdl(A, k2_ainv_kernel<0>, A.g_k2, kBlock, row_smem(A, A.g_k2, 1), st, A, par, init);
}
void launch_k3_ainv(const KArgs& A, int par, int init, cudaStream_t st) {
    if (A.dia_q > 8) launch_pdl(A, k3_ainv_kernel<16>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
    else if (A.dia_q > 4) launch_pdl(A, k3_ainv_kernel<8>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
    else if (A.dia_q > 0) launch_pdl(A, k3_ainv_kernel<4>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
    else if (A.dc && A.z.col16) launch_pdl(A, k3_ainv_kernel<-1, true>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
    else if (A.dc) launch_pdl(A, k3_ainv_kernel<0, true>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
    else if (A.z.col16) launch_pdl(A, k3_ainv_kernel<-1>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
    else launch_pdl(A, k3_ainv_kernel<0>, A.g_k3, kBlock, row_smem(A, A.g_k3, 1), st, A, par, init);
}
void launch_k2_diag(const KArgs& A, int par, int init, int none, cudaStream_t st) {
    if (A.dc) launch_pdl(A, k2_diag_kernel<true>, A.g_kd, kBlock, row_smem(A, A.g_kd, 2), st, A, par, init, none);
    else launch_pdl(A, k2_diag_kernel<false>, A.g_kd, kBlock, row_smem(A, A.g_kd, 2), st, A, par, init, none);
}
void launch_prep(const KArgs& A, cudaStream_t st) {
    const int64_t n = (int64_t)(A.nloc + 2 * A.halo) * A.pitch;
    const int64_t G = std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 16);
    prep_kernel<<<(unsigned)G, kBlock, 0, st>>>(A);
}
void launch_init_residual(const KArgs& A, cudaStream_t st) {
    init_residual_kernel<<<A.g_row, kBlock, row_smem(A, A.g_row, 1), st>>>(A);
}
void launch_fin(const KArgs& A, cudaStream_t st) { fin_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A); }
void launch_true_residual(const KArgs& A, cudaStream_t st) {
    true_residual_kernel<<<A.g_row, kBlock, row_smem(A, A.g_row, 1), st>>>(A);
}
void launch_apply(const KArgs& A, const double* x, double* y, cudaStream_t st) {
    apply_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A, x, y);
}
void launch_scalar(const KArgs& A, int step, cudaStream_t st) { scalar_kernel<<<1, 1, 0, st>>>(A, step); }
void launch_extrapolate(const double* xt, const double* xm, double* x0, int64_t n, cudaStream_t st) {
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 8));
    extrapolate_kernel<<<(unsigned)G, kBlock, 0, st>>>(xt, xm, x0, n);
}
cudaError_t launch_loop(const KArgs& A, cudaStream_t st) {
    void* args[] = {(void*)&A};
    const void* fn = A.sigma ? (const void*)loop_kernel<true> : (const void*)loop_kernel<false>;
    return cudaLaunchCooperativeKernel(fn, dim3(A.g_loop), dim3(kBlock), args, 0, st);
}
void launch_set_cond(cudaGraphConditionalHandle h, cudaStream_t st) { set_cond_kernel<<<1, 1, 0, st>>>(h); }

}  // namespace pcg

#ifdef PCG_TIMELINE
// Diagnostic build only: copy the block timeline of the last K1/K2/K3 launches to the host.
extern "C" int pcg_diag_timeline(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, pcg::g_timeline, sizeof(pcg::g_timeline));
}
extern "C" int pcg_diag_tail(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, pcg::g_tail, sizeof(pcg::g_tail));
}
extern "C" int pcg_diag_units(unsigned* out, int reset) {
    int e = (int)cudaMemcpyFromSymbol(out, pcg::g_units, sizeof(pcg::g_units));
    if (reset) {
        static unsigned z[2048] = {};
        cudaMemcpyToSymbol(pcg::g_units, z, sizeof(z));
    }
    return e;
}
#endif
