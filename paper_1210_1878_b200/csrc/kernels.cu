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
//   * SELL rows: acc = 0, fma over the stored entries in ascending column order; K2 then
//     divides by Dhat;
//   * updates: x = fma(alpha, d, x); r = fma(-alpha, q, r); d = fma(beta, d_old, s);
//   * dot products: one element per thread, fl(a*b); 256-thread block = shuffle-down tree
//     (16,8,4,2,1) per warp, then the same tree over the 8 warp sums; the last block sums the
//     block partials t, t+256, ... left to right per thread and applies the block tree.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"
#include "kernels.h"

namespace pcg {

namespace {

__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
    return v;
}

// Block tree (kBlock threads): result valid in thread 0.
__device__ __forceinline__ double block_tree(double v) {
    __shared__ double ws[kBlock / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_tree(v);
    __syncthreads();                       // ws may still be read by a previous call
    if (lane == 0) ws[w] = v;
    __syncthreads();
    double u = 0.0;
    if (w == 0) {
        u = lane < kBlock / 32 ? ws[lane] : 0.0;
        u = warp_tree(u);
    }
    return u;
}

// Publish this block's partial and report whether it is the last block to finish.
__device__ __forceinline__ bool publish_partial(double part, double* partial, uint32_t* counter) {
    __shared__ bool am_last;
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = part;
        __threadfence();
        const uint32_t t = atomicAdd(counter, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return am_last;
}

// In the last block: thread t sums partials t, t+B, ... then the block tree.
__device__ __forceinline__ double final_sum(const double* partial, int G) {
    __threadfence();
    double acc = 0.0;
    for (int m = threadIdx.x; m < G; m += kBlock) acc = __dadd_rn(acc, __ldcg(partial + m));
    return block_tree(acc);
}

// tree over the per-rank sums in rank order, zero padded to 32
__device__ double rank_tree(const double* gath, int nranks, int slot) {
    double u[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) u[l] = l < nranks ? gath[l * 4 + slot] : 0.0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
        for (int l = 0; l + off < 32; ++l) u[l] = __dadd_rn(u[l], u[l + off]);
    return u[0];
}

__device__ __forceinline__ void set_cond(const KArgs& A, int v) {
    if (A.use_cond) cudaGraphSetConditional(A.cond, (unsigned)v);
}

__device__ __forceinline__ void stop(const KArgs& A, int status) {
    DevScalars* sc = A.sc;
    sc->status = status;
    sc->active = 0;
    set_cond(A, 0);
}

__device__ __forceinline__ bool is_active(const KArgs& A) {
    return *(volatile int32_t*)&A.sc->active != 0;
}

// ---- scalar updates (one thread) --------------------------------------------------------
__device__ void fin_bb(const KArgs& A, double bb) {
    DevScalars* sc = A.sc;
    sc->nb = __dsqrt_rn(bb);
    sc->bzero = sc->nb == 0.0;
    sc->alpha = 0.0; sc->beta = 0.0; sc->k = 0; sc->status = kStOk; sc->xpend = 0;
    sc->active = 1;                       // provisional: decided after s0 (fin_init)
}

__device__ void fin_init(const KArgs& A, double rho0, double rr0) {
    DevScalars* sc = A.sc;
    if (sc->bzero) {
        A.hist[0] = 0.0;
        sc->active = 0;
        set_cond(A, 0);
        return;
    }
    sc->rho = rho0;
    sc->beta = 0.0;
    const double h = __ddiv_rn(__dsqrt_rn(rr0), sc->nb);
    A.hist[0] = h;
    const int act = (h > sc->tol) && (sc->maxit > 0);
    sc->active = act;
    set_cond(A, act);
}

__device__ void fin_iter(const KArgs& A, double rho_new, double rr) {
    DevScalars* sc = A.sc;
    const int k = sc->k + 1;
    sc->k = k;
    if (!isfinite(rho_new) || !isfinite(rr)) {
        if (k < A.hist_cap) A.hist[k] = NAN;
        stop(A, kStBreakdown);
        return;
    }
    sc->beta = __ddiv_rn(rho_new, sc->rho);
    sc->rho = rho_new;
    const double h = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
    if (k < A.hist_cap) A.hist[k] = h;
    const int act = (h > sc->tol) && (k < sc->maxit);
    sc->active = act;
    set_cond(A, act);
}

// alpha of the current iteration from the global (d, q); false on breakdown
__device__ __forceinline__ bool get_alpha(const KArgs& A, int init, double& alpha) {
    if (init) { alpha = 0.0; return true; }
    const double gamma = A.sc->red[0];
    if (!(gamma > 0.0) || !isfinite(gamma)) return false;
    alpha = __ddiv_rn(A.sc->rho, gamma);
    return true;
}

// ---- K1: d = s + beta d_old ; x += alpha_prev d_old ; q = A d ; (d, q) --------------------
template <bool SIGMA>
__global__ void __launch_bounds__(kBlock) k1_kernel(const KArgs A, const int par) {
    if (!is_active(A)) return;
    const double beta = A.sc->beta, alpha = A.sc->alpha;
    const double* __restrict__ dold = A.d[par];
    double* __restrict__ dnew = A.d[par ^ 1];
    const double* __restrict__ s = A.s;
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double v = 0.0;
    if (e < A.nel) {
        const int32_t i = (int32_t)(e % A.pitch);
        if (i < A.ni) {
            const int64_t a = e + A.pitch;
            const int64_t aw = i == 0 ? a + (A.ni - 1) : a - 1;
            const int64_t ae = i == A.ni - 1 ? a - (A.ni - 1) : a + 1;
            const int64_t as = a - A.pitch, an = a + A.pitch;
            const double dop = dold[a];
            const double dp = __fma_rn(beta, dop, s[a]);
            const double dw = __fma_rn(beta, dold[aw], s[aw]);
            const double de = __fma_rn(beta, dold[ae], s[ae]);
            const double ds = __fma_rn(beta, dold[as], s[as]);
            const double dn = __fma_rn(beta, dold[an], s[an]);
            A.x[a] = __fma_rn(alpha, dop, A.x[a]);
            const double cep = A.cE[a], cew = A.cE[aw];
            const double cnr = A.cN[a];
            const bool land = signbit(cnr);
            const double cnp = fabs(cnr), cns = fabs(A.cN[as]);
            double app = __dadd_rn(__dadd_rn(__dadd_rn(cep, cew), cnp), cns);
            if (SIGMA) app = __dadd_rn(app, A.sigma[a]);
            double acc = __dmul_rn(app, dp);
            acc = __fma_rn(-cew, dw, acc);
            acc = __fma_rn(-cep, de, acc);
            acc = __fma_rn(-cns, ds, acc);
            acc = __fma_rn(-cnp, dn, acc);
            const double qv = land ? 0.0 : acc;
            dnew[a] = dp;
            A.q[a] = qv;
            v = __dmul_rn(dp, qv);
            // d on the halo rows (needed by the next K1 of a multi-rank solve)
            if (e < A.pitch) dnew[as] = ds;
            if (e >= A.nel - A.pitch) dnew[an] = dn;
        }
    }
    const double part = block_tree(v);
    if (publish_partial(part, A.partial[0], &A.sc->counter[0])) {
        const double tot = final_sum(A.partial[0], gridDim.x);
        if (threadIdx.x == 0) {
            if (A.multi) A.sc->loc[0] = tot;
            else A.sc->red[0] = tot;
            A.sc->xpend = 0;
            A.sc->counter[0] = 0;
        }
    }
}

// ---- K2 (AINV): r -= alpha q ; t = Dhat^-1 Z^T r ; (r, r) --------------------------------
__global__ void __launch_bounds__(kBlock) k2_ainv_kernel(const KArgs A, const int par, const int init) {
    if (!is_active(A)) return;
    double alpha;
    if (!get_alpha(A, init, alpha)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) stop(A, kStBreakdown);
        return;
    }
    const double* __restrict__ ro = A.r[par];
    double* __restrict__ rn = A.r[par ^ 1];
    const double* __restrict__ q = A.q;
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double v = 0.0;
    if (e < A.nel) {
        const int64_t a = e + A.pitch;
        const int64_t sl = e >> 5;
        const int lane = (int)(e & 31);
        const double rnew = __fma_rn(-alpha, q[a], ro[a]);
        const int64_t off = A.zt_off[sl];
        const int64_t L = (A.zt_off[sl + 1] - off) >> 5;
        double acc = 0.0;
        for (int64_t m = 0; m < L; ++m) {
            const int64_t slot = off + (m << 5) + lane;
            const int32_t c = __ldg(A.zt_col + slot);
            const double z = __ldg(A.zt_val + slot);
            acc = __fma_rn(z, __fma_rn(-alpha, q[c], ro[c]), acc);
        }
        A.t[a] = __ddiv_rn(acc, A.piv[a]);
        rn[a] = rnew;
        v = __dmul_rn(rnew, rnew);
    }
    const double part = block_tree(v);
    if (publish_partial(part, A.partial[1], &A.sc->counter[1])) {
        const double tot = final_sum(A.partial[1], gridDim.x);
        if (threadIdx.x == 0) {
            if (A.multi) A.sc->loc[2] = tot;
            else A.sc->red[2] = tot;
            A.sc->alpha = alpha;
            A.sc->xpend = init ? 0 : 1;
            A.sc->counter[1] = 0;
        }
    }
}

// ---- K3 (AINV): s = Z t ; (s, r) ; beta / history / flag -----------------------------------
__global__ void __launch_bounds__(kBlock) k3_ainv_kernel(const KArgs A, const int par, const int init) {
    if (!is_active(A)) return;
    const double* __restrict__ rn = A.r[par ^ 1];
    const double* __restrict__ t = A.t;
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double v = 0.0;
    if (e < A.nel) {
        const int64_t a = e + A.pitch;
        const int64_t sl = e >> 5;
        const int lane = (int)(e & 31);
        const int64_t off = A.z_off[sl];
        const int64_t L = (A.z_off[sl + 1] - off) >> 5;
        double acc = 0.0;
        for (int64_t m = 0; m < L; ++m) {
            const int64_t slot = off + (m << 5) + lane;
            acc = __fma_rn(__ldg(A.z_val + slot), t[__ldg(A.z_col + slot)], acc);
        }
        A.s[a] = acc;
        v = __dmul_rn(acc, rn[a]);
    }
    const double part = block_tree(v);
    if (publish_partial(part, A.partial[2], &A.sc->counter[2])) {
        const double tot = final_sum(A.partial[2], gridDim.x);
        if (threadIdx.x == 0) {
            A.sc->counter[2] = 0;
            if (A.multi) A.sc->loc[1] = tot;
            else if (init) fin_init(A, tot, A.sc->red[2]);
            else fin_iter(A, tot, A.sc->red[2]);
        }
    }
}

// ---- K2 (Jacobi / none): r -= alpha q ; s = r / A_pp (or r) ; (r, r), (s, r) ---------------
__global__ void __launch_bounds__(kBlock) k2_diag_kernel(const KArgs A, const int par, const int init,
                                                         const int none) {
    if (!is_active(A)) return;
    double alpha;
    if (!get_alpha(A, init, alpha)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) stop(A, kStBreakdown);
        return;
    }
    const double* __restrict__ ro = A.r[par];
    double* __restrict__ rn = A.r[par ^ 1];
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double v1 = 0.0, v2 = 0.0;
    if (e < A.nel) {
        const int64_t a = e + A.pitch;
        const double rnew = __fma_rn(-alpha, A.q[a], ro[a]);
        const double sv = none ? rnew : __ddiv_rn(rnew, A.diag[a]);
        A.s[a] = sv;
        rn[a] = rnew;
        v1 = __dmul_rn(rnew, rnew);
        v2 = __dmul_rn(sv, rnew);
    }
    const double p1 = block_tree(v1);
    const double p2 = block_tree(v2);
    __shared__ bool am_last;
    if (threadIdx.x == 0) {
        A.partial[1][blockIdx.x] = p1;
        A.partial[2][blockIdx.x] = p2;
        __threadfence();
        am_last = atomicAdd(&A.sc->counter[1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (am_last) {
        const double rr = final_sum(A.partial[1], gridDim.x);
        const double rs = final_sum(A.partial[2], gridDim.x);
        if (threadIdx.x == 0) {
            A.sc->counter[1] = 0;
            A.sc->alpha = alpha;
            A.sc->xpend = init ? 0 : 1;
            if (A.multi) { A.sc->loc[2] = rr; A.sc->loc[1] = rs; }
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

// prep: zero land entries of x and b (land is not an unknown, reading R20), zero d[0] everywhere
__global__ void __launch_bounds__(kBlock) prep_kernel(const KArgs A) {
    const int64_t n = (int64_t)(A.nloc + 2) * A.pitch;
    for (int64_t a = (int64_t)blockIdx.x * kBlock + threadIdx.x; a < n; a += (int64_t)gridDim.x * kBlock) {
        A.d[0][a] = 0.0;
        const int64_t row = a / A.pitch;
        if (row >= 1 && row <= A.nloc) {
            if (signbit(A.cN[a])) { A.x[a] = 0.0; A.b[a] = 0.0; }
        }
    }
}

// a3: r0 = b - A x0 into r[1]; (b, b)
__global__ void __launch_bounds__(kBlock) init_residual_kernel(const KArgs A) {
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double v = 0.0;
    if (e < A.nel) {
        const int32_t i = (int32_t)(e % A.pitch);
        if (i < A.ni) {
            const int64_t a = e + A.pitch;
            bool land;
            const double ax = stencil(A, A.x, a, i, land);
            const double bv = A.b[a];
            A.r[1][a] = land ? 0.0 : __dadd_rn(bv, -ax);
            v = __dmul_rn(bv, bv);
        }
    }
    const double part = block_tree(v);
    if (publish_partial(part, A.partial[0], &A.sc->counter[3])) {
        const double tot = final_sum(A.partial[0], gridDim.x);
        if (threadIdx.x == 0) {
            A.sc->counter[3] = 0;
            if (A.multi) A.sc->loc[3] = tot;
            else fin_bb(A, tot);
        }
    }
}

// a9: pending x update (or x = 0 when b = 0)
__global__ void __launch_bounds__(kBlock) fin_kernel(const KArgs A) {
    const DevScalars* sc = A.sc;
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (e >= A.nel) return;
    const int32_t i = (int32_t)(e % A.pitch);
    if (i >= A.ni) return;
    const int64_t a = e + A.pitch;
    if (sc->bzero) { A.x[a] = 0.0; return; }
    if (sc->xpend) A.x[a] = __fma_rn(sc->alpha, A.d[sc->k & 1][a], A.x[a]);
}

// a9: ||b - A x|| / ||b||
__global__ void __launch_bounds__(kBlock) true_residual_kernel(const KArgs A) {
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double v = 0.0;
    if (e < A.nel) {
        const int32_t i = (int32_t)(e % A.pitch);
        if (i < A.ni) {
            const int64_t a = e + A.pitch;
            bool land;
            const double ax = stencil(A, A.x, a, i, land);
            const double r = land ? 0.0 : __dadd_rn(A.b[a], -ax);
            v = __dmul_rn(r, r);
        }
    }
    const double part = block_tree(v);
    if (publish_partial(part, A.partial[0], &A.sc->counter[3])) {
        const double tot = final_sum(A.partial[0], gridDim.x);
        if (threadIdx.x == 0) {
            A.sc->counter[3] = 0;
            if (A.multi) A.sc->loc[3] = tot;
            else A.sc->true_rel = A.sc->bzero ? 0.0 : __ddiv_rn(__dsqrt_rn(tot), A.sc->nb);
        }
    }
}

__global__ void __launch_bounds__(kBlock) apply_kernel(const KArgs A, const double* __restrict__ x,
                                                       double* __restrict__ y) {
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (e >= A.nel) return;
    const int32_t i = (int32_t)(e % A.pitch);
    if (i >= A.ni) return;
    const int64_t a = e + A.pitch;
    bool land;
    const double ax = stencil(A, x, a, i, land);
    y[a] = land ? 0.0 : ax;
}

__global__ void scalar_kernel(const KArgs A, const int step) {
    DevScalars* sc = A.sc;
    const int P = A.nranks;
    switch (step) {
        case kSsBB: fin_bb(A, rank_tree(A.gath, P, 3)); break;
        case kSsGamma: sc->red[0] = rank_tree(A.gath, P, 0); break;
        case kSsInit: if (sc->active) fin_init(A, rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2)); break;
        case kSsIter: if (sc->active) fin_iter(A, rank_tree(A.gath, P, 1), rank_tree(A.gath, P, 2)); break;
        case kSsTrue: {
            const double tot = rank_tree(A.gath, P, 3);
            sc->true_rel = sc->bzero ? 0.0 : __ddiv_rn(__dsqrt_rn(tot), sc->nb);
        } break;
    }
}

__global__ void set_cond_kernel(cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1u); }

}  // namespace

int64_t grid_blocks(const KArgs& A) { return (A.nel + kBlock - 1) / kBlock; }

void launch_k1(const KArgs& A, int par, cudaStream_t st) {
    const unsigned G = (unsigned)grid_blocks(A);
    if (A.sigma) k1_kernel<true><<<G, kBlock, 0, st>>>(A, par);
    else k1_kernel<false><<<G, kBlock, 0, st>>>(A, par);
}
void launch_k2_ainv(const KArgs& A, int par, int init, cudaStream_t st) {
    k2_ainv_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A, par, init);
}
void launch_k3_ainv(const KArgs& A, int par, int init, cudaStream_t st) {
    k3_ainv_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A, par, init);
}
void launch_k2_diag(const KArgs& A, int par, int init, int none, cudaStream_t st) {
    k2_diag_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A, par, init, none);
}
void launch_prep(const KArgs& A, cudaStream_t st) {
    const int64_t n = (int64_t)(A.nloc + 2) * A.pitch;
    const int64_t G = std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 16);
    prep_kernel<<<(unsigned)G, kBlock, 0, st>>>(A);
}
void launch_init_residual(const KArgs& A, cudaStream_t st) {
    init_residual_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A);
}
void launch_fin(const KArgs& A, cudaStream_t st) { fin_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A); }
void launch_true_residual(const KArgs& A, cudaStream_t st) {
    true_residual_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A);
}
void launch_apply(const KArgs& A, const double* x, double* y, cudaStream_t st) {
    apply_kernel<<<(unsigned)grid_blocks(A), kBlock, 0, st>>>(A, x, y);
}
void launch_scalar(const KArgs& A, int step, cudaStream_t st) { scalar_kernel<<<1, 1, 0, st>>>(A, step); }
void launch_set_cond(cudaGraphConditionalHandle h, cudaStream_t st) { set_cond_kernel<<<1, 1, 0, st>>>(h); }

}  // namespace pcg
