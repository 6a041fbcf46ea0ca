// rs.cu -- the resident-strip PCG loop: one persistent cooperative kernel runs every iteration of
// Alg. 1 (d = s + beta d, R6) on one GPU.
//
// Why: the three-kernel iteration (kernels.cu K1 / K2 / K3) is latency-bound at ORCA025 size --
// every element's row sum waits on a DRAM load, then on L2 gathers of its neighbours, and every
// kernel boundary drains and refills the machine.  Here each of the 148 blocks (one per SM) owns a
// contiguous range of units (256-column row segments, row-major) per phase and copies the vector
// that phase gathers from -- d for the stencil, r_new for Z^T r, t for Z t -- for its range plus
// the halo its stencil / Z rows reach into shared memory.  Every gather is then a shared-memory
// load; global memory sees coalesced streams of 32-element chunks, several per warp in flight.
//
// Per iteration (block b, phase-1 units [ua1, ub1), phase-2 units [ua2, ub2)):
//   1a  d = s + beta d_old over the range +- one grid row -> smem; own: d -> global, x += alpha d_old
//   1b  q = A d (5-point, E-W wrap) on own ocean points from smem; (d, q) warp sums      Alg.1 l.6
//   --  grid barrier; every block forms the canonical (d, q) sum -> alpha               (reduce 1)
//   2A  r_new = r - alpha q over [lo2, range end) -> smem; own: r_new -> global, (r, r)   l.7
//   2B  t = Dhat^-1 Z^T r_new (ELL(4) slots + overflow) on own ocean points -> global t
//   --  t-ready stamp of b
//   2C  own t -> smem; wait for the stamps of the blocks whose t this block's Z rows reach, then
//       their t over [range end, hi2) -> smem
//   2D  s = Z t (ELL(4) + overflow) on own ocean points -> global; (s, r_new) warp sums
//   --  grid barrier; every block forms (r, r) and (s, r) -> beta, history, stop test    (reduce 2)
// Jacobi / none: phase 2 is one pointwise pass (s = r_new / A_pp or r_new).
// Land chunks (ocean bit mask 0) issue no loads at all.  The overflow entries of Z / Z^T (rows
// longer than the 4 ELL slots: the long E-W tails of the pole rows) are read in rounds of RS_OVF
// coalesced loads with the next round in flight, after bulk prefetches of the block's overflow
// range into L2 at the start of phase 2.
//
// ARITHMETIC: bitwise the canonical order of DESIGN.md §5 (the same per-point expressions as
// kernels.cu, the same per-(row, segment) partials and final sums), so this driver is compared
// against the oracle's canonical mode like the others.  Vectors written by other blocks inside the
// kernel are read with ld.global.cg (L2), never through L1.  Array indices are 32-bit (setup
// requires fewer than 2^31 elements).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "internal.h"
#include "kernels.h"
#include "dev_common.cuh"

namespace pcg {
namespace {

// Per block size: chunks per warp in flight in the vector passes (1a, 2A, 2C, Jacobi: VU), the
// stencil pass (1b: K1C) and the Z / Z^T passes (2B, 2D: ZC), overflow entries per round (OVF,
// two rounds in flight), partial loads in flight per thread in the final sums (NB: (d, q); NB2:
// per array for (r, r), (s, r)).  512 threads get 128 registers, 768 threads 80 (measured at
// cfg4: 768 threads 75.7 vs 76.6 us per iteration for AINV(0.1), 34.2 vs 36.7 for Jacobi; at
// cfg2 / cfg3 AINV 16.0 / 19.8 vs 14.9 / 17.9 -- setup_rs picks per problem).  NB = 24 puts a
// cfg4-sized (d, q) sum (6126 partials, 24 per thread) in one round of loads.
template <int NT, int PC>
struct RsCfg;
template <int PC>
struct RsCfg<512, PC> {
    static constexpr int VU = 8, K1C = 4, ZC = 2, OVF = 8, NB = 24, NB2 = 12;
};
// 768 threads (tuning hooks RS768_* for the factored instantiation, RS768D_* for Jacobi / none)
#ifndef RS768_VU
#define RS768_VU 4
#endif
#ifndef RS768_K1C
#define RS768_K1C 4
#endif
#ifndef RS768_ZC
#define RS768_ZC 2
#endif
#ifndef RS768_OVF
#define RS768_OVF 4
#endif
#ifndef RS768_NB
#define RS768_NB 24
#endif
#ifndef RS768_NB2
#define RS768_NB2 8
#endif
#ifndef RS768D_VU
#define RS768D_VU 4
#endif
#ifndef RS768D_K1C
#define RS768D_K1C 2
#endif
#ifndef RS768D_NB
#define RS768D_NB 24
#endif
#ifndef RS768D_NB2
#define RS768D_NB2 12
#endif
template <int PC>
struct RsCfg<768, PC> {
    static constexpr bool F = PC == 0;
    static constexpr int VU = F ? RS768_VU : RS768D_VU, K1C = F ? RS768_K1C : RS768D_K1C, ZC = RS768_ZC,
                         OVF = RS768_OVF, NB = F ? RS768_NB : RS768D_NB, NB2 = F ? RS768_NB2 : RS768D_NB2;
};

// Diagnostic build only (-DRS_TIMELINE): per-block globaltimer durations of each pass, summed over
// the iterations (read back with pcg_rs_timeline).
#ifdef RS_TIMELINE
__device__ unsigned long long g_rs_tl[160][12];
__device__ __forceinline__ unsigned long long rs_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RS_T(slot)                                                  \
    do {                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 160) {                 \
            const unsigned long long now_ = rs_now();               \
            g_rs_tl[blockIdx.x][slot] += now_ - tl_prev;            \
            tl_prev = now_;                                         \
        }                                                           \
    } while (0)
#else
#define RS_T(slot) ((void)0)
#endif
// a block barrier that is also a timeline point
#define RS_TS(slot)      \
    do {                 \
        __syncthreads(); \
        RS_T(slot);      \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// bulk prefetch of [p, p + bytes) into L2 (bytes a multiple of 16, p 16-byte aligned), in pieces
// of at most 64 KB
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t bytes) {
    const char* q = static_cast<const char*>(p);
    for (uint64_t o = 0; o < bytes; o += 65536) {
        const uint32_t n = (uint32_t)min((uint64_t)65536, bytes - o);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q + o), "r"(n) : "memory");
    }
}

// Watchdog of the spin waits: a wait that outlives ~4 s of polling records (block, site, value,
// target) in g_rs_hang and traps, so a protocol error ends the kernel with an error instead of
// hanging the GPU.
__device__ unsigned g_rs_hang[4];
__device__ __forceinline__ void rs_spin(const unsigned* p, unsigned target, unsigned site) {
    unsigned long long n = 0;
    unsigned v;
    while ((v = ld_acquire_u32(p)) < target) {
        if (++n > (1ull << 27)) {
            g_rs_hang[0] = blockIdx.x; g_rs_hang[1] = site; g_rs_hang[2] = v; g_rs_hang[3] = target;
            __threadfence_system();
            __trap();
        }
    }
}

// Grid barrier of co-resident blocks: thread 0 publishes the block's writes (bar.sync orders the
// block's threads before it; the gpu-scope fence makes them visible) and waits for every block.
__device__ __forceinline__ void rs_grid_sync(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        rs_spin(ctr, target, 0u);
    }
    __syncthreads();
}

// array index of the first element of unit m (row-major units: m = row * nbx + segment); units
// tile the rows, so unit_a0(m + 1) is the end of unit m
__device__ __forceinline__ int32_t unit_a0(const KArgs& A, int32_t m) {
    const int32_t j = m / A.nbx, bx = m - j * A.nbx;
    return (j + A.halo) * A.pitch + bx * kBlock;
}

// canonical final sum in every thread of the block
template <int NB>
__device__ __forceinline__ double rs_final(const double* partial, int64_t G, double* bc) {
    const double v = final_sum<NB>(partial, G);
    if (threadIdx.x == 0) *bc = v;
    __syncthreads();
    const double r = *bc;
    __syncthreads();
    return r;
}

// canonical final sums of two partial arrays in one walk (each in final_sum's order: bitwise the
// same), in every thread of the block
template <int NB>
__device__ __forceinline__ void rs_final2(const double* p1, const double* p2, int64_t G, double* bc, double& s1,
                                          double& s2) {
    double a1 = 0.0, a2 = 0.0;
    int64_t m = threadIdx.x < kBlock ? (int64_t)threadIdx.x : G;
    for (; m < G; m += NB * kBlock) {
        double u1[NB], u2[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const bool in = m + u * kBlock < G;
            u1[u] = in ? __ldcg(p1 + m + u * kBlock) : 0.0;
            u2[u] = in ? __ldcg(p2 + m + u * kBlock) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NB; ++u)
            if (m + u * kBlock < G) { a1 = __dadd_rn(a1, u1[u]); a2 = __dadd_rn(a2, u2[u]); }
    }
    const double t1 = block_tree(a1);
    if (threadIdx.x == 0) bc[0] = t1;
    const double t2 = block_tree(a2);
    if (threadIdx.x == 0) bc[1] = t2;
    __syncthreads();
    s1 = bc[0];
    s2 = bc[1];
    __syncthreads();
}

// unit partials of units [ua, ua + nu) from their chunk warp sums (second level of the block
// tree); uc[u] = first chunk of unit ua + u relative to unit ua (uc[nu] = end)
template <int NW>
__device__ __forceinline__ void rs_partials(int32_t ua, int32_t nu, const int32_t* uc, const double* ws, double* partial) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int32_t u = warp; u < nu; u += NW) {
        const int32_t c0 = uc[u], nc = uc[u + 1] - c0;
        double v = lane < nc ? ws[c0 + lane] : 0.0;
        v = warp_tree(v);
        if (lane == 0) partial[ua + u] = v;
    }
}

// One Z / Z^T row: the 4 preloaded ELL slots (z, cw: int16 offsets from the element's own array
// index a; zero / own index on land lanes), then the row's entries in the SELL-32 overflow of its
// slice (o0 = first entry, L per lane; entry m of lane l at o0 + 32 m + l, coalesced per warp).
// Gathers from shared memory: xb[c] is the gathered vector at array index c.  acc = 0, fma over
// the entries in ascending column order, padding included (as kernels.cu's
// overflow_sum).
template <int RS_OVF>
__device__ __forceinline__ double rs_row(const double (&z)[kEll], uint2 cw, int64_t o0, int L, int32_t a,
                                         const double* xb, const double* __restrict__ ov, const int32_t* __restrict__ oc) {
    const int32_t c0 = a + (int32_t)(int16_t)(cw.x & 0xffffu), c1 = a + (int32_t)(int16_t)(cw.x >> 16);
    const int32_t c2 = a + (int32_t)(int16_t)(cw.y & 0xffffu), c3 = a + (int32_t)(int16_t)(cw.y >> 16);
    double acc = __fma_rn(z[0], xb[c0], 0.0);
    acc = __fma_rn(z[1], xb[c1], acc);
    acc = __fma_rn(z[2], xb[c2], acc);
    acc = __fma_rn(z[3], xb[c3], acc);
    if (L == 0) return acc;
    const int lane = threadIdx.x & 31;
    const double* vp = ov + o0 + lane;
    const int32_t* cp = oc + o0 + lane;
    // two rounds of RS_OVF entries in flight: round A is consumed while round B's loads are out,
    // then A is refilled two rounds ahead (entries past L re-read the last entry, never used)
    double za[RS_OVF], zb[RS_OVF];
    int32_t ca[RS_OVF], cb[RS_OVF];
#pragma unroll
    for (int u = 0; u < RS_OVF; ++u) {
        const int m = min(u, L - 1) << 5, n = min(RS_OVF + u, L - 1) << 5;
        za[u] = __ldg(vp + m);
        ca[u] = __ldg(cp + m);
        zb[u] = __ldg(vp + n);
        cb[u] = __ldg(cp + n);
    }
    for (int m0 = 0; m0 < L; m0 += 2 * RS_OVF) {
#pragma unroll
        for (int u = 0; u < RS_OVF; ++u)
            if (m0 + u < L) acc = __fma_rn(za[u], xb[ca[u]], acc);
        if (m0 + 2 * RS_OVF < L) {
#pragma unroll
            for (int u = 0; u < RS_OVF; ++u) {
                const int m = min(m0 + 2 * RS_OVF + u, L - 1) << 5;
                za[u] = __ldg(vp + m);
                ca[u] = __ldg(cp + m);
            }
        }
#pragma unroll
        for (int u = 0; u < RS_OVF; ++u)
            if (m0 + RS_OVF + u < L) acc = __fma_rn(zb[u], xb[cb[u]], acc);
        if (m0 + 3 * RS_OVF < L) {
#pragma unroll
            for (int u = 0; u < RS_OVF; ++u) {
                const int m = min(m0 + 3 * RS_OVF + u, L - 1) << 5;
                zb[u] = __ldg(vp + m);
                cb[u] = __ldg(cp + m);
            }
        }
    }
    return acc;
}


// Every pass below walks the warp's chunks (c = warp + NW q) in batches of D: the loads of D
// chunks are issued into register slots before any of them is consumed.  Every slot is assigned
// on every batch (zeros for masked chunks), so no value is carried across batches.

// PC: 0 = factored Z Dhat^-1 Z^T (AINV, P_B2, FSAI through the ELL form), 1 = Jacobi, 2 = none
template <bool SIGMA, int PC, int NT>
__global__ void __launch_bounds__(NT, 1) rs_loop_kernel(const KArgs A) {
    using C = RsCfg<NT, PC>;
    extern __shared__ __align__(16) double sm[];
    __shared__ double bc[2];
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    const unsigned nblk = gridDim.x;
    DevScalars* sc = A.sc;
    const int32_t P = A.pitch, ni = A.ni;
    const int64_t U = (int64_t)A.nloc * A.nbx;
    uint32_t* const rs_sync = A.rs.sync;
    const int32_t cap = A.rs.cap, maxu1 = A.rs.maxu1, maxu2 = A.rs.maxu2, maxnx = A.rs.maxnx;
    const int32_t ua1 = A.rs.ub1[b], ub1 = A.rs.ub1[b + 1], ua2 = A.rs.ub2[b], ub2 = A.rs.ub2[b + 1];
    const int32_t nu1 = ub1 - ua1, nu2 = ub2 - ua2;
    const int32_t e0 = unit_a0(A, ua1), e1 = unit_a0(A, ub1);
    const int32_t f0 = unit_a0(A, ua2), f1 = unit_a0(A, ub2);
    const int32_t lo2 = (int32_t)A.rs.lo2[b];
    const int32_t hi2 = (int32_t)((A.rs.hi2[b] + 31) & ~(int64_t)31);   // t buffer end, whole chunks
    const int32_t wait2 = A.rs.wait2[b];
    double* buf = sm;
    double* ws1 = buf + cap;
    double* ws2 = ws1 + (size_t)maxu1 * kWarps;
    double* ws3 = ws2 + (size_t)maxu2 * kWarps;
    uint32_t* cm = reinterpret_cast<uint32_t*>(ws3 + (size_t)maxu2 * kWarps);
    int32_t* uc1 = reinterpret_cast<int32_t*>(cm + maxnx);
    int32_t* uc2 = uc1 + maxu1 + 1;
    uint16_t* cc = reinterpret_cast<uint16_t*>(uc2 + maxu2 + 1);
    // per-chunk tables of the elements each phase touches -- K1: [e0 - P, e1 + P), K2/K3: [lo2,
    // hi2) -- the ocean bit mask (cm; 0 outside the owned rows) and the grid column of the chunk's
    // first element (cc), so the passes need no integer division
    const int32_t nx1 = e1 > e0 ? (e1 - e0 + 2 * P) >> 5 : 0;
    const int32_t nx2 = f1 > f0 ? (hi2 - lo2) >> 5 : 0;
    for (int q = tid; q < nx1 + nx2; q += NT) {
        const int32_t e = (q < nx1 ? e0 - P + 32 * q : lo2 + 32 * (q - nx1)) - (int32_t)A.hoff;
        uint32_t m = 0u;
        int32_t i = 0;
        if (e >= 0 && e < A.nloc * P) {
            const int32_t j = e / P;
            i = e - j * P;
            m = __ldg(A.ocean + ((int64_t)j * A.nbx + (i >> 8)) * kWarps + ((i & (kBlock - 1)) >> 5));
        }
        cm[q] = m;
        cc[q] = (uint16_t)i;
    }
    for (int u = tid; u <= nu1; u += NT) uc1[u] = (unit_a0(A, ua1 + u) - e0) >> 5;
    for (int u = tid; u <= nu2; u += NT) uc2[u] = (unit_a0(A, ua2 + u) - f0) >> 5;
    double rho = sc->rho, beta = sc->beta, alpha = sc->alpha;
    const double nb = sc->nb, tol = sc->tol;
    int k = sc->k, status = sc->status, xpend = 0;
    const int maxit = sc->maxit;
    bool active = sc->active != 0;
    const bool lead = b == 0 && tid == 0;
    unsigned bar = 0;
    int par = 0;
    __syncthreads();
#ifdef RS_TIMELINE
    unsigned long long tl_prev = rs_now();
#endif
    while (active) {
        RS_T(0);
        // ------------------------------------------------------------------ phase 1 (K1)
        if (e1 > e0) {
            const double* __restrict__ dold = A.d[par];
            double* __restrict__ dnew = A.d[par ^ 1];
            const int32_t D0 = e0 - P;
            const int nD = (e1 - e0 + 2 * P) >> 5, own0 = P >> 5, own1 = own0 + ((e1 - e0) >> 5);
            const int cmD = 0;
            // 1a: d over [D0, D0 + 32 nD) -> buf (land chunks: 0, no loads); own chunks: d -> global,
            // x += alpha_prev d_old
            for (int c0 = warp; c0 < nD; c0 += C::VU * NW) {
                double sv[C::VU], dv[C::VU], xv[C::VU];
                uint32_t m[C::VU];
#pragma unroll
                for (int u = 0; u < C::VU; ++u) {
                    const int c = c0 + u * NW;
                    const int32_t a = D0 + 32 * c + lane;
                    m[u] = c < nD ? cm[cmD + c] : 0u;
                    sv[u] = m[u] ? __ldcg(A.s + a) : 0.0;
                    dv[u] = m[u] ? __ldcg(dold + a) : 0.0;
                    xv[u] = (m[u] && c >= own0 && c < own1) ? __ldcg(A.x + a) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < C::VU; ++u) {
                    const int c = c0 + u * NW;
                    if (c >= nD) break;
                    const int32_t a = D0 + 32 * c + lane;
                    const double d = m[u] ? __fma_rn(beta, dv[u], sv[u]) : 0.0;
                    buf[a - D0] = d;
                    if (m[u] && c >= own0 && c < own1) {
                        dnew[a] = d;
                        A.x[a] = __fma_rn(alpha, dv[u], xv[u]);
                    }
                }
            }
            RS_TS(1);
            // 1b: q = A d on own ocean points, (d, q) warp sums; C::K1C chunks per
            // warp with all their loads issued before any computes
            const double* bd = buf - D0;
            const int nch = (e1 - e0) >> 5, cm1 = P >> 5;
            for (int c0 = warp; c0 < nch; c0 += C::K1C * NW) {
                double cEp[C::K1C], cNr[C::K1C], cNs[C::K1C], cEw[C::K1C], sg[C::K1C];
                uint32_t m[C::K1C];
                int32_t ic[C::K1C];
#pragma unroll
                for (int u = 0; u < C::K1C; ++u) {
                    const int c = c0 + u * NW;
                    const int32_t a = e0 + 32 * c + lane;
                    m[u] = c < nch ? cm[cm1 + c] : 0u;
                    ic[u] = c < nch ? cc[cm1 + c] + lane : 0;
                    const bool ld = m[u] && ic[u] < ni;
                    cEp[u] = ld ? __ldg(A.cE + a) : 0.0;
                    cNr[u] = ld ? __ldg(A.cN + a) : 0.0;
                    cNs[u] = ld ? __ldg(A.cN + a - P) : 0.0;
                    cEw[u] = (ld && (lane == 0 || ic[u] == 0)) ? __ldg(A.cE + (ic[u] == 0 ? a + (ni - 1) : a - 1)) : 0.0;
                    sg[u] = (SIGMA && ld) ? __ldg(A.sigma + a) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < C::K1C; ++u) {
                    const int c = c0 + u * NW;
                    if (c >= nch) break;
                    const int32_t a = e0 + 32 * c + lane, i = ic[u];
                    double v = 0.0;
                    if (m[u]) {
                        const double cEl = __shfl_up_sync(kFull, cEp[u], 1);
                        const double cw = (lane == 0 || i == 0) ? cEw[u] : cEl;
                        if ((m[u] >> lane) & 1u) {
                            const int32_t aw = i == 0 ? a + (ni - 1) : a - 1;
                            const int32_t ae = i == ni - 1 ? a - (ni - 1) : a + 1;
                            const double dC = bd[a], dW = bd[aw], dE = bd[ae], dS = bd[a - P], dN = bd[a + P];
                            const double cNp = fabs(cNr[u]), cNsp = fabs(cNs[u]);
                            double app = __dadd_rn(__dadd_rn(__dadd_rn(cEp[u], cw), cNp), cNsp);
                            if (SIGMA) app = __dadd_rn(app, sg[u]);
                            double acc = __dmul_rn(app, dC);
                            acc = __fma_rn(-cw, dW, acc);
                            acc = __fma_rn(-cEp[u], dE, acc);
                            acc = __fma_rn(-cNsp, dS, acc);
                            acc = __fma_rn(-cNp, dN, acc);
                            A.q[a] = acc;
                            v = __dmul_rn(dC, acc);
                        }
                    }
                    v = warp_tree(v);
                    if (lane == 0) ws1[c] = v;
                }
            }
            __syncthreads();
            rs_partials<NW>(ua1, nu1, uc1, ws1, A.partial[0]);
        }
        RS_T(2);
        xpend = 0;                                           // x += alpha_prev d_old done
        bar += nblk;
        rs_grid_sync(rs_sync, bar);
        RS_T(3);
        const double gamma = rs_final<C::NB>(A.partial[0], U, bc);
        RS_T(4);
        if (!(gamma > 0.0) || !isfinite(gamma)) { status = kStBreakdown; break; }
        alpha = __ddiv_rn(rho, gamma);
        // ------------------------------------------------------------------ phase 2 (K2, K3)
        // (no emptiness guard: a block without phase-2 units still publishes its t-ready stamp,
        // which the blocks to its south may wait for; every loop below is then empty)
        {
            const double* __restrict__ ro = A.r[par];
            double* __restrict__ rn = A.r[par ^ 1];
            const int nch = (f1 - f0) >> 5;
            const int cmF = nx1 + ((f0 - lo2) >> 5);
            if (PC == 0) {
                if (tid == 0 && nch > 0) {                      // this block's overflow rows -> L2
                    const int64_t* pf = A.rs.pf + 4 * (int64_t)b;
                    if (pf[1] > 0) {
                        prefetch_l2(A.zt.oval + pf[0], (uint64_t)pf[1] * 8);
                        prefetch_l2(A.zt.ocol + pf[0], (uint64_t)pf[1] * 4);
                    }
                    if (pf[3] > 0) {
                        prefetch_l2(A.z.oval + pf[2], (uint64_t)pf[3] * 8);
                        prefetch_l2(A.z.ocol + pf[2], (uint64_t)pf[3] * 4);
                    }
                }
                // 2A: r_new over [lo2, f1) -> buf; own chunks: r_new -> global, (r, r) warp sums
                const int nR = (f1 - lo2) >> 5, own0 = (f0 - lo2) >> 5, cmR = nx1;
                for (int c0 = warp; c0 < nR; c0 += C::VU * NW) {
                    double qv[C::VU], rv[C::VU];
                    uint32_t m[C::VU];
#pragma unroll
                    for (int u = 0; u < C::VU; ++u) {
                        const int c = c0 + u * NW;
                        const int32_t a = lo2 + 32 * c + lane;
                        m[u] = c < nR ? cm[cmR + c] : 0u;
                        qv[u] = m[u] ? __ldcg(A.q + a) : 0.0;
                        rv[u] = m[u] ? __ldcg(ro + a) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < C::VU; ++u) {
                        const int c = c0 + u * NW;
                        if (c >= nR) break;
                        const int32_t a = lo2 + 32 * c + lane;
                        const double rnew = m[u] ? __fma_rn(-alpha, qv[u], rv[u]) : 0.0;
                        buf[a - lo2] = rnew;
                        if (c >= own0) {
                            const bool live = (m[u] >> lane) & 1u;
                            if (live) rn[a] = rnew;
                            const double v = warp_tree(live ? __dmul_rn(rnew, rnew) : 0.0);
                            if (lane == 0) ws2[c - own0] = v;
                        }
                    }
                }
                RS_TS(5);
                // 2B: t = Dhat^-1 Z^T r_new on own ocean points, C::ZC chunks per warp in flight
                const double* rb = buf - lo2;
                for (int c0 = warp; c0 < nch; c0 += C::ZC * NW) {
                    double z[C::ZC][kEll], pv[C::ZC];
                    uint2 cw[C::ZC];
                    int32_t o0[C::ZC], ol[C::ZC];
                    uint32_t m[C::ZC];
#pragma unroll
                    for (int u = 0; u < C::ZC; ++u) {
                        const int c = c0 + u * NW;
                        const int32_t a = f0 + 32 * c + lane, e = a - (int32_t)A.hoff;
                        m[u] = c < nch ? cm[cmF + c] : 0u;
                        const bool live = (m[u] >> lane) & 1u;
                        z[u][0] = z[u][1] = z[u][2] = z[u][3] = 0.0;
                        if (live) ld_nc_f64x4(A.zt.val + (int64_t)e * kEll, z[u]);
                        cw[u] = live ? __ldg(reinterpret_cast<const uint2*>(A.zt.col16) + e) : make_uint2(0u, 0u);
                        pv[u] = live ? __ldg(A.piv + a) : 1.0;
                        const int64_t oa = m[u] ? __ldg(A.zt.ooff + (e >> 5)) : 0;
                        const int64_t ob = m[u] ? __ldg(A.zt.ooff + (e >> 5) + 1) : 0;
                        o0[u] = (int32_t)oa;
                        ol[u] = (int32_t)((ob - oa) >> 5);
                    }
#pragma unroll
                    for (int u = 0; u < C::ZC; ++u) {
                        if (!m[u]) continue;
                        const int32_t a = f0 + 32 * (c0 + u * NW) + lane;
                        const double acc = rs_row<C::OVF>(z[u], cw[u], o0[u], ol[u], a, rb, A.zt.oval, A.zt.ocol);
                        if ((m[u] >> lane) & 1u) A.t[a] = __ddiv_rn(acc, pv[u]);
                    }
                }
                // publish this block's t; copy it to buf while the blocks its Z rows reach finish
                // theirs, then wait for their stamps and copy their t
                RS_TS(6);
                const unsigned stamp = (unsigned)k + 1u;
                if (tid == 0) {
                    __threadfence();
                    st_release_u32(rs_sync + 1 + b, stamp);
                }
                // 2C: t over [f0, hi2) -> buf (land chunks: 0); the own chunks [0, nOwn) first
                const int nT = (hi2 - f0) >> 5, nOwn = (f1 - f0) >> 5;
#pragma unroll 1
                for (int pass = 0; pass < 2; ++pass) {              // own chunks, then the rest
                    const int cbeg = pass ? nOwn : 0, cend = pass ? nT : nOwn;
                    for (int c0 = cbeg + warp; c0 < cend; c0 += C::VU * NW) {
                        double tv[C::VU];
#pragma unroll
                        for (int u = 0; u < C::VU; ++u) {
                            const int c = c0 + u * NW;
                            tv[u] = (c < cend && cm[cmF + c]) ? __ldcg(A.t + f0 + 32 * c + lane) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < C::VU; ++u) {
                            const int c = c0 + u * NW;
                            if (c < cend) buf[32 * c + lane] = tv[u];
                        }
                    }
                    if (pass == 0) {
                        if (tid == 0)
                            for (int bb = b + 1; bb <= wait2; ++bb) rs_spin(rs_sync + 1 + bb, stamp, 1u + (unsigned)bb);
                        RS_TS(7);
                    }
                }
                RS_TS(8);
                // 2D: s = Z t on own ocean points, (s, r_new) warp sums, C::ZC chunks per warp in flight
                const double* tb = buf - f0;
                for (int c0 = warp; c0 < nch; c0 += C::ZC * NW) {
                    double z[C::ZC][kEll], rv[C::ZC];
                    uint2 cw[C::ZC];
                    int32_t o0[C::ZC], ol[C::ZC];
                    uint32_t m[C::ZC];
#pragma unroll
                    for (int u = 0; u < C::ZC; ++u) {
                        const int c = c0 + u * NW;
                        const int32_t a = f0 + 32 * c + lane, e = a - (int32_t)A.hoff;
                        m[u] = c < nch ? cm[cmF + c] : 0u;
                        const bool live = (m[u] >> lane) & 1u;
                        z[u][0] = z[u][1] = z[u][2] = z[u][3] = 0.0;
                        if (live) ld_nc_f64x4(A.z.val + (int64_t)e * kEll, z[u]);
                        cw[u] = live ? __ldg(reinterpret_cast<const uint2*>(A.z.col16) + e) : make_uint2(0u, 0u);
                        rv[u] = live ? __ldcg(rn + a) : 0.0;
                        const int64_t oa = m[u] ? __ldg(A.z.ooff + (e >> 5)) : 0;
                        const int64_t ob = m[u] ? __ldg(A.z.ooff + (e >> 5) + 1) : 0;
                        o0[u] = (int32_t)oa;
                        ol[u] = (int32_t)((ob - oa) >> 5);
                    }
#pragma unroll
                    for (int u = 0; u < C::ZC; ++u) {
                        const int c = c0 + u * NW;
                        if (c >= nch) break;
                        const int32_t a = f0 + 32 * c + lane;
                        double v = 0.0;
                        if (m[u]) {
                            const double acc = rs_row<C::OVF>(z[u], cw[u], o0[u], ol[u], a, tb, A.z.oval, A.z.ocol);
                            if ((m[u] >> lane) & 1u) {
                                A.s[a] = acc;
                                v = __dmul_rn(acc, rv[u]);
                            }
                        }
                        v = warp_tree(v);
                        if (lane == 0) ws3[c] = v;
                    }
                }
            } else {
                // Jacobi / none: r_new, s = r_new / A_pp (or r_new), (r, r), (s, r) in one pass
                for (int c0 = warp; c0 < nch; c0 += C::VU * NW) {
                    double qv[C::VU], rv[C::VU], dv[C::VU];
                    uint32_t m[C::VU];
#pragma unroll
                    for (int u = 0; u < C::VU; ++u) {
                        const int c = c0 + u * NW;
                        const int32_t a = f0 + 32 * c + lane;
                        m[u] = c < nch ? cm[cmF + c] : 0u;
                        qv[u] = m[u] ? __ldcg(A.q + a) : 0.0;
                        rv[u] = m[u] ? __ldcg(ro + a) : 0.0;
                        dv[u] = (PC == 1 && m[u]) ? __ldg(A.diag + a) : 1.0;
                    }
#pragma unroll
                    for (int u = 0; u < C::VU; ++u) {
                        const int c = c0 + u * NW;
                        if (c >= nch) break;
                        const int32_t a = f0 + 32 * c + lane;
                        double v1 = 0.0, v2 = 0.0;
                        if (m[u]) {
                            const double rnew = __fma_rn(-alpha, qv[u], rv[u]);
                            const double sv = PC == 2 ? rnew : __ddiv_rn(rnew, dv[u]);
                            A.s[a] = sv;
                            rn[a] = rnew;
                            v1 = __dmul_rn(rnew, rnew);
                            v2 = __dmul_rn(sv, rnew);
                        }
                        v1 = warp_tree(v1);
                        v2 = warp_tree(v2);
                        if (lane == 0) { ws2[c] = v1; ws3[c] = v2; }
                    }
                }
            }
            __syncthreads();
            rs_partials<NW>(ua2, nu2, uc2, ws2, A.partial[1]);
            rs_partials<NW>(ua2, nu2, uc2, ws3, A.partial[2]);
        }
        RS_T(9);
        bar += nblk;
        rs_grid_sync(rs_sync, bar);
        RS_T(10);
        double rr, rho_new;
        rs_final2<C::NB2>(A.partial[1], A.partial[2], U, bc, rr, rho_new);
        RS_T(11);
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

template <bool SIGMA, int NT>
const void* rs_fn(int pc) {
    if (pc == 1) return (const void*)rs_loop_kernel<SIGMA, 1, NT>;
    if (pc == 2) return (const void*)rs_loop_kernel<SIGMA, 2, NT>;
    return (const void*)rs_loop_kernel<SIGMA, 0, NT>;
}

}  // namespace

// diagnostic: copy (and reset) the per-block pass durations of -DRS_TIMELINE builds; 0 otherwise
int rs_timeline(unsigned long long* out, int nblk) {
#ifdef RS_TIMELINE
    const size_t n = (size_t)std::min(nblk, 160) * 12;
    cudaMemcpyFromSymbol(out, g_rs_tl, n * sizeof(unsigned long long));
    static unsigned long long zero[160 * 12];
    cudaMemcpyToSymbol(g_rs_tl, zero, sizeof(zero));
    return 1;
#else
    (void)out; (void)nblk;
    return 0;
#endif
}

size_t rs_smem_bytes(int32_t cap, int32_t maxu1, int32_t maxu2, int32_t maxnx) {
    return (size_t)cap * 8 + (size_t)(maxu1 + 2 * maxu2) * kWarps * 8 + (size_t)maxnx * 4 +
           (size_t)(maxu1 + maxu2 + 2) * 4 + (size_t)maxnx * 2 + 16;
}

const void* rs_kernel_fn(const KArgs& A) {
    if (A.rs.nt == 768) return A.sigma ? rs_fn<true, 768>(A.precond) : rs_fn<false, 768>(A.precond);
    return A.sigma ? rs_fn<true, 512>(A.precond) : rs_fn<false, 512>(A.precond);
}

cudaError_t launch_rs(const KArgs& A, cudaStream_t st) {
    const void* fn = rs_kernel_fn(A);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)A.rs.smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)A.rs.nblk);
    cfg.blockDim = dim3((unsigned)A.rs.nt);
    cfg.dynamicSmemBytes = A.rs.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned n = 0;
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
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
    void* args[] = {(void*)&A};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace pcg
