// dev_common.cuh -- device helpers shared by the iteration kernels (kernels.cu) and the
// resident-strip solver (rs.cu): the canonical reduction trees of DESIGN.md §5.2 and the
// 256-bit non-coherent load.  Included inside an anonymous namespace of each translation unit.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace pcg {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = kBlock / 32;

__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(kFull, v, off));
    return v;
}

// Block tree (kBlock threads): result valid in thread 0.
// Threads beyond kBlock (the producer warp of the TMA kernels) take part in the barriers only.
__device__ __forceinline__ double block_tree(double v) {
    __shared__ double wsb[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_tree(v);
    __syncthreads();                       // wsb may still be read by a previous call
    if (lane == 0 && w < kWarps) wsb[w] = v;
    __syncthreads();
    double u = 0.0;
    if (w == 0) {
        u = lane < kWarps ? wsb[lane] : 0.0;
        u = warp_tree(u);
    }
    return u;
}

// In the last block: thread t sums partials t, t+B, ... left to right, then the block tree.
// NB loads per thread are issued before their adds (NB = 32: G <= 8192 in one L2 round trip);
// kernels with a tight register budget use a smaller NB so the walk does not force spills into
// their main loop.
template <int NB = 32>
__device__ __forceinline__ double final_sum(const double* partial, int64_t G) {
    double acc = 0.0;
    int64_t m = threadIdx.x < kBlock ? (int64_t)threadIdx.x : G;
    for (; m < G; m += NB * kBlock) {
        double p[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) p[u] = m + u * kBlock < G ? __ldcg(partial + m + u * kBlock) : 0.0;
#pragma unroll
        for (int u = 0; u < NB; ++u)
            if (m + u * kBlock < G) acc = __dadd_rn(acc, p[u]);
    }
    return block_tree(acc);
}

__device__ __forceinline__ void ld_nc_f64x4(const double* p, double (&z)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(z[0]), "=d"(z[1]), "=d"(z[2]), "=d"(z[3]) : "l"(p));
}

}  // namespace
}  // namespace pcg
