// ellbench.cu -- attribution microbenchmark for the K3 shape (ELL(4) gather + dot product) on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ellbench tools/ellbench.cu && ./tools/ellbench
// Variants (all read val[4][n], col[4][n], rn[n], write s[n]):
//   A  stream: x = t[e] (no gather), no reduction
//   B  gather: x = t[e + off(col)], no reduction
//   C  B + per-block reduction (block tree, fence, atomic ticket), one element per thread
//   D  B + persistent grid-stride, warp sums in shared memory, one ticket per block
//   E  D with 2 units per loop iteration
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int B = 256;
__device__ unsigned g_counter;
__device__ double g_sink;

__device__ __forceinline__ double warp_tree(double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

template <bool GATHER>
__device__ __forceinline__ double row(const double* __restrict__ val, const int32_t* __restrict__ col,
                                      const double* __restrict__ t, long n, long e, int P) {
    int32_t c[4]; double z[4], x[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) { c[m] = __ldg(col + m * n + e); z[m] = __ldg(val + m * n + e); }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        long g = GATHER ? e + (c[m] & 3) + (long)(c[m] >> 2) * P : e;
        x[m] = __ldg(t + g);
    }
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) acc = fma(z[m], x[m], acc);
    return acc;
}

template <bool GATHER>
__global__ void kA(const double* val, const int32_t* col, const double* t, const double* rn, double* s, long n, int P) {
    long e = blockIdx.x * (long)B + threadIdx.x;
    if (e >= n) return;
    double acc = row<GATHER>(val, col, t, n, e, P);
    s[e] = acc;
    if (acc * rn[e] == 1234.5) g_sink = acc;
}

__global__ void kC(const double* val, const int32_t* col, const double* t, const double* rn, double* s, double* part, long n, int P) {
    __shared__ double ws[8];
    __shared__ bool last;
    long e = blockIdx.x * (long)B + threadIdx.x;
    double v = 0.0;
    if (e < n) { double acc = row<true>(val, col, t, n, e, P); s[e] = acc; v = acc * rn[e]; }
    v = warp_tree(v);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double u = threadIdx.x < 8 ? ws[threadIdx.x] : 0.0;
        u = warp_tree(u);
        if (threadIdx.x == 0) { part[blockIdx.x] = u; __threadfence(); last = atomicAdd(&g_counter, 1u) == gridDim.x - 1; }
    }
    __syncthreads();
    if (last && threadIdx.x == 0) g_counter = 0;
}

template <int UNROLL>
__global__ void kD(const double* val, const int32_t* col, const double* t, const double* rn, double* s, double* part, long n, int P) {
    extern __shared__ double ws[];
    __shared__ bool last;
    long units = (n + B - 1) / B;
    int k = 0;
    for (long u = blockIdx.x; u < units; u += (long)gridDim.x * UNROLL) {
        double v[UNROLL];
#pragma unroll
        for (int q = 0; q < UNROLL; ++q) {
            long uu = u + (long)q * gridDim.x;
            long e = uu * B + threadIdx.x;
            v[q] = 0.0;
            if (uu < units && e < n) { double acc = row<true>(val, col, t, n, e, P); s[e] = acc; v[q] = acc * rn[e]; }
        }
#pragma unroll
        for (int q = 0; q < UNROLL; ++q) {
            double w = warp_tree(v[q]);
            if ((threadIdx.x & 31) == 0) ws[(k + q) * 8 + (threadIdx.x >> 5)] = w;
        }
        k += UNROLL;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        for (int kk = 0; kk < k; ++kk) {
            double u = threadIdx.x < 8 ? ws[kk * 8 + threadIdx.x] : 0.0;
            u = warp_tree(u);
            if (threadIdx.x == 0) part[blockIdx.x * 64 + kk] = u;
        }
        if (threadIdx.x == 0) { __threadfence(); last = atomicAdd(&g_counter, 1u) == gridDim.x - 1; }
    }
    __syncthreads();
    if (last && threadIdx.x == 0) g_counter = 0;
}

template <class F>
float timed(cudaStream_t st, F launch) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < 30; ++k) launch();
    cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    return best * 1e3f / 30.0f;
}

int main() {
    const int P = 1472;
    const long n = (long)P * 1021;
    double *val, *t, *rn, *s, *part; int32_t* col;
    cudaMalloc(&val, 4 * n * 8); cudaMalloc(&col, 4 * n * 4); cudaMalloc(&t, (n + 8 * P) * 8);
    cudaMalloc(&rn, n * 8); cudaMalloc(&s, n * 8); cudaMalloc(&part, 1 << 24);
    cudaMemset(val, 0, 4 * n * 8); cudaMemset(t, 0, (n + 8 * P) * 8); cudaMemset(rn, 0, n * 8);
    // columns: offsets (0,0) (1,0) (0,1) (0,2) as (di + 4*dj)
    int32_t* hc = new int32_t[4 * n];
    for (long e = 0; e < n; ++e) { hc[e] = 0; hc[n + e] = 1; hc[2 * n + e] = 4; hc[3 * n + e] = 8; }
    cudaMemcpy(col, hc, 4 * n * 4, cudaMemcpyHostToDevice);
    cudaStream_t st; cudaStreamCreate(&st);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned G = (unsigned)((n + B - 1) / B);
    const double bytes = n * (4 * 8 + 4 * 4 + 8 + 8 + 8.0);
    auto rep = [&](const char* name, float us) { printf("%-34s %7.2f us  %7.1f GB/s (alg %.0f MB)\n", name, us, bytes / (us * 1e-6) / 1e9, bytes / 1e6); };
    rep("A stream (no gather, no reduce)", timed(st, [&] { kA<false><<<G, B, 0, st>>>(val, col, t, rn, s, n, P); }));
    rep("B gather, no reduce", timed(st, [&] { kA<true><<<G, B, 0, st>>>(val, col, t, rn, s, n, P); }));
    rep("C gather + per-block ticket", timed(st, [&] { kC<<<G, B, 0, st>>>(val, col, t, rn, s, part, n, P); }));
    for (int occ : {2, 4, 6, 8}) {
        unsigned g = sms * occ;
        char nm[64];
        snprintf(nm, 64, "D persistent grid=%d", g);
        rep(nm, timed(st, [&] { kD<1><<<g, B, 64 * 8 * 8, st>>>(val, col, t, rn, s, part, n, P); }));
        snprintf(nm, 64, "E persistent x2 grid=%d", g);
        rep(nm, timed(st, [&] { kD<2><<<g, B, 64 * 8 * 8, st>>>(val, col, t, rn, s, part, n, P); }));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
