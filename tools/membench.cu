// membench.cu -- calibration of achievable bandwidth for K1-like traffic on B200 (fp64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu && ./membench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_stream(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ c,
                         const double* __restrict__ d, const double* __restrict__ e, double* __restrict__ x,
                         double* __restrict__ y, double* __restrict__ z, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        double s = a[i] + b[i] * c[i] + d[i] - e[i];
        x[i] = s; y[i] = s * 2.0; z[i] = s * 3.0;
    }
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ x, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) x[i] = a[i];
}

__global__ void k_empty() {}

int main() {
    const long n = 1472L * 1023;     // cfg4 pitched elements incl. halos
    double* buf[8];
    for (int k = 0; k < 8; ++k) { cudaMalloc(&buf[k], n * 8); cudaMemset(buf[k], 0, n * 8); }
    double* big; cudaMalloc(&big, 512L << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int grid : {sms * 2, sms * 4, sms * 8, (int)((n + 255) / 256)}) {
        for (int flush = 0; flush < 2; ++flush) {
            float best = 1e9;
            for (int rep = 0; rep < 20; ++rep) {
                if (flush) cudaMemset(big, rep, 512L << 20);
                cudaEventRecord(e0);
                k_stream<<<grid, 256>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], n);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
            }
            printf("stream5r3w grid=%6d flushL2=%d : %7.2f us  %7.1f GB/s\n", grid, flush, best * 1e3, 8.0 * 8 * n / (best * 1e-3) / 1e9);
        }
    }
    // big copy for the HBM reference
    const long nb = (256L << 20) / 8;
    double* src = big; double* dst = big + nb;
    float best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(e0); k_copy<<<sms * 8, 256>>>(src, dst, nb); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("copy 256MB: %7.2f us  %7.1f GB/s\n", best * 1e3, 2.0 * 8 * nb / (best * 1e-3) / 1e9);
    best = 1e9;
    for (int rep = 0; rep < 50; ++rep) {
        cudaEventRecord(e0); k_empty<<<1, 32>>>(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("empty kernel: %7.2f us\n", best * 1e3);
    // 3 back-to-back stream kernels (K1,K2,K3-like) in a graph: launch gaps
    cudaStream_t st; cudaStreamCreate(&st);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < 30; ++k) k_stream<<<sms * 8, 256, 0, st>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], n);
    cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
    best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("30 stream kernels in a graph: %7.2f us per kernel  %7.1f GB/s\n", best * 1e3 / 30, 30 * 8.0 * 8 * n / (best * 1e-3) / 1e9);
    return 0;
}
