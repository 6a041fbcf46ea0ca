// devcomm.cu -- setup of the device-comm window (PCG_FLAG_DEVICE_COMM) and the
// protocol self-test of dev_comm.cuh.
//
// The window is one symmetric NCCL window per context (ncclMemAlloc + ncclCommWindowRegister,
// collective over the communicator); the peer pointers of every rank are read once, on the
// device, with ncclGetPeerPointer and kept in a small device array that the reduction kernels
// index directly.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "dev_comm.cuh"
#include "../../include/libpcg.h"

namespace pcg {
void set_thread_error(const std::string& m);

namespace {

__global__ void dc_peer_kernel(ncclWindow_t win, int P, char** out, int rank, int64_t south_off, int64_t north_off,
                               double** halo) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) out[p] = static_cast<char*>(ncclGetPeerPointer(win, 0, p));
    if (threadIdx.x == 0) {
        halo[0] = south_off >= 0 ? static_cast<double*>(ncclGetPeerPointer(win, (size_t)south_off, rank - 1)) : nullptr;
        halo[1] = north_off >= 0 ? static_cast<double*>(ncclGetPeerPointer(win, (size_t)north_off, rank + 1)) : nullptr;
    }
}

// P virtual ranks in one cooperative launch (block r = rank r, thread 0 does the protocol), over
// P windows carved from one device buffer.  Round k: rank r's four sums are v(k, r, q) (a fixed
// hash, so every rank knows every value); each rank gathers and forms the canonical rank tree of
// every slot into out[k][r][q].
__device__ double dc_test_value(uint64_t seed, int k, int r, int q) {
    uint64_t x = seed ^ (0x9e3779b97f4a7c15ull * (uint64_t)(k * 131 + r * 7 + q + 1));
    x ^= x >> 31; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 29; x *= 0x94d049bb133111ebull; x ^= x >> 32;
    return (double)(int64_t)(x & 0xfffffffffffffull) * 0x1p-40 - 2048.0;
}

__global__ void dc_selftest_kernel(char* base, int P, int rounds, uint64_t seed, uint32_t* seqs, double* gath,
                                   double* out) {
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x;
    char* peer[kDcMaxRanks];
    for (int p = 0; p < P; ++p) peer[p] = base + (size_t)p * kDcWindowBytes;
    double* g = gath + (size_t)me * kDcMaxRanks * 4;
    for (int k = 0; k < rounds; ++k) {
        double loc[4];
        for (int q = 0; q < 4; ++q) loc[q] = dc_test_value(seed, k, me, q);
        if (k & 1) {
            dc_publish(peer, P, me, seqs + me, loc);        // the pipelined split form
            dc_collect(peer, P, me, seqs + me, g);
        } else {
            dc_allgather(peer, P, me, seqs + me, loc, g);
        }
        for (int q = 0; q < 4; ++q) {
            double u[32];
            for (int l = 0; l < 32; ++l) u[l] = l < P ? g[l * 4 + q] : 0.0;
            for (int off = 16; off >= 1; off >>= 1)
                for (int l = 0; l + off < 32; ++l) u[l] = __dadd_rn(u[l], u[l + off]);
            out[((size_t)k * P + me) * 4 + q] = u[0];
        }
    }
}

}  // namespace

// window + peer pointers of one context; called collectively by every rank of the communicator.
// With halo stores (DcHalo::on) the window also holds this rank's s array (the vector K3 writes
// and the next K1's stencil reads on the halo rows): region [kDcSOffset, kDcSOffset + 8 * max_r
// nel_r) on every rank, and the pointers to the rows of the neighbours' s arrays this rank's first
// and last owned rows are copied into (their northern / southern halo rows) are read here once.
int dc_setup(ncclComm_t comm, int nranks, int rank, const DcHalo& h, DcOut& out, cudaStream_t st, std::string& err) {
    if (nranks > kDcMaxRanks) { err = "device comm: at most 32 ranks"; return PCG_ERR_ARG; }
    const ncclTeam_t lsa = ncclTeamLsa(comm);
    if (lsa.nRanks != nranks) {
        err = "device comm: every rank must be load/store reachable (one NVLink domain); LSA team has " +
              std::to_string(lsa.nRanks) + " of " + std::to_string(nranks) + " ranks";
        return PCG_ERR_COMM;
    }
    // every rank's (nloc, nel) -- the neighbours' halo rows and the largest s array
    int64_t* dinfo = nullptr;
    if (cudaMalloc(&dinfo, sizeof(int64_t) * 2 * nranks) != cudaSuccess) { err = "device comm: cudaMalloc failed"; return PCG_ERR_CUDA; }
    const int64_t mine[2] = {h.nloc, h.nel};
    cudaMemcpyAsync(dinfo + 2 * rank, mine, sizeof(mine), cudaMemcpyHostToDevice, st);
    ncclResult_t r = ncclAllGather(dinfo + 2 * rank, dinfo, 2, ncclInt64, comm, st);
    std::vector<int64_t> info((size_t)2 * nranks);
    if (r != ncclSuccess || cudaMemcpyAsync(info.data(), dinfo, sizeof(int64_t) * 2 * nranks, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        cudaFree(dinfo);
        err = std::string("device comm: setup allgather failed: ") + ncclGetErrorString(r);
        return PCG_ERR_COMM;
    }
    cudaFree(dinfo);
    int64_t max_nel = 0;
    for (int q = 0; q < nranks; ++q) max_nel = std::max<int64_t>(max_nel, info[(size_t)2 * q + 1]);
    const size_t bytes = h.on ? kDcSOffset + (size_t)max_nel * sizeof(double) : kDcWindowBytes;
    void* buf = nullptr;
    r = ncclMemAlloc(&buf, bytes);
    if (r != ncclSuccess) { err = std::string("ncclMemAlloc: ") + ncclGetErrorString(r); return PCG_ERR_COMM; }
    if (cudaMemsetAsync(buf, 0, bytes, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        ncclMemFree(buf);
        err = "device comm: window memset failed";
        return PCG_ERR_CUDA;
    }
    ncclWindow_t w = nullptr;
    r = ncclCommWindowRegister(comm, buf, bytes, &w, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        ncclMemFree(buf);
        err = std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r);
        return PCG_ERR_COMM;
    }
    char** pp = nullptr;
    uint32_t* sq = nullptr;
    double** hp = nullptr;
    if (cudaMalloc(&pp, sizeof(char*) * nranks) != cudaSuccess || cudaMalloc(&sq, sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&hp, 2 * sizeof(double*)) != cudaSuccess) {
        ncclCommWindowDeregister(comm, w);
        ncclMemFree(buf);
        err = "device comm: cudaMalloc failed";
        return PCG_ERR_CUDA;
    }
    cudaMemsetAsync(sq, 0, sizeof(uint32_t), st);
    // neighbours' halo rows: rank-1's northern one (array row H + nloc_{r-1}), rank+1's southern
    // one (array row H - 1); the pitch and H are the same on every rank
    const int64_t south_off = rank > 0 ? (int64_t)kDcSOffset + (h.halo + info[(size_t)2 * (rank - 1)]) * h.pitch * 8 : -1;
    const int64_t north_off = rank < nranks - 1 ? (int64_t)kDcSOffset + (int64_t)(h.halo - 1) * h.pitch * 8 : -1;
    dc_peer_kernel<<<1, 32, 0, st>>>(w, nranks, pp, rank, h.on ? south_off : -1, h.on ? north_off : -1, hp);
    double* hh[2] = {nullptr, nullptr};
    if (cudaMemcpyAsync(hh, hp, sizeof(hh), cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        err = "device comm: peer pointers";
        return PCG_ERR_CUDA;
    }
    cudaFree(hp);
    // every rank's window is zero before any rank can store into it
    r = ncclAllReduce(sq, sq, 1, ncclUint32, ncclSum, comm, st);   // sq = 0 on every rank: stays 0
    if (r != ncclSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        err = std::string("device comm: setup barrier failed: ") + ncclGetErrorString(r);
        return PCG_ERR_COMM;
    }
    out.win_buf = buf; out.win = (void*)w; out.peers = pp; out.seq = sq;
    out.s = h.on ? reinterpret_cast<double*>(static_cast<char*>(buf) + kDcSOffset) : nullptr;
    out.south = hh[0]; out.north = hh[1];
    return PCG_OK;
}

void dc_free(ncclComm_t comm, void* win_buf, void* win, char** peers, uint32_t* seq) {
    if (win) ncclCommWindowDeregister(comm, (ncclWindow_t)win);
    if (win_buf) ncclMemFree(win_buf);
    if (peers) cudaFree(peers);
    if (seq) cudaFree(seq);
}

}  // namespace pcg

extern "C" pcg_status pcg_devcomm_selftest(int32_t nranks, int32_t rounds, uint64_t seed, double* out) {
    using namespace pcg;
    if (nranks < 1 || nranks > kDcMaxRanks || rounds < 1 || !out) return PCG_ERR_ARG;
    char* base = nullptr;
    uint32_t* seqs = nullptr;
    double *gath = nullptr, *dout = nullptr;
    const size_t nout = (size_t)rounds * nranks * 4;
    pcg_status rc = PCG_OK;
    if (cudaMalloc(&base, kDcWindowBytes * nranks) != cudaSuccess || cudaMalloc(&seqs, sizeof(uint32_t) * nranks) != cudaSuccess ||
        cudaMalloc(&gath, sizeof(double) * nranks * kDcMaxRanks * 4) != cudaSuccess ||
        cudaMalloc(&dout, sizeof(double) * nout) != cudaSuccess) {
        rc = PCG_ERR_CUDA;
    } else {
        cudaMemset(base, 0, kDcWindowBytes * nranks);
        cudaMemset(seqs, 0, sizeof(uint32_t) * nranks);
        int P = nranks, R = rounds;
        void* args[] = {(void*)&base, (void*)&P, (void*)&R, (void*)&seed, (void*)&seqs, (void*)&gath, (void*)&dout};
        // cooperative: all P blocks co-resident, so ranks that wait on one another make progress
        if (cudaLaunchCooperativeKernel((const void*)dc_selftest_kernel, dim3(nranks), dim3(32), args, 0, 0) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess ||
            cudaMemcpy(out, dout, sizeof(double) * nout, cudaMemcpyDeviceToHost) != cudaSuccess) {
            set_thread_error("pcg_devcomm_selftest: " + std::string(cudaGetErrorString(cudaGetLastError())));
            rc = PCG_ERR_CUDA;
        }
    }
    cudaFree(base); cudaFree(seqs); cudaFree(gath); cudaFree(dout);
    return rc;
}
