// dev_comm.cuh -- device-side allgather of the per-rank sums (PCG_FLAG_DEVICE_COMM).
//
// Every reduction of Alg. 1 ((d, q) before line 7, (s, r) and (r, r) before
// line 8) ends, on each rank, in the last block of the kernel that formed the rank's block-tree
// sums (DevScalars::loc).  With device comm that block's thread 0 stores the four sums straight
// into every rank's window over NVLink (peer pointers from ncclGetPeerPointer on a symmetric
// NCCL window), publishes a stamp, waits for every rank's stamp in its own window and leaves the
// gathered sums in A.gath in rank order -- the layout ncclAllGather produces -- so the canonical
// rank tree and the scalar step run inline, bitwise as after the host-enqueued
// allgather.  No NCCL call, no scalar-kernel launch, no host round trip.
//
// Window layout (bytes, identical on every rank): [0, 256) stamps u32 [2][32] (slot parity x
// source rank); [256, 2304) sums double [2][32][4].  Reduction n (a per-context sequence number
// every rank advances identically) uses slot n & 1 and stamp n.  A rank can be at most one
// reduction ahead of any other (it cannot pass reduction n+1 before every rank published n+1, and
// a rank publishes n+1 only after reading n), so the two slots never hold a value still unread.
#pragma once
#include <cstdint>

namespace pcg {

constexpr int kDcMaxRanks = 32;
constexpr size_t kDcStampBytes = 2 * kDcMaxRanks * sizeof(uint32_t);
constexpr size_t kDcWindowBytes = kDcStampBytes + 2 * kDcMaxRanks * 4 * sizeof(double);
constexpr size_t kDcSOffset = 4096;                 // the s array in the window (halo stores)

// host side of the window setup (devcomm.cu)
struct DcHalo {
    bool on;                                        // s in the window, halo rows stored by K3
    int64_t nloc, nel, pitch, halo;                 // this rank's owned rows, s elements, pitch, halo rows
};
struct DcOut {
    void *win_buf = nullptr, *win = nullptr;
    char** peers = nullptr;                         // [nranks] window bases (device array)
    uint32_t* seq = nullptr;
    double* s = nullptr;                            // this rank's s array inside the window
    double *south = nullptr, *north = nullptr;      // rank-1's northern / rank+1's southern halo row of s
};

#ifdef __CUDACC__
__device__ __forceinline__ void dc_st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dc_ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double dc_ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Watchdog: a rank that waits ~4 s for a stamp records (rank, source, stamp seen, expected) and
// traps, so a protocol error ends the kernel with an error instead of hanging the GPU.
static __device__ unsigned g_dc_hang[4];

// One thread.  peer[p] = base of rank p's window (peer[me] = this rank's own), seq = this rank's
// reduction counter, loc = the 4 sums of this rank, gath = [P][4] out.
// dc_publish advances the counter and stores this rank's sums + stamp at every rank; dc_collect
// waits for every rank's stamp of the current reduction in the own window and reads the sums.
// Pipelined PCG publishes at the end of KPC and collects in the next KPA (the wait overlaps the
// other blocks' work); every other reduction does both at once (dc_allgather).
__device__ __forceinline__ void dc_publish(char* const* peer, int P, int me, uint32_t* seq, const double* loc) {
    const uint32_t n = *seq + 1u;
    *seq = n;
    const int s = (int)(n & 1u);
    const double l0 = loc[0], l1 = loc[1], l2 = loc[2], l3 = loc[3];
    for (int p = 0; p < P; ++p) {
        double* v = reinterpret_cast<double*>(peer[p] + kDcStampBytes) + ((size_t)s * kDcMaxRanks + me) * 4;
        v[0] = l0; v[1] = l1; v[2] = l2; v[3] = l3;
    }
    __threadfence_system();                             // the sums before any stamp, at every peer
    for (int p = 0; p < P; ++p)
        dc_st_release_sys(reinterpret_cast<uint32_t*>(peer[p]) + s * kDcMaxRanks + me, n);
}

__device__ __forceinline__ void dc_collect(char* const* peer, int P, int me, const uint32_t* seq, double* gath) {
    const uint32_t n = *seq;
    const int s = (int)(n & 1u);
    const uint32_t* st = reinterpret_cast<const uint32_t*>(peer[me]) + s * kDcMaxRanks;
    const double* vals = reinterpret_cast<const double*>(peer[me] + kDcStampBytes) + (size_t)s * kDcMaxRanks * 4;
    for (int r = 0; r < P; ++r) {
        unsigned long long spin = 0;
        uint32_t got;
        while ((got = dc_ld_acquire_sys(st + r)) != n) {
            if (++spin > (1ull << 27)) {
                g_dc_hang[0] = (unsigned)me; g_dc_hang[1] = (unsigned)r; g_dc_hang[2] = got; g_dc_hang[3] = n;
                __threadfence_system();
                __trap();
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) gath[r * 4 + q] = dc_ld_relaxed_sys(vals + r * 4 + q);
    }
}

__device__ __forceinline__ void dc_allgather(char* const* peer, int P, int me, uint32_t* seq, const double* loc,
                                             double* gath) {
    dc_publish(peer, P, me, seq, loc);
    dc_collect(peer, P, me, seq, gath);
}
#endif

}  // namespace pcg
