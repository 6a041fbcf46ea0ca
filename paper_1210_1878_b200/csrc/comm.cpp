// comm.cpp -- NCCL plumbing of the C ABI: unique id, communicator init/destroy.  The
// per-iteration collectives (allgather of rank sums, halo send/recv) live in solver.cu.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "../../include/libpcg.h"

namespace pcg {
void set_thread_error(const std::string& m);
}

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

extern "C" {

pcg_status pcg_comm_unique_id(char* out128) {
    if (!out128) return PCG_ERR_ARG;
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) { pcg::set_thread_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r)); return PCG_ERR_COMM; }
    std::memcpy(out128, &id, 128);
    return PCG_OK;
}

pcg_status pcg_comm_init_rank(const char* id128, int32_t nranks, int32_t rank, int32_t device, void** comm) {
    if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return PCG_ERR_ARG;
    if (cudaSetDevice(device) != cudaSuccess) { pcg::set_thread_error("pcg_comm_init_rank: cudaSetDevice failed"); return PCG_ERR_CUDA; }
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t c = nullptr;
    ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) { pcg::set_thread_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r)); return PCG_ERR_COMM; }
    *comm = (void*)c;
    return PCG_OK;
}

pcg_status pcg_comm_destroy(void* comm) {
    if (!comm) return PCG_OK;
    ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
    return r == ncclSuccess ? PCG_OK : PCG_ERR_COMM;
}

}  // extern "C"
