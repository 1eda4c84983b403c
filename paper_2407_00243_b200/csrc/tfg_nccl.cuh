// tfg_nccl.cuh -- NCCL entry points resolved at run time.
//
// libtfg does not link NCCL: a process that drives the multi-GPU path
// already has one loaded (the host's own, or the one torch.distributed
// brought in), and the communicator handle the caller passes must be used
// with that same library.  So the entry points are looked up in the process
// first (dlsym RTLD_DEFAULT) and only then from libnccl.so.2.
#pragma once
#include <nccl.h>

namespace tfg {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Throws tfg::runtime_error when no NCCL library can be found.
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // namespace tfg
