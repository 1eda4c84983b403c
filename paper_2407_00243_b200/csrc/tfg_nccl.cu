// tfg_nccl.cu -- run-time NCCL binding (tfg_nccl.cuh) and the communicator
// helpers of the C-ABI (include/tfg.h, multi-GPU section).
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "tfg_common.cuh"
#include "tfg_nccl.cuh"

namespace tfg {

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    void* h = RTLD_DEFAULT;
    if (!dlsym(h, "ncclSend")) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto get = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(get("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(get("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(get("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(get("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(get("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(get("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(get("ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(get("ncclGetErrorString"));
    ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart &&
         api.GroupEnd && api.Send && api.Recv;
  });
  if (!ok) throw runtime_error("NCCL not available (no ncclSend in the process, no libnccl.so.2)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "unknown";
  throw runtime_error(std::string("NCCL error in ") + what + ": " + m);
}

}  // namespace tfg

using namespace tfg;

extern "C" {

tfg_status tfg_nccl_unique_id(void* id_out, size_t cap) {
  return guard([&] {
    if (!id_out || cap < sizeof(ncclUniqueId)) throw invalid_argument("nccl_unique_id: buffer < 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof id);
  });
}

tfg_status tfg_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, void** comm) {
  return guard([&] {
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
      throw invalid_argument("nccl_comm_init: bad arguments");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
    *comm = c;
  });
}

tfg_status tfg_nccl_comm_destroy(void* comm) {
  return guard([&] {
    if (comm) nccl_check(nccl().CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

}  // extern "C"
