// nccl_ex.cu — native NCCL exchange for the N > 1 protocols (include/gim.h gim_set_nccl).
//
// The protocols' collectives (count / decrement all-reduce, replicated-pool all-gather,
// node-sharded reduce-scatter) are issued by the library itself on its stream
// through an NCCL communicator it owns, instead of a per-step callback into Python (whose host
// round trip dominated the per-step cost of the dense and node-sharded protocols). NCCL is the
// copy already loaded in the process (torch's), found with dlopen(RTLD_NOLOAD), else the
// system's; the library does not link against it, so nothing changes for callers that never
// call gim_set_nccl.
#include <dlfcn.h>
#include <nccl.h>
#include <cstring>
#include "gim_internal.h"

namespace gim {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  bool ok = false;
};

static const NcclApi& api() {
  static const NcclApi a = [] {
    NcclApi x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    x.all_reduce = reinterpret_cast<decltype(x.all_reduce)>(dlsym(h, "ncclAllReduce"));
    x.all_gather = reinterpret_cast<decltype(x.all_gather)>(dlsym(h, "ncclAllGather"));
    x.reduce_scatter = reinterpret_cast<decltype(x.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
    x.ok = x.get_unique_id && x.comm_init_rank && x.comm_destroy && x.all_reduce && x.all_gather && x.reduce_scatter;
    return x;
  }();
  return a;
}

bool nccl_available() { return api().ok; }

int nccl_unique_id(void* out) {
  if (!api().ok) return 1;
  ncclUniqueId id;
  if (api().get_unique_id(&id) != ncclSuccess) return 1;
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int nccl_comm_init(void** comm, const void* id_bytes, int rank, int world) {
  if (!api().ok) return 1;
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t c = nullptr;
  if (api().comm_init_rank(&c, world, id, rank) != ncclSuccess) return 1;
  *comm = c;
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm && api().ok) api().comm_destroy(static_cast<ncclComm_t>(comm));
}

// the gim_*_fn hook signatures; user = the communicator
int nccl_allreduce_i32(void* buf, uint64_t count, void* stream, void* comm) {
  return api().all_reduce(buf, buf, count, ncclInt32, ncclSum, static_cast<ncclComm_t>(comm),
                          static_cast<cudaStream_t>(stream)) != ncclSuccess;
}
int nccl_allgather_bytes(const void* send, uint64_t bytes, void* recv, void* stream, void* comm) {
  return api().all_gather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(comm),
                          static_cast<cudaStream_t>(stream)) != ncclSuccess;
}
int nccl_reducescatter_i32(void* send, void* recv, uint64_t recv_count, void* stream, void* comm) {
  return api().reduce_scatter(send, recv, recv_count, ncclInt32, ncclSum, static_cast<ncclComm_t>(comm),
                              static_cast<cudaStream_t>(stream)) != ncclSuccess;
}

}  // namespace gim
