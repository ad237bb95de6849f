// NCCL communicator for multi-rank contexts (one process per GPU).
//
// libnccl is dlopen'ed on first use instead of linked: the same process may
// already carry PyTorch's bundled NCCL (a different minor version with the
// same soname), and a link-time dependency would pin whichever loads first.
// Only three entry points are needed: unique-id, init-rank and all-gather.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "lgp_internal.h"

namespace lgp {

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(a.h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(a.h, "ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(a.h, "ncclCommDestroy");
    a.all_gather = (decltype(a.all_gather))dlsym(a.h, "ncclAllGather");
    a.get_error_string = (decltype(a.get_error_string))dlsym(a.h, "ncclGetErrorString");
  });
  if (!a.h || !a.get_unique_id || !a.comm_init_rank || !a.all_gather)
    throw Error(LGP_E_NCCL, "libnccl.so.2 could not be loaded");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().get_error_string ? api().get_error_string(r) : "?";
    throw Error(LGP_E_NCCL, std::string(what) + ": " + s);
  }
}
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

void comm_unique_id(uint8_t* out128) {
  ncclUniqueId id;
  check(api().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
}

Comm* comm_create(int rank, int world, const uint8_t* id128, cudaStream_t stream) {
  (void)stream;
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  Comm* c = new Comm;
  c->rank = rank;
  c->world = world;
  ncclResult_t r = api().comm_init_rank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    check(r, "ncclCommInitRank");
  }
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm && api().comm_destroy) api().comm_destroy(c->comm);
  delete c;
}

void comm_allgather_inplace(Comm* c, double* buf, size_t count, cudaStream_t stream) {
  check(api().all_gather(buf + (size_t)c->rank * count, buf, count, ncclFloat64, c->comm, stream),
        "ncclAllGather");
}

}  // namespace lgp
