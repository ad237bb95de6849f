// NCCL communicator for multi-rank contexts (one process per GPU).
//
// libnccl is dlopen'ed on first use instead of linked: the same process may
// already carry PyTorch's bundled NCCL (a different minor version with the
// same soname), and a link-time dependency would pin whichever loads first.
// Only three entry points are needed: unique-id, init-rank and all-gather.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <iterator>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

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
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
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
    a.all_reduce = (decltype(a.all_reduce))dlsym(a.h, "ncclAllReduce");
    a.get_error_string = (decltype(a.get_error_string))dlsym(a.h, "ncclGetErrorString");
  });
  if (!a.h || !a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.all_reduce)
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

// Loopback group (TEST ONLY): the ranks of one process, each with its own
// context / stream on the same GPU, run by host threads. The all-gather is
// host-mediated (stream sync, host barrier, device-to-device copies of the
// peers' slices, barrier): no kernel ever waits on another rank, so the ranks
// need not be co-scheduled. It exercises the engine's multi-rank bookkeeping
// (row partitions, padded slices, offsets) on one GPU. Selected by an id whose
// first 12 bytes are "LGP-LOOPBACK"; bytes 12.. name the group.
namespace {
constexpr char kLoopMagic[] = "LGP-LOOPBACK";
struct Loopback {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<double*> bufs;
  std::vector<double*> tmp;  // per-rank sum buffers (all-reduce)
  std::vector<size_t> tmp_n;
  std::vector<double*> hvals;  // per-rank host values (max all-reduce)
  void barrier() {
    std::unique_lock<std::mutex> l(mu);
    const long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(l, std::chrono::seconds(120), [&] { return gen != g; }))
      throw Error(LGP_E_NCCL, "loopback all-gather: a rank did not arrive within 120 s");
  }
};
std::mutex g_loop_mu;
std::map<std::string, std::weak_ptr<Loopback>> g_loop;
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  std::shared_ptr<Loopback> loop;
};

void comm_unique_id(uint8_t* out128) {
  ncclUniqueId id;
  check(api().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
}

Comm* comm_create(int rank, int world, const uint8_t* id128, cudaStream_t stream) {
  (void)stream;
  if (std::memcmp(id128, kLoopMagic, sizeof(kLoopMagic) - 1) == 0) {
    const std::string key(reinterpret_cast<const char*>(id128), 128);
    std::lock_guard<std::mutex> g(g_loop_mu);
    for (auto it = g_loop.begin(); it != g_loop.end();)  // drop finished groups
      it = it->second.expired() ? g_loop.erase(it) : std::next(it);
    std::shared_ptr<Loopback> lb = g_loop[key].lock();
    if (!lb) {
      lb = std::make_shared<Loopback>();
      lb->world = world;
      lb->bufs.assign(world, nullptr);
      lb->tmp.assign(world, nullptr);
      lb->tmp_n.assign(world, 0);
      lb->hvals.assign(world, nullptr);
      g_loop[key] = lb;
    }
    if (lb->world != world) throw Error(LGP_E_ARG, "loopback group world size mismatch");
    Comm* c = new Comm;
    c->rank = rank;
    c->world = world;
    c->loop = lb;
    return c;
  }
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
  if (c->loop) {
    std::lock_guard<std::mutex> g(c->loop->mu);
    if (c->loop->tmp[c->rank]) cudaFree(c->loop->tmp[c->rank]);
    c->loop->tmp[c->rank] = nullptr;
    c->loop->tmp_n[c->rank] = 0;
  }
  if (c->comm && !c->loop && api().comm_destroy) api().comm_destroy(c->comm);
  delete c;
}

void comm_allgather_inplace(Comm* c, double* buf, size_t count, cudaStream_t stream) {
  if (c->loop) {
    Loopback& lb = *c->loop;
    {
      std::lock_guard<std::mutex> g(lb.mu);
      lb.bufs[c->rank] = buf;
    }
    LGP_CUDA_CHECK(cudaStreamSynchronize(stream));  // own slice written
    lb.barrier();                                   // every slice written, every buffer known
    for (int q = 0; q < c->world; ++q)
      if (q != c->rank)
        LGP_CUDA_CHECK(cudaMemcpyAsync(buf + (size_t)q * count, lb.bufs[q] + (size_t)q * count,
                                       count * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    LGP_CUDA_CHECK(cudaStreamSynchronize(stream));
    lb.barrier();  // every peer has read this rank's slice
    return;
  }
  check(api().all_gather(buf + (size_t)c->rank * count, buf, count, ncclFloat64, c->comm, stream),
        "ncclAllGather");
}

void comm_allreduce_sum_inplace(Comm* c, double* buf, size_t count, cudaStream_t stream) {
  if (c->loop) {
    // every rank sums all ranks' buffers in rank order into its own scratch
    // (identical bits everywhere), then copies the sum over its buffer once
    // no peer reads it any more
    Loopback& lb = *c->loop;
    double* tmp = nullptr;
    {
      std::lock_guard<std::mutex> g(lb.mu);
      lb.bufs[c->rank] = buf;
      if (lb.tmp_n[c->rank] < count) {
        if (lb.tmp[c->rank]) cudaFree(lb.tmp[c->rank]);
        LGP_CUDA_CHECK(cudaMalloc(&lb.tmp[c->rank], count * sizeof(double)));
        lb.tmp_n[c->rank] = count;
      }
      tmp = lb.tmp[c->rank];
    }
    LGP_CUDA_CHECK(cudaStreamSynchronize(stream));
    lb.barrier();
    LGP_CUDA_CHECK(cudaMemcpyAsync(tmp, lb.bufs[0], count * sizeof(double), cudaMemcpyDeviceToDevice,
                                   stream));
    for (int q = 1; q < c->world; ++q) vec::add_inplace(tmp, lb.bufs[q], (int64_t)count, stream);
    LGP_CUDA_CHECK(cudaStreamSynchronize(stream));
    lb.barrier();
    LGP_CUDA_CHECK(cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    return;
  }
  check(api().all_reduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, stream), "ncclAllReduce");
}

void comm_allreduce_max_host(Comm* c, double* vals, int count, cudaStream_t stream) {
  if (count <= 0) return;
  if (c->loop) {
    Loopback& lb = *c->loop;
    std::vector<double> m(vals, vals + count);
    {
      std::lock_guard<std::mutex> g(lb.mu);
      lb.hvals[c->rank] = vals;
    }
    lb.barrier();
    for (int q = 0; q < c->world; ++q)
      for (int i = 0; i < count; ++i) m[i] = std::max(m[i], lb.hvals[q][i]);
    lb.barrier();  // every rank has read every other rank's values
    std::memcpy(vals, m.data(), (size_t)count * sizeof(double));
    return;
  }
  double* d = nullptr;
  LGP_CUDA_CHECK(cudaMallocAsync(&d, (size_t)count * sizeof(double), stream));
  LGP_CUDA_CHECK(cudaMemcpyAsync(d, vals, (size_t)count * sizeof(double), cudaMemcpyHostToDevice, stream));
  check(api().all_reduce(d, d, (size_t)count, ncclFloat64, ncclMax, c->comm, stream), "ncclAllReduce(max)");
  LGP_CUDA_CHECK(cudaMemcpyAsync(vals, d, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, stream));
  LGP_CUDA_CHECK(cudaFreeAsync(d, stream));
  LGP_CUDA_CHECK(cudaStreamSynchronize(stream));
}

}  // namespace lgp
