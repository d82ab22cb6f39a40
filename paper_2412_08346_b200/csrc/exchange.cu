// Particle-sharding exchange backends (see exchange.cuh).
#include "exchange.cuh"

#include <dlfcn.h>
#include <nccl.h>  // types only; the library is resolved at run time

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

void asicp_group::barrier() {
  std::unique_lock<std::mutex> lock(mu);
  if (aborted) throw std::runtime_error("asicp exchange: another rank of the group failed");
  const unsigned long long g = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lock, [&] { return generation != g || aborted; });
    if (aborted) throw std::runtime_error("asicp exchange: another rank of the group failed");
  }
}

// A rank that fails between the two barriers of an allgather releases the
// others (they throw instead of waiting forever); the group is then unusable.
void asicp_group::abort() {
  std::lock_guard<std::mutex> lock(mu);
  aborted = true;
  cv.notify_all();
}

namespace asicp {
namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("asicp exchange: ") + what + ": " + cudaGetErrorString(e));
}

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api = [] {
      NcclApi a;
      for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        a.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (a.handle) break;
      }
      if (!a.handle) return a;
      a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.handle, "ncclGetUniqueId"));
      a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.handle, "ncclCommInitRank"));
      a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.handle, "ncclAllGather"));
      a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.handle, "ncclCommDestroy"));
      a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.handle, "ncclGetErrorString"));
      return a;
    }();
    if (!api.handle || !api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy)
      throw std::runtime_error("asicp exchange: NCCL (libnccl.so.2) is not available");
    return api;
  }

  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw std::runtime_error(std::string("asicp exchange: ") + what + ": " +
                               (error_string ? error_string(r) : "NCCL error"));
  }
};

class NcclExchange final : public Exchange {
 public:
  NcclExchange(int device, int r, int w, const unsigned char id[128]) {
    rank = r;
    world = w;
    NcclApi& api = NcclApi::get();
    ncclUniqueId uid;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&uid, id, sizeof(uid));
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    api.check(api.comm_init_rank(&comm_, w, uid, r), "ncclCommInitRank");
  }
  ~NcclExchange() override {
    if (comm_) NcclApi::get().comm_destroy(comm_);
  }
  // NCCL collectives may be captured into a CUDA graph: every rank captures
  // the same solve (same problem, same partition) and replays it once per
  // solve, so each replay's all-gathers stay collective.  A re-prepare that
  // changes the shape re-captures on every rank alike.  ASICP_NCCL_GRAPH=0
  // launches the sharded solve eagerly instead.
  bool capturable() const override {
    static const bool on = [] {
      const char* e = std::getenv("ASICP_NCCL_GRAPH");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    NcclApi& api = NcclApi::get();
    api.check(api.all_gather(send, recv, bytes, ncclUint8, comm_, st), "ncclAllGather");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

class GroupExchange final : public Exchange {
 public:
  GroupExchange(asicp_group* g, int r) : g_(g) {
    rank = r;
    world = g->world;
  }
  bool capturable() const override { return false; }  // host round trip: never inside a graph
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    try {
      exchange(send, recv, bytes, st);
    } catch (...) {
      g_->abort();
      throw;
    }
  }

 private:
  void exchange(const void* send, void* recv, size_t bytes, cudaStream_t st) {
    std::vector<char>& mine = g_->slot[rank];
    mine.resize(bytes);
    if (bytes) cuda_ok(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_ok(cudaStreamSynchronize(st), "sync");
    g_->barrier();  // every rank's slot is filled
    for (int r = 0; r < world; ++r) {
      if (g_->slot[r].size() != bytes) throw std::runtime_error("asicp exchange: ranks disagree on the gather size");
      if (bytes)
        cuda_ok(cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(r) * bytes, g_->slot[r].data(),
                                bytes, cudaMemcpyHostToDevice, st),
                "H2D");
    }
    cuda_ok(cudaStreamSynchronize(st), "sync");
    g_->barrier();  // every rank has read every slot
  }

  asicp_group* g_;
};

}  // namespace

void nccl_unique_id(unsigned char id[128]) {
  NcclApi& api = NcclApi::get();
  ncclUniqueId uid;
  api.check(api.get_unique_id(&uid), "ncclGetUniqueId");
  std::memcpy(id, &uid, sizeof(uid));
}

std::unique_ptr<Exchange> make_nccl_exchange(int device, int rank, int world, const unsigned char id[128]) {
  return std::make_unique<NcclExchange>(device, rank, world, id);
}

std::unique_ptr<Exchange> make_group_exchange(asicp_group* group, int rank) {
  return std::make_unique<GroupExchange>(group, rank);
}

}  // namespace asicp
