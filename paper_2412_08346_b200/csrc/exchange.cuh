// Particle-sharding exchange: one allgather of the
// ranks' [theta, drift] rows per Stein iteration and one of the particle
// summaries after the final ranking.
//
//  * NcclExchange: NCCL over NVLink/NVSwitch, one process per GPU.  NCCL is
//    dlopen'ed (libnccl.so.2 — torch's copy when torch already loaded it), so
//    libasicp.so carries no link-time NCCL dependency.
//  * GroupExchange: contexts of ONE process (one host thread each) exchanging
//    through host memory with a barrier.  It serves several GPUs driven from
//    one process, and on a single GPU it lets the sharded path be checked
//    against the unsharded solve (the streams never wait on each other on the
//    device: each rank synchronises its own stream before the host barrier).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <memory>
#include <mutex>
#include <vector>

struct asicp_group {
  explicit asicp_group(int w) : world(w), slot(static_cast<size_t>(w)) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  bool aborted = false;  // a rank failed mid-exchange: every barrier throws from now on
  std::vector<std::vector<char>> slot;
  void barrier();
  void abort();
};

namespace asicp {

struct Exchange {
  int rank = 0;
  int world = 1;
  virtual ~Exchange() = default;
  // Whether the allgather may be recorded into a CUDA graph.
  virtual bool capturable() const = 0;
  // recv[r * bytes .. (r + 1) * bytes) = rank r's send, enqueued on st.
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
};

// 128-byte ncclUniqueId (NCCL_UNIQUE_ID_BYTES).
void nccl_unique_id(unsigned char id[128]);
std::unique_ptr<Exchange> make_nccl_exchange(int device, int rank, int world, const unsigned char id[128]);
std::unique_ptr<Exchange> make_group_exchange(asicp_group* group, int rank);

}  // namespace asicp
