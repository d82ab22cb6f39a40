// Host orchestration of the B200 AS-ICP solver and the C-ABI (include/asicp.h).
//
// asicp_prepare mirrors GraspProblem::validate (grasp.cpp:20-31) and the
// requires the reference raises inside its loop, then uploads the problem;
// asicp_run replays optimize_grasp (grasp.cpp:132-307) as a fixed sequence
// of kernels per iteration (optionally captured once into a CUDA graph:
// every size that varies with k — the minibatch ramp m(k), the annealing
// gamma(k), the phase — is a host-side function of k, and every data-
// dependent branch is resolved on the device through work lists).
#include "asicp.h"
#include "asicp_debug.h"
#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"
#include "mt64.cuh"
#include "register.cuh"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using namespace asicp;

// NVTX ranges on the host API (header-only NVTX 3: no cost without a tool
// attached): prepare, capture / graph launch / eager enqueue, wait.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


constexpr int kSubRows = kSub;
constexpr int kStats = 256;  // [0..15] NN counters, [16..255] full rescans per iteration

struct InvalidArgument : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void require(bool cond, const char* msg) {
  if (!cond) throw InvalidArgument(msg);
}

#define CUDA_OK(expr)                                                                             \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw DeviceError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + \
                        ":" + std::to_string(__LINE__));                                          \
  } while (0)

void copy_err(const std::string& msg, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = '\0';
  }
}

// spatial_index.cpp:133-139
int64_t minibatch_schedule(int64_t k, int64_t k_max, int64_t n_ref) {
  const double saturation = 2.0 * static_cast<double>(k_max) / 3.0;
  const double ramp = std::min(static_cast<double>(k), saturation) / saturation;
  const auto m = static_cast<int64_t>(std::llround(static_cast<double>(n_ref) * ramp));
  return std::clamp<int64_t>(m, 1, n_ref);
}

// optim.cpp:158-164
double annealing(int64_t t, int64_t T, int64_t C, double p) {
  const double period = static_cast<double>(T) / static_cast<double>(C);
  const double phase = std::fmod(static_cast<double>(t), period) / period;
  return std::pow(phase, p);
}

// A device allocation that grows on demand.
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (n == 0) return;
    CUDA_OK(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

struct asicp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nn_mode = 0;
  int use_graph = 1;
  int profile = 0;
  // Forward / final NN filter on the tensor cores (nn.cu nn_tc_kernel);
  // ASICP_NN_TC=1 selects it.
  bool nn_tc = [] {
    const char* e = std::getenv("ASICP_NN_TC");
    return e && e[0] == '1';
  }();
  int num_sms = 148;
  int nn_grid = 296;
  int max_chunks = 16;
  int window_pool = 0;  // ASICP_OPT_WINDOW_POOL (0: automatic)
  int throughput = 0;   // ASICP_OPT_THROUGHPUT: the NN split model of a shared GPU

  // Prepared problem (host side).
  bool prepared = false;
  int J = 0, n_obj = 0, n_obj_pad = 0, n_scene = 0, n_pre = 0, k_max = 0, k_stein = 0, max_pop = 0;
  int max_ns = 0;
  int max_coarse = 0;
  int64_t total_surf = 0;
  int record_trace = 0;
  double n_ref = 0, eta_stein = 0;
  std::vector<double> gammas;
  std::vector<int64_t> ms;
  std::vector<int> part_pre;
  std::vector<double> init_theta;
  uint64_t seed = 0;
  int target_items = 0;

  // Particle sharding within populations (asicp_set_partition_*): this ctx
  // owns global particles [j_lo, j_lo + J) of J_glob; rows_per_rank pads the
  // allgather blocks to equal size.  Unsharded: xchg null, J_glob = J.
  std::unique_ptr<asicp::Exchange> xchg;
  int J_glob = 0, j_lo = 0, rows_per_rank = 0, final_stride = 0;
  Buf theta_all, drift_all, xsend, xrecv, fsend, frecv, gpop_off_d, med_hist, med_state, kofs_d, kmat;
  int med_big_grid = 0, max_gpop = 0, med_mid = 0;
  double* host_gath = nullptr;
  size_t host_gath_bytes = 0;
  char* pin = nullptr;  // pinned upload staging (upload())
  size_t pin_cap = 0, pin_off = 0;

  DevProblem P{};
  DevState S{};

  // Device buffers.
  Buf obj64, obj_meta, obj_cand, obj_cand4, obj_tc, tc_top, scene64, surf64, pre_surf_off, pre_tcp, pre_sdf, grids, sdf_values, part_pre_d,
      part_surf_off, part_pop, pop_off, pop_logk1, init_theta_d, scene32, sdf_coarse;
  // Collision clusters (collide.cu) and the scratch of their Morton sort.
  Buf scene_box, scene_code, scene_idx, scene_tmp, clusters, subclusters, scene_s32, scene_perm;
  int n_clusters = 0;
  Buf theta, theta_next, loss, prev_loss, in_col, converged, active, n_col, grad, drift, h, S64, Sq32, Sc32,
      Bs, ctr, colc, col_lists, col_idx, col_q, res_fwd, res_rev, rng_state, rng_mti, pool_idx, pool32, fy_scratch, fy_par, items0,
      items1,
      item_count, item_off, item_counter, partials, amb_pool, amb_n, amb_count, refine_list, refine_count,
      stats, iter_stats, trace_theta,
      trace_loss, trace_col,
      final_loss, final_free;

  // SGD-ICP registration batches (register.cu), created on first use.
  std::unique_ptr<asicp::RegBatch> reg;

  cudaGraphExec_t graph_exec = nullptr;
  bool graph_valid = false;
  std::vector<char> graph_sig;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t side = nullptr;  // forked work inside an iteration (median bandwidth)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t rev_side = nullptr;  // the reverse match beside the minibatch draw / forward filter
  cudaEvent_t ev_rev_fork = nullptr, ev_rev_join = nullptr, ev_fill = nullptr;
  bool fork_rev = [] {  // ASICP_FORK_REV=0: the reverse match in line
    const char* e = std::getenv("ASICP_FORK_REV");
    return !(e && e[0] == '0');
  }();
  // Profile mode (ASICP_OPT_PROFILE, eager launches): per-stage event pairs.
  enum Stage { kStNn = 0, kStCollide, kStMinibatch, kStCost, kStSvgd, kStages };
  struct ProfEvent {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<ProfEvent> prof_events;
  asicp_stats last_stats{};
  double nn_pairs_planned = 0.0;
  int64_t launches = 0;
  unsigned long long raw_stats[kStats] = {};

  // Pinned host staging for the per-particle summaries, so a launched solve
  // returns control to the host (asicp_run_async) and several contexts on
  // different streams overlap on one GPU.
  struct Staging {
    double* theta = nullptr;
    double* floss = nullptr;
    int* ffree = nullptr;
    int* conv = nullptr;
    unsigned long long* stats = nullptr;
    int* refine_total = nullptr;
    int cap = 0;
  } host;
  bool in_flight = false;

  void ensure_staging(int J) {
    if (J <= host.cap) return;
    free_staging();
    const size_t j = static_cast<size_t>(J);
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host.theta), 7 * j * 8));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host.floss), j * 8));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host.ffree), j * 4));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host.conv), j * 4));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host.stats), kStats * 8));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host.refine_total), 4));
    host.cap = J;
  }
  void free_staging() {
    void* all[] = {host.theta, host.floss, host.ffree, host.conv, host.stats, host.refine_total};
    for (void* p : all)
      if (p) cudaFreeHost(p);
    host = Staging{};
  }

  void ensure_gath(size_t bytes) {
    if (bytes <= host_gath_bytes) return;
    if (host_gath) cudaFreeHost(host_gath);
    host_gath = nullptr;
    host_gath_bytes = 0;
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&host_gath), bytes));
    host_gath_bytes = bytes;
  }

  ~asicp_ctx() {
    if (in_flight && stream) cudaStreamSynchronize(stream);
    free_staging();
    if (host_gath) cudaFreeHost(host_gath);
    if (pin) cudaFreeHost(pin);
    xchg.reset();
    reg.reset();
    Buf* shard_bufs[] = {&theta_all, &drift_all, &xsend,    &xrecv,  &fsend, &frecv,
                         &gpop_off_d, &med_hist, &med_state, &kofs_d, &kmat};
    for (Buf* b : shard_bufs) b->release();
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (auto& e : prof_events) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (ev_rev_fork) cudaEventDestroy(ev_rev_fork);
    if (ev_rev_join) cudaEventDestroy(ev_rev_join);
    if (ev_fill) cudaEventDestroy(ev_fill);
    if (rev_side) cudaStreamDestroy(rev_side);
    Buf* all[] = {&obj64, &obj_meta, &obj_cand, &obj_cand4, &obj_tc, &tc_top, &scene64, &surf64, &pre_surf_off, &pre_tcp, &pre_sdf, &grids, &sdf_values,
                  &part_pre_d, &part_surf_off, &part_pop, &pop_off, &pop_logk1, &init_theta_d,
                  &scene32, &sdf_coarse, &scene_box, &scene_code, &scene_idx, &scene_tmp, &clusters, &subclusters,
                  &scene_s32, &scene_perm, &theta,
                  &theta_next, &loss, &prev_loss, &in_col, &converged, &active, &n_col, &grad, &drift, &h,
                  &S64, &Sq32, &Sc32, &Bs, &ctr, &colc, &col_lists, &col_idx, &col_q, &res_fwd, &res_rev, &rng_state, &rng_mti,
                  &pool_idx, &pool32, &fy_scratch, &fy_par, &items0, &items1, &item_count, &item_off,
                  &item_counter,
                  &partials, &amb_pool, &amb_n, &amb_count, &refine_list, &refine_count, &stats, &iter_stats, &trace_theta,
                  &trace_loss, &trace_col,
                  &final_loss, &final_free};
    for (Buf* b : all) b->release();
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

namespace {

// Host -> device through the ctx's pinned staging buffer: a memcpy into
// pinned memory, then a true async DMA.  Pageable copies made the driver pin
// pages on the fly, and asicp_prepare's time varied from 1 to 80 ms on the
// bench boxes (tools/prepare_timing.py).  Staged copies stay in flight until
// the stream synchronizes at the end of asicp_prepare; a full buffer
// synchronizes and restarts.
// Copy `bytes` from host `src` to device `dst` through the pinned staging.
void stage_copy(asicp_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st);

template <typename T>
void upload(asicp_ctx* c, Buf& b, const T* src, size_t n, cudaStream_t st) {
  b.ensure(std::max<size_t>(n, 1) * sizeof(T));
  if (!n) return;
  stage_copy(c, b.p, src, n * sizeof(T), st);
}

void stage_copy(asicp_ctx* c, void* dst_dev, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  const size_t need = (bytes + 255) / 256 * 256;
  if (c->pin_off + need > c->pin_cap) {
    CUDA_OK(cudaStreamSynchronize(st));
    c->pin_off = 0;
    if (need > c->pin_cap) {
      if (c->pin) cudaFreeHost(c->pin);
      c->pin = nullptr;
      c->pin_cap = 0;
      const size_t cap = std::max<size_t>(need, size_t(16) << 20);
      CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&c->pin), cap));
      c->pin_cap = cap;
    }
  }
  char* dst = c->pin + c->pin_off;
  std::memcpy(dst, src, bytes);
  CUDA_OK(cudaMemcpyAsync(dst_dev, dst, bytes, cudaMemcpyHostToDevice, st));
  c->pin_off += need;
}

// GraspProblem::validate (grasp.cpp:20-31) + Preshape::validate (:13-18),
// then the requires the reference hits inside its first iteration.
void validate(const asicp_problem& p) {
  require(p.n_object > 0, "GraspProblem: empty object cloud");
  require(p.n_scene > 0, "GraspProblem: empty scene cloud");
  require(p.n_preshapes > 0, "GraspProblem: no preshapes");
  require(p.n_init_lists == p.n_preshapes, "GraspProblem: one initialization list per preshape required");
  require(p.k_stein <= p.k_max, "GraspProblem: k_stein must not exceed k_max");
  for (int64_t i = 0; i < p.n_preshapes; ++i) {
    const asicp_preshape& s = p.preshapes[i];
    require(s.n_surface > 0, "Preshape: empty inner surface cloud");
    require(s.n_full > 0, "Preshape: empty full cloud");
    // tool_centre_point = centroid (geometry.cpp:86-96): sum in order, / n.
    double c[3] = {0.0, 0.0, 0.0};
    for (int64_t k = 0; k < s.n_surface; ++k)
      for (int a = 0; a < 3; ++a) c[a] = c[a] + s.inner_surface[3 * k + a];
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = s.tcp[a] - c[a] / static_cast<double>(s.n_surface);
    require(std::sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]) <= 1e-9,
            "Preshape: tcp must be the contact-surface centroid");
    require(s.sdf_index >= 0 && s.sdf_index < p.n_sdf_grids, "GraspProblem: preshape sdf_index out of range");
  }
  int64_t J = 0;
  for (int64_t i = 0; i < p.n_init_lists; ++i) J += p.init_counts[i];
  require(J >= 1, "optimize_grasp: no initial poses");
  // First evaluation of particle 0 (grasp.cpp:171-194): unit quaternion
  // (geometry.cpp:19), then the prior (optim.cpp:150); then the others.
  auto unit_ok = [&](int64_t j) {
    const double* q = p.init_poses + 7 * j + 3;
    const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
    return std::abs(std::sqrt(n2) - 1.0) <= 1e-6;
  };
  if (p.k_max > 0) {
    require(unit_ok(0), "rotation_matrix: quaternion is not unit-norm");
    for (int a = 0; a < 3; ++a)
      require(p.prior_t_sigma[a] * p.prior_t_sigma[a] > 0.0, "prior_log_gradient: t_sigma must be positive");
    for (int64_t j = 1; j < J; ++j) require(unit_ok(j), "rotation_matrix: quaternion is not unit-norm");
    if (p.k_stein > 0) {
      require(p.anneal_cycles >= 1 && p.anneal_period_total >= p.anneal_cycles, "annealing: need T >= C >= 1");
      require(p.anneal_exponent > 0.0, "annealing: exponent must be positive");
      bool coupled = false;
      for (int64_t i = 0; i < p.n_init_lists; ++i) coupled = coupled || p.init_counts[i] >= 2;
      if (coupled && p.bandwidth_mode == ASICP_BANDWIDTH_FIXED)
        require(p.fixed_bandwidth > 0.0, "rbf_kernel: bandwidth must be positive");
    }
  } else {
    // Final ranking still transforms every particle (grasp.cpp:271-277).
    for (int64_t j = 0; j < J; ++j) require(unit_ok(j), "rotation_matrix: quaternion is not unit-norm");
  }
  for (int64_t g = 0; g < p.n_sdf_grids; ++g)
    for (int a = 0; a < 3; ++a) require(p.sdf_grids[g].dims[a] >= 2, "asicp: SDF grid needs >= 2 nodes per axis");
  require(p.n_object < (1ll << 30) && p.n_scene < (1ll << 30), "asicp: cloud too large");
  // The collision kernel keeps one bit per scene point in shared memory.
  require(p.n_scene <= 1600000, "asicp: scene cloud above 1,600,000 points");
}

void prepare(asicp_ctx* c, const asicp_problem& p) {
  NvtxRange range("asicp_prepare");
  // ASICP_PREPARE_TIMING=1: host-side section times to stderr (diagnostics).
  static const bool timing = std::getenv("ASICP_PREPARE_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "prepare %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  validate(p);
  mark("validate");
  c->pin_off = 0;
  CUDA_OK(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const int n_pre = static_cast<int>(p.n_preshapes);
  c->n_pre = n_pre;
  c->n_obj = static_cast<int>(p.n_object);
  c->n_scene = static_cast<int>(p.n_scene);
  c->k_max = static_cast<int>(p.k_max);
  c->k_stein = static_cast<int>(p.k_stein);
  c->record_trace = p.record_trace ? 1 : 0;
  c->seed = p.seed;
  c->n_ref = static_cast<double>(p.n_object);
  c->eta_stein = p.step_scale / c->n_ref;  // grasp.cpp:154

  // Object cloud: FP64 rows; the re-centred FP32 candidates (pair-interleaved
  // and plain, rows padded to the NN subtile with +inf) are built on the device.
  c->n_obj_pad = static_cast<int>((p.n_object + kSubRows - 1) / kSubRows * kSubRows);
  upload(c, c->obj64, p.object_cloud, 3 * p.n_object, st);
  c->obj_meta.ensure(4 * sizeof(double));
  c->obj_cand.ensure(static_cast<size_t>(c->n_obj_pad) * sizeof(float4));
  c->obj_cand4.ensure(static_cast<size_t>(c->n_obj_pad) * sizeof(float4));
  launch_object_prepare(c->obj64.as<double>(), c->n_obj, c->n_obj_pad, c->obj_meta.as<double>(),
                        c->obj_cand.as<float4>(), c->obj_cand4.as<float4>(), st);
  if (c->nn_tc) {
    c->obj_tc.ensure(static_cast<size_t>(c->n_obj) * 3 * sizeof(float4));
    launch_obj_tc(c->obj_cand4.as<float4>(), c->n_obj, c->obj_tc.as<float4>(), st);
  }
  upload(c, c->scene64, p.scene_cloud, 3 * p.n_scene, st);
  {
    // FP32 scene copy and the collision clusters, built on the device
    // (collide.cu: Morton sort, cluster centres and radii).
    const int n = c->n_scene;
    c->n_clusters = (n + kClusterPts - 1) / kClusterPts;
    const size_t npad = static_cast<size_t>(c->n_clusters) * kClusterPts;
    c->scene32.ensure(static_cast<size_t>(n) * sizeof(float4));
    c->scene_box.ensure(6 * sizeof(double));
    c->scene_code.ensure(2 * static_cast<size_t>(n) * sizeof(unsigned int));
    c->scene_idx.ensure(2 * static_cast<size_t>(n) * sizeof(int));
    const size_t tb = scene_sort_temp_bytes(n);
    c->scene_tmp.ensure(std::max<size_t>(tb, 16));
    c->clusters.ensure(static_cast<size_t>(c->n_clusters) * sizeof(float4));
    c->subclusters.ensure(static_cast<size_t>(c->n_clusters) * kSubPerCluster * sizeof(float4));
    c->scene_s32.ensure(npad * sizeof(float4));
    c->scene_perm.ensure(npad * sizeof(int));
    launch_scene_prepare(c->scene64.as<double>(), n, c->scene32.as<float4>(), c->scene_box.as<double>(),
                         c->scene_code.as<unsigned int>(), c->scene_code.as<unsigned int>() + n,
                         c->scene_idx.as<int>(), c->scene_idx.as<int>() + n, c->scene_tmp.p, c->scene_tmp.bytes,
                         c->clusters.as<float4>(), c->subclusters.as<float4>(), c->scene_s32.as<float4>(),
                         c->scene_perm.as<int>(), st);
  }

  // Preshapes.
  std::vector<double> surf;
  std::vector<int> pre_off(n_pre + 1, 0), pre_sdf(n_pre);
  std::vector<double> tcp(3 * n_pre);
  c->max_ns = 0;
  c->max_pop = 0;
  for (int i = 0; i < n_pre; ++i) {
    const asicp_preshape& s = p.preshapes[i];
    pre_off[i] = static_cast<int>(surf.size() / 3);
    surf.insert(surf.end(), s.inner_surface, s.inner_surface + 3 * s.n_surface);
    pre_sdf[i] = static_cast<int>(s.sdf_index);
    for (int a = 0; a < 3; ++a) tcp[3 * i + a] = s.tcp[a];
    c->max_ns = std::max(c->max_ns, static_cast<int>(s.n_surface));
  }
  pre_off[n_pre] = static_cast<int>(surf.size() / 3);
  upload(c, c->surf64, surf.data(), surf.size(), st);
  upload(c, c->pre_surf_off, pre_off.data(), pre_off.size(), st);
  upload(c, c->pre_tcp, tcp.data(), tcp.size(), st);
  upload(c, c->pre_sdf, pre_sdf.data(), pre_sdf.size(), st);

  // SDF grids.
  std::vector<Grid> grids(p.n_sdf_grids);
  int64_t values_total = 0;
  for (int64_t g = 0; g < p.n_sdf_grids; ++g)
    values_total += static_cast<int64_t>(p.sdf_grids[g].dims[0]) * p.sdf_grids[g].dims[1] * p.sdf_grids[g].dims[2];
  c->sdf_values.ensure(static_cast<size_t>(std::max<int64_t>(values_total, 1)) * sizeof(float));
  int64_t values_off = 0;
  int64_t coarse_total = 0;
  for (int64_t g = 0; g < p.n_sdf_grids; ++g) {
    const asicp_sdf_grid& s = p.sdf_grids[g];
    Grid& d = grids[g];
    for (int a = 0; a < 3; ++a) {
      d.dims[a] = s.dims[a];
      d.origin[a] = s.origin[a];
      d.offset[a] = s.offset[a];
    }
    d.voxel = s.voxel;
    d.boundary_max_abs = s.boundary_max_abs;
    d.values_offset = values_off;
    const size_t total = static_cast<size_t>(s.dims[0]) * s.dims[1] * s.dims[2];
    stage_copy(c, c->sdf_values.as<float>() + values_off, s.values, total * sizeof(float), st);  // grid by grid
    values_off += static_cast<int64_t>(total);
    // Bounds of the collision kernel's FP32 pre-test (lip, vmax and the
    // dilated 4^3-block maxima) are computed on the device below.
    d.lip = 0.0;
    d.vmax = 0.0;
    for (int a = 0; a < 3; ++a) d.cdims[a] = (s.dims[a] - 1 + kCoarse - 1) / kCoarse;
    d.coarse_offset = coarse_total;
    coarse_total += static_cast<int64_t>(d.cdims[0]) * d.cdims[1] * d.cdims[2];
  }
  mark("host-build");
  upload(c, c->grids, grids.data(), grids.size(), st);
  mark("sdf-upload");
  c->sdf_coarse.ensure(static_cast<size_t>(std::max<int64_t>(coarse_total, 1)) * sizeof(float));
  launch_grid_bounds(c->grids.as<Grid>(), static_cast<int>(p.n_sdf_grids), c->sdf_values.as<float>(),
                     c->sdf_coarse.as<float>(), st);
  c->max_coarse = 0;
  for (const Grid& g : grids)
    c->max_coarse = std::max(c->max_coarse, g.cdims[0] * g.cdims[1] * g.cdims[2]);

  // Particles (preshape-major flattening, grasp.cpp:135-145).  Sharded, this
  // ctx keeps the contiguous slice [lo, hi) = [r J / R, (r + 1) J / R) of the
  // global order; each particle's RNG stream stays seeded by its GLOBAL index
  // (seed + j, grasp.cpp:148-151) through the seed offset below.
  std::vector<int> gpop_off(n_pre + 1, 0);
  int64_t Jg = 0;
  for (int i = 0; i < n_pre; ++i) {
    gpop_off[i] = static_cast<int>(Jg);
    Jg += p.init_counts[i];
  }
  gpop_off[n_pre] = static_cast<int>(Jg);
  const int world = c->xchg ? c->xchg->world : 1, rank = c->xchg ? c->xchg->rank : 0;
  const int lo = static_cast<int>(static_cast<int64_t>(rank) * Jg / world);
  const int hi = static_cast<int>(static_cast<int64_t>(rank + 1) * Jg / world);
  require(hi > lo, "asicp: particle partition leaves a rank without particles (fewer particles than ranks)");
  std::vector<int> part_pre, part_pop, pop_off(n_pre + 1, 0), part_pre_glob;
  std::vector<int64_t> part_surf_off;
  std::vector<double> logk1(n_pre);
  int64_t so = 0;
  for (int i = 0; i < n_pre; ++i) {
    pop_off[i] = static_cast<int>(part_pre.size());
    int local = 0;
    for (int64_t k = 0; k < p.init_counts[i]; ++k) {
      const int64_t g = gpop_off[i] + k;
      part_pre_glob.push_back(i);
      if (g < lo || g >= hi) continue;
      part_pre.push_back(i);
      part_pop.push_back(i);
      part_surf_off.push_back(so);
      so += (p.preshapes[i].n_surface + kSubRows - 1) / kSubRows * kSubRows;  // rows padded to the subtile
      ++local;
    }
    logk1[i] = std::log(static_cast<double>(p.init_counts[i]) + 1.0);  // optim.cpp:143 (global K)
    c->max_pop = std::max(c->max_pop, local);
  }
  pop_off[n_pre] = static_cast<int>(part_pre.size());
  part_surf_off.push_back(so);
  const int J = static_cast<int>(part_pre.size());
  c->J = J;
  c->J_glob = static_cast<int>(Jg);
  c->j_lo = lo;
  c->seed = p.seed + static_cast<uint64_t>(lo);
  c->rows_per_rank = static_cast<int>((Jg + world - 1) / world);
  c->total_surf = so;
  c->part_pre = part_pre_glob;
  upload(c, c->part_pre_d, part_pre.data(), part_pre.size(), st);
  upload(c, c->part_pop, part_pop.data(), part_pop.size(), st);
  upload(c, c->pop_off, pop_off.data(), pop_off.size(), st);
  upload(c, c->gpop_off_d, gpop_off.data(), gpop_off.size(), st);
  // Split SVGD (kernel matrix, then ordered sums) while the K x K_local
  // matrices stay under 8 M pairs (128 MB); the fused kernel otherwise.
  std::vector<long long> kofs(n_pre, 0);
  long long ktot = 0;
  c->max_gpop = 0;
  for (int i = 0; i < n_pre; ++i) {
    kofs[i] = ktot;
    ktot += static_cast<long long>(p.init_counts[i]) * (pop_off[i + 1] - pop_off[i]);
    c->max_gpop = std::max(c->max_gpop, static_cast<int>(p.init_counts[i]));
  }
  const bool svgd_split = c->k_stein > 0 && ktot > 0 && ktot <= (8ll << 20);
  if (svgd_split) c->kmat.ensure(static_cast<size_t>(ktot) * sizeof(double2));
  upload(c, c->kofs_d, kofs.data(), kofs.size(), st);
  upload(c, c->pop_logk1, logk1.data(), logk1.size(), st);
  // Median select: populations below kMedBigK in one CTA, up to kMedClusterK
  // in one 8-CTA cluster (median.cu), larger ones grid-wide over 128 x 128
  // tiles of the pair triangle (kernels.cu).
  long long big_tiles = 0;
  c->med_mid = 0;
  for (int i = 0; i < n_pre; ++i) {
    const long long K = p.init_counts[i];
    if (K >= kMedBigK && K <= kMedClusterK) c->med_mid = 1;
    if (K > kMedClusterK) {
      const long long nb = (K + 127) / 128;
      big_tiles = std::max(big_tiles, nb * (nb + 1) / 2);
    }
  }
  c->med_big_grid = static_cast<int>(std::min<long long>(big_tiles, 8ll * c->num_sms));
  c->med_hist.ensure(static_cast<size_t>(n_pre) * 4096 * 4);
  c->med_state.ensure(static_cast<size_t>(n_pre) * sizeof(MedState));
  upload(c, c->part_surf_off, part_surf_off.data(), part_surf_off.size(), st);
  c->init_theta.assign(p.init_poses + 7 * static_cast<int64_t>(lo), p.init_poses + 7 * static_cast<int64_t>(hi));
  upload(c, c->init_theta_d, c->init_theta.data(), c->init_theta.size(), st);

  // Schedules (host-exact: llround / fmod / pow of the reference).
  c->ms.resize(c->k_max);
  c->gammas.resize(c->k_max);
  for (int k = 0; k < c->k_max; ++k) {
    c->ms[k] = minibatch_schedule(k, p.k_max, p.n_object);
    c->gammas[k] = k < c->k_stein ? annealing(k, p.anneal_period_total, p.anneal_cycles, p.anneal_exponent) : 0.0;
  }

  // Forward work: base_items query blocks; the device splits the candidates
  // so that (query blocks of the particles matching) x splits ~ target_items,
  // i.e. the persistent grid gets several items per CTA in every iteration.
  int base_items = 0;
  for (int i = 0; i < n_pre; ++i)
    base_items += static_cast<int>(p.init_counts[i] * ((p.preshapes[i].n_surface + kNnQB - 1) / kNnQB));
  c->target_items = 4 * c->nn_grid;
  const size_t fwd_slots = static_cast<size_t>(base_items) + c->target_items;  // >= T x splits

  // State buffers.
  const size_t Jz = static_cast<size_t>(J);
  c->theta.ensure(Jz * 7 * 8);
  c->theta_next.ensure(Jz * 7 * 8);
  c->loss.ensure(Jz * 8);
  c->prev_loss.ensure(Jz * 8);
  c->in_col.ensure(Jz * 4);
  c->converged.ensure(Jz * 4);
  c->active.ensure(Jz * 4);
  c->n_col.ensure(Jz * 4);
  c->grad.ensure(Jz * 7 * 8);
  c->drift.ensure(Jz * 7 * 8);
  c->h.ensure(static_cast<size_t>(n_pre) * 8);
  c->S64.ensure(static_cast<size_t>(so) * 24);
  c->Sq32.ensure(static_cast<size_t>(so) * 16);
  c->Sc32.ensure(static_cast<size_t>(so) * 16);
  c->Bs.ensure(Jz * 8);
  c->ctr.ensure(Jz * 3 * 8);
  c->colc.ensure(Jz * sizeof(ColConst));
  const size_t jscene = Jz * static_cast<size_t>(c->n_scene);
  c->col_idx.ensure(jscene * 4);
  c->col_q.ensure(jscene * 16);
  c->res_rev.ensure(jscene * 4);
  c->res_fwd.ensure(static_cast<size_t>(so) * 4);
  c->rng_state.ensure(Jz * mt::kN * 8);
  c->rng_mti.ensure(Jz * 4);
  const size_t jobj = Jz * static_cast<size_t>(c->n_obj_pad);
  c->pool_idx.ensure(jobj * 4);
  c->pool32.ensure(jobj * 16);
  if (static_cast<size_t>(c->n_obj) * 4 > static_cast<size_t>(minibatch_smem_cap()))
    c->fy_scratch.ensure(Jz * static_cast<size_t>(c->n_obj) * 4);
  // Parallel Fisher-Yates scratch (5 int arrays per particle) when it takes at
  // most a quarter of the free HBM; the serial kernel covers the rest.
  mark("particles");
  // Parallel Fisher-Yates scratch: 5 int arrays per particle, for the whole
  // population when that takes at most a quarter of the free HBM, else for a
  // batch of particles the minibatch launches cover in turn (large clouds,
  // SURVEY cfg5 at 50k-200k points).  cudaMemGetInfo costs 1-11 ms of host
  // time on the bench boxes: ask only when the scratch grows.
  const size_t fy_per = 5 * static_cast<size_t>(c->n_obj_pad) * 4;
  int fy_batch = J;
  if (Jz * fy_per > c->fy_par.bytes) {
    size_t free_b = 0, total_b = 0;
    CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
    const size_t budget = c->fy_par.bytes + free_b / 4;
    fy_batch = static_cast<int>(std::min<size_t>(Jz, budget / fy_per));
  }
  if (const char* e = std::getenv("ASICP_FY_BATCH"))  // test knob: force particle batches of the scratch
    fy_batch = std::max(1, std::min(fy_batch, std::atoi(e)));
  const bool fy_par_on = fy_batch >= 1;
  if (fy_par_on) c->fy_par.ensure(static_cast<size_t>(fy_batch) * fy_per);
  if (fy_par_on && static_cast<size_t>(fy_batch) * fy_per < c->fy_par.bytes)  // an earlier, larger scratch
    fy_batch = static_cast<int>(std::min<size_t>(Jz, c->fy_par.bytes / fy_per));
  mark("memgetinfo");
  // Work items: forward < base_items + target_items (T x splits, see
  // fwd_split); reverse <= sum ceil(n_col / 32) <= J * ceil(n_scene / 32).
  c->items0.ensure((fwd_slots + Jz) * sizeof(NnItem));
  c->items1.ensure((Jz * ((c->n_scene + kRevWQ - 1) / kRevWQ) + Jz) * sizeof(NnItem));
  c->item_count.ensure(2 * (Jz + 1) * 4);
  c->item_off.ensure(2 * (Jz + 1) * 4);
  c->item_counter.ensure(4 * 4);  // [0..1] item counters, [2..3] device split (nn_dyn)
  c->partials.ensure(fwd_slots * kNnQB * sizeof(NnPartial));
  if (c->nn_tc) c->tc_top.ensure(fwd_slots * kNnQB * 2 * sizeof(float4));
  // Ambiguous windows: ~0.3 % of queries on cfg2, but up to ~15 % for dense
  // clouds matched from far (100k points, queries 25 cm out).  A (query,
  // split) allocates at most one block while the pool lasts, so a quarter of
  // all slots (64 k floor) keeps exhaustion — and with it the full FP64
  // rescan of the affected queries — out of every tested workload.
  const int amb_cap = c->window_pool > 0 ? c->window_pool
                                         : static_cast<int>(std::min<size_t>(
                                               std::max<size_t>(65536, fwd_slots * kNnQB / 4), 1u << 26));
  c->amb_pool.ensure(static_cast<size_t>(amb_cap) * kWinCap * sizeof(int2));
  c->amb_n.ensure(static_cast<size_t>(amb_cap) * sizeof(int));
  c->amb_count.ensure(sizeof(int));
  const size_t refine_cap = std::min<size_t>(static_cast<size_t>(so) + jscene, 64ull << 20);
  c->refine_list.ensure(refine_cap * sizeof(int4));
  c->refine_count.ensure(4);
  c->stats.ensure(kStats * sizeof(unsigned long long));
  c->iter_stats.ensure(4 * static_cast<size_t>(c->k_max + 1) * sizeof(unsigned long long));
  if (c->record_trace) {
    const size_t rows = static_cast<size_t>(c->k_max) * Jz;
    c->trace_theta.ensure(std::max<size_t>(rows, 1) * 7 * 8);
    c->trace_loss.ensure(std::max<size_t>(rows, 1) * 8);
    c->trace_col.ensure(std::max<size_t>(rows, 1) * 4);
  }
  c->final_loss.ensure(Jz * 8);
  c->final_free.ensure(Jz * 4);
  if (c->xchg) {
    const size_t rows = static_cast<size_t>(c->rows_per_rank), wr = static_cast<size_t>(world) * rows;
    c->theta_all.ensure(static_cast<size_t>(Jg) * 7 * 8);
    c->drift_all.ensure(static_cast<size_t>(Jg) * 7 * 8);
    c->xsend.ensure(rows * 14 * 8);
    c->xrecv.ensure(wr * 14 * 8);
    c->final_stride = 10 + (c->record_trace ? 9 * c->k_max : 0);
    c->fsend.ensure(rows * c->final_stride * 8);
    c->frecv.ensure(wr * c->final_stride * 8);
    // Padding rows of the send blocks are never read back, but keep them defined.
    CUDA_OK(cudaMemsetAsync(c->xsend.p, 0, c->xsend.bytes, st));
    CUDA_OK(cudaMemsetAsync(c->fsend.p, 0, c->fsend.bytes, st));
  }

  // Device views.
  DevProblem& P = c->P;
  P.J = J;
  P.n_obj = c->n_obj;
  P.n_obj_pad = c->n_obj_pad;
  P.n_scene = c->n_scene;
  P.n_pop = n_pre;
  P.obj64 = c->obj64.as<double>();
  P.obj_cand = c->obj_cand.as<float4>();
  P.obj_cand4 = c->obj_cand4.as<float4>();
  P.obj_tc = c->nn_tc ? c->obj_tc.as<float4>() : nullptr;
  P.scene64 = c->scene64.as<double>();
  P.scene32 = c->scene32.as<float4>();
  P.n_clusters = c->n_clusters;
  P.med_mid = c->med_mid;
  P.col_lists_global = 0;
  P.col_lists_global = collide_lists_global(P) ? 1 : 0;
  P.throughput = c->throughput;
  P.clusters = c->clusters.as<float4>();
  P.subclusters = c->subclusters.as<float4>();
  P.scene_s32 = c->scene_s32.as<float4>();
  P.scene_perm = c->scene_perm.as<int>();
  P.surf64 = c->surf64.as<double>();
  P.pre_surf_off = c->pre_surf_off.as<int>();
  P.pre_tcp = c->pre_tcp.as<double>();
  P.pre_sdf = c->pre_sdf.as<int>();
  P.grids = c->grids.as<Grid>();
  P.sdf_values = c->sdf_values.as<float>();
  P.sdf_coarse = c->sdf_coarse.as<float>();
  P.max_coarse = c->max_coarse;
  P.part_pre = c->part_pre_d.as<int>();
  P.part_surf_off = c->part_surf_off.as<int64_t>();
  P.part_pop = c->part_pop.as<int>();
  P.pop_off = c->pop_off.as<int>();
  P.pop_logk1 = c->pop_logk1.as<double>();
  P.gpop_off = c->gpop_off_d.as<int>();
  P.j_lo = lo;
  P.kofs = c->kofs_d.as<long long>();
  P.obj_meta = c->obj_meta.as<double>();
  for (int a = 0; a < 3; ++a) {
    P.com[a] = p.com[a];
    P.prior_t_mean[a] = p.prior_t_mean[a];
    P.prior_t_sigma[a] = p.prior_t_sigma[a];
  }
  P.contact_tolerance = p.contact_tolerance;
  for (int a = 0; a < 4; ++a) {
    P.prior_q_location[a] = p.prior_q_location[a];
    P.prior_q_kappa[a] = p.prior_q_kappa[a];
  }
  P.bandwidth_mode = p.bandwidth_mode == ASICP_BANDWIDTH_FIXED ? 1 : 0;
  P.fixed_bandwidth = p.fixed_bandwidth;
  for (int i = 0; i < 49; ++i) P.A[i] = p.A[i];
  P.lr = p.learning_rate;
  P.conv_thr = p.convergence_threshold;

  DevState& S = c->S;
  S.theta = c->theta.as<double>();
  S.theta_next = c->theta_next.as<double>();
  S.loss = c->loss.as<double>();
  S.prev_loss = c->prev_loss.as<double>();
  S.in_col = c->in_col.as<int>();
  S.converged = c->converged.as<int>();
  S.active = c->active.as<int>();
  S.n_col = c->n_col.as<int>();
  S.grad = c->grad.as<double>();
  S.drift = c->drift.as<double>();
  S.theta_all = c->xchg ? c->theta_all.as<double>() : S.theta;
  S.drift_all = c->xchg ? c->drift_all.as<double>() : S.drift;
  S.h = c->h.as<double>();
  S.kmat = svgd_split ? c->kmat.as<double2>() : nullptr;
  S.med_hist = c->med_hist.as<unsigned int>();
  S.med_state = c->med_state.as<MedState>();
  S.S64 = c->S64.as<double>();
  S.Sq32 = c->Sq32.as<float4>();
  S.Sc32 = c->Sc32.as<float4>();
  S.Bs = c->Bs.as<double>();
  S.ctr = c->ctr.as<double>();
  S.colc = c->colc.as<ColConst>();
  if (P.col_lists_global)
    c->col_lists.ensure(Jz * (1 + kSubPerCluster) * static_cast<size_t>(c->n_clusters) * sizeof(int));
  S.col_lists = P.col_lists_global ? c->col_lists.as<int>() : nullptr;
  S.col_idx = c->col_idx.as<int>();
  S.col_q = c->col_q.as<float4>();
  S.res_fwd = c->res_fwd.as<int>();
  S.res_rev = c->res_rev.as<int>();
  S.rng_state = c->rng_state.as<uint64_t>();
  S.rng_mti = c->rng_mti.as<int>();
  S.pool_idx = c->pool_idx.as<int>();
  S.pool32 = c->pool32.as<float4>();
  S.fy_scratch = c->fy_scratch.as<int>();
  S.fy_par = fy_par_on ? c->fy_par.as<int>() : nullptr;
  S.fy_stride = 5 * static_cast<int64_t>(c->n_obj_pad);
  S.fy_batch = fy_par_on ? fy_batch : 0;
  S.pool_map = nullptr;
  S.items[0] = c->items0.as<NnItem>();
  S.items[1] = c->items1.as<NnItem>();
  S.item_count[0] = c->item_count.as<int>();
  S.item_count[1] = c->item_count.as<int>() + (Jz + 1);
  S.item_off[0] = c->item_off.as<int>();
  S.item_off[1] = c->item_off.as<int>() + (Jz + 1);
  S.item_counter = c->item_counter.as<int>();
  S.nn_dyn = c->item_counter.as<int>() + 2;
  S.partials = c->partials.as<NnPartial>();
  S.tc_top = c->nn_tc ? c->tc_top.as<float4>() : nullptr;
  S.amb_pool = c->amb_pool.as<int2>();
  S.amb_n = c->amb_n.as<int>();
  S.amb_count = c->amb_count.as<int>();
  S.amb_cap = amb_cap;
  S.refine_list = c->refine_list.as<int4>();
  S.refine_count = c->refine_count.as<int>();
  S.refine_cap = static_cast<int>(refine_cap);
  S.stats = c->stats.as<unsigned long long>();
  S.iter_stats = c->iter_stats.as<unsigned long long>();
  S.trace_theta = c->trace_theta.as<double>();
  S.trace_loss = c->trace_loss.as<double>();
  S.trace_col = c->trace_col.as<int>();
  S.final_loss = c->final_loss.as<double>();
  S.final_free = c->final_free.as<int>();
  mark("buffers");
  CUDA_OK(cudaStreamSynchronize(st));
  c->pin_off = 0;  // every staged copy has landed: the next prepare reuses the buffer from the start
  mark("sync");
  // The captured graph bakes DevProblem/DevState and the k schedule into its
  // kernel parameters: keep it only if all of them are unchanged.
  std::vector<char> sig(sizeof(DevProblem) + sizeof(DevState));
  std::memcpy(sig.data(), &P, sizeof(DevProblem));
  std::memcpy(sig.data() + sizeof(DevProblem), &S, sizeof(DevState));
  auto push = [&](const void* ptr, size_t n) {
    const char* b = static_cast<const char*>(ptr);
    sig.insert(sig.end(), b, b + n);
  };
  push(c->ms.data(), c->ms.size() * sizeof(int64_t));
  push(c->gammas.data(), c->gammas.size() * sizeof(double));
  // Host-side launch shapes the capture bakes in as well (grids of the Stein
  // kernels, whether the grid-wide median runs and kmat is forked, the NN
  // plan / merge shapes, the partition).
  const int64_t extra[13] = {c->k_max,        c->k_stein,      c->record_trace,  c->max_chunks,
                             static_cast<int64_t>(c->seed),     c->max_pop,      c->max_gpop,
                             c->med_big_grid, c->max_ns,       c->target_items,  c->nn_grid,
                             c->J_glob,       c->rows_per_rank};
  push(extra, sizeof(extra));
  push(&c->eta_stein, sizeof(double));
  if (sig != c->graph_sig) {
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
    c->graph_valid = false;
    c->graph_sig = std::move(sig);
  }
  c->prepared = true;
}

// Profile mode: bracket a stage's launches with an event pair on the ctx stream.
struct StageTimer {
  asicp_ctx* c;
  cudaEvent_t b = nullptr;
  StageTimer(asicp_ctx* ctx, int stage, bool capture) : c(ctx) {
    if (!c->profile || capture) return;
    asicp_ctx::ProfEvent e{stage, nullptr, nullptr};
    CUDA_OK(cudaEventCreate(&e.a));
    CUDA_OK(cudaEventCreate(&e.b));
    c->prof_events.push_back(e);
    CUDA_OK(cudaEventRecord(e.a, c->stream));
    b = e.b;
  }
  ~StageTimer() {
    if (b) cudaEventRecord(b, c->stream);
  }
};

NnPlan make_plan(const asicp_ctx* c, int kind, int64_t m, bool pooled) {
  NnPlan plan{};
  plan.kind = kind;
  plan.pooled = pooled ? 1 : 0;
  plan.m = static_cast<int>(m);
  plan.fp64_mode = c->nn_mode == 1 ? 1 : 0;
  // Upper bound of the device-chosen split (nn.cu fwd_split): splits keep at
  // least 2 tiles of candidates each.
  plan.nchunks = std::max(1, std::min(c->max_chunks, static_cast<int>(m / (2 * kNnTile))));
  plan.target_items = c->target_items;
  static const int item_overhead = [] {  // ASICP_NN_ITEM_OVERHEAD: split-model experiments
    const char* e = std::getenv("ASICP_NN_ITEM_OVERHEAD");
    return e ? std::max(0, std::atoi(e)) : 1024;  // swept 128-2048: 1024 best on cfg2/cfg3/cfg4
  }();
  plan.item_overhead = item_overhead;
  plan.throughput = c->throughput;
  plan.max_ns = c->max_ns;
  plan.use_tc = c->nn_tc && !plan.fp64_mode ? 1 : 0;
  return plan;
}

// Enqueue one NN round (plan, optional minibatch, filter(s), merge, refine).
// In profile mode the forward/final filter launch is bracketed by events
// (the roofline kernel of bench.py).
void enqueue_nn(asicp_ctx* c, const NnPlan& plan, int minibatch_m, bool capture) {
  cudaStream_t st = c->stream;
  // The reverse match (colliding particles) needs neither the minibatch pools
  // nor the forward filter: fork it so it fills the SMs the draw leaves idle.
  // The item fill (both lists) depends only on the collision test, so it
  // goes on the fork too, ahead of the reverse match, and the forward filter
  // waits for it after the draw.
  const bool fork_rev = plan.kind == 0 && c->fork_rev && !c->profile;
  const bool fork_fill = fork_rev && minibatch_m > 0;
  if (fork_fill) {
    CUDA_OK(cudaEventRecord(c->ev_rev_fork, st));
    CUDA_OK(cudaStreamWaitEvent(c->rev_side, c->ev_rev_fork, 0));
    launch_nn_plan(c->P, c->S, plan, c->rev_side);
    CUDA_OK(cudaEventRecord(c->ev_fill, c->rev_side));
  } else {
    launch_nn_plan(c->P, c->S, plan, st);
  }
  int mb_launches = 0;
  if (minibatch_m > 0) {
    StageTimer t(c, asicp_ctx::kStMinibatch, capture);
    mb_launches = launch_minibatch(c->P, c->S, minibatch_m, st);
  }
  if (fork_rev) {
    if (!fork_fill) {  // the fill ran on the main stream: fork after it
      CUDA_OK(cudaEventRecord(c->ev_rev_fork, st));
      CUDA_OK(cudaStreamWaitEvent(c->rev_side, c->ev_rev_fork, 0));
    }
    launch_nn_rev(c->P, c->S, plan, 2 * c->num_sms, c->rev_side);
    CUDA_OK(cudaEventRecord(c->ev_rev_join, c->rev_side));
    if (fork_fill) CUDA_OK(cudaStreamWaitEvent(st, c->ev_fill, 0));
  }
  asicp_ctx::ProfEvent e{asicp_ctx::kStNn, nullptr, nullptr};
  if (c->profile && !capture) {
    CUDA_OK(cudaEventCreate(&e.a));
    CUDA_OK(cudaEventCreate(&e.b));
    c->prof_events.push_back(e);
  }
  const int n = launch_nn(c->P, c->S, plan, c->nn_grid, 2 * c->num_sms, st, e.a, e.b,
                          fork_rev ? c->ev_rev_join : nullptr);
  c->launches += 1 + n + mb_launches + (fork_rev ? 1 : 0);  // fill (plan fused) + filter(s), merge, refine + minibatch
}

// The whole optimize_grasp as a kernel sequence on c->stream.
void enqueue_solve(asicp_ctx* c, bool capture) {
  cudaStream_t st = c->stream;
  DevProblem& P = c->P;
  DevState& S = c->S;
  c->launches = 0;
  CUDA_OK(cudaMemcpyAsync(S.theta, c->init_theta_d.p, static_cast<size_t>(c->J) * 7 * 8, cudaMemcpyDeviceToDevice,
                          st));
  CUDA_OK(cudaMemsetAsync(S.stats, 0, kStats * sizeof(unsigned long long), st));
  CUDA_OK(cudaMemsetAsync(S.iter_stats, 0, c->iter_stats.bytes, st));
  // ASICP_DEBUG_SYNC=1 (eager runs only): synchronise after every stage and
  // name the stage a device fault surfaced in.
  static const bool dbg_sync = [] {
    const char* e = std::getenv("ASICP_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  int dbg_k = -1;
  auto stage = [&](const char* name) {
    if (!dbg_sync || capture) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
      throw DeviceError(std::string("asicp: device fault after ") + name + " (iteration " + std::to_string(dbg_k) +
                        "): " + cudaGetErrorString(e));
  };
  launch_init_state(P, S, st);
  launch_seed_rng(P, S, c->seed, st);
  c->launches += 2;
  stage("init");
  for (int k = 0; k < c->k_max; ++k) {
    dbg_k = k;
    const bool stein = k < c->k_stein;
    const int64_t m = c->ms[k];
    const bool pooled = m < c->n_obj;
    // The small-population median bandwidth reads only the poses at the start
    // of the iteration: fork it onto the side stream so its few CTAs overlap
    // the collision test / matching / cost (unsharded runs; sharded ones need
    // the pose all-gather first).  Joined before the Stein update.
    const bool fork_median = stein && !c->xchg && !dbg_sync && !c->profile;  // profile: every stage on one stream
    if (fork_median) {
      CUDA_OK(cudaEventRecord(c->ev_fork, st));
      CUDA_OK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
      launch_median_small(P, S, c->side);
      ++c->launches;
      if (S.kmat && c->med_big_grid == 0) {  // the split SVGD's kernel matrix: poses and h only
        launch_svgd_kmat(P, S, c->max_pop, c->max_gpop, c->side);
        ++c->launches;
      }
      CUDA_OK(cudaEventRecord(c->ev_join, c->side));
    }
    launch_pose_prep(P, S, 0, st);
    stage("pose_prep");
    {
      StageTimer t(c, asicp_ctx::kStCollide, capture);
      launch_collide(P, S, 0, 0, st);
    }
    stage("collide");
    S.pool_map = pooled ? S.pool_idx : nullptr;
    NnPlan plan = make_plan(c, 0, m, pooled);
    plan.iter = k;
    if (dbg_sync && !capture) {
      launch_nn_plan(c->P, c->S, plan, st);
      stage("nn_plan");
      if (pooled) {
        launch_minibatch(c->P, c->S, static_cast<int>(m), st);
        stage("minibatch");
      }
      launch_nn(c->P, c->S, plan, c->nn_grid, 2 * c->num_sms, st, nullptr, nullptr);
      stage("nn");
    } else {
      enqueue_nn(c, plan, pooled ? static_cast<int>(m) : 0, capture);
    }
    {
      StageTimer t(c, asicp_ctx::kStCost, capture);
      launch_cost(P, S, 0, st);
    }
    stage("cost");
    c->launches += 3;
    if (c->record_trace) {
      launch_trace(P, S, k, st);
      ++c->launches;
    }
    if (stein) {
      StageTimer t(c, asicp_ctx::kStSvgd, capture);
      launch_drift(P, S, c->gammas[k], c->n_ref, st);
      if (c->xchg) {
        // The population's poses and drifts from every rank, in global order.
        launch_pack_stein(P, S, c->xsend.as<double>(), st);
        c->xchg->allgather(c->xsend.p, c->xrecv.p, static_cast<size_t>(c->rows_per_rank) * 14 * 8, st);
        launch_unpack_stein(c->xrecv.as<double>(), c->theta_all.as<double>(), c->drift_all.as<double>(), c->J_glob,
                            c->xchg->world, c->rows_per_rank, st);
        c->launches += 2;
      }
      if (fork_median) CUDA_OK(cudaStreamWaitEvent(st, c->ev_join, 0));
      c->launches +=
          1 + launch_stein_update(P, S, c->eta_stein, c->max_pop, c->max_gpop, c->med_big_grid, st, !fork_median);
      stage("stein");
    } else {
      launch_sgd(P, S, st);
      ++c->launches;
    }
    launch_bookkeeping(P, S, stein ? 1 : 0, (k + 1) < c->k_stein ? 1 : 0, st);
    ++c->launches;
    stage("bookkeeping");
  }
  dbg_k = c->k_max;
  // Final ranking on the full reference cloud (grasp.cpp:260-281).
  S.pool_map = nullptr;
  launch_pose_prep(P, S, 1, st);
  stage("final pose_prep");
  launch_collide(P, S, 1, 1, st);
  stage("final collide");
  NnPlan fin = make_plan(c, 2, c->n_obj, false);
  fin.iter = c->k_max;
  enqueue_nn(c, fin, 0, capture);
  stage("final nn");
  launch_cost(P, S, 1, st);
  stage("final cost");
  c->launches += 3;
  if (c->xchg) {
    // Every rank receives every particle's summary (and trace): the solution
    // each rank returns is the whole population's.
    launch_pack_final(P, S, c->fsend.as<double>(), c->final_stride, c->k_max, c->record_trace, st);
    c->xchg->allgather(c->fsend.p, c->frecv.p, static_cast<size_t>(c->rows_per_rank) * c->final_stride * 8, st);
    ++c->launches;
  }
  CUDA_OK(cudaGetLastError());
}

// Enqueue one solve (graph replay) plus the D2H of the particle summaries
// into pinned staging; returns without waiting.
void launch(asicp_ctx* c) {
  NvtxRange range("asicp_run: launch");
  if (!c->prepared) throw InvalidArgument("asicp_run: no prepared problem");
  if (c->in_flight) throw InvalidArgument("asicp_run_async: a solve is already in flight (call asicp_wait)");
  CUDA_OK(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  for (auto& e : c->prof_events) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  c->prof_events.clear();
  CUDA_OK(cudaEventRecord(c->ev0, st));
  const bool graph = c->use_graph && !c->profile && (!c->xchg || c->xchg->capturable());
  if (graph) {
    if (!c->graph_valid) {
      NvtxRange capture_range("asicp_run: capture the solve graph");
      cudaGraph_t g;
      CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_solve(c, true);
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        throw;
      }
      CUDA_OK(cudaStreamEndCapture(st, &g));
      CUDA_OK(cudaGraphInstantiate(&c->graph_exec, g, 0));
      cudaGraphDestroy(g);
      c->graph_valid = true;
    }
    CUDA_OK(cudaGraphLaunch(c->graph_exec, st));
  } else {
    NvtxRange eager_range("asicp_run: eager enqueue");
    enqueue_solve(c, false);
  }
  CUDA_OK(cudaEventRecord(c->ev1, st));

  const size_t J = static_cast<size_t>(c->J);
  c->ensure_staging(c->J_glob);
  if (c->xchg) {
    const size_t bytes = static_cast<size_t>(c->xchg->world) * c->rows_per_rank * c->final_stride * 8;
    c->ensure_gath(bytes);
    CUDA_OK(cudaMemcpyAsync(c->host_gath, c->frecv.p, bytes, cudaMemcpyDeviceToHost, st));
  } else {
    CUDA_OK(cudaMemcpyAsync(c->host.theta, c->S.theta, 7 * J * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(c->host.floss, c->S.final_loss, J * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(c->host.ffree, c->S.final_free, J * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(c->host.conv, c->S.converged, J * 4, cudaMemcpyDeviceToHost, st));
  }
  CUDA_OK(cudaMemcpyAsync(c->host.stats, c->S.stats, kStats * 8, cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaMemcpyAsync(c->host.refine_total, c->S.refine_count, 4, cudaMemcpyDeviceToHost, st));
  c->in_flight = true;
}

// Wait for the launched solve and fill `out` (traces are copied here).
void finish(asicp_ctx* c, asicp_solution* out) {
  NvtxRange range("asicp_wait");
  if (!c->in_flight) throw InvalidArgument("asicp_wait: no solve in flight");
  cudaStream_t st = c->stream;
  c->in_flight = false;
  CUDA_OK(cudaStreamSynchronize(st));
  const int J = c->J_glob;
  const double* theta = c->host.theta;
  const double* floss = c->host.floss;
  const int* ffree = c->host.ffree;
  const int* conv = c->host.conv;
  const unsigned long long* stats = c->host.stats;
  const size_t rows = static_cast<size_t>(c->k_max) * J;
  if (c->xchg) {
    // Gathered summaries (rank-major blocks of rows_per_rank rows) -> global order.
    const int world = c->xchg->world, stride = c->final_stride;
    for (int r = 0; r < world; ++r) {
      const int lo = static_cast<int>(static_cast<int64_t>(r) * J / world);
      const int hi = static_cast<int>(static_cast<int64_t>(r + 1) * J / world);
      for (int i = 0; i < hi - lo; ++i) {
        const double* row = c->host_gath + (static_cast<size_t>(r) * c->rows_per_rank + i) * stride;
        const int g = lo + i;
        for (int a = 0; a < 7; ++a) c->host.theta[7 * g + a] = row[a];
        c->host.floss[g] = row[7];
        c->host.ffree[g] = static_cast<int>(row[8]);
        c->host.conv[g] = static_cast<int>(row[9]);
        if (!c->record_trace) continue;
        for (int k = 0; k < c->k_max; ++k) {
          const double* t = row + 10 + 9 * k;
          const size_t tr = static_cast<size_t>(k) * J + g;
          if (out->trace_theta)
            for (int a = 0; a < 7; ++a) out->trace_theta[7 * tr + a] = t[a];
          if (out->trace_loss) out->trace_loss[tr] = t[7];
          if (out->trace_in_collision) out->trace_in_collision[tr] = static_cast<int32_t>(t[8]);
        }
      }
    }
  } else if (c->record_trace && rows) {
    if (out->trace_theta)
      CUDA_OK(cudaMemcpyAsync(out->trace_theta, c->S.trace_theta, rows * 7 * 8, cudaMemcpyDeviceToHost, st));
    if (out->trace_loss)
      CUDA_OK(cudaMemcpyAsync(out->trace_loss, c->S.trace_loss, rows * 8, cudaMemcpyDeviceToHost, st));
    if (out->trace_in_collision)
      CUDA_OK(cudaMemcpyAsync(out->trace_in_collision, c->S.trace_col, rows * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  }
  if (*c->host.refine_total > c->S.refine_cap) throw DeviceError("asicp: FP64 refine list overflow");

  float ms = 0.0f;
  CUDA_OK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  asicp_stats& s = c->last_stats;
  s = asicp_stats{};
  s.solve_ms = ms;
  for (auto& e : c->prof_events) {
    float t = 0.0f;
    CUDA_OK(cudaEventElapsedTime(&t, e.a, e.b));
    switch (e.stage) {
      case asicp_ctx::kStNn:
        s.nn_ms += t;
        ++s.nn_launches;
        break;
      case asicp_ctx::kStCollide:
        s.collide_ms += t;
        break;
      case asicp_ctx::kStMinibatch:
        s.minibatch_ms += t;
        break;
      case asicp_ctx::kStCost:
        s.cost_ms += t;
        break;
      default:
        s.svgd_ms += t;
        break;
    }
  }
  s.kernel_launches = c->launches;

  // Final selection (grasp.cpp:283-306): strict < over collision-free
  // particles, else the best attempt with kNoGraspFound.
  out->n_particles = J;
  int best = -1;
  for (int j = 0; j < J; ++j) {
    if (!ffree[j]) continue;
    if (best < 0 || floss[j] < floss[best]) best = j;
  }
  if (best < 0) {
    out->status = ASICP_STATUS_NO_GRASP_FOUND;
    for (int j = 0; j < J; ++j)
      if (best < 0 || floss[j] < floss[best]) best = j;
  } else {
    out->status = ASICP_STATUS_FOUND;
  }
  for (int a = 0; a < 7; ++a) out->theta[a] = theta[7 * best + a];
  out->preshape_id = c->part_pre[best];
  out->final_loss = floss[best];
  out->converged = conv[best];
  for (int j = 0; j < J; ++j) {
    if (out->particle_theta)
      for (int a = 0; a < 7; ++a) out->particle_theta[7 * j + a] = theta[7 * j + a];
    if (out->particle_loss) out->particle_loss[j] = floss[j];
    if (out->particle_collision_free) out->particle_collision_free[j] = ffree[j];
    if (out->particle_converged) out->particle_converged[j] = conv[j];
    if (out->particle_preshape) out->particle_preshape[j] = c->part_pre[j];
  }
  out->nn_uncertified = static_cast<int64_t>(stats[0]);
  out->nn_full_refines = static_cast<int64_t>(stats[1]);
  out->nn_queries = static_cast<int64_t>(stats[2]);
  out->nn_pool_ties = static_cast<int64_t>(stats[3]);
  std::memcpy(c->raw_stats, stats, sizeof(c->raw_stats));
  out->nn_pairs = static_cast<double>(stats[4]);
  s.nn_pairs = static_cast<double>(stats[12]);  // pairs of the event-timed (forward/final) filter launches
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return ASICP_OK;
  } catch (const InvalidArgument& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_DEVICE_ERROR;
  }
}

}  // namespace

extern "C" {

int asicp_abi_version(void) { return ASICP_ABI_VERSION; }

asicp_ctx* asicp_create(int device, void* stream, char* err, size_t errlen) {
  asicp_ctx* c = new asicp_ctx();
  const int rc = guarded(err, errlen, [&] {
    c->device = device;
    CUDA_OK(cudaSetDevice(device));
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CUDA_OK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    nn_set_attrs();
    set_all_kernel_attrs();
    CUDA_OK(cudaEventCreate(&c->ev0));
    CUDA_OK(cudaEventCreate(&c->ev1));
    CUDA_OK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CUDA_OK(cudaStreamCreateWithFlags(&c->rev_side, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_rev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_rev_join, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_fill, cudaEventDisableTiming));
    c->nn_grid = c->num_sms * std::max(1, nn_blocks_per_sm());
  });
  if (rc != ASICP_OK) {
    delete c;
    return nullptr;
  }
  return c;
}

void asicp_destroy(asicp_ctx* ctx) { delete ctx; }

int asicp_set_option(asicp_ctx* ctx, int option, int64_t value) {
  if (!ctx) return ASICP_INVALID_ARGUMENT;
  switch (option) {
    case ASICP_OPT_NN_MODE:
      ctx->nn_mode = static_cast<int>(value);
      break;
    case ASICP_OPT_USE_GRAPH:
      ctx->use_graph = static_cast<int>(value);
      break;
    case ASICP_OPT_MAX_CHUNKS:
      ctx->max_chunks = std::max<int>(1, static_cast<int>(value));
      break;
    case ASICP_OPT_WINDOW_POOL:
      ctx->window_pool = std::max<int>(0, static_cast<int>(value));
      ctx->prepared = false;  // buffers are sized at prepare
      break;
    case ASICP_OPT_PROFILE:
      ctx->profile = static_cast<int>(value);
      break;
    case ASICP_OPT_NN_TC:
      ctx->nn_tc = value != 0;
      ctx->prepared = false;  // the TF32 candidate rows and the top-3 buffer are built at prepare
      break;
    case ASICP_OPT_THROUGHPUT:
      ctx->throughput = value ? 1 : 0;
      ctx->P.throughput = ctx->throughput;  // a prepared problem keeps its buffers; the graph is re-captured
      break;
    default:
      return ASICP_INVALID_ARGUMENT;
  }
  ctx->graph_valid = false;
  ctx->graph_sig.clear();
  if (ctx->graph_exec) {
    cudaGraphExecDestroy(ctx->graph_exec);
    ctx->graph_exec = nullptr;
  }
  return ASICP_OK;
}

int asicp_prepare(asicp_ctx* ctx, const asicp_problem* problem, char* err, size_t errlen) {
  if (!ctx || !problem) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] {
    if (ctx->in_flight) throw InvalidArgument("asicp_prepare: a solve is in flight (call asicp_wait)");
    prepare(ctx, *problem);
  });
}

int asicp_run(asicp_ctx* ctx, asicp_solution* solution, char* err, size_t errlen) {
  if (!ctx || !solution) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] {
    launch(ctx);
    finish(ctx, solution);
  });
}

int asicp_build_sdf(asicp_ctx* ctx, const double* cloud, int64_t n, double voxel, double padding, double band,
                    int32_t* dims, double* meta, float* values, char* err, size_t errlen) {
  if (!ctx || !cloud || !dims || !meta) return ASICP_INVALID_ARGUMENT;
  int rc = ASICP_OK;
  const int g = guarded(err, errlen, [&] {
    std::string msg;
    rc = build_sdf_device(ctx->device, ctx->stream, cloud, n, voxel, padding, band, dims, meta, values, &msg);
    if (rc != ASICP_OK) throw InvalidArgument(msg);
  });
  return g;
}

int asicp_nccl_unique_id(unsigned char* id, char* err, size_t errlen) {
  if (!id) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] { nccl_unique_id(id); });
}

static void reset_partition(asicp_ctx* ctx) {
  if (ctx->in_flight) throw InvalidArgument("asicp_set_partition: a solve is in flight (call asicp_wait)");
  ctx->xchg.reset();
  ctx->prepared = false;
  ctx->graph_valid = false;
  ctx->graph_sig.clear();
  if (ctx->graph_exec) {
    cudaGraphExecDestroy(ctx->graph_exec);
    ctx->graph_exec = nullptr;
  }
}

int asicp_set_partition_nccl(asicp_ctx* ctx, int rank, int world, const unsigned char* id, char* err, size_t errlen) {
  if (!ctx || !id || world < 1 || rank < 0 || rank >= world) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] {
    reset_partition(ctx);
    ctx->xchg = make_nccl_exchange(ctx->device, rank, world, id);
  });
}

asicp_group* asicp_group_create(int world) { return world >= 1 ? new asicp_group(world) : nullptr; }

void asicp_group_destroy(asicp_group* group) { delete group; }

int asicp_set_partition_group(asicp_ctx* ctx, asicp_group* group, int rank, char* err, size_t errlen) {
  if (!ctx || !group || rank < 0 || rank >= group->world) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] {
    reset_partition(ctx);
    ctx->xchg = make_group_exchange(group, rank);
  });
}

int asicp_clear_partition(asicp_ctx* ctx) {
  if (!ctx) return ASICP_INVALID_ARGUMENT;
  return guarded(nullptr, 0, [&] { reset_partition(ctx); });
}

int asicp_run_async(asicp_ctx* ctx, char* err, size_t errlen) {
  if (!ctx) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] { launch(ctx); });
}

int asicp_wait(asicp_ctx* ctx, asicp_solution* solution, char* err, size_t errlen) {
  if (!ctx || !solution) return ASICP_INVALID_ARGUMENT;
  return guarded(err, errlen, [&] { finish(ctx, solution); });
}

int asicp_optimize_grasp(asicp_ctx* ctx, const asicp_problem* problem, asicp_solution* solution, char* err,
                         size_t errlen) {
  const int rc = asicp_prepare(ctx, problem, err, errlen);
  if (rc != ASICP_OK) return rc;
  return asicp_run(ctx, solution, err, errlen);
}

int asicp_register_prepare(asicp_ctx* ctx, int64_t n_problems, const double* sources, const int64_t* source_offsets,
                           const double* references, const int64_t* reference_offsets, const double* initial,
                           const uint64_t* seeds, const asicp_sgd_config* cfg, char* err, size_t errlen) {
  if (!ctx || !cfg) return ASICP_INVALID_ARGUMENT;
  std::string msg;
  int rc = ASICP_OK;
  try {
    if (!ctx->reg) ctx->reg = std::make_unique<RegBatch>(ctx->device, ctx->stream);
    rc = ctx->reg->prepare(n_problems, sources, source_offsets, references, reference_offsets, initial, seeds, *cfg,
                           &msg);
  } catch (const std::exception& e) {
    msg = e.what();
    rc = ASICP_DEVICE_ERROR;
  }
  if (rc != ASICP_OK) copy_err(msg, err, errlen);
  return rc;
}

int asicp_register_run(asicp_ctx* ctx, asicp_registration* results, char* err, size_t errlen) {
  if (!ctx) return ASICP_INVALID_ARGUMENT;
  if (!ctx->reg) {
    copy_err("asicp: no registration batch prepared", err, errlen);
    return ASICP_INVALID_ARGUMENT;
  }
  std::string msg;
  const int rc = ctx->reg->run(results, &msg);
  if (rc != ASICP_OK) copy_err(msg, err, errlen);
  if (rc == ASICP_OK) {
    ctx->last_stats = asicp_stats{};
    ctx->last_stats.solve_ms = ctx->reg->last_kernel_ms();
    ctx->last_stats.kernel_launches = ctx->reg->launches();
  }
  return rc;
}

int asicp_register_sgd_icp_batch(asicp_ctx* ctx, int64_t n_problems, const double* sources,
                                 const int64_t* source_offsets, const double* references,
                                 const int64_t* reference_offsets, const double* initial, const uint64_t* seeds,
                                 const asicp_sgd_config* cfg, asicp_registration* results, char* err,
                                 size_t errlen) {
  const int rc = asicp_register_prepare(ctx, n_problems, sources, source_offsets, references, reference_offsets,
                                        initial, seeds, cfg, err, errlen);
  if (rc != ASICP_OK) return rc;
  return asicp_register_run(ctx, results, err, errlen);
}

int asicp_register_sgd_icp(asicp_ctx* ctx, const double* source, int64_t n_source, const double* reference,
                           int64_t n_reference, const double* initial, const asicp_sgd_config* cfg, uint64_t seed,
                           asicp_registration* result, char* err, size_t errlen) {
  const int64_t so[2] = {0, n_source}, ro[2] = {0, n_reference};
  return asicp_register_sgd_icp_batch(ctx, 1, source, so, reference, ro, initial, &seed, cfg, result, err, errlen);
}

int asicp_icp_closed_form_step_batch(asicp_ctx* ctx, int64_t n_problems, const double* sources,
                                     const int64_t* source_offsets, const double* references,
                                     const int64_t* reference_offsets, const double* thetas,
                                     asicp_icp_step* results, char* err, size_t errlen) {
  if (!ctx) return ASICP_INVALID_ARGUMENT;
  std::string msg;
  int rc = ASICP_OK;
  try {
    if (!ctx->reg) ctx->reg = std::make_unique<RegBatch>(ctx->device, ctx->stream);
    rc = ctx->reg->icp_step(n_problems, sources, source_offsets, references, reference_offsets, thetas, results,
                            &msg);
  } catch (const std::exception& e) {
    msg = e.what();
    rc = ASICP_DEVICE_ERROR;
  }
  if (rc != ASICP_OK) copy_err(msg, err, errlen);
  return rc;
}

int asicp_icp_closed_form_step(asicp_ctx* ctx, const double* source, int64_t n_source, const double* reference,
                               int64_t n_reference, const double* theta, asicp_icp_step* result, char* err,
                               size_t errlen) {
  const int64_t so[2] = {0, n_source}, ro[2] = {0, n_reference};
  return asicp_icp_closed_form_step_batch(ctx, 1, source, so, reference, ro, theta, result, err, errlen);
}

int asicp_get_stats(asicp_ctx* ctx, asicp_stats* stats) {
  if (!ctx || !stats) return ASICP_INVALID_ARGUMENT;
  *stats = ctx->last_stats;
  return ASICP_OK;
}

int64_t asicp_minibatch_schedule(int64_t k, int64_t k_max, int64_t n_ref) {
  return minibatch_schedule(k, k_max, n_ref);
}

double asicp_annealing(int64_t t, int64_t T, int64_t C, double p) { return annealing(t, T, C, p); }

double asicp_dbg_ffma_tflops(int iters) { return run_ffma_peak(iters); }
double asicp_dbg_dfma_tflops(int iters) { return run_dfma_peak(iters); }

int asicp_dbg_minibatch(uint64_t seed, int64_t n, const int64_t* ms, int64_t calls, int32_t parallel, int32_t* out) {
  const bool par = parallel != 0;
  // One particle stream (seed), `calls` consecutive minibatch draws of sizes
  // ms[c]; pool indices written back to back into out.
  try {
    set_all_kernel_attrs();
    DevProblem P{};
    DevState S{};
    P.J = 1;
    P.n_obj = static_cast<int>(n);
    P.n_obj_pad = static_cast<int>((n + kSubRows - 1) / kSubRows * kSubRows);
    Buf cand, active, ncol, st, mti, pidx, p32, fy;
    cand.ensure(static_cast<size_t>(P.n_obj_pad) * 16);
    CUDA_OK(cudaMemset(cand.p, 0, static_cast<size_t>(P.n_obj_pad) * 16));
    active.ensure(4);
    ncol.ensure(4);
    const int one = 1, zero = 0;
    CUDA_OK(cudaMemcpy(active.p, &one, 4, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(ncol.p, &zero, 4, cudaMemcpyHostToDevice));
    st.ensure(mt::kN * 8);
    mti.ensure(4);
    pidx.ensure(static_cast<size_t>(P.n_obj_pad) * 4);
    p32.ensure(static_cast<size_t>(P.n_obj_pad) * 16);
    fy.ensure(static_cast<size_t>(n) * 4);
    Buf fyp;
    if (par) fyp.ensure(5 * static_cast<size_t>(P.n_obj_pad) * 4);
    S.fy_par = par ? fyp.as<int>() : nullptr;
    S.fy_stride = 5 * static_cast<int64_t>(P.n_obj_pad);
    S.fy_batch = P.J;
    P.obj_cand = cand.as<float4>();
    P.obj_cand4 = cand.as<float4>();  // all-zero candidates: either layout
    S.active = active.as<int>();
    S.n_col = ncol.as<int>();
    S.rng_state = st.as<uint64_t>();
    S.rng_mti = mti.as<int>();
    S.pool_idx = pidx.as<int>();
    S.pool32 = p32.as<float4>();
    S.fy_scratch = fy.as<int>();
    launch_seed_rng(P, S, seed, nullptr);
    int64_t o = 0;
    for (int64_t c = 0; c < calls; ++c) {
      launch_minibatch(P, S, static_cast<int>(ms[c]), nullptr);
      CUDA_OK(cudaGetLastError());
      CUDA_OK(cudaMemcpy(out + o, S.pool_idx, static_cast<size_t>(ms[c]) * 4, cudaMemcpyDeviceToHost));
      o += ms[c];
    }
    const Buf* bufs[] = {&cand, &active, &ncol, &st, &mti, &pidx, &p32, &fy, &fyp};
    for (const Buf* b : bufs) const_cast<Buf*>(b)->release();
    return ASICP_OK;
  } catch (const std::exception&) {
    return ASICP_DEVICE_ERROR;
  }
}

int asicp_dbg_raw_stats(asicp_ctx* ctx, uint64_t* out16) {
  if (!ctx || !out16) return ASICP_INVALID_ARGUMENT;
  for (int i = 0; i < kStats; ++i) out16[i] = ctx->raw_stats[i];
  return ASICP_OK;
}

int64_t asicp_dbg_iter_stats(asicp_ctx* ctx, uint64_t* out, int64_t n) {
  if (!ctx || !ctx->prepared) return -1;
  const int64_t total = 4 * static_cast<int64_t>(ctx->k_max + 1);
  if (out && n > 0) {
    if (ctx->in_flight) return -1;
    if (cudaMemcpy(out, ctx->iter_stats.p, static_cast<size_t>(std::min(n, total)) * 8, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      return -1;
  }
  return total;
}

void asicp_dbg_exp_host(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = host_glibc_exp(x[i]);
}

int asicp_dbg_exp_device(const double* x, double* y, int64_t n) {
  double *dx = nullptr, *dy = nullptr;
  const size_t bytes = static_cast<size_t>(n) * sizeof(double);
  if (cudaMalloc(&dx, bytes) != cudaSuccess) return ASICP_DEVICE_ERROR;
  if (cudaMalloc(&dy, bytes) != cudaSuccess) {
    cudaFree(dx);
    return ASICP_DEVICE_ERROR;
  }
  cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice);
  launch_dbg_exp(dx, dy, n, nullptr);
  const cudaError_t e = cudaMemcpy(y, dy, bytes, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dy);
  return e == cudaSuccess ? ASICP_OK : ASICP_DEVICE_ERROR;
}

}  // extern "C"
