// Device-side problem / state layout of the B200 AS-ICP solver and the host
// launchers of its kernels (kernels.cu, nn.cu).  See DESIGN.md §3 for the HBM
// layout.
#pragma once

#include "dmath.cuh"
#include "nn.cuh"

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace asicp {

// Read-only problem data (uploaded once per asicp_prepare).
struct DevProblem {
  int J;            // particles (all preshapes, preshape-major)
  int n_obj;        // |R|
  int n_obj_pad;    // |R| rounded up to the NN subtile (padding rows are +inf)
  int n_scene;      // |C|
  int n_pop;        // Stein populations (= preshapes)
  const double* obj64;      // R, n_obj x 3
  const float4* obj_cand;   // R as FP32 NN candidates (-2b, |b|^2), b = r - center
  const float4* obj_cand4;  // the same candidates one float4 per point (minibatch pool gathers)
  const float4* obj_tc;     // their TF32 splits, 3 x float4 per point (tensor-core filter, nn.cu)
  const double* scene64;    // C, n_scene x 3
  const float4* scene32;    // C rounded to FP32 (x, y, z, |p|_1 rounded up), for the collision pre-test
  // Collision clusters (collide.cu): the scene sorted along a Morton curve and
  // cut into clusters of kClusterPts points; FP32 centre + radius per cluster.
  int n_clusters;
  const float4* clusters;   // (cx, cy, cz, r), r >= max |p - c|
  const float4* subclusters;  // n_clusters x kSubPerCluster spheres of kSubPts points
  const float4* scene_s32;  // scene32 in sorted order, n_clusters x kClusterPts
  const int* scene_perm;    // sorted position -> scene index (-1: padding)
  int col_lists_global;     // the collision kernel's cluster lists live in DevState::col_lists (large scenes)
  int throughput;           // the context shares the GPU with other solves (ASICP_OPT_THROUGHPUT)
  const double* surf64;     // concatenated preshape contact surfaces (gripper frame)
  const int* pre_surf_off;  // preshape -> offset into surf64 rows (n_pre + 1)
  const double* pre_tcp;    // preshape tcp, 3 per preshape
  const int* pre_sdf;       // preshape -> grid index
  const Grid* grids;
  const float* sdf_values;
  const float* sdf_coarse;  // per grid: dilated 4x4x4-block maxima (collision pre-test)
  int max_coarse;           // largest coarse grid (blocks)
  const int* part_pre;      // particle -> preshape
  const int64_t* part_surf_off;  // particle -> first surface row (rows padded to 32) (J + 1)
  const int* part_pop;      // particle -> population
  const int* pop_off;       // population -> first particle (n_pop + 1)
  const double* pop_logk1;  // log(K + 1) per population (host std::log)
  // Particle sharding: this context owns global particles
  // [j_lo, j_lo + J); populations span gpop_off in the global order, whose
  // poses and drifts the exchange gathers into DevState::theta_all/drift_all.
  // Unsharded: j_lo = 0, gpop_off = pop_off, theta_all = theta.
  const int* gpop_off;      // population -> first global particle (n_pop + 1)
  int j_lo;
  int med_mid;              // some population takes the cluster median (kMedBigK <= K <= kMedClusterK)
  const long long* kofs;    // population -> offset of its K x K_local block in DevState::kmat (split SVGD)
  // Forward-match re-centring (built on the device, launch_object_prepare):
  // [0..2] origin (the object centroid), [3] B_obj >= max |r - origin|.
  const double* obj_meta;
  double com[3];
  double contact_tolerance;
  double prior_t_mean[3];
  double prior_t_sigma[3];
  double prior_q_location[4];
  double prior_q_kappa[4];
  int bandwidth_mode;
  double fixed_bandwidth;
  double A[49];
  double lr;
  double conv_thr;
};

// Per-particle constants of the collision kernel's FP32 tests (collide.cu),
// derived in pose_prep_kernel from the FP64 inverse pose and the grid.
struct ColConst {
  float r[9], t[3];     // FP32 rotation / translation of the inverse pose
  float lo[3], cx[3], hx[3];  // grid box: origin, centre, half extent
  float d0;             // per-axis transform error bound, without the |p|_1 term
  float inv_vox;
  float tol32, tol_dn;  // float(tol), and the largest float <= tol
  float cut32;          // the largest float below the coarse cut
  float vm_pos, vm_c;   // value margins: per unit of position error, constant
  float lip;
  int cull_ok;
};

// Median select: populations below kMedBigK in one CTA, up to kMedClusterK
// in one thread-block cluster (median.cu), larger ones grid-wide (kernels.cu).
constexpr int kMedBigK = 320;
constexpr int kMedClusterK = 1536;
struct MedState {
  unsigned long long prefix, mask;
  long long rank;
};

// Mutable solver state (device pointers).
struct DevState {
  double2* kmat;           // split SVGD: (rbf, |q.q|) per (partner, own) pair, or null
  unsigned int* med_hist;  // n_pop x 4096 (grid-wide median select)
  MedState* med_state;     // n_pop
  double* theta;       // J x 7
  double* theta_next;  // J x 7 (SVGD double buffer)
  double* loss;
  double* prev_loss;
  int* in_col;
  int* converged;
  int* active;
  int* n_col;
  double* grad;        // J x 7 likelihood gradient
  double* drift;       // J x 7
  const double* theta_all;  // global J x 7 poses (SVGD partners / median)
  const double* drift_all;  // global J x 7 drifts
  double* h;           // per population bandwidth
  double* S64;         // transformed contact surface, padded rows x 3
  float4* Sq32;        // its FP32 forward queries (x, y, z, margin), object-centred
  float4* Sc32;        // its FP32 reverse candidates (-2b, |b|^2), particle-centred, pair-interleaved (pc_index)
  double* ctr;         // J x 3 per-particle reverse-match centre (TCP in world)
  double* Bs;          // per particle max |s - ctr|
  ColConst* colc;      // per particle collision-test constants
  int* col_lists;      // J x 5 x n_clusters cluster lists (only when DevProblem::col_lists_global)
  int* col_idx;        // J x n_scene colliding scene indices (scene order)
  float4* col_q;       // J x n_scene FP32 reverse queries (particle-centred)
  int* res_fwd;        // per surface row: NN position in the candidate set
  int* res_rev;        // J x n_scene: nearest surface index per colliding point
  uint64_t* rng_state; // J x 312
  int* rng_mti;        // J
  int* pool_idx;       // J x n_obj_pad minibatch object indices (sample order)
  float4* pool32;      // J x n_obj_pad gathered FP32 candidates (+inf padded)
  int* fy_scratch;     // J x n_obj Fisher-Yates scratch (large clouds only)
  int* fy_par;         // fy_batch x fy_stride scratch of the parallel Fisher-Yates (or null)
  int64_t fy_stride;   // 5 x n_obj_pad
  int fy_batch;        // particles the scratch covers (the minibatch launches in batches of these)
  const int* pool_map; // = pool_idx when this iteration's forward match is pooled
  NnItem* items[2];    // work lists: [0] forward / final, [1] reverse
  int* item_count[2];  // J + 1 each
  int* item_off[2];    // J + 1 each
  int* item_counter;   // 2 ints
  int* nn_dyn;         // device-chosen forward split: [0] splits, [1] forward items
  NnPartial* partials; // padded surface rows x max chunks
  float4* tc_top;      // tensor-core filter: per (query, split) top-3 subtile minima (b1, b2, b3, s1 | s2 << 16)
  int2* amb_pool;      // ambiguous-window member lists (kWinCap entries per block)
  int* amb_n;          // members per block (> kWinCap: overflow)
  int* amb_count;      // blocks allocated in the current NN round
  int amb_cap;         // blocks available
  int4* refine_list;
  int* refine_count;
  int refine_cap;
  unsigned long long* stats;  // [0] windows > 1, [1] full refines, [2] queries, [3] canonical-order ties, [4] pairs
  unsigned long long* iter_stats;  // per iteration k (k_max = final): [4k + list] pairs, [4k + 2 + list] queries
  double* trace_theta;
  double* trace_loss;
  int* trace_col;
  double* final_loss;
  int* final_free;
};

struct NnPlan {
  int kind;      // 0 iteration match, 2 final ranking
  int pooled;    // forward candidates are the particle's minibatch pool
  int m;         // forward candidate count
  int nchunks;   // upper bound on forward candidate splits (split-K); the device picks <= this
  int target_items;  // forward items the device split aims for (fills the persistent grid)
  int item_overhead; // per-item cost of the split model, in candidates (fwd_split)
  int throughput;    // split model for a GPU shared with other solves (ASICP_OPT_THROUGHPUT)
  int fp64_mode; // resolve every query by FP64 brute force (validation mode)
  int max_ns;    // largest contact surface (merge grid)
  int iter;      // iteration index (diagnostic counters)
  int use_tc;    // forward / final filter on the tensor cores (nn_tc_kernel)
};

// Per-device kernel attributes (opt-in shared memory), set for every context.
void kernels_set_attrs();
void collide_set_attrs();
void median_set_attrs();
void minibatch_set_attrs();
inline void set_all_kernel_attrs() {
  kernels_set_attrs();
  collide_set_attrs();
  median_set_attrs();
  minibatch_set_attrs();
}
void launch_grid_bounds(Grid* grids, int n_grids, const float* values, float* coarse, cudaStream_t st);
// Object cloud -> centroid, B_obj and the FP32 NN candidates (-2b, |b|^2),
// b = r - centroid: pair-interleaved (cand, n_pad rows, +inf padded) and plain
// (cand4).  meta = [centroid x, y, z, B_obj].
void launch_obj_tc(const float4* cand4, int n, float4* tc, cudaStream_t st);  // nn.cu
void launch_object_prepare(const double* obj64, int n, int n_pad, double* meta, float4* cand, float4* cand4,
                           cudaStream_t st);
// sdf_build.cu: graspmatch::build_sdf on the device (returns ASICP_OK or
// ASICP_INVALID_ARGUMENT with the reference message in *err; throws on CUDA
// errors).  values == null: geometry only (dims, meta = origin[3], voxel, 0).
int build_sdf_device(int device, cudaStream_t st, const double* cloud, int64_t n, double voxel, double padding,
                     double band, int32_t* dims, double* meta, float* values, std::string* err);
void launch_seed_rng(const DevProblem& P, DevState& S, uint64_t seed, cudaStream_t st);
void launch_init_state(const DevProblem& P, DevState& S, cudaStream_t st);
void launch_pose_prep(const DevProblem& P, DevState& S, int all, cudaStream_t st);
void launch_collide(const DevProblem& P, DevState& S, int all, int count_only, cudaStream_t st);  // collide.cu
bool collide_lists_global(const DevProblem& P);  // the lists do not fit the kernel's shared memory
constexpr int kClusterPts = 32;
constexpr int kSubPts = 8;
constexpr int kSubPerCluster = kClusterPts / kSubPts;
size_t scene_sort_temp_bytes(int n);
// Builds scene32 (original order) and the collision clusters from scene64 on
// the device: box, Morton codes, a stable radix sort, per-cluster centre and
// radius.  code/idx buffers: n each; temp: scene_sort_temp_bytes(n).
void launch_scene_prepare(const double* scene64, int n, float4* s32, double* box, unsigned int* code_in,
                          unsigned int* code_out, int* idx_in, int* perm, void* temp, size_t temp_bytes,
                          float4* clusters, float4* subclusters, float4* s32s, int* perm_pad, cudaStream_t st);
// Both return the number of launches (0: the parallel path does not apply).
int launch_minibatch(const DevProblem& P, DevState& S, int m, cudaStream_t st);
int launch_minibatch_par(const DevProblem& P, DevState& S, int m, cudaStream_t st);  // minibatch.cu
int minibatch_smem_cap();
void launch_cost(const DevProblem& P, DevState& S, int final_pass, cudaStream_t st);
void launch_trace(const DevProblem& P, DevState& S, int k, cudaStream_t st);
void launch_drift(const DevProblem& P, DevState& S, double gamma, double n_ref, cudaStream_t st);
void launch_median_small(const DevProblem& P, DevState& S, cudaStream_t st);  // median.cu (K < kMedBigK)
// big_grid > 0: some population has K >= kMedBigK; the grid-wide select runs
// with big_grid CTAs per population (returns the launch count).
// S.kmat != null selects the split SVGD (kmat + accumulate kernels);
// max_pop / max_gpop: largest local / global population.
void launch_svgd_kmat(const DevProblem& P, DevState& S, int max_pop, int max_gpop, cudaStream_t st);
// small_median = false: the caller already launched launch_median_small (and,
// for the split SVGD without a grid-wide median, launch_svgd_kmat)
// (e.g. on a forked stream, overlapping the iteration's matching).
int launch_stein_update(const DevProblem& P, DevState& S, double eta, int max_pop, int max_gpop, int big_grid,
                        cudaStream_t st, bool small_median = true);
// Particle-sharding exchange helpers: pack local rows [theta(7), drift(7)]
// into `send` (stride 14 doubles), and scatter a gathered world x rows_per_rank
// block back into global order (rank r's rows start at floor(r * J_glob / world)).
void launch_pack_stein(const DevProblem& P, const DevState& S, double* send, cudaStream_t st);
void launch_unpack_stein(const double* gathered, double* theta_all, double* drift_all, int J_glob, int world,
                         int rows_per_rank, cudaStream_t st);
// Final-summary pack: [theta(7), final_loss, final_free, converged] + trace
// (k_max x [theta(7), loss, in_collision]) per local row, stride `stride`.
void launch_pack_final(const DevProblem& P, const DevState& S, double* send, int stride, int k_max, int with_trace,
                       cudaStream_t st);
void launch_sgd(const DevProblem& P, DevState& S, cudaStream_t st);
void launch_bookkeeping(const DevProblem& P, DevState& S, int stein_phase, int next_stein, cudaStream_t st);
void launch_dbg_exp(const double* x, double* y, int64_t n, cudaStream_t st);
double host_glibc_exp(double x);
double run_ffma_peak(int iters);

// nn.cu
void launch_nn_plan(const DevProblem& P, DevState& S, const NnPlan& plan, cudaStream_t st);
int nn_smem_bytes();
void nn_set_attrs();
int nn_blocks_per_sm();
// Launches the forward/final list (and the reverse list when kind == 0),
// the merge (nchunks > 1) and the FP64 refine.  Returns the launch count.
int launch_nn(const DevProblem& P, DevState& S, const NnPlan& plan, int grid, int refine_grid, cudaStream_t st,
              cudaEvent_t ev_begin, cudaEvent_t ev_end, cudaEvent_t rev_done = nullptr);
// The reverse match alone (forked beside the minibatch draw and the forward
// filter; launch_nn then joins it through rev_done).
void launch_nn_rev(const DevProblem& P, DevState& S, const NnPlan& plan, int refine_grid, cudaStream_t st);

}  // namespace asicp
