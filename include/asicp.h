/*
 * asicp.h — C-ABI of the B200-native AS-ICP grasp optimiser.
 *
 * This is the drop-in boundary for the reference hot path
 *   graspmatch::GraspSolution graspmatch::optimize_grasp(const GraspProblem&)
 *   (/root/reference/proj/include/graspmatch/grasp.hpp:141, defined at
 *    /root/reference/proj/src/grasp.cpp:132-307).
 * It also replaces the registration entry points of SURVEY.md §8(f) rank 4,
 *   graspmatch::register_sgd_icp (optim.hpp:170-176, optim.cpp:274-321) and
 *   graspmatch::icp_closed_form_step (optim.hpp:87-91, optim.cpp:51-90),
 * declared further below.
 * The reference has no FFI layer of its own; its C++ entry point is replaced
 * at link time by the adapter in paper_2412_08346_b200/csrc/graspmatch_adapter.cpp,
 * which marshals GraspProblem into the POD structs below.
 *
 * Plain C: no torch/Eigen/CUDA types cross this boundary.  All point arrays are
 * row-major xyz float64 (n x 3); poses are 7-vectors (tx, ty, tz, qw, qx, qy, qz)
 * exactly like graspmatch::PoseParams::as_vector (types.hpp:24-41).
 *
 * Return codes of every int-returning entry point:
 *   ASICP_OK (0)            success
 *   ASICP_INVALID_ARGUMENT  contract violation; the message graspmatch would
 *                           have thrown as InvalidArgument is copied into err
 *   ASICP_DEVICE_ERROR      CUDA failure (message in err)
 */
#ifndef ASICP_H_
#define ASICP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASICP_ABI_VERSION 1

#define ASICP_OK 0
#define ASICP_INVALID_ARGUMENT 1
#define ASICP_DEVICE_ERROR 2

/* graspmatch::GraspStatus (grasp.hpp:76) */
#define ASICP_STATUS_FOUND 0
#define ASICP_STATUS_NO_GRASP_FOUND 1

/* graspmatch::BandwidthMode (optim.hpp:56) */
#define ASICP_BANDWIDTH_MEDIAN 0
#define ASICP_BANDWIDTH_FIXED 1

/* Context options (asicp_set_option). */
#define ASICP_OPT_NN_MODE 1        /* 0 = FP32 filter + FP64 certification (default), 1 = FP64 brute force */
#define ASICP_OPT_USE_GRAPH 2      /* 1 = capture the iteration loop in a CUDA graph (default 1) */
#define ASICP_OPT_PROFILE 3        /* 1 = record per-kernel CUDA events (asicp_get_stats) */
#define ASICP_OPT_MAX_CHUNKS 4     /* cap on the forward match's candidate split (default 16) */
#define ASICP_OPT_THROUGHPUT 6     /* 1 = this context shares the GPU with other solves (batch): the forward
                                      match splits its candidates for throughput, not for one solve's latency */
#define ASICP_OPT_NN_TC 7          /* 1 = forward / final NN filter on the tensor cores (tcgen05 TF32 split,
                                      bit-identical; default 0 = packed FFMA2) */
#define ASICP_OPT_WINDOW_POOL 5    /* ambiguous-window blocks per NN round (0 = sized automatically);
                                      an exhausted pool falls back to full FP64 rescans (testing) */

/* One voxel grid of the stacked gripper SDF (graspmatch::SdfGrid, sdf.hpp:23-39,
 * plus its StackedSdf offset, sdf.hpp:43-47). */
typedef struct asicp_sdf_grid {
  int32_t dims[3];           /* node counts per axis */
  double origin[3];
  double voxel;
  double boundary_max_abs;
  double offset[3];          /* StackedSdf::offsets[i] */
  const float* values;       /* dims[0]*dims[1]*dims[2], x-major ((ix*ny)+iy)*nz+iz */
} asicp_sdf_grid;

/* graspmatch::Preshape (grasp.hpp:16-24). */
typedef struct asicp_preshape {
  const double* inner_surface; /* S: n_surface x 3, gripper frame */
  int64_t n_surface;
  const double* full_cloud;    /* G: validated non-empty only (grasp.cpp:15) */
  int64_t n_full;
  double tcp[3];
  int64_t sdf_index;
} asicp_preshape;

/* graspmatch::GraspProblem (grasp.hpp:27-44) with SgdConfig / SteinConfig
 * (optim.hpp:28-76) flattened.  Caller-owned; never retained after return. */
typedef struct asicp_problem {
  const double* object_cloud;  /* R: n_object x 3 */
  int64_t n_object;
  const double* scene_cloud;   /* C: n_scene x 3 */
  int64_t n_scene;
  const asicp_preshape* preshapes;
  int64_t n_preshapes;
  const asicp_sdf_grid* sdf_grids;
  int64_t n_sdf_grids;
  double com[3];
  /* initializations: per preshape p, init_counts[p] poses; rows concatenated
   * preshape-major (the global particle order of grasp.cpp:135-145). */
  const double* init_poses;    /* J x 7 */
  const int64_t* init_counts;  /* n_init_lists entries */
  int64_t n_init_lists;        /* GraspProblem::initializations.size(); must equal n_preshapes */
  /* SgdConfig */
  double learning_rate;
  double A[49];                /* row-major 7x7 preconditioner */
  double convergence_threshold;
  /* SteinConfig */
  int32_t bandwidth_mode;
  double fixed_bandwidth;
  double prior_t_mean[3];
  double prior_t_sigma[3];
  double prior_q_location[4];
  double prior_q_kappa[4];
  int64_t anneal_period_total; /* AnnealingSchedule::period_total (T) */
  int64_t anneal_cycles;       /* C */
  double anneal_exponent;      /* p */
  double step_scale;
  /* GraspProblem scalars */
  int64_t k_stein;
  int64_t k_max;
  double contact_tolerance;
  uint64_t seed;
  int32_t workers;             /* accepted and ignored (results are worker-count invariant) */
  int32_t record_trace;
} asicp_problem;

/* graspmatch::GraspSolution (grasp.hpp:78-86).  Scalars are filled by the
 * library; every array pointer is caller-allocated and may be NULL. */
typedef struct asicp_solution {
  int32_t status;              /* ASICP_STATUS_* */
  double theta[7];
  int64_t preshape_id;
  double final_loss;
  int32_t converged;
  int64_t n_particles;         /* J (filled) */
  /* ParticleSummary (grasp.hpp:67-74), global particle order, J entries */
  double* particle_theta;      /* J x 7 */
  double* particle_loss;       /* J: full_cloud_loss */
  int32_t* particle_collision_free;
  int32_t* particle_converged;
  int64_t* particle_preshape;
  /* TraceRecord (grasp.hpp:57-65), row-major iteration x particle, k_max*J
   * entries, written only when record_trace != 0.  iteration / particle /
   * preshape / phase follow from the row index and the problem. */
  double* trace_theta;         /* (k_max*J) x 7, pre-update pose */
  double* trace_loss;          /* k_max*J */
  int32_t* trace_in_collision; /* k_max*J */
  /* Diagnostics (not part of the reference contract). */
  int64_t nn_queries;          /* nearest-neighbour queries resolved */
  int64_t nn_uncertified;      /* queries the FP32 filter could not certify alone */
  int64_t nn_full_refines;     /* queries that needed a full FP64 rescan */
  int64_t nn_pool_ties;        /* exact FP64 ties between distinct points resolved by canonical order */
  double nn_pairs;             /* (query, candidate) pairs evaluated by the NN kernels */
} asicp_solution;

/* Per-stage device timing collected when ASICP_OPT_PROFILE is set (the solve
 * then runs eagerly on the ctx stream, every stage bracketed by CUDA events);
 * only solve_ms and kernel_launches are filled otherwise. */
typedef struct asicp_stats {
  double solve_ms;             /* device time of the last asicp_run (events on the ctx stream) */
  double nn_ms;                /* summed device time of forward/final NN filter launches */
  int64_t nn_launches;
  double nn_pairs;             /* candidate pairs processed by those launches */
  double collide_ms;           /* collision test (colliding_points) launches */
  double minibatch_ms;         /* minibatch sampling + pool gather launches */
  double cost_ms;              /* cost / gradient launches of the iterations */
  double svgd_ms;              /* Stein step (drift, exchange, median, kernel matrix, update) */
  int64_t kernel_launches;     /* kernels enqueued by the last asicp_run */
} asicp_stats;

typedef struct asicp_ctx asicp_ctx;

/* ABI version check. */
int asicp_abi_version(void);

/* Create a context on CUDA device `device`.  `stream` is a cudaStream_t to
 * launch on (NULL: the context creates its own non-blocking stream).
 * Device buffers persist across calls. Returns NULL on failure (message in err). */
asicp_ctx* asicp_create(int device, void* stream, char* err, size_t errlen);
void asicp_destroy(asicp_ctx* ctx);

int asicp_set_option(asicp_ctx* ctx, int option, int64_t value);

/* Validate (GraspProblem::validate, grasp.cpp:20-31, plus the in-loop
 * requires) and upload the problem into device memory. */
int asicp_prepare(asicp_ctx* ctx, const asicp_problem* problem, char* err, size_t errlen);

/* Run optimize_grasp on the prepared, device-resident problem and fill the
 * solution (synchronous with respect to the host). */
int asicp_run(asicp_ctx* ctx, asicp_solution* solution, char* err, size_t errlen);

/* asicp_run split in two: enqueue the solve on the ctx stream and return
 * (per-particle summaries land in pinned staging), then wait and fill the
 * solution.  Contexts on different streams overlap on one GPU (batched
 * objects / preshape units).  One solve in flight per ctx. */
int asicp_run_async(asicp_ctx* ctx, char* err, size_t errlen);
int asicp_wait(asicp_ctx* ctx, asicp_solution* solution, char* err, size_t errlen);

/* Particle sharding within a population (no reference
 * counterpart — the reference runs one process).  Every rank prepares the SAME
 * full problem; rank r owns global particles [r J / R, (r + 1) J / R) and,
 * each Stein iteration, all-gathers the population's poses and drifts (the
 * median bandwidth and the Stein sums then read the whole population in the
 * reference order).  After the final ranking the particle summaries are
 * gathered, so every rank's asicp_solution is the full, unsharded answer.
 *
 * NCCL backend (one process per GPU): rank 0 makes the 128-byte id, the
 * caller broadcasts it, then every rank calls asicp_set_partition_nccl
 * (collective).  Group backend: contexts of one process, one host thread per
 * rank, exchanging through host memory.  Setting or clearing a partition
 * drops the prepared problem. */
/* graspmatch::build_sdf(cloud, voxel, {padding, surface_band}) (sdf.hpp,
 * sdf.cpp:48-175) on the ctx's device: exact FP64 node distances and the
 * widest-path sign, bit-identical to the reference field.  Fills dims and
 * meta = {origin x, y, z, voxel, boundary_max_abs}; values (dims[0] * dims[1]
 * * dims[2] floats, x-major) only when non-NULL — call once with NULL to size
 * the buffer.  padding < 0 selects the reference default (4 voxels).
 * ASICP_INVALID_ARGUMENT with the reference message for a non-positive voxel
 * or fewer than 4 / coplanar points. */
int asicp_build_sdf(asicp_ctx* ctx, const double* cloud, int64_t n, double voxel, double padding, double band,
                    int32_t* dims, double* meta, float* values, char* err, size_t errlen);

/* graspmatch::export_trace (io.hpp:94, io.cpp:691-710): write a solution's
 * per-iteration trace (record_trace) in the reference's 13-field text format
 * — "iteration particle preshape phase loss in_collision tx ty tz qw qx qy qz",
 * k-major like asicp_solution's trace arrays; phase = "stein" for
 * iterations < k_stein, else "sgd".  Host-only (no ctx).  Errors:
 * ASICP_INVALID_ARGUMENT "cannot write trace: <path>". */
int asicp_export_trace(const char* path, int64_t k_max, int64_t n_particles, int64_t k_stein,
                       const int64_t* particle_preshape, const double* trace_theta, const double* trace_loss,
                       const int32_t* trace_in_collision, char* err, size_t errlen);

typedef struct asicp_group asicp_group;
int asicp_nccl_unique_id(unsigned char* id /* 128 bytes */, char* err, size_t errlen);
int asicp_set_partition_nccl(asicp_ctx* ctx, int rank, int world, const unsigned char* id, char* err,
                             size_t errlen);
asicp_group* asicp_group_create(int world);
void asicp_group_destroy(asicp_group* group);
int asicp_set_partition_group(asicp_ctx* ctx, asicp_group* group, int rank, char* err, size_t errlen);
int asicp_clear_partition(asicp_ctx* ctx);

/* ------------------------------------------------------------------------
 * SGD-ICP registration: the drop-in for
 *   graspmatch::RegistrationResult graspmatch::register_sgd_icp(
 *       const PointCloud& source, const PointCloud& reference,
 *       const PoseParams& initial, const SgdConfig& cfg, std::uint64_t seed)
 *   (/root/reference/proj/include/graspmatch/optim.hpp:170-176, defined at
 *    /root/reference/proj/src/optim.cpp:274-321), bit-identical.
 * ------------------------------------------------------------------------ */

/* graspmatch::PreconditionerMode (optim.hpp:14-27) */
#define ASICP_PRECOND_FIXED 0
#define ASICP_PRECOND_GAUSS_NEWTON_ROTATION 1

/* graspmatch::SgdConfig (optim.hpp:29-43), every field. */
typedef struct asicp_sgd_config {
  double learning_rate;
  double A[49];                  /* row-major 7x7 */
  int64_t max_iterations;
  double convergence_threshold;  /* < 0 disables early stopping */
  int32_t preconditioner_mode;   /* ASICP_PRECOND_* */
  double gn_damping;
  int64_t minibatch_size;
} asicp_sgd_config;

/* graspmatch::RegistrationResult (optim.hpp:163-168). */
typedef struct asicp_registration {
  double theta[7];
  int64_t iterations;
  double final_loss;
  int32_t converged;
} asicp_registration;

/* One registration.  Errors (ASICP_INVALID_ARGUMENT, the reference message):
 * "register_sgd_icp: empty cloud", SgdConfig::validate (kFixed only),
 * "sample_minibatch: m out of range" (minibatch_size 0), "rotation_matrix:
 * quaternion is not unit-norm" (initial pose, or a pose that left the unit
 * sphere mid-run — the reference throws at that iteration too). */
int asicp_register_sgd_icp(asicp_ctx* ctx, const double* source, int64_t n_source, const double* reference,
                           int64_t n_reference, const double* initial /* 7 */, const asicp_sgd_config* cfg,
                           uint64_t seed, asicp_registration* result, char* err, size_t errlen);

/* A batch of independent registrations with one config (no reference
 * counterpart: the reference calls register_sgd_icp once per problem, e.g.
 * the 20 trials of test_acceptance.cpp:256-292).  Problem i registers
 * sources[source_offsets[i] .. source_offsets[i+1]) (rows of 3 doubles) into
 * references[reference_offsets[i] .. +1) from initial[7 i ..] with seeds[i];
 * results[i] is exactly what register_sgd_icp returns for it.  Problems are
 * validated in order; the first failure's message is returned. */
int asicp_register_sgd_icp_batch(asicp_ctx* ctx, int64_t n_problems, const double* sources,
                                 const int64_t* source_offsets, const double* references,
                                 const int64_t* reference_offsets, const double* initial, const uint64_t* seeds,
                                 const asicp_sgd_config* cfg, asicp_registration* results, char* err,
                                 size_t errlen);

/* The batch call split like asicp_prepare / asicp_run: validate + upload once,
 * then solve the device-resident batch (repeatable; each run restarts from the
 * uploaded initial poses and seeds). */
int asicp_register_prepare(asicp_ctx* ctx, int64_t n_problems, const double* sources, const int64_t* source_offsets,
                           const double* references, const int64_t* reference_offsets, const double* initial,
                           const uint64_t* seeds, const asicp_sgd_config* cfg, char* err, size_t errlen);
int asicp_register_run(asicp_ctx* ctx, asicp_registration* results, char* err, size_t errlen);

/* graspmatch::ClosedFormStepResult (optim.hpp:82-85). */
typedef struct asicp_icp_step {
  double theta[7];
  int32_t degenerate;
} asicp_icp_step;

/* graspmatch::icp_closed_form_step(source, reference, theta, index)
 * (optim.hpp:87-91, optim.cpp:51-90): match every transformed source point,
 * then the closed-form Kabsch/SVD step; bit-identical (the reference's
 * JacobiSVD is the oracle/shim one).  The NnIndex argument of the reference
 * is replaced by the reference cloud.  Errors: "icp_closed_form_step: empty
 * cloud", "rotation_matrix: quaternion is not unit-norm". */
int asicp_icp_closed_form_step(asicp_ctx* ctx, const double* source, int64_t n_source, const double* reference,
                               int64_t n_reference, const double* theta /* 7 */, asicp_icp_step* result, char* err,
                               size_t errlen);
/* n independent steps in one launch (one CTA each). */
int asicp_icp_closed_form_step_batch(asicp_ctx* ctx, int64_t n_problems, const double* sources,
                                     const int64_t* source_offsets, const double* references,
                                     const int64_t* reference_offsets, const double* thetas,
                                     asicp_icp_step* results, char* err, size_t errlen);

/* prepare + run: the drop-in for graspmatch::optimize_grasp. */
int asicp_optimize_grasp(asicp_ctx* ctx, const asicp_problem* problem, asicp_solution* solution,
                         char* err, size_t errlen);

int asicp_get_stats(asicp_ctx* ctx, asicp_stats* stats);

/* Host-side reference helpers used by the adapter/tests (pure functions). */
int64_t asicp_minibatch_schedule(int64_t k, int64_t k_max, int64_t n_ref); /* spatial_index.cpp:133-139 */
double asicp_annealing(int64_t t, int64_t T, int64_t C, double p);        /* optim.cpp:158-164 */

#ifdef __cplusplus
}
#endif

#endif /* ASICP_H_ */
