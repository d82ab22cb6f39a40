// Drop-in definition of graspmatch::optimize_grasp (grasp.hpp:141) on the B200.
//
// This is the file a maintainer adds to the reference build in place of the
// definition at proj/src/grasp.cpp:132-307: it keeps the
// reference signature and error behaviour — GraspProblem::validate() runs on
// the host first (grasp.cpp:133), contract violations surface as
// graspmatch::InvalidArgument with the message the library reports — marshals
// the problem into the POD structs of include/asicp.h and fills the
// GraspSolution (particle summaries and the optional trace) from the device
// result.  `workers` is accepted and ignored: results are worker-count
// invariant in the reference too (test_acceptance.cpp:659-680).
//
// Built here only as test infrastructure (oracle/Makefile, against the
// reference headers and the Eigen shim) to run the reference's own
// optimize_grasp tests on the GPU path.
#include "asicp.h"
#include "graspmatch/grasp.hpp"
#include "graspmatch/optim.hpp"

#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace graspmatch {

namespace {

std::vector<double> flatten(const PointCloud& c) {
  std::vector<double> out;
  out.reserve(3 * c.size());
  for (const Vec3& p : c) {
    out.push_back(p[0]);
    out.push_back(p[1]);
    out.push_back(p[2]);
  }
  return out;
}

// One context per thread: device buffers and the captured CUDA graph are
// reused across calls (the reference call is stateless, so is this one).
asicp_ctx* thread_context() {
  thread_local struct Holder {
    asicp_ctx* ctx = nullptr;
    ~Holder() {
      if (ctx) asicp_destroy(ctx);
    }
  } holder;
  if (!holder.ctx) {
    char err[512] = {0};
    holder.ctx = asicp_create(0, nullptr, err, sizeof(err));
    if (!holder.ctx) throw std::runtime_error(std::string("asicp_create: ") + err);
  }
  return holder.ctx;
}

}  // namespace

GraspSolution optimize_grasp(const GraspProblem& problem) {
  problem.validate();  // grasp.cpp:133, identical messages

  // Marshal (FP64 throughout; the device keeps the reference's arithmetic).
  const std::vector<double> object = flatten(problem.object_cloud);
  const std::vector<double> scene = flatten(problem.scene_cloud);
  std::vector<std::vector<double>> surf, full;
  std::vector<asicp_preshape> pre;
  for (const Preshape& p : problem.preshapes) {
    surf.push_back(flatten(p.inner_surface_cloud));
    full.push_back(flatten(p.full_cloud));
  }
  for (size_t i = 0; i < problem.preshapes.size(); ++i) {
    const Preshape& p = problem.preshapes[i];
    asicp_preshape s{};
    s.inner_surface = surf[i].data();
    s.n_surface = static_cast<int64_t>(p.inner_surface_cloud.size());
    s.full_cloud = full[i].data();
    s.n_full = static_cast<int64_t>(p.full_cloud.size());
    for (int a = 0; a < 3; ++a) s.tcp[a] = p.tcp[a];
    s.sdf_index = static_cast<int64_t>(p.sdf_index);
    pre.push_back(s);
  }
  std::vector<asicp_sdf_grid> grids;
  for (size_t i = 0; i < problem.sdf.grids.size(); ++i) {
    const SdfGrid& g = problem.sdf.grids[i];
    asicp_sdf_grid s{};
    for (int a = 0; a < 3; ++a) {
      s.dims[a] = g.dims[a];
      s.origin[a] = g.origin[a];
      s.offset[a] = i < problem.sdf.offsets.size() ? problem.sdf.offsets[i][a] : 0.0;
    }
    s.voxel = g.voxel;
    s.boundary_max_abs = g.boundary_max_abs;
    s.values = g.values.data();
    grids.push_back(s);
  }
  std::vector<double> inits;
  std::vector<int64_t> counts;
  for (const auto& list : problem.initializations) {
    counts.push_back(static_cast<int64_t>(list.size()));
    for (const PoseParams& p : list) {
      const Vec7 v = p.as_vector();
      for (int a = 0; a < 7; ++a) inits.push_back(v[a]);
    }
  }
  asicp_problem ap{};
  ap.object_cloud = object.data();
  ap.n_object = static_cast<int64_t>(problem.object_cloud.size());
  ap.scene_cloud = scene.data();
  ap.n_scene = static_cast<int64_t>(problem.scene_cloud.size());
  ap.preshapes = pre.data();
  ap.n_preshapes = static_cast<int64_t>(pre.size());
  ap.sdf_grids = grids.data();
  ap.n_sdf_grids = static_cast<int64_t>(grids.size());
  for (int a = 0; a < 3; ++a) ap.com[a] = problem.com[a];
  ap.init_poses = inits.data();
  ap.init_counts = counts.data();
  ap.n_init_lists = static_cast<int64_t>(counts.size());
  ap.learning_rate = problem.sgd.learning_rate;
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) ap.A[7 * r + c] = problem.sgd.A(r, c);
  ap.convergence_threshold = problem.sgd.convergence_threshold;
  ap.bandwidth_mode =
      problem.stein.bandwidth_mode == BandwidthMode::kFixed ? ASICP_BANDWIDTH_FIXED : ASICP_BANDWIDTH_MEDIAN;
  ap.fixed_bandwidth = problem.stein.fixed_bandwidth;
  for (int a = 0; a < 3; ++a) {
    ap.prior_t_mean[a] = problem.stein.prior.t_mean[a];
    ap.prior_t_sigma[a] = problem.stein.prior.t_sigma[a];
  }
  for (int a = 0; a < 4; ++a) {
    ap.prior_q_location[a] = problem.stein.prior.q_location[a];
    ap.prior_q_kappa[a] = problem.stein.prior.q_kappa[a];
  }
  ap.anneal_period_total = static_cast<int64_t>(problem.stein.annealing.period_total);
  ap.anneal_cycles = static_cast<int64_t>(problem.stein.annealing.cycles);
  ap.anneal_exponent = problem.stein.annealing.exponent;
  ap.step_scale = problem.stein.step_scale;
  ap.k_stein = static_cast<int64_t>(problem.k_stein);
  ap.k_max = static_cast<int64_t>(problem.k_max);
  ap.contact_tolerance = problem.contact_tolerance;
  ap.seed = problem.seed;
  ap.workers = problem.workers;
  ap.record_trace = problem.record_trace ? 1 : 0;

  size_t J = 0;
  for (int64_t c : counts) J += static_cast<size_t>(c);
  std::vector<double> theta(7 * J), loss(J);
  std::vector<int32_t> free_(J), conv(J);
  std::vector<int64_t> pre_id(J);
  const size_t rows = problem.record_trace ? problem.k_max * J : 0;
  std::vector<double> tr_theta(7 * rows), tr_loss(rows);
  std::vector<int32_t> tr_col(rows);
  asicp_solution out{};
  out.particle_theta = theta.data();
  out.particle_loss = loss.data();
  out.particle_collision_free = free_.data();
  out.particle_converged = conv.data();
  out.particle_preshape = pre_id.data();
  if (rows) {
    out.trace_theta = tr_theta.data();
    out.trace_loss = tr_loss.data();
    out.trace_in_collision = tr_col.data();
  }
  char err[512] = {0};
  const int rc = asicp_optimize_grasp(thread_context(), &ap, &out, err, sizeof(err));
  if (rc == ASICP_INVALID_ARGUMENT) throw InvalidArgument(err);
  if (rc != ASICP_OK) throw std::runtime_error(std::string("asicp_optimize_grasp: ") + err);

  auto pose = [](const double* v) {
    Vec7 x;
    for (int a = 0; a < 7; ++a) x[a] = v[a];
    return PoseParams::from_vector(x);
  };
  GraspSolution sol;
  sol.status = out.status == ASICP_STATUS_FOUND ? GraspStatus::kFound : GraspStatus::kNoGraspFound;
  sol.theta = pose(out.theta);
  sol.preshape_id = static_cast<size_t>(out.preshape_id);
  sol.final_loss = out.final_loss;
  sol.converged = out.converged != 0;
  sol.particles.resize(J);
  for (size_t j = 0; j < J; ++j) {
    ParticleSummary& s = sol.particles[j];
    s.particle = j;
    s.preshape_id = static_cast<size_t>(pre_id[j]);
    s.theta = pose(&theta[7 * j]);
    s.full_cloud_loss = loss[j];
    s.collision_free = free_[j] != 0;
    s.converged = conv[j] != 0;
  }
  for (size_t r = 0; r < rows; ++r) {  // row-major iteration x particle (grasp.cpp:197-209)
    TraceRecord rec;
    rec.iteration = r / J;
    rec.particle = r % J;
    rec.preshape_id = static_cast<size_t>(pre_id[r % J]);
    rec.loss = tr_loss[r];
    rec.in_collision = tr_col[r] != 0;
    rec.phase = rec.iteration < problem.k_stein ? ParticlePhase::kStein : ParticlePhase::kSgd;
    rec.theta = pose(&tr_theta[7 * r]);
    sol.trace.push_back(rec);
  }
  return sol;
}

// Drop-in definition of graspmatch::register_sgd_icp (optim.hpp:170-176) in
// place of optim.cpp:274-321: same signature, same InvalidArgument messages,
// bit-identical RegistrationResult (csrc/register.cu).
RegistrationResult register_sgd_icp(const PointCloud& source, const PointCloud& reference, const PoseParams& initial,
                                    const SgdConfig& cfg, std::uint64_t seed) {
  asicp_sgd_config c{};
  c.learning_rate = cfg.learning_rate;
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) c.A[7 * i + j] = cfg.A(i, j);
  c.max_iterations = static_cast<int64_t>(cfg.max_iterations);
  c.convergence_threshold = cfg.convergence_threshold;
  c.preconditioner_mode = cfg.preconditioner_mode == PreconditionerMode::kGaussNewtonRotation
                              ? ASICP_PRECOND_GAUSS_NEWTON_ROTATION
                              : ASICP_PRECOND_FIXED;
  c.gn_damping = cfg.gn_damping;
  c.minibatch_size = static_cast<int64_t>(cfg.minibatch_size);
  const std::vector<double> src = flatten(source), ref = flatten(reference);
  const double init[7] = {initial.t[0], initial.t[1], initial.t[2], initial.q[0],
                          initial.q[1], initial.q[2], initial.q[3]};
  asicp_registration r{};
  char err[512] = {0};
  const int rc = asicp_register_sgd_icp(thread_context(), src.data(), static_cast<int64_t>(source.size()), ref.data(),
                                        static_cast<int64_t>(reference.size()), init, &c, seed, &r, err, sizeof(err));
  if (rc == ASICP_INVALID_ARGUMENT) throw InvalidArgument(err);
  if (rc != ASICP_OK) throw std::runtime_error(std::string("asicp_register_sgd_icp: ") + err);
  RegistrationResult out;
  out.theta.t = Vec3(r.theta[0], r.theta[1], r.theta[2]);
  out.theta.q = Vec4(r.theta[3], r.theta[4], r.theta[5], r.theta[6]);
  out.iterations = static_cast<std::size_t>(r.iterations);
  out.final_loss = r.final_loss;
  out.converged = r.converged != 0;
  return out;
}

// Drop-in definition of graspmatch::build_sdf (sdf.hpp:60-61) in place of
// sdf.cpp:48-175: the field is built on the GPU (csrc/sdf_build.cu), value for
// value the reference's, so everything downstream — stack_preshapes, the
// scenario front end's GMSDF001 cache files (io.cpp:555-580, save_sdf at
// sdf.cpp:256-285), the collision queries — sees identical bytes.
SdfGrid build_sdf(const PointCloud& cloud, double voxel, const SdfBuildOptions& options) {
  const std::vector<double> pts = flatten(cloud);
  int32_t dims[3] = {0, 0, 0};
  double meta[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  char err[512] = {0};
  const int64_t n = static_cast<int64_t>(cloud.size());
  // First call sizes the grid (values == NULL), the second fills it.
  int rc = asicp_build_sdf(thread_context(), pts.data(), n, voxel, options.padding, options.surface_band, dims, meta,
                           nullptr, err, sizeof(err));
  if (rc == ASICP_INVALID_ARGUMENT) throw InvalidArgument(err);
  if (rc != ASICP_OK) throw std::runtime_error(std::string("asicp_build_sdf: ") + err);
  SdfGrid grid;
  grid.values.resize(static_cast<size_t>(dims[0]) * static_cast<size_t>(dims[1]) * static_cast<size_t>(dims[2]));
  rc = asicp_build_sdf(thread_context(), pts.data(), n, voxel, options.padding, options.surface_band, dims, meta,
                       grid.values.data(), err, sizeof(err));
  if (rc == ASICP_INVALID_ARGUMENT) throw InvalidArgument(err);
  if (rc != ASICP_OK) throw std::runtime_error(std::string("asicp_build_sdf: ") + err);
  for (int a = 0; a < 3; ++a) grid.dims[a] = dims[a];
  grid.origin = Vec3(meta[0], meta[1], meta[2]);
  grid.voxel = meta[3];
  grid.boundary_max_abs = meta[4];
  return grid;
}

// Drop-in definition of graspmatch::icp_closed_form_step (optim.hpp:87-91)
// in place of optim.cpp:51-90.  The NnIndex argument is not needed: the GPU
// matches against the reference cloud itself (same answers, the kd-tree's
// tie rule).
ClosedFormStepResult icp_closed_form_step(const PointCloud& source, const PointCloud& reference,
                                          const PoseParams& theta, const NnIndex& /*index*/) {
  const std::vector<double> src = flatten(source), ref = flatten(reference);
  const double th[7] = {theta.t[0], theta.t[1], theta.t[2], theta.q[0], theta.q[1], theta.q[2], theta.q[3]};
  asicp_icp_step r{};
  char err[512] = {0};
  const int rc = asicp_icp_closed_form_step(thread_context(), src.data(), static_cast<int64_t>(source.size()),
                                            ref.data(), static_cast<int64_t>(reference.size()), th, &r, err,
                                            sizeof(err));
  if (rc == ASICP_INVALID_ARGUMENT) throw InvalidArgument(err);
  if (rc != ASICP_OK) throw std::runtime_error(std::string("asicp_icp_closed_form_step: ") + err);
  ClosedFormStepResult out;
  out.theta.t = Vec3(r.theta[0], r.theta[1], r.theta[2]);
  out.theta.q = Vec4(r.theta[3], r.theta[4], r.theta[5], r.theta[6]);
  out.degenerate = r.degenerate != 0;
  return out;
}

}  // namespace graspmatch
