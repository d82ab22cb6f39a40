// Oracle bridge — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference (compiled from /root/reference/proj/src by
// oracle/Makefile) through the same POD structs as the product C-ABI
// (include/asicp.h), so tests and bench.py's CPU-baseline leg can run the
// reference graspmatch::optimize_grasp (grasp.cpp:132-307) on exactly the
// inputs the CUDA path receives.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load this library.
#include "asicp.h"
#include "graspmatch/geometry.hpp"
#include "graspmatch/grasp.hpp"
#include "graspmatch/io.hpp"
#include "graspmatch/optim.hpp"
#include "graspmatch/sdf.hpp"
#include "graspmatch/spatial_index.hpp"
#include "graspmatch/synthetic.hpp"

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

using namespace graspmatch;

namespace {

void copy_err(const std::string& msg, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = '\0';
  }
}

PointCloud to_cloud(const double* xyz, int64_t n) {
  PointCloud c;
  c.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) c.push_back(Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]));
  return c;
}

GraspProblem to_problem(const asicp_problem& p) {
  GraspProblem g;
  g.object_cloud = to_cloud(p.object_cloud, p.n_object);
  g.scene_cloud = to_cloud(p.scene_cloud, p.n_scene);
  for (int64_t i = 0; i < p.n_preshapes; ++i) {
    const asicp_preshape& s = p.preshapes[i];
    Preshape pre;
    pre.id = "preshape-" + std::to_string(i);
    pre.inner_surface_cloud = to_cloud(s.inner_surface, s.n_surface);
    pre.full_cloud = to_cloud(s.full_cloud, s.n_full);
    pre.tcp = Vec3(s.tcp[0], s.tcp[1], s.tcp[2]);
    pre.sdf_index = static_cast<size_t>(s.sdf_index);
    g.preshapes.push_back(pre);
  }
  double eps = 0.0;
  for (int64_t i = 0; i < p.n_sdf_grids; ++i) {
    const asicp_sdf_grid& s = p.sdf_grids[i];
    SdfGrid grid;
    grid.origin = Vec3(s.origin[0], s.origin[1], s.origin[2]);
    grid.voxel = s.voxel;
    grid.dims = {s.dims[0], s.dims[1], s.dims[2]};
    const size_t total = static_cast<size_t>(s.dims[0]) * s.dims[1] * s.dims[2];
    grid.values.assign(s.values, s.values + total);
    grid.boundary_max_abs = s.boundary_max_abs;
    g.sdf.grids.push_back(grid);
    g.sdf.offsets.push_back(Vec3(s.offset[0], s.offset[1], s.offset[2]));
  }
  g.sdf.epsilon = eps;
  g.com = Vec3(p.com[0], p.com[1], p.com[2]);
  int64_t row = 0;
  for (int64_t i = 0; i < p.n_init_lists; ++i) {
    std::vector<PoseParams> poses;
    for (int64_t k = 0; k < p.init_counts[i]; ++k, ++row) {
      Vec7 v;
      for (int a = 0; a < 7; ++a) v[a] = p.init_poses[7 * row + a];
      poses.push_back(PoseParams::from_vector(v));
    }
    g.initializations.push_back(poses);
  }
  g.sgd.learning_rate = p.learning_rate;
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) g.sgd.A(r, c) = p.A[7 * r + c];
  g.sgd.convergence_threshold = p.convergence_threshold;
  g.stein.bandwidth_mode =
      p.bandwidth_mode == ASICP_BANDWIDTH_FIXED ? BandwidthMode::kFixed : BandwidthMode::kMedianHeuristic;
  g.stein.fixed_bandwidth = p.fixed_bandwidth;
  for (int a = 0; a < 3; ++a) {
    g.stein.prior.t_mean[a] = p.prior_t_mean[a];
    g.stein.prior.t_sigma[a] = p.prior_t_sigma[a];
  }
  for (int a = 0; a < 4; ++a) {
    g.stein.prior.q_location[a] = p.prior_q_location[a];
    g.stein.prior.q_kappa[a] = p.prior_q_kappa[a];
  }
  g.stein.annealing.period_total = static_cast<size_t>(p.anneal_period_total);
  g.stein.annealing.cycles = static_cast<size_t>(p.anneal_cycles);
  g.stein.annealing.exponent = p.anneal_exponent;
  g.stein.step_scale = p.step_scale;
  g.k_stein = static_cast<size_t>(p.k_stein);
  g.k_max = static_cast<size_t>(p.k_max);
  g.contact_tolerance = p.contact_tolerance;
  g.seed = p.seed;
  g.workers = p.workers;
  g.record_trace = p.record_trace != 0;
  return g;
}

// Owns everything an asicp_problem view points into.
struct Holder {
  PointCloud object, scene;
  std::vector<std::vector<double>> surf, full;
  std::vector<std::vector<float>> values;
  std::vector<double> object_flat, scene_flat, inits;
  std::vector<int64_t> counts;
  std::vector<asicp_preshape> pre;
  std::vector<asicp_sdf_grid> grids;
  asicp_problem view{};
};

std::vector<double> flat(const PointCloud& c) {
  std::vector<double> out;
  out.reserve(3 * c.size());
  for (const Vec3& p : c) {
    out.push_back(p[0]);
    out.push_back(p[1]);
    out.push_back(p[2]);
  }
  return out;
}

Holder* hold(const GraspProblem& g) {
  auto* h = new Holder();
  h->object_flat = flat(g.object_cloud);
  h->scene_flat = flat(g.scene_cloud);
  for (const Preshape& p : g.preshapes) {
    h->surf.push_back(flat(p.inner_surface_cloud));
    h->full.push_back(flat(p.full_cloud));
  }
  for (size_t i = 0; i < g.preshapes.size(); ++i) {
    asicp_preshape s{};
    s.inner_surface = h->surf[i].data();
    s.n_surface = static_cast<int64_t>(g.preshapes[i].inner_surface_cloud.size());
    s.full_cloud = h->full[i].data();
    s.n_full = static_cast<int64_t>(g.preshapes[i].full_cloud.size());
    for (int a = 0; a < 3; ++a) s.tcp[a] = g.preshapes[i].tcp[a];
    s.sdf_index = static_cast<int64_t>(g.preshapes[i].sdf_index);
    h->pre.push_back(s);
  }
  for (size_t i = 0; i < g.sdf.grids.size(); ++i) h->values.push_back(g.sdf.grids[i].values);
  for (size_t i = 0; i < g.sdf.grids.size(); ++i) {
    const SdfGrid& gr = g.sdf.grids[i];
    asicp_sdf_grid s{};
    for (int a = 0; a < 3; ++a) {
      s.dims[a] = gr.dims[a];
      s.origin[a] = gr.origin[a];
      s.offset[a] = g.sdf.offsets[i][a];
    }
    s.voxel = gr.voxel;
    s.boundary_max_abs = gr.boundary_max_abs;
    s.values = h->values[i].data();
    h->grids.push_back(s);
  }
  for (const auto& poses : g.initializations) {
    h->counts.push_back(static_cast<int64_t>(poses.size()));
    for (const PoseParams& p : poses) {
      const Vec7 v = p.as_vector();
      for (int a = 0; a < 7; ++a) h->inits.push_back(v[a]);
    }
  }
  asicp_problem& v = h->view;
  v.object_cloud = h->object_flat.data();
  v.n_object = static_cast<int64_t>(g.object_cloud.size());
  v.scene_cloud = h->scene_flat.data();
  v.n_scene = static_cast<int64_t>(g.scene_cloud.size());
  v.preshapes = h->pre.data();
  v.n_preshapes = static_cast<int64_t>(h->pre.size());
  v.sdf_grids = h->grids.data();
  v.n_sdf_grids = static_cast<int64_t>(h->grids.size());
  for (int a = 0; a < 3; ++a) v.com[a] = g.com[a];
  v.init_poses = h->inits.data();
  v.init_counts = h->counts.data();
  v.n_init_lists = static_cast<int64_t>(h->counts.size());
  v.learning_rate = g.sgd.learning_rate;
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) v.A[7 * r + c] = g.sgd.A(r, c);
  v.convergence_threshold = g.sgd.convergence_threshold;
  v.bandwidth_mode = g.stein.bandwidth_mode == BandwidthMode::kFixed ? ASICP_BANDWIDTH_FIXED
                                                                     : ASICP_BANDWIDTH_MEDIAN;
  v.fixed_bandwidth = g.stein.fixed_bandwidth;
  for (int a = 0; a < 3; ++a) {
    v.prior_t_mean[a] = g.stein.prior.t_mean[a];
    v.prior_t_sigma[a] = g.stein.prior.t_sigma[a];
  }
  for (int a = 0; a < 4; ++a) {
    v.prior_q_location[a] = g.stein.prior.q_location[a];
    v.prior_q_kappa[a] = g.stein.prior.q_kappa[a];
  }
  v.anneal_period_total = static_cast<int64_t>(g.stein.annealing.period_total);
  v.anneal_cycles = static_cast<int64_t>(g.stein.annealing.cycles);
  v.anneal_exponent = g.stein.annealing.exponent;
  v.step_scale = g.stein.step_scale;
  v.k_stein = static_cast<int64_t>(g.k_stein);
  v.k_max = static_cast<int64_t>(g.k_max);
  v.contact_tolerance = g.contact_tolerance;
  v.seed = g.seed;
  v.workers = g.workers;
  v.record_trace = g.record_trace ? 1 : 0;
  return h;
}

}  // namespace

extern "C" {

// graspmatch::optimize_grasp (grasp.cpp:132) on an asicp_problem.
int ref_optimize_grasp(const asicp_problem* p, asicp_solution* out, char* err, size_t errlen) {
  try {
    const GraspProblem g = to_problem(*p);
    const GraspSolution s = optimize_grasp(g);
    out->status = s.status == GraspStatus::kFound ? ASICP_STATUS_FOUND : ASICP_STATUS_NO_GRASP_FOUND;
    const Vec7 th = s.theta.as_vector();
    for (int a = 0; a < 7; ++a) out->theta[a] = th[a];
    out->preshape_id = static_cast<int64_t>(s.preshape_id);
    out->final_loss = s.final_loss;
    out->converged = s.converged ? 1 : 0;
    out->n_particles = static_cast<int64_t>(s.particles.size());
    for (size_t j = 0; j < s.particles.size(); ++j) {
      const ParticleSummary& ps = s.particles[j];
      const Vec7 v = ps.theta.as_vector();
      if (out->particle_theta)
        for (int a = 0; a < 7; ++a) out->particle_theta[7 * j + a] = v[a];
      if (out->particle_loss) out->particle_loss[j] = ps.full_cloud_loss;
      if (out->particle_collision_free) out->particle_collision_free[j] = ps.collision_free ? 1 : 0;
      if (out->particle_converged) out->particle_converged[j] = ps.converged ? 1 : 0;
      if (out->particle_preshape) out->particle_preshape[j] = static_cast<int64_t>(ps.preshape_id);
    }
    for (size_t r = 0; r < s.trace.size(); ++r) {
      const TraceRecord& t = s.trace[r];
      const Vec7 v = t.theta.as_vector();
      if (out->trace_theta)
        for (int a = 0; a < 7; ++a) out->trace_theta[7 * r + a] = v[a];
      if (out->trace_loss) out->trace_loss[r] = t.loss;
      if (out->trace_in_collision) out->trace_in_collision[r] = t.in_collision ? 1 : 0;
    }
    return ASICP_OK;
  } catch (const InvalidArgument& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_DEVICE_ERROR;
  }
}

// graspmatch::optimize_grasp with record_trace, then graspmatch::export_trace
// (io.cpp:691-710) of its trace to `path` — the reference trace file.
int ref_optimize_and_export_trace(const asicp_problem* p, const char* path, char* err, size_t errlen) {
  try {
    GraspProblem g = to_problem(*p);
    g.record_trace = true;
    const GraspSolution s = optimize_grasp(g);
    export_trace(s.trace, path);
    return ASICP_OK;
  } catch (const InvalidArgument& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_DEVICE_ERROR;
  }
}

// The desk scenario (synthetic.cpp) solved with the given schedule and its
// trace exported by graspmatch::export_trace — callable without any other
// C++ runtime in the process (the library links libstdc++ statically, and
// its iostreams must not meet a second libstdc++, e.g. numpy's).
int ref_desk_export_trace(uint64_t seed, int64_t n_init, int64_t n_top, int64_t k_max, int64_t k_stein,
                          int64_t anneal_total, const char* path) {
  try {
    GraspProblem g = synthetic::desk_grasp_problem(seed, 0, static_cast<size_t>(n_init), static_cast<size_t>(n_top));
    g.k_max = static_cast<size_t>(k_max);
    g.k_stein = static_cast<size_t>(k_stein);
    g.stein.annealing.period_total = static_cast<size_t>(anneal_total);
    g.record_trace = true;
    const GraspSolution s = optimize_grasp(g);
    export_trace(s.trace, path);
    return ASICP_OK;
  } catch (const std::exception&) {
    return ASICP_DEVICE_ERROR;
  }
}

// Reference fixtures (synthetic.cpp) as an owned asicp_problem view.
void* ref_desk_problem(uint64_t seed, int workers, int64_t n_init, int64_t n_top) {
  const GraspProblem g = synthetic::desk_grasp_problem(seed, workers, static_cast<size_t>(n_init),
                                                       static_cast<size_t>(n_top));
  return hold(g);
}

// Reference self-matching problem of test_grasp.cpp:46-57 (two-finger contact
// surface as object, far-away scene).
void* ref_self_matching_problem() {
  const auto two_finger = synthetic::two_finger_preshape();
  GraspProblem problem;
  problem.object_cloud = two_finger.preshape.inner_surface_cloud;
  problem.scene_cloud = PointCloud{Vec3(10.0, 10.0, 10.0)};
  problem.preshapes = {two_finger.preshape};
  problem.sdf = stack_preshapes({build_sdf(two_finger.preshape.full_cloud, 0.005)}, 0.05);
  problem.com = two_finger.preshape.tcp;
  problem.workers = 1;
  problem.initializations = {{PoseParams::identity()}};
  return hold(problem);
}

asicp_problem* ref_problem_view(void* h) { return &static_cast<Holder*>(h)->view; }
void ref_problem_free(void* h) { delete static_cast<Holder*>(h); }

// Building blocks for component-level goldens.
void ref_cylinder_cloud(double radius, double height, int n, uint64_t seed, double* out) {
  const auto c = synthetic::cylinder_cloud(radius, height, n, seed);
  for (size_t i = 0; i < c.size(); ++i)
    for (int a = 0; a < 3; ++a) out[3 * i + a] = c[i][a];
}

int ref_sample_minibatch_indices(uint64_t seed, int64_t skip, int64_t n, int64_t m, int64_t* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < skip; ++i) rng.next_u64();
  try {
    const auto idx = sample_minibatch_indices(static_cast<size_t>(n), static_cast<size_t>(m), rng);
    for (size_t i = 0; i < idx.size(); ++i) out[i] = static_cast<int64_t>(idx[i]);
  } catch (const InvalidArgument&) {
    return ASICP_INVALID_ARGUMENT;
  }
  return ASICP_OK;
}

// graspmatch::register_sgd_icp (optim.cpp:274-321) on the C-ABI's structs.
int ref_register_sgd_icp(const double* source, int64_t n_source, const double* reference, int64_t n_reference,
                         const double* initial, const asicp_sgd_config* c, uint64_t seed, asicp_registration* out,
                         char* err, size_t errlen) {
  SgdConfig cfg;
  cfg.learning_rate = c->learning_rate;
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) cfg.A(i, j) = c->A[7 * i + j];
  cfg.max_iterations = static_cast<size_t>(c->max_iterations);
  cfg.convergence_threshold = c->convergence_threshold;
  cfg.preconditioner_mode = c->preconditioner_mode == ASICP_PRECOND_GAUSS_NEWTON_ROTATION
                                ? PreconditionerMode::kGaussNewtonRotation
                                : PreconditionerMode::kFixed;
  cfg.gn_damping = c->gn_damping;
  cfg.minibatch_size = static_cast<size_t>(c->minibatch_size);
  PoseParams init;
  init.t = Vec3(initial[0], initial[1], initial[2]);
  init.q = Vec4(initial[3], initial[4], initial[5], initial[6]);
  try {
    const RegistrationResult r =
        register_sgd_icp(to_cloud(source, n_source), to_cloud(reference, n_reference), init, cfg, seed);
    for (int i = 0; i < 3; ++i) out->theta[i] = r.theta.t[i];
    for (int i = 0; i < 4; ++i) out->theta[3 + i] = r.theta.q[i];
    out->iterations = static_cast<int64_t>(r.iterations);
    out->final_loss = r.final_loss;
    out->converged = r.converged ? 1 : 0;
  } catch (const InvalidArgument& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_INVALID_ARGUMENT;
  }
  return ASICP_OK;
}

// graspmatch::icp_closed_form_step (optim.cpp:51-90).
int ref_icp_closed_form_step(const double* source, int64_t n_source, const double* reference, int64_t n_reference,
                             const double* theta, asicp_icp_step* out, char* err, size_t errlen) {
  try {
    const PointCloud ref = to_cloud(reference, n_reference);
    PoseParams th;
    th.t = Vec3(theta[0], theta[1], theta[2]);
    th.q = Vec4(theta[3], theta[4], theta[5], theta[6]);
    if (ref.empty()) {  // build_index would throw its own message first; the reference test passes an index
      copy_err("icp_closed_form_step: empty cloud", err, errlen);
      return ASICP_INVALID_ARGUMENT;
    }
    const NnIndex index = build_index(ref);
    const ClosedFormStepResult r = icp_closed_form_step(to_cloud(source, n_source), ref, th, index);
    for (int i = 0; i < 3; ++i) out->theta[i] = r.theta.t[i];
    for (int i = 0; i < 4; ++i) out->theta[3 + i] = r.theta.q[i];
    out->degenerate = r.degenerate ? 1 : 0;
  } catch (const InvalidArgument& e) {
    copy_err(e.what(), err, errlen);
    return ASICP_INVALID_ARGUMENT;
  }
  return ASICP_OK;
}

// test_acceptance.cpp:48-52 + 256-282: the C2 trial inputs, from the
// reference's own generators.
void ref_c2_trial(int trial, int n, double* source, double* reference, double* truth7) {
  const PointCloud ref = synthetic::box_surface_cloud(n, Vec3(0.05, 0.03, 0.02), 42);
  Rng rng(100 + trial);
  Vec3 axis(rng.normal(), rng.normal(), rng.normal());
  const double angle = rng.uniform(0.0, M_PI / 6.0);
  axis.normalize();
  const double sh = std::sin(angle / 2.0);
  PoseParams truth;
  truth.q = Vec4(std::cos(angle / 2.0), sh * axis.x(), sh * axis.y(), sh * axis.z());
  Vec3 dir(rng.normal(), rng.normal(), rng.normal());
  dir.normalize();
  truth.t = dir * rng.uniform(0.0, 0.2);
  const Mat3 r_true = rotation_matrix(truth.q);
  for (size_t i = 0; i < ref.size(); ++i) {
    const Vec3 s = r_true.transpose() * (ref[i] - truth.t);
    for (int a = 0; a < 3; ++a) {
      source[3 * i + a] = s[a];
      reference[3 * i + a] = ref[i][a];
    }
  }
  for (int i = 0; i < 3; ++i) truth7[i] = truth.t[i];
  for (int i = 0; i < 4; ++i) truth7[3 + i] = truth.q[i];
}

void ref_blob_cloud(int n, double radius, uint64_t seed, double* out) {
  const auto c = synthetic::blob_cloud(n, radius, seed);
  for (size_t i = 0; i < c.size(); ++i)
    for (int a = 0; a < 3; ++a) out[3 * i + a] = c[i][a];
}

double ref_quaternion_angle(const double* q1, const double* q2) {
  return quaternion_angle(Vec4(q1[0], q1[1], q1[2], q1[3]), Vec4(q2[0], q2[1], q2[2], q2[3]));
}

int64_t ref_nearest(const double* cloud, int64_t n, const double* q, double* dist) {
  const NnIndex idx = build_index(to_cloud(cloud, n));
  const NearestResult r = idx.nearest(Vec3(q[0], q[1], q[2]));
  if (dist) *dist = r.distance;
  return static_cast<int64_t>(r.index);
}

// Colliding scene indices for a pose (sdf.cpp:227-243): returns N_col and
// writes a 0/1 flag per scene point.
int64_t ref_colliding_flags(const asicp_problem* p, int64_t preshape, const double* theta7,
                            int32_t* flags) {
  const GraspProblem g = to_problem(*p);
  Vec7 v;
  for (int a = 0; a < 7; ++a) v[a] = theta7[a];
  const PoseParams th = PoseParams::from_vector(v);
  const auto inv = inverse(th);
  const Mat3 r = rotation_matrix(inv.q);
  const Vec3 offset = g.sdf.offsets[static_cast<size_t>(preshape)];
  int64_t n = 0;
  for (size_t i = 0; i < g.scene_cloud.size(); ++i) {
    const Vec3 local = r * g.scene_cloud[i] + inv.t + offset;
    const bool hit = query(g.sdf, static_cast<size_t>(preshape), local) > g.contact_tolerance;
    flags[i] = hit ? 1 : 0;
    n += hit ? 1 : 0;
  }
  return n;
}

double ref_sdf_query(const asicp_problem* p, int64_t preshape, const double* xyz) {
  const GraspProblem g = to_problem(*p);
  return query(g.sdf, static_cast<size_t>(preshape), Vec3(xyz[0], xyz[1], xyz[2]));
}

// build_sdf (sdf.cpp:48-175) for fixture parity: returns node count; fills
// meta = {origin xyz, voxel, boundary_max_abs} and dims; values must hold
// the node count (call once with values == NULL to size).
int64_t ref_build_sdf(const double* cloud, int64_t n, double voxel, double padding, double band,
                      int32_t* dims, double* meta, float* values) {
  SdfBuildOptions opt;
  opt.padding = padding;
  opt.surface_band = band;
  const SdfGrid g = build_sdf(to_cloud(cloud, n), voxel, opt);
  for (int a = 0; a < 3; ++a) {
    dims[a] = g.dims[a];
    meta[a] = g.origin[a];
  }
  meta[3] = g.voxel;
  meta[4] = g.boundary_max_abs;
  if (values) std::memcpy(values, g.values.data(), g.values.size() * sizeof(float));
  return static_cast<int64_t>(g.values.size());
}

}  // extern "C"
