/*
 * asicp_fixtures.h — deterministic synthetic problems for tests and bench.py.
 *
 * Not part of the optimize_grasp drop-in: these are the input generators the
 * reference keeps in proj/src/synthetic.cpp (desk scenario, synthetic.cpp:179-206)
 * plus the bench workloads SURVEY.md §8(d) defines (KG3 three-finger gripper,
 * cylinder / partial-view objects).  Re-implemented here (host C++, same
 * std::mt19937_64 streams and arithmetic) so bench inputs never come from the
 * oracle; tests check them bit-for-bit against the reference fixtures.
 *
 * Each constructor returns an owning handle; asicp_fx_view() exposes it as the
 * asicp_problem the solver consumes (valid until asicp_fx_free()).
 */
#ifndef ASICP_FIXTURES_H_
#define ASICP_FIXTURES_H_

#include "asicp.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct asicp_fixture asicp_fixture;

/* graspmatch::synthetic::desk_grasp_problem(seed, workers, n_init, n_top). */
asicp_fixture* asicp_fx_desk(uint64_t seed, int64_t n_init, int64_t n_top);

/* Bench workloads.  cfg: 1 = KG3 x1 vs 2k cylinder, 64
 * particles, 50 iters; 2 = 3 KG3 preshapes x 256 vs 10k cylinder, 64^3 SDF,
 * 100 iters (38 Stein); 3 = noisy 40 %-occluded 20k partial view, 3 x 1024,
 * 40 iters.  `particles_per_preshape` <= 0 keeps the config's count;
 * `n_object` <= 0 keeps its object size. */
asicp_fixture* asicp_fx_config(int cfg, uint64_t seed, int64_t particles_per_preshape, int64_t n_object);

asicp_problem* asicp_fx_view(asicp_fixture* fx);
void asicp_fx_free(asicp_fixture* fx);

/* Building blocks (for fixture parity tests). */
void asicp_fx_cylinder_cloud(double radius, double height, int n, uint64_t seed, double* out);
/* Acceptance C2 (test_acceptance.cpp:256-282) trial inputs: n-point source /
 * reference clouds (n x 3 each) and the truth pose (7). */
void asicp_fx_c2_trial(int trial, int n, double* source, double* reference, double* truth7);
void asicp_fx_blob_cloud(int n, double radius, uint64_t seed, double* out);
/* Returns the node count; dims/meta (origin xyz, voxel, boundary_max_abs)
 * filled; values written when non-NULL. */
int64_t asicp_fx_build_sdf(const double* cloud, int64_t n, double voxel, double padding, double band,
                           int32_t* dims, double* meta, float* values);

#ifdef __cplusplus
}
#endif

#endif /* ASICP_FIXTURES_H_ */
