// Oracle check tool — TEST INFRASTRUCTURE ONLY.
// Runs the reference desk scenario (synthetic.cpp:179-206) through the
// reference optimize_grasp and prints the README summary line
// (proj/README.md:43-46) so the shim build can be pinned against it.
#include "graspmatch/grasp.hpp"
#include "graspmatch/synthetic.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

using namespace graspmatch;

int main(int argc, char** argv) {
  const unsigned long long seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 0;
  const int workers = argc > 2 ? std::atoi(argv[2]) : 0;
  GraspProblem problem = synthetic::desk_grasp_problem(seed, workers);
  const auto t0 = std::chrono::steady_clock::now();
  const GraspSolution sol = optimize_grasp(problem);
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  int free_count = 0;
  for (const auto& p : sol.particles) free_count += p.collision_free ? 1 : 0;
  std::printf("%s (preshape %zu, %d/%zu collision-free particles, %.2fs)\n",
              sol.status == GraspStatus::kFound ? "grasp found" : "no grasp found", sol.preshape_id,
              free_count, sol.particles.size(), secs);
  std::printf("  t = [%9.6f %9.6f %9.6f]\n", sol.theta.t[0], sol.theta.t[1], sol.theta.t[2]);
  std::printf("  q = [%9.6f %9.6f %9.6f %9.6f]\n", sol.theta.q[0], sol.theta.q[1], sol.theta.q[2],
              sol.theta.q[3]);
  std::printf("  loss = %.11f, converged = %s\n", sol.final_loss, sol.converged ? "yes" : "no");
  return 0;
}
