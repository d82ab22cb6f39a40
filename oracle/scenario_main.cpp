// Scenario front end end to end — TEST INFRASTRUCTURE ONLY.
//
//   scenario_{ref,b200} DIR [TRACE]
//
// Writes the reference's bundled demo scenario into DIR
// (graspmatch::write_demo_scenario, io.cpp:712), loads it
// (load_scenario_config), runs graspmatch::run_scenario (io.cpp:608-666: cloud
// I/O, cached collision fields, initial poses, optimize_grasp, trace export)
// and prints report_to_json with wall_seconds zeroed.  Built twice by
// oracle/Makefile: scenario_ref with the reference optimize_grasp, and
// scenario_b200 with the B200 drop-in adapter (the
// reference's own front end running on the GPU path).
#include "graspmatch/io.hpp"

#include <cstdio>
#include <iostream>

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s DIR [TRACE]\n", argv[0]);
    return 2;
  }
  try {
    const auto config_path = graspmatch::write_demo_scenario(argv[1]);
    graspmatch::ScenarioConfig config = graspmatch::load_scenario_config(config_path);
    if (argc > 2) config.trace_path = argv[2];
    graspmatch::GraspReport report = graspmatch::run_scenario(config);
    report.wall_seconds = 0.0;
    std::cout << graspmatch::report_to_json(report) << '\n';
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
