"""The oracle is pinned before it is trusted (CPU).

1. The reference compiled verbatim against the Eigen/doctest shims passes the
   reference's own unit suite (103 doctest cases) and all 9 acceptance criteria.
2. Its desk seed-0 solve prints exactly proj/README.md:43-46.
3. The plain-C restatement (oracle/port) is bit-identical to it, and both
   reproduce the committed golden vectors.
"""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import ref
from paper_2412_08346_b200 import fixtures

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
REF = ROOT / "oracle" / "_ref"

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
needs_port = pytest.mark.skipif(not ref.port_available(), reason="oracle port not built (make -C oracle port)")


@needs_ref
def test_reference_unit_suite_passes():
    r = subprocess.run([str(REF / "unit_tests")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "103 passed | 0 failed" in r.stdout


@needs_ref
def test_reference_acceptance_criteria_pass():
    r = subprocess.run([str(REF / "acceptance_tests")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout
    assert "acceptance: 9/9 criteria passed" in r.stdout


@needs_ref
def test_readme_desk_seed0():
    """proj/README.md:43-46."""
    sol = ref.optimize_grasp(ref.desk(0))
    assert int(sol.status) == 0 and sol.preshape_id == 0
    assert int(sol.particle_collision_free.sum()) == 16 and len(sol.particle_loss) == 100
    assert "[%9.6f %9.6f %9.6f]" % tuple(sol.theta[:3]) == "[ 0.005176  0.000263  0.103996]"
    assert "[%9.6f %9.6f %9.6f %9.6f]" % tuple(sol.theta[3:]) == "[ 0.995938 -0.005412  0.089213 -0.010885]"
    assert "%.11f" % sol.final_loss == "0.00022030658"
    assert not sol.converged


def _check_golden(sol, name):
    g = np.load(GOLD / name)
    assert int(sol.status) == int(g["status"])
    assert sol.preshape_id == int(g["preshape_id"])
    assert np.array_equal(sol.theta, g["theta"])
    assert sol.final_loss == float(g["final_loss"])
    assert np.array_equal(sol.particle_theta, g["particle_theta"])
    assert np.array_equal(sol.particle_loss, g["particle_loss"])
    assert np.array_equal(sol.particle_collision_free, g["particle_collision_free"])
    assert np.array_equal(sol.particle_converged, g["particle_converged"])
    assert np.array_equal(sol.trace_theta, g["trace_theta"])
    assert np.array_equal(sol.trace_loss, g["trace_loss"], equal_nan=True)
    assert np.array_equal(sol.trace_in_collision, g["trace_in_collision"])


def _smoke_fx():
    return fixtures.desk(0, n_init=32, n_top=4).set(k_max=12, k_stein=5, anneal_period_total=12, record_trace=1)


@needs_ref
def test_reference_matches_golden():
    _check_golden(ref.optimize_grasp(_smoke_fx()), "smoke_desk32.npz")
    _check_golden(ref.optimize_grasp(fixtures.desk(0).set(record_trace=1)), "desk_seed0.npz")


@needs_port
def test_port_matches_golden():
    _check_golden(ref.port_optimize_grasp(_smoke_fx()), "smoke_desk32.npz")
    fx = fixtures.config(1, seed=3, particles_per_preshape=24).set(k_max=20, k_stein=8, anneal_period_total=20,
                                                                   record_trace=1)
    _check_golden(ref.port_optimize_grasp(fx), "cfg1_small.npz")


@needs_port
@needs_ref
@pytest.mark.parametrize("seed", [1, 5])
def test_port_bit_identical_to_reference(seed):
    fx = fixtures.desk(seed, n_init=24, n_top=4).set(record_trace=1)
    a = ref.port_optimize_grasp(fx)
    b = ref.optimize_grasp(fx)
    assert np.array_equal(a.trace_theta, b.trace_theta)
    assert np.array_equal(a.particle_loss, b.particle_loss)
    assert a.final_loss == b.final_loss and a.status == b.status


@needs_ref
def test_minibatch_golden():
    g = np.load(GOLD / "minibatch.npz")
    for i, (s, n, m, skip) in enumerate(g["cases"]):
        assert np.array_equal(ref.sample_minibatch_indices(int(s), int(n), int(m), int(skip)), g[f"idx_{i}"])


def test_reference_cli_builds_on_the_cli11_shim(tmp_path):
    """oracle/shim/CLI11.hpp carries the reference's command-line front end
    (proj/tools/graspmatch_cli.cpp, unmodified): make-demo + grasp -c print
    README.md:43-46, options are validated like CLI11 (exit codes)."""
    import subprocess

    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "graspmatch_ref"
    if not exe.exists():
        pytest.skip("oracle/_ref/graspmatch_ref not built (make -C oracle ref)")
    run = lambda *a: subprocess.run([str(exe), *a], capture_output=True, text=True, timeout=300,  # noqa: E731
                                    cwd=tmp_path)
    assert run("make-demo", "-d", "demo").returncode == 0
    r = run("grasp", "-c", "demo/scenario.json")
    assert r.returncode == 0, r.stderr
    assert "grasp found (preshape 0, 16/100 collision-free particles" in r.stdout
    assert "t = [ 0.005176  0.000263  0.103996]" in r.stdout
    assert "q = [ 0.995938 -0.005412  0.089213 -0.010885]" in r.stdout
    assert "loss = 0.00022030658, converged = no" in r.stdout
    assert run("bogus").returncode != 0
    bad = run("sdf", "--cloud", "demo/gripper_full.ply", "--voxel", "-1", "-o", "f.bin")
    assert bad.returncode != 0 and "positive" in bad.stderr
    assert run("grasp").returncode != 0  # -c is required
