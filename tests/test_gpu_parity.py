"""GPU parity of the B200 optimize_grasp against the reference oracle.

The reference (oracle/_ref, the unmodified /root/reference sources) and the
CUDA path run on identical inputs; the bar is BIT-IDENTITY of every pose, loss
and flag of every particle at every iteration (the CUDA path evaluates the
reference's FP64 arithmetic in the same order, exp() is the glibc algorithm,
and the FP32 nearest-neighbour filter is certified by an FP64 decision,
DESIGN.md §4).  TOL = 0.
"""
import numpy as np
import pytest

from paper_2412_08346_b200 import GraspStatus, InvalidArgument, fixtures

pytestmark = pytest.mark.gpu

TOL = 0.0  # bit-identical, see module docstring


def cpu_oracle(fx):
    """The reference itself (oracle/_ref) wherever it is built, else the C
    restatement pinned to it (oracle/port, tests/test_oracle.py)."""
    from oracle import ref

    if ref.available():
        return ref.optimize_grasp(fx)
    if not ref.port_available():
        pytest.skip("neither oracle/_ref nor the oracle port is built")
    return ref.port_optimize_grasp(fx)


def assert_same_solution(got, want, tol=TOL):
    assert got.status == want.status
    assert got.preshape_id == want.preshape_id
    np.testing.assert_array_equal(got.particle_collision_free, want.particle_collision_free)
    np.testing.assert_array_equal(got.particle_converged, want.particle_converged)
    np.testing.assert_allclose(got.particle_theta, want.particle_theta, rtol=tol, atol=tol)
    np.testing.assert_allclose(got.particle_loss, want.particle_loss, rtol=tol, atol=1e-15)
    np.testing.assert_allclose(got.theta, want.theta, rtol=tol, atol=tol)
    np.testing.assert_allclose(got.final_loss, want.final_loss, rtol=tol)


@pytest.mark.parametrize("seed", [0, 4])
def test_desk_matches_reference(solver, oracle, seed):
    fx = fixtures.desk(seed).set(record_trace=1)
    want = oracle.optimize_grasp(fx)
    got = solver.optimize(fx)
    np.testing.assert_array_equal(got.trace_in_collision, want.trace_in_collision)
    np.testing.assert_allclose(got.trace_theta, want.trace_theta, rtol=TOL, atol=TOL)
    np.testing.assert_allclose(got.trace_loss, want.trace_loss, rtol=TOL, atol=1e-15)
    assert_same_solution(got, want)


def test_desk_seed0_readme(solver):
    """proj/README.md:43-46: preshape 0, 16/100 collision-free, printed pose."""
    sol = solver.optimize(fixtures.desk(0))
    assert sol.status == GraspStatus.kFound
    assert sol.preshape_id == 0
    assert int(sol.particle_collision_free.sum()) == 16
    np.testing.assert_allclose(sol.theta[:3], [0.005176, 0.000263, 0.103996], atol=5e-7)
    np.testing.assert_allclose(sol.theta[3:], [0.995938, -0.005412, 0.089213, -0.010885], atol=5e-7)
    assert f"{sol.final_loss:.11f}" == "0.00022030658"
    assert not sol.converged


def test_rerun_bit_identical(solver):
    a = solver.optimize(fixtures.desk(2))
    b = solver.optimize(fixtures.desk(2))
    np.testing.assert_array_equal(a.particle_theta, b.particle_theta)
    assert a.final_loss == b.final_loss


def test_fp64_mode_matches_certified(oracle):
    from paper_2412_08346_b200 import Solver

    s = Solver(nn_mode=1)
    fx = fixtures.desk(1)
    got = s.optimize(fx)
    want = oracle.optimize_grasp(fx)
    assert_same_solution(got, want)
    s.close()


def test_cfg1_small_matches_reference(solver, oracle):
    fx = fixtures.config(1, seed=3, particles_per_preshape=24)
    fx.set(k_max=20, k_stein=8, anneal_period_total=20, record_trace=1)
    want = oracle.optimize_grasp(fx)
    got = solver.optimize(fx)
    np.testing.assert_array_equal(got.trace_in_collision, want.trace_in_collision)
    np.testing.assert_allclose(got.trace_theta, want.trace_theta, rtol=TOL, atol=TOL)
    assert_same_solution(got, want)


def test_self_matching_identity(solver, oracle):
    """test_grasp.cpp:348-369 on the GPU."""
    fx = oracle.self_matching()
    p = fx.problem()
    p.initializations = [np.array([[0.002, -0.001, 0.001, *(np.array([1.0, 0.008, -0.006, 0.01]) /
                                                           np.linalg.norm([1.0, 0.008, -0.006, 0.01]))]])]
    p.k_stein = 0
    p.k_max = 100
    p.sgd.convergence_threshold = -1.0
    p.sgd.A = np.eye(7)
    p.sgd.A[3:, 3:] = np.eye(4) * 20.0
    p.seed = 5
    sol = solver.optimize(p)
    want = oracle.optimize_grasp(p)
    assert_same_solution(sol, want)
    assert sol.status == GraspStatus.kFound
    assert sol.final_loss <= 1e-4
    assert np.linalg.norm(sol.theta[:3]) <= 1e-3


def test_collision_escape(solver, oracle):
    """test_grasp.cpp:371-396: starts penetrating, escapes via the reverse match."""
    p = fixtures.desk(0).problem()
    p.initializations = [np.array([[0.0, 0.02, 0.145, 1.0, 0.0, 0.0, 0.0]])]
    p.k_stein = 0
    p.k_max = 40
    p.record_trace = True
    sol = solver.optimize(p)
    want = oracle.optimize_grasp(p)
    assert sol.trace_in_collision[0, 0]
    assert not sol.trace_in_collision[-1, 0]
    np.testing.assert_array_equal(sol.trace_in_collision, want.trace_in_collision)
    np.testing.assert_allclose(sol.trace_theta, want.trace_theta, rtol=TOL, atol=TOL)
    assert_same_solution(sol, want)


def test_invalid_arguments_match_reference(solver, oracle):
    base = fixtures.desk(0).problem()
    cases = []
    p = fixtures.desk(0).problem(); p.object_cloud = np.zeros((0, 3)); cases.append(p)
    p = fixtures.desk(0).problem(); p.k_stein, p.k_max = 50, 40; cases.append(p)
    p = fixtures.desk(0).problem(); p.initializations = []; cases.append(p)
    p = fixtures.desk(0).problem(); p.preshapes[0].sdf_index = 3; cases.append(p)
    p = fixtures.desk(0).problem(); p.preshapes[0].tcp = p.preshapes[0].tcp + 1e-3; cases.append(p)
    p = fixtures.desk(0).problem(); p.initializations[0][0, 3] = 2.0; p.workers = 1; cases.append(p)
    for p in cases:
        with pytest.raises(InvalidArgument) as e_got:
            solver.optimize(p)
        with pytest.raises(InvalidArgument) as e_want:
            oracle.optimize_grasp(p)
        assert str(e_got.value) == str(e_want.value)
    del base


def test_preshape_sharding_on_gpu_is_bit_identical(solver):
    """Object/preshape sharding (shard.py) with the B200 solver: three
    simulated ranks solve their (object, preshape) units independently; the
    combined answers equal the unsharded B200 solves bit for bit."""
    from paper_2412_08346_b200 import shard

    problems = []
    for seed in (0, 1):
        problems.append(fixtures.config(2, seed=seed, particles_per_preshape=6).set(
            k_max=10, k_stein=4, anneal_period_total=10).problem())
    world = 3
    parts = [shard.solve_local(problems, solver.optimize, r, world) for r in range(world)]
    got = shard.combine(problems, parts)
    for res, p in zip(got, problems):
        want = solver.optimize(p)
        assert int(res["status"]) == int(want.status)
        assert np.array_equal(res["theta"], want.theta)
        assert res["final_loss"] == want.final_loss
        assert np.array_equal(res["particle_theta"], want.particle_theta)


def test_golden_vectors_without_oracle(solver):
    """The committed golden vectors (reference outputs) on the GPU path."""
    from pathlib import Path

    gold = Path(__file__).resolve().parent / "golden"
    cases = [("smoke_desk32.npz", fixtures.desk(0, n_init=32, n_top=4).set(k_max=12, k_stein=5, anneal_period_total=12)),
             ("desk_seed0.npz", fixtures.desk(0)),
             ("cfg1_small.npz", fixtures.config(1, seed=3, particles_per_preshape=24).set(
                 k_max=20, k_stein=8, anneal_period_total=20))]
    for name, fx in cases:
        g = np.load(gold / name)
        got = solver.optimize(fx.set(record_trace=1))
        assert np.array_equal(got.trace_theta, g["trace_theta"]), name
        assert np.array_equal(got.trace_loss, g["trace_loss"], equal_nan=True), name
        assert np.array_equal(got.particle_theta, g["particle_theta"]), name
        assert np.array_equal(got.particle_loss, g["particle_loss"]), name
        assert got.final_loss == float(g["final_loss"]) and int(got.status) == int(g["status"]), name


def test_device_exp_is_glibc_exact():
    import ctypes as C
    import math

    from paper_2412_08346_b200 import _lib as L

    lib = C.CDLL(str(L.LIB_PATH))
    rng = np.random.default_rng(3)
    x = np.concatenate([-rng.uniform(0, 40, 400_000), -rng.exponential(3.0, 100_000)])
    y = np.zeros_like(x)
    assert lib.asicp_dbg_exp_device(x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), C.c_int64(len(x))) == 0
    want = np.array([math.exp(v) for v in x])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("seed", [0, 1])
def test_cfg2_reduced_matches_port(solver, seed):
    """cfg2 shape (3 KG3 preshapes, 64^3 SDFs, 10k cylinder) with 8 particles per
    preshape and 12 iterations, against the reference (cpu_oracle)."""
    fx = fixtures.config(2, seed=seed, particles_per_preshape=8).set(k_max=12, k_stein=5, anneal_period_total=12,
                                                                     record_trace=1)
    want = cpu_oracle(fx)
    got = solver.optimize(fx)
    assert np.array_equal(got.trace_theta, want.trace_theta)
    assert_same_solution(got, want)


@pytest.mark.parametrize("cfg,seed,ppp,k_max", [(3, 0, 8, 12), (3, 2, 6, 24), (4, 3, 8, 12), (4, 6, 16, 40),
                                                 (4, 8, 8, 12)])
def test_partial_view_and_batch_objects_match_port(solver, cfg, seed, ppp, k_max):
    """cfg3 (noisy occluded scan) and cfg4 batch objects (box / sphere / blob)
    at reduced particle counts, full trace against the reference (cpu_oracle)."""
    fx = fixtures.config(cfg, seed=seed, particles_per_preshape=ppp)
    fx.set(k_max=k_max, k_stein=min(15, k_max // 2), anneal_period_total=k_max, record_trace=1)
    want = cpu_oracle(fx)
    got = solver.optimize(fx)
    np.testing.assert_array_equal(got.trace_in_collision, want.trace_in_collision)
    assert np.array_equal(got.trace_theta, want.trace_theta)
    assert_same_solution(got, want)


def test_large_population_grid_median_matches_port(solver):
    """A population above kMedBigK (2048) takes the grid-wide median select;
    2100 particles leave ragged 128-row tiles.  Full trace against the reference."""
    fx = fixtures.config(5, seed=2, particles_per_preshape=2100, n_object=500)  # grid-wide median
    fx.set(k_max=5, k_stein=3, anneal_period_total=5, record_trace=1)  # T >= C = 5 cycles
    want = cpu_oracle(fx)
    got = solver.optimize(fx)
    assert np.array_equal(got.trace_theta, want.trace_theta)
    assert_same_solution(got, want)


@pytest.mark.parametrize("ppp", [250, 700])
def test_mid_population_median_and_split_svgd_match_port(solver, ppp):
    """K = 250 takes the sampled-bracket median (M > 8192) and the split SVGD;
    K = 700 the grid-wide median.  Full trace against the reference."""
    fx = fixtures.config(5, seed=4, particles_per_preshape=ppp, n_object=600)
    fx.set(k_max=6, k_stein=5, anneal_period_total=6, record_trace=1)
    want = cpu_oracle(fx)
    got = solver.optimize(fx)
    assert np.array_equal(got.trace_theta, want.trace_theta)
    assert_same_solution(got, want)


@pytest.mark.parametrize("pool", [1, 64])
def test_exhausted_window_pool_stays_exact(pool, oracle):
    """With the ambiguous-window pool nearly empty, ambiguous queries go
    listless and are settled by the full FP64 rescan — including windows that
    carry over sub-chunks of a 10k-point cloud.  Still bit-identical."""
    from oracle import ref
    from paper_2412_08346_b200 import Solver

    s = Solver(window_pool=pool)
    fx = fixtures.desk(5).set(record_trace=1)
    got = s.optimize(fx)
    want = oracle.optimize_grasp(fx)
    assert np.array_equal(got.trace_theta, want.trace_theta)
    assert_same_solution(got, want)
    if pool == 1:
        assert got.diagnostics["nn_full_refines"] > 0  # the fallback really ran
    if ref.port_available():
        fx2 = fixtures.config(2, seed=3, particles_per_preshape=6).set(k_max=10, k_stein=5, anneal_period_total=10,
                                                                       record_trace=1)
        got2 = s.optimize(fx2)
        want2 = ref.port_optimize_grasp(fx2)
        assert np.array_equal(got2.trace_theta, want2.trace_theta)
        assert_same_solution(got2, want2)
    s.close()
