"""The tensor-core forward/final NN filter (ASICP_NN_TC=1, nn.cu nn_tc_kernel:
tcgen05 kind::tf32 MMAs with a three-term TF32 split, FP32 accumulators in
TMEM, certified by nn_tc_window_kernel) against the reference itself.

The path is opt-in (it is parity-exact but not yet faster
than the FFMA2 filter), so these tests create their solvers with the switch
set; the bar is the same BIT-IDENTITY as everywhere else (TOL = 0)."""
import numpy as np
import pytest

from paper_2412_08346_b200 import Solver, fixtures

pytestmark = pytest.mark.gpu


@pytest.fixture
def tc_solver(monkeypatch):
    monkeypatch.setenv("ASICP_NN_TC", "1")  # read when the context is created
    s = Solver()
    yield s
    s.close()


def _ref():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return ref


def _same(got, want):
    assert int(got.status) == int(want.status) and got.preshape_id == want.preshape_id
    assert np.array_equal(got.theta, want.theta) and got.final_loss == want.final_loss
    assert np.array_equal(got.particle_theta, want.particle_theta)
    assert np.array_equal(got.particle_loss, want.particle_loss)
    assert np.array_equal(got.particle_collision_free, want.particle_collision_free)
    assert np.array_equal(got.particle_converged, want.particle_converged)


@pytest.mark.parametrize("cfg,seed,ppp,k_max", [(2, 0, 16, 30), (3, 1, 8, 16), (4, 6, 16, 40)])
def test_tensor_core_filter_trace_matches_reference(tc_solver, cfg, seed, ppp, k_max):
    """Reduced populations, every iteration's poses: pooled minibatches of
    every size (m = 1 .. n), splits, and the unpooled final ranking."""
    ref = _ref()
    fx = fixtures.config(cfg, seed=seed, particles_per_preshape=ppp)
    fx.set(k_max=k_max, k_stein=min(15, k_max // 2), anneal_period_total=k_max, record_trace=1)
    want = ref.optimize_grasp(fx)
    got = tc_solver.optimize(fx)
    assert np.array_equal(got.trace_in_collision, want.trace_in_collision)
    assert np.array_equal(got.trace_theta, want.trace_theta)
    _same(got, want)


def test_tensor_core_filter_full_cfg2(tc_solver):
    """The full cfg2 solve (3 x 256 particles, 100 iterations)."""
    ref = _ref()
    fx = fixtures.config(2, seed=0)
    want = ref.optimize_grasp(fx)
    got = tc_solver.optimize(fx)
    _same(got, want)
    st = tc_solver.raw_stats()
    assert st[2] > 0 and st[12] > 0  # the filter ran (queries, forward pairs)


def test_tensor_core_filter_through_the_context_option():
    """The same path selected per context (ASICP_OPT_NN_TC, Solver(nn_tc=True))
    next to a default context: both bit-identical to the reference."""
    ref = _ref()
    fx = fixtures.config(4, seed=3, particles_per_preshape=8).set(k_max=12, k_stein=6, anneal_period_total=12)
    want = ref.optimize_grasp(fx)
    for tc in (True, False):
        s = Solver(nn_tc=tc)
        try:
            _same(s.optimize(fx), want)
        finally:
            s.close()
