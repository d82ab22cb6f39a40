"""register_sgd_icp on the GPU (csrc/register.cu) against the reference,
bit for bit: acceptance C2 batched in one launch, the unit-test cases, the
shared-memory / global-memory layouts, mixed batches and the error paths."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))
import reg_cases  # noqa: E402
from test_registration import error_cases  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2412_08346_b200 import (InvalidArgument, PreconditionerMode, RegistrationBatch, SgdConfig,  # noqa: E402
                                   fixtures, register_sgd_icp, register_sgd_icp_batch)

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden" / "registration.npz"


@pytest.fixture(scope="module")
def golden():
    g = np.load(GOLDEN)
    return {str(n): (g["theta"][i], int(g["iterations"][i]), float(g["final_loss"][i]), bool(g["converged"][i]))
            for i, n in enumerate(g["names"])}


def check(r, want):
    theta, iters, loss, conv = want
    assert np.array_equal(r.theta, theta), (r.theta, theta)
    assert r.iterations == iters and r.final_loss == loss and r.converged == conv


def same(a, b):
    check(a, (b.theta, b.iterations, b.final_loss, b.converged))


def test_c2_batch_matches_reference(solver, golden):
    cases = reg_cases.c2_cases()
    res = register_sgd_icp_batch([c[1] for c in cases], [c[2] for c in cases], [c[3] for c in cases],
                                 reg_cases.c2_config(), [c[5] for c in cases], solver=solver)
    for c, r in zip(cases, res):
        check(r, golden[c[0]])


@pytest.mark.parametrize("case", reg_cases.unit_cases(), ids=lambda c: c[0])
def test_single_matches_reference(solver, golden, case):
    name, src, rf, init, cfg, seed, _ = case
    check(register_sgd_icp(src, rf, init, cfg, seed, solver=solver), golden[name])


def test_repeated_runs_identical(solver, golden):
    cases = reg_cases.c2_cases()[:6]
    b = RegistrationBatch(solver, [c[1] for c in cases], [c[2] for c in cases], [c[3] for c in cases],
                          [c[5] for c in cases], reg_cases.c2_config())
    for _ in range(3):
        for c, r in zip(cases, b.run()):
            check(r, golden[c[0]])


def _port():
    if not ref.port_available():
        pytest.skip("oracle port not built")
    return ref.port_register_sgd_icp


def test_global_memory_layouts(solver):
    """Reference clouds beyond the shared-memory stage (> 3072 points) and
    sources beyond the shared Fisher-Yates array (> 16384 indices)."""
    port = _port()
    big_src = fixtures.blob_cloud(20000, 0.08, 4)
    big_ref = fixtures.blob_cloud(5000, 0.08, 5)
    small_src, small_ref, _ = fixtures.c2_trial(1)
    cfg = reg_cases.c2_config()
    cfg.max_iterations = 25
    srcs = [big_src, small_src, small_src[:90]]
    refs = [big_ref, small_ref, big_ref]
    inits = [reg_cases.IDENTITY] * 3
    seeds = [1, 2, 3]
    res = register_sgd_icp_batch(srcs, refs, inits, cfg, seeds, solver=solver)
    for s, r, i, sd, got in zip(srcs, refs, inits, seeds, res):
        same(got, port(s, r, i, cfg, sd))


def test_mixed_batch_fixed_preconditioner(solver):
    """Different cloud sizes, minibatch >= |source| for some problems (full
    batch, early stop), non-identity starts."""
    port = _port()
    rng = np.random.default_rng(0)
    srcs, refs, inits, seeds = [], [], [], []
    for i in range(12):
        n = int(rng.integers(20, 400))
        s = fixtures.blob_cloud(n, 0.05, 100 + i)
        shift = rng.normal(scale=0.004, size=3)
        srcs.append(s)
        refs.append(s + shift)
        q = np.array([1.0, *rng.normal(scale=0.02, size=3)])
        q = q / np.sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3])
        inits.append(np.concatenate([[0.0, 0.0, 0.0], q]))
        seeds.append(int(rng.integers(0, 2**63)))
    cfg = SgdConfig(learning_rate=0.9, max_iterations=150, convergence_threshold=0.01, minibatch_size=128)
    res = register_sgd_icp_batch(srcs, refs, inits, cfg, seeds, solver=solver)
    for s, r, i, sd, got in zip(srcs, refs, inits, seeds, res):
        same(got, port(s, r, i, cfg, sd))
    gn = SgdConfig(preconditioner_mode=PreconditionerMode.kGaussNewtonRotation, max_iterations=80,
                   minibatch_size=200, convergence_threshold=0.005)
    res = register_sgd_icp_batch(srcs, refs, inits, gn, seeds, solver=solver)
    for s, r, i, sd, got in zip(srcs, refs, inits, seeds, res):
        same(got, port(s, r, i, gn, sd))


@pytest.mark.parametrize("case", error_cases(), ids=lambda c: c[0])
def test_errors_match_reference(solver, case):
    _, src, rf, init, cfg = case
    port = _port()
    try:
        want = port(src, rf, init, cfg, 0)
        want_err = None
    except InvalidArgument as e:
        want_err = str(e)
    try:
        got = register_sgd_icp(src, rf, init, cfg, 0, solver=solver)
        got_err = None
    except InvalidArgument as e:
        got_err = str(e)
    assert got_err == want_err
    if want_err is None:
        same(got, want)


def test_empty_batch(solver):
    assert register_sgd_icp_batch([], [], np.zeros((0, 7)), SgdConfig(), [], solver=solver) == []


# ---------------------------------------------------------------------------
# icp_closed_form_step (optim.cpp:51-90)
# ---------------------------------------------------------------------------
from paper_2412_08346_b200 import icp_closed_form_step, icp_closed_form_step_batch  # noqa: E402

ICP_GOLDEN = Path(__file__).resolve().parent / "golden" / "icp_step.npz"


@pytest.fixture(scope="module")
def icp_golden():
    g = np.load(ICP_GOLDEN)
    return {str(n): (g["theta"][i], bool(g["degenerate"][i])) for i, n in enumerate(g["names"])}


def test_icp_step_batch_matches_reference(solver, icp_golden):
    cases = reg_cases.icp_cases()
    res = icp_closed_form_step_batch([c[1] for c in cases], [c[2] for c in cases], [c[3] for c in cases],
                                     solver=solver)
    for c, r in zip(cases, res):
        assert np.array_equal(r.theta, icp_golden[c[0]][0]), c[0]
        assert r.degenerate == icp_golden[c[0]][1], c[0]


def test_icp_step_chain_matches_port(solver):
    """Ten chained steps (test_optim.cpp:79-95) and a large-cloud case
    (reference beyond any shared-memory stage)."""
    src = fixtures.blob_cloud(200, 0.05, 42)
    rf = src + np.array([0.01, 0.0, 0.0])
    a = b = reg_cases.IDENTITY
    for _ in range(10):
        a = icp_closed_form_step(src, rf, a, solver=solver).theta
        b = ref.port_icp_closed_form_step(src, rf, b).theta if ref.port_available() else a
        assert np.array_equal(a, b)
    big_s, big_r = fixtures.blob_cloud(6000, 0.08, 7), fixtures.blob_cloud(9000, 0.08, 8)
    got = icp_closed_form_step(big_s, big_r, reg_cases.IDENTITY, solver=solver)
    if ref.port_available():
        want = ref.port_icp_closed_form_step(big_s, big_r, reg_cases.IDENTITY)
        assert np.array_equal(got.theta, want.theta) and got.degenerate == want.degenerate


def test_icp_step_errors(solver):
    src = np.zeros((5, 3))
    bad = reg_cases.IDENTITY.copy()
    bad[3] = 1.2
    with pytest.raises(InvalidArgument, match="icp_closed_form_step: empty cloud"):
        icp_closed_form_step(np.zeros((0, 3)), src, reg_cases.IDENTITY, solver=solver)
    with pytest.raises(InvalidArgument, match="quaternion is not unit-norm"):
        icp_closed_form_step(src, src + 1.0, bad, solver=solver)


def test_large_minibatch_global_buffers(solver):
    """Minibatches beyond the shared-memory batch buffers (m > 2048) and the
    gathered-point stage (m > 256): the double buffer and the draws live in
    global memory."""
    port = _port()
    src = fixtures.blob_cloud(5000, 0.06, 21)
    rf = fixtures.blob_cloud(3000, 0.06, 22)
    cfg = SgdConfig(preconditioner_mode=PreconditionerMode.kGaussNewtonRotation, minibatch_size=3000,
                    max_iterations=6)
    got = register_sgd_icp(src, rf, reg_cases.IDENTITY, cfg, 77, solver=solver)
    same(got, port(src, rf, reg_cases.IDENTITY, cfg, 77))
