"""register_sgd_icp parity cases shared by the golden generator and the tests.

Inputs come from the product fixtures (paper_2412_08346_b200.fixtures), which
reproduce the reference generators bit for bit (tests/test_registration.py
checks that against oracle/_ref).
"""
import numpy as np

from paper_2412_08346_b200 import PreconditionerMode, SgdConfig, fixtures

IDENTITY = np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0])


def _normalized(q):
    q = np.asarray(q, dtype=np.float64)
    return q / np.sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3])


def _apply(theta, cloud):
    """geometry.cpp:68-74 apply_transform (R p + t, the shim's evaluation order)."""
    w, x, y, z = theta[3:]
    r = np.array([[w * w + x * x - y * y - z * z, 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)],
                  [2.0 * (x * y + w * z), w * w - x * x + y * y - z * z, 2.0 * (y * z - w * x)],
                  [2.0 * (x * z - w * y), 2.0 * (y * z + w * x), w * w - x * x - y * y + z * z]])
    n2 = ((w * w + x * x) + y * y) + z * z
    r = r / n2
    out = np.empty_like(cloud)
    for a in range(3):
        out[:, a] = ((r[a, 0] * cloud[:, 0] + r[a, 1] * cloud[:, 1]) + r[a, 2] * cloud[:, 2]) + theta[a]
    return out


def c2_config() -> SgdConfig:
    """test_acceptance.cpp:277-280."""
    return SgdConfig(preconditioner_mode=PreconditionerMode.kGaussNewtonRotation, minibatch_size=100,
                     max_iterations=500)


def c2_cases():
    """The 20 trials of acceptance C2 (test_acceptance.cpp:256-292)."""
    out = []
    for trial in range(20):
        src, ref, truth = fixtures.c2_trial(trial)
        out.append((f"c2_{trial}", src, ref, IDENTITY, c2_config(), 1000 + trial, truth))
    return out


def unit_cases():
    """test_optim.cpp:540-584 plus fixed-preconditioner / chunking variants."""
    cases = []
    src = fixtures.blob_cloud(150, 0.05, 58)
    truth = np.concatenate([[0.005, -0.003, 0.004], _normalized([1.0, 0.015, -0.01, 0.02])])
    ref = _apply(truth, src)
    cfg = SgdConfig(preconditioner_mode=PreconditionerMode.kGaussNewtonRotation, max_iterations=120,
                    convergence_threshold=-1.0)
    cases.append(("small_offset_gn", src, ref, IDENTITY, cfg, 7, truth))
    src = fixtures.blob_cloud(50, 0.05, 59)
    start = IDENTITY.copy()
    start[0] = 0.002
    cases.append(("full_batch_converges", src, src.copy(), start, SgdConfig(max_iterations=300,
                                                                             convergence_threshold=0.02), 11, None))
    cases.append(("full_batch_never", src, src.copy(), start, SgdConfig(max_iterations=300,
                                                                        convergence_threshold=-1.0), 11, None))
    # Fixed preconditioner with a non-identity SPD A and a smaller step.
    A = np.eye(7)
    A[0, 1] = A[1, 0] = 0.1
    A[3, 4] = A[4, 3] = -0.05
    A[6, 6] = 0.5
    s2, r2, t2 = fixtures.c2_trial(3)
    cases.append(("fixed_spd", s2, r2, IDENTITY, SgdConfig(learning_rate=0.7, A=A, max_iterations=200), 5, t2))
    # Minibatches larger than one 128-pair accumulation chunk.
    cfg = c2_config()
    cfg.minibatch_size = 300
    cfg.max_iterations = 60
    cases.append(("gn_m300", s2, r2, IDENTITY, cfg, 9, t2))
    # Full batch under Gauss-Newton (the early-stop branch with m == |source|).
    cfg = c2_config()
    cfg.minibatch_size = 1000
    cfg.max_iterations = 200
    cfg.convergence_threshold = 1e-3
    cases.append(("gn_full_batch", s2, r2, IDENTITY, cfg, 13, t2))
    return cases


def all_cases():
    return c2_cases() + unit_cases()


def icp_cases():
    """icp_closed_form_step inputs: test_optim.cpp:69-124 and variants that
    reach every branch of the SVD / Kabsch / quaternion tail."""
    cases = []
    blob = fixtures.blob_cloud(100, 0.05, 41)
    cases.append(("aligned", blob, blob.copy(), IDENTITY))
    src = fixtures.blob_cloud(200, 0.05, 42)
    cases.append(("translation", src, src + np.array([0.01, 0.0, 0.0]), IDENTITY))
    cases.append(("single_point", np.array([[0.0, 0.0, 0.0]]), np.array([[0.05, 0.0, 0.0]]), IDENTITY))
    cases.append(("two_points", src[:2], src[:2] + 0.01, IDENTITY))
    rng = np.random.default_rng(43)
    s120, r150 = fixtures.blob_cloud(120, 0.05, 44), fixtures.blob_cloud(150, 0.06, 45)
    for k in range(6):
        q = _normalized(np.concatenate([[1.0], rng.normal(scale=0.3, size=3)]))
        cases.append((f"random_pose_{k}", s120, r150, np.concatenate([rng.normal(scale=0.03, size=3), q])))
    for k in range(3):  # large rotations: the other Shepperd branches
        q = _normalized(rng.normal(size=4))
        s2, r2, _ = fixtures.c2_trial(k)
        cases.append((f"c2_big_rotation_{k}", s2, r2, np.concatenate([[0.0, 0.0, 0.0], q])))
    # Exact 150-degree rotations about x, y, z started at the truth: the
    # Kabsch rotation has a negative trace (the three non-trace branches).
    for ax in range(3):
        half = np.deg2rad(150.0) / 2.0
        q = np.zeros(4)
        q[0] = np.cos(half)
        q[1 + ax] = np.sin(half)
        q = _normalized(q)
        truth = np.concatenate([[0.01, -0.02, 0.005], q])
        cases.append((f"rot150_axis{ax}", s120, _apply(truth, s120), truth))
    g = np.stack(np.meshgrid(np.linspace(-0.05, 0.05, 7), np.linspace(-0.03, 0.03, 5)), -1).reshape(-1, 2)
    plane = np.concatenate([g, np.zeros((len(g), 1))], axis=1)
    cases.append(("planar", plane, plane + np.array([0.001, -0.002, 0.003]), IDENTITY))
    line = np.outer(np.linspace(-0.05, 0.05, 9), [1.0, 0.5, 0.25])
    cases.append(("collinear", line, line + 0.01, IDENTITY))
    return cases
