"""Generate the committed golden vectors from the reference oracle.

Run where /root/reference exists (oracle/_ref built by `make -C oracle`):
    python tests/golden/make_golden.py
Every file is produced by the UNMODIFIED reference graspmatch::optimize_grasp
(grasp.cpp:132-307) / sample_minibatch_indices (spatial_index.cpp:111-123) /
register_sgd_icp (optim.cpp:274-321)
on the bit-identical fixtures of include/asicp_fixtures.h.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_2412_08346_b200 import fixtures  # noqa: E402

OUT = Path(__file__).resolve().parent


def save_solution(name, fx, sol, **extra):
    np.savez_compressed(
        OUT / name,
        status=np.int32(sol.status), theta=sol.theta, preshape_id=np.int64(sol.preshape_id),
        final_loss=np.float64(sol.final_loss), converged=np.int32(sol.converged),
        particle_theta=sol.particle_theta, particle_loss=sol.particle_loss,
        particle_collision_free=sol.particle_collision_free, particle_converged=sol.particle_converged,
        trace_theta=sol.trace_theta, trace_loss=sol.trace_loss, trace_in_collision=sol.trace_in_collision,
        **extra)
    print("wrote", name)


def main():
    assert ref.available(), "build oracle/_ref first (make -C oracle)"
    # smoke(): desk scenario, 32 particles x 12 iterations (5 Stein).
    fx = fixtures.desk(0, n_init=32, n_top=4).set(k_max=12, k_stein=5, anneal_period_total=12, record_trace=1)
    save_solution("smoke_desk32.npz", fx, ref.optimize_grasp(fx))
    # The reference desk run (README.md:43-46), full trace.
    fx = fixtures.desk(0).set(record_trace=1)
    save_solution("desk_seed0.npz", fx, ref.optimize_grasp(fx))
    # cfg1 (KG3 gripper, 2k cylinder), reduced: 24 particles x 20 iterations.
    fx = fixtures.config(1, seed=3, particles_per_preshape=24).set(k_max=20, k_stein=8, anneal_period_total=20,
                                                                   record_trace=1)
    save_solution("cfg1_small.npz", fx, ref.optimize_grasp(fx))
    # Minibatch draws (seed, n, m, skip).
    cases = [(0, 1500, 1, 0), (7, 1500, 844, 0), (13, 900, 439, 5), (42, 20000, 5000, 311), (3, 64, 64, 0)]
    arrays = {}
    for i, (s, n, m, skip) in enumerate(cases):
        arrays[f"idx_{i}"] = ref.sample_minibatch_indices(s, n, m, skip)
    np.savez_compressed(OUT / "minibatch.npz", cases=np.array(cases, dtype=np.int64), **arrays)
    print("wrote minibatch.npz")
    # register_sgd_icp (optim.cpp:274-321): acceptance C2's 20 trials and the
    # unit-test / variant cases of tests/reg_cases.py.
    sys.path.insert(0, str(ROOT / "tests"))
    import reg_cases

    names, theta, iters, loss, conv = [], [], [], [], []
    for name, src, rf, init, cfg, seed, _ in reg_cases.all_cases():
        r = ref.register_sgd_icp(src, rf, init, cfg, seed)
        names.append(name)
        theta.append(r.theta)
        iters.append(r.iterations)
        loss.append(r.final_loss)
        conv.append(int(r.converged))
    np.savez_compressed(OUT / "registration.npz", names=np.array(names), theta=np.array(theta),
                        iterations=np.array(iters, dtype=np.int64), final_loss=np.array(loss),
                        converged=np.array(conv, dtype=np.int32))
    print("wrote registration.npz")
    # icp_closed_form_step (optim.cpp:51-90).
    names, theta, degen = [], [], []
    for name, src, rf, th in reg_cases.icp_cases():
        r = ref.icp_closed_form_step(src, rf, th)
        names.append(name)
        theta.append(r.theta)
        degen.append(int(r.degenerate))
    np.savez_compressed(OUT / "icp_step.npz", names=np.array(names), theta=np.array(theta),
                        degenerate=np.array(degen, dtype=np.int32))
    print("wrote icp_step.npz")


if __name__ == "__main__":
    main()
