"""Particle sharding within a population on one GPU.

Every rank prepares the full problem and owns the slice [r J / R, (r+1) J / R)
of the global particle order; per Stein iteration the ranks all-gather the
population's poses and drifts, and the final summaries are gathered so each
rank returns the whole answer.  Here the ranks are contexts of one process
driven by one host thread each, exchanging through host memory (the group
backend: each rank synchronises its own stream before the host barrier, so no
kernel waits on another rank's kernel).  The sharded answer — every particle,
every iteration — must equal the unsharded solve bit for bit.  The NCCL backend
is exercised at world size 1 (one GPU available).
"""
import threading

import numpy as np
import pytest

from paper_2412_08346_b200 import Solver, fixtures
from paper_2412_08346_b200.grasp import Group, nccl_unique_id

pytestmark = pytest.mark.gpu


def sharded_solve(fx, world):
    group = Group(world)
    out, errs = [None] * world, []
    solvers = [Solver() for _ in range(world)]

    def rank_main(r):
        try:
            solvers[r].set_partition_group(group, r)
            out[r] = solvers[r].optimize(fx)
        except Exception as e:  # surfaced below
            errs.append(e)

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    for s in solvers:
        s.close()
    group.close()
    assert not errs, errs
    return out


def assert_identical(a, b):
    assert int(a.status) == int(b.status) and a.preshape_id == b.preshape_id
    assert np.array_equal(a.theta, b.theta) and a.final_loss == b.final_loss
    assert np.array_equal(a.particle_theta, b.particle_theta)
    assert np.array_equal(a.particle_loss, b.particle_loss)
    assert np.array_equal(a.particle_collision_free, b.particle_collision_free)
    assert np.array_equal(a.particle_converged, b.particle_converged)
    assert np.array_equal(a.trace_theta, b.trace_theta)
    assert np.array_equal(a.trace_loss, b.trace_loss, equal_nan=True)
    assert np.array_equal(a.trace_in_collision, b.trace_in_collision)


@pytest.mark.parametrize("world", [2, 4])
def test_group_sharding_matches_unsharded_multi_population(solver, world):
    # 3 populations x 7 particles: the rank slices straddle population borders.
    fx = fixtures.config(2, seed=1, particles_per_preshape=7).set(k_max=14, k_stein=8, anneal_period_total=14,
                                                                   record_trace=1)
    want = solver.optimize(fx)
    for got in sharded_solve(fx, world):
        assert_identical(got, want)


def test_group_sharding_desk_population(solver):
    fx = fixtures.desk(3).set(record_trace=1)
    want = solver.optimize(fx)
    for got in sharded_solve(fx, 3):
        assert_identical(got, want)


def test_group_sharding_cfg5_shape(solver):
    """One population (cfg5 shape) of 256 particles against a 20k-point cylinder."""
    fx = fixtures.config(5, seed=0, particles_per_preshape=256, n_object=20000).set(
        k_max=16, k_stein=10, anneal_period_total=16, record_trace=1)
    want = solver.optimize(fx)
    for got in sharded_solve(fx, 2):
        assert_identical(got, want)


def test_nccl_backend_world1(solver):
    fx = fixtures.config(2, seed=0, particles_per_preshape=5).set(k_max=10, k_stein=6, anneal_period_total=10,
                                                                   record_trace=1)
    want = solver.optimize(fx)
    s = Solver()
    s.set_partition_nccl(0, 1, nccl_unique_id())
    got = s.optimize(fx)
    got2 = s.optimize(fx)  # the communicator is reused across solves
    s.close()
    assert_identical(got, want)
    assert_identical(got2, want)


def test_partition_needs_a_particle_per_rank():
    from paper_2412_08346_b200 import InvalidArgument

    fx = fixtures.desk(0, n_init=2, n_top=0)
    group = Group(3)
    s = Solver()
    s.set_partition_group(group, 0)  # J = 2 over 3 ranks: rank 0's slice [0, 0) is empty
    with pytest.raises(InvalidArgument, match="without particles"):
        s.prepare(fx)
    s.close()
    group.close()


def test_group_sharding_large_population(solver):
    """cfg5 shape above the grid-wide median threshold, sharded over 2 ranks."""
    fx = fixtures.config(5, seed=1, particles_per_preshape=2600, n_object=4000).set(
        k_max=6, k_stein=5, anneal_period_total=6, record_trace=1)
    want = solver.optimize(fx)
    for got in sharded_solve(fx, 2):
        assert_identical(got, want)
