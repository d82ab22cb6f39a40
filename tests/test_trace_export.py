"""graspmatch::export_trace (io.cpp:691-710) — SURVEY.md §8(f) rank 3.

The native writer (csrc/trace_io.cpp, asicp_export_trace) must produce the
reference's file byte for byte: the schema header and one 13-field line per
(iteration, particle) record, doubles in shortest round-trip form.  On CPU
the records come from the reference solve itself (oracle/_ref); on the GPU
from the B200 solve, whose trajectories are bit-identical.
"""
import numpy as np
import pytest

from oracle import ref
from paper_2412_08346_b200 import GraspSolution, GraspStatus, export_trace, fixtures

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@needs_ref
def test_writer_matches_reference_file_on_reference_trace(tmp_path):
    fx = ref.desk(1, n_init=24, n_top=3).set(k_max=15, k_stein=6, anneal_period_total=15, record_trace=1)
    sol = ref.optimize_grasp(fx)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    export_trace(sol, ours)
    ref.desk_trace_file(theirs, seed=1, n_init=24, n_top=3, k_max=15, k_stein=6, anneal_total=15)
    a, b = ours.read_bytes(), theirs.read_bytes()
    assert a == b
    lines = a.decode().splitlines()
    assert len(lines) == 1 + 15 * fx.J and lines[0].startswith("#")
    assert all(len(line.split()) == 13 for line in lines[1:])
    assert lines[1].split()[3] == "stein" and lines[-1].split()[3] == "sgd"


def test_unit_records_and_empty_trace(tmp_path):
    """test_io.cpp:426-464: 3 iterations x 2 particles, t = (0.1, 0.2, 0.3),
    identity quaternion; and an empty trace gives the header alone."""
    k, J = 3, 2
    th = np.zeros((k, J, 7))
    th[:, :, :3] = [0.1, 0.2, 0.3]
    th[:, :, 3] = 1.0
    loss = np.array([[0.5 * (i + 1)] * J for i in range(k)])
    col = np.array([[i == 0] * J for i in range(k)])
    sol = GraspSolution(GraspStatus.kFound, th[0, 0], 0, 0.0, False, th[-1], loss[-1], ~col[-1], col[-1],
                        np.zeros(J, dtype=np.int64), th, loss, col, k_stein=1)
    p = tmp_path / "trace.txt"
    export_trace(sol, p)
    lines = p.read_text().splitlines()
    assert len(lines) == 7 and lines[0][0] == "#"
    for i, line in enumerate(lines[1:]):
        f = line.split()
        assert len(f) == 13
        assert f[0] == str(i // J) and f[1] == str(i % J) and f[2] == "0"
        assert f[3] == ("stein" if i // J < 1 else "sgd")
        assert f[5] == ("1" if i // J == 0 else "0")
        assert f[6] == "0.1" and f[9] == "1"
    sol.trace_theta = sol.trace_loss = sol.trace_in_collision = None
    export_trace(sol, tmp_path / "empty.txt")
    assert len((tmp_path / "empty.txt").read_text().splitlines()) == 1


@needs_ref
@pytest.mark.gpu
def test_gpu_trace_file_is_the_reference_file(tmp_path):
    from paper_2412_08346_b200 import Solver

    fx = fixtures.desk(0).set(record_trace=1)
    s = Solver()
    sol = s.optimize(fx)
    s.close()
    export_trace(sol, tmp_path / "b200.txt")
    ref.desk_trace_file(tmp_path / "ref.txt", seed=0)
    assert (tmp_path / "b200.txt").read_bytes() == (tmp_path / "ref.txt").read_bytes()
