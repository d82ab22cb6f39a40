"""The drop-in, exercised by the reference's OWN test suites on the GPU.

oracle/_ref/unit_tests_b200 and acceptance_tests_b200 are the reference's
doctest suite (103 cases) and acceptance binary (criteria C1-C9) linked against
paper_2412_08346_b200/csrc/graspmatch_adapter.cpp — i.e. every
graspmatch::optimize_grasp call in them (test_grasp.cpp:348-458, acceptance C7
desk grasp over 10 seeds and C9 worker-count determinism) and every
graspmatch::register_sgd_icp / icp_closed_form_step call (test_optim.cpp:69-124,
540-584, acceptance C2's 20 recovery trials) and every graspmatch::build_sdf
call (test_sdf.cpp, the desk scenario, the scenario front end's field cache)
runs on the B200 through the C-ABI.  Built here by `make -C oracle dropin`; the binaries travel
to the GPU box with the repo.
"""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def _run(name, timeout):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (make -C oracle dropin)")
    return subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout)


def test_reference_unit_suite_on_b200():
    r = _run("unit_tests_b200", 900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "103 passed | 0 failed" in r.stdout


def test_reference_acceptance_on_b200():
    r = _run("acceptance_tests_b200", 1800)
    assert r.returncode == 0, r.stdout
    assert "acceptance: 9/9 criteria passed" in r.stdout


def test_reference_scenario_front_end_on_b200(tmp_path):
    """the reference's scenario front end —
    write_demo_scenario, load_scenario_config, run_scenario (cloud I/O, cached
    collision fields, initial poses, export_trace), report_to_json — driving
    the B200 build_sdf and optimize_grasp through the drop-in.  Report (wall_seconds zeroed)
    and trace file must equal the reference's own run byte for byte."""
    for name in ("scenario_ref", "scenario_b200"):
        if not (REF / name).exists():
            pytest.skip(f"{REF / name} not built (make -C oracle ref dropin)")
    d, trace = tmp_path / "demo", tmp_path / "trace.txt"  # same paths: the report echoes them
    ref = subprocess.run([str(REF / "scenario_ref"), str(d), str(trace)], capture_output=True, text=True, timeout=600)
    ref_trace = trace.read_bytes()
    # The reference's GMSDF001 field cache (io.cpp:555-580, save_sdf at
    # sdf.cpp:256-285): remove it so the B200 run rebuilds every field through
    # the drop-in graspmatch::build_sdf (csrc/sdf_build.cu), then compare bytes.
    cache = d / "cache"
    ref_fields = {f.name: f.read_bytes() for f in sorted(cache.iterdir())}
    assert ref_fields, "the demo scenario wrote no cached field"
    for f in cache.iterdir():
        f.unlink()
    b200 = subprocess.run([str(REF / "scenario_b200"), str(d), str(trace)], capture_output=True, text=True,
                          timeout=600)
    assert ref.returncode == 0 and b200.returncode == 0, ref.stderr + b200.stderr
    assert '"pose"' in b200.stdout
    assert b200.stdout == ref.stdout
    assert trace.read_bytes() == ref_trace
    assert {f.name: f.read_bytes() for f in sorted(cache.iterdir())} == ref_fields


def test_reference_cli_on_b200(tmp_path):
    """SURVEY.md §8(f) rank 2 end to end: the reference's OWN command-line
    front end (proj/tools/graspmatch_cli.cpp, unmodified; CLI11 from
    oracle/shim) built on the reference library (graspmatch_ref) and on the
    B200 drop-in (graspmatch_b200).  `grasp -c scenario.json` (cloud I/O,
    fields built on the GPU into the GMSDF001 cache, solve, report, trace),
    `sdf` (a field file) and the error path must match the reference's own
    run byte for byte (wall-clock seconds masked)."""
    import json
    import re

    exes = {k: REF / f"graspmatch_{k}" for k in ("ref", "b200")}
    for e in exes.values():
        if not e.exists():
            pytest.skip(f"{e} not built (make -C oracle ref dropin)")

    def run(kind, *args):
        return subprocess.run([str(exes[kind]), *args], capture_output=True, text=True, timeout=600, cwd=tmp_path)

    assert run("ref", "make-demo", "-d", "demo").returncode == 0
    cfg = "demo/scenario.json"
    ref = run("ref", "grasp", "-c", cfg, "--trace", "trace.txt", "--report", "report.json")
    assert ref.returncode == 0, ref.stderr
    ref_trace = (tmp_path / "trace.txt").read_bytes()
    ref_report = json.loads((tmp_path / "report.json").read_text())
    cache = tmp_path / "demo" / "cache"
    ref_fields = {f.name: f.read_bytes() for f in sorted(cache.iterdir())}
    for f in cache.iterdir():
        f.unlink()
    b200 = run("b200", "grasp", "-c", cfg, "--trace", "trace.txt", "--report", "report.json")
    assert b200.returncode == 0, b200.stderr
    mask = lambda s: re.sub(r"\d+\.\d\ds\)", "T s)", s)  # noqa: E731  (the wall-clock seconds)
    assert "grasp found (preshape 0, 16/100 collision-free particles" in b200.stdout
    assert mask(b200.stdout) == mask(ref.stdout)
    assert (tmp_path / "trace.txt").read_bytes() == ref_trace
    got_report = json.loads((tmp_path / "report.json").read_text())
    for rep in (ref_report, got_report):
        rep.pop("wall_seconds", None)
    assert got_report == ref_report
    assert {f.name: f.read_bytes() for f in sorted(cache.iterdir())} == ref_fields
    # `sdf`: a field file from the gripper cloud, built on the GPU.
    for kind in ("ref", "b200"):
        r = run(kind, "sdf", "--cloud", "demo/gripper_full.ply", "--voxel", "0.004", "-o", f"field_{kind}.bin")
        assert r.returncode == 0, r.stderr
    assert (tmp_path / "field_b200.bin").read_bytes() == (tmp_path / "field_ref.bin").read_bytes()
    # Error path: same message, same exit code.
    ref_err, b200_err = run("ref", "grasp", "-c", "missing.json"), run("b200", "grasp", "-c", "missing.json")
    assert ref_err.returncode == b200_err.returncode != 0 and ref_err.stderr == b200_err.stderr
