"""Parity oracle — TEST INFRASTRUCTURE ONLY.

ctypes access to oracle/_ref/libgraspmatch_ref.so: the UNMODIFIED reference
(/root/reference/proj/src/*.cpp, built by oracle/Makefile against the Eigen /
doctest subset shims) plus a bridge taking the product's asicp_problem struct
(oracle/ref_bridge.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs use this module — it is the checker, never the product.

Pinning (tests/test_oracle.py): the reference's own 103 unit tests and 9/9
acceptance criteria pass on this build, and the desk seed-0 solve reproduces
proj/README.md:43-46 to every printed digit.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2412_08346_b200 import _lib as L
from paper_2412_08346_b200.grasp import (CProblem, GraspProblem, GraspSolution, InvalidArgument, SolutionBuffers,
                                         problem_from_c)

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libgraspmatch_ref.so"
_LIB = None


def available() -> bool:
    return LIB_PATH.exists()


def load() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        lib = C.CDLL(str(LIB_PATH))
        lib.ref_optimize_grasp.argtypes = [C.POINTER(L.Problem), C.POINTER(L.Solution), C.c_char_p, C.c_size_t]
        lib.ref_desk_problem.restype = C.c_void_p
        lib.ref_desk_problem.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64]
        lib.ref_self_matching_problem.restype = C.c_void_p
        lib.ref_problem_view.restype = C.POINTER(L.Problem)
        lib.ref_problem_view.argtypes = [C.c_void_p]
        lib.ref_problem_free.argtypes = [C.c_void_p]
        lib.ref_cylinder_cloud.argtypes = [C.c_double, C.c_double, C.c_int, C.c_uint64, L.c_double_p]
        lib.ref_sample_minibatch_indices.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, L.c_i64_p]
        lib.ref_nearest.restype = C.c_int64
        lib.ref_nearest.argtypes = [L.c_double_p, C.c_int64, L.c_double_p, L.c_double_p]
        lib.ref_colliding_flags.restype = C.c_int64
        lib.ref_colliding_flags.argtypes = [C.POINTER(L.Problem), C.c_int64, L.c_double_p, L.c_i32_p]
        lib.ref_sdf_query.restype = C.c_double
        lib.ref_sdf_query.argtypes = [C.POINTER(L.Problem), C.c_int64, L.c_double_p]
        lib.ref_build_sdf.restype = C.c_int64
        lib.ref_build_sdf.argtypes = [L.c_double_p, C.c_int64, C.c_double, C.c_double, C.c_double, L.c_i32_p,
                                      L.c_double_p, L.c_float_p]
        _LIB = lib
    return _LIB


def optimize_grasp(problem) -> GraspSolution:
    """Reference graspmatch::optimize_grasp on a GraspProblem / CProblem / Fixture."""
    lib = load()
    cp = problem if hasattr(problem, "ptr") else CProblem(problem)
    bufs = SolutionBuffers(cp.J, cp.k_max, cp.record_trace)
    err = C.create_string_buffer(512)
    rc = lib.ref_optimize_grasp(cp.ptr(), C.byref(bufs.struct), err, 512)
    if rc == L.ASICP_INVALID_ARGUMENT:
        raise InvalidArgument(err.value.decode())
    if rc != L.ASICP_OK:
        raise RuntimeError(err.value.decode())
    return bufs.solution(cp.k_stein)


class RefFixture:
    def __init__(self, handle):
        self.lib = load()
        self.handle = handle
        self._view = self.lib.ref_problem_view(handle)

    @property
    def struct(self):
        return self._view.contents

    def ptr(self):
        return self._view

    @property
    def J(self):
        v = self.struct
        return int(sum(v.init_counts[i] for i in range(v.n_init_lists)))

    @property
    def k_max(self):
        return int(self.struct.k_max)

    @property
    def k_stein(self):
        return int(self.struct.k_stein)

    @property
    def record_trace(self):
        return bool(self.struct.record_trace)

    def set(self, **fields):
        for k, v in fields.items():
            setattr(self.struct, k, v)
        return self

    def problem(self) -> GraspProblem:
        return problem_from_c(self.struct)

    def __del__(self):
        try:
            if self.handle:
                self.lib.ref_problem_free(self.handle)
        except Exception:
            pass


def desk(seed: int = 0, workers: int = 0, n_init: int = 100, n_top: int = 6) -> RefFixture:
    return RefFixture(load().ref_desk_problem(seed, workers, n_init, n_top))


def self_matching() -> RefFixture:
    return RefFixture(load().ref_self_matching_problem())


def sample_minibatch_indices(seed: int, n: int, m: int, skip: int = 0) -> np.ndarray:
    out = np.zeros(m, dtype=np.int64)
    rc = load().ref_sample_minibatch_indices(seed, skip, n, m, out.ctypes.data_as(L.c_i64_p))
    if rc != 0:
        raise InvalidArgument("sample_minibatch: m out of range")
    return out


def cylinder_cloud(radius=0.03, height=0.12, n=1500, seed=1) -> np.ndarray:
    out = np.zeros((n, 3))
    load().ref_cylinder_cloud(radius, height, n, seed, out.ctypes.data_as(L.c_double_p))
    a_side = 2.0 * np.pi * radius * height
    a_cap = np.pi * radius * radius
    n_side = int(n * a_side / (a_side + 2.0 * a_cap))
    return out[: n_side + 2 * ((n - n_side) // 2)]


def build_sdf(cloud, voxel, padding=-1.0, band=0.003):
    cloud = np.ascontiguousarray(cloud, dtype=np.float64)
    dims = (C.c_int32 * 3)()
    meta = (C.c_double * 5)()
    lib = load()
    n = lib.ref_build_sdf(cloud.ctypes.data_as(L.c_double_p), len(cloud), voxel, padding, band, dims, meta, None)
    vals = np.zeros(n, dtype=np.float32)
    lib.ref_build_sdf(cloud.ctypes.data_as(L.c_double_p), len(cloud), voxel, padding, band, dims, meta,
                      vals.ctypes.data_as(L.c_float_p))
    return tuple(dims), np.array(meta[:3]), meta[3], meta[4], vals


# ---------------------------------------------------------------------------
# Oracle-side build of the synthetic-input generators (csrc/fixtures.cu compiled
# by oracle/Makefile into _build/libasicp_fixtures_oracle.so): the reference arm
# of bench.py builds its inputs with it, so that arm maps oracle libraries only.
# Same source, same C-ABI as the product-side libasicp_fixtures.so.
# ---------------------------------------------------------------------------
FIXTURES_PATH = HERE / "_build" / "libasicp_fixtures_oracle.so"
_FX = None


def fixtures_lib() -> C.CDLL:
    global _FX
    if _FX is None:
        if not FIXTURES_PATH.exists():
            raise RuntimeError(f"{FIXTURES_PATH} missing: run `make -C oracle port`")
        _FX = L.declare_fixtures(C.CDLL(str(FIXTURES_PATH)))
    return _FX


class OracleFixture(RefFixture):
    """A fixture owned by the oracle-side generator library."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("unknown fixture")
        self.lib = fixtures_lib()
        self.handle = handle
        self._view = self.lib.asicp_fx_view(handle)

    def __del__(self):
        try:
            if self.handle:
                self.lib.asicp_fx_free(self.handle)
                self.handle = None
        except Exception:
            pass


def fixture_config(cfg: int, seed: int = 0, particles_per_preshape: int = 0, n_object: int = 0) -> OracleFixture:
    """asicp_fx_config (include/asicp_fixtures.h) from the oracle-side library."""
    return OracleFixture(fixtures_lib().asicp_fx_config(cfg, seed, particles_per_preshape, n_object))


# ---------------------------------------------------------------------------
# The plain-C restatement (oracle/port/asicp_port.c) — available wherever the
# repo is built, even without /root/reference.
# ---------------------------------------------------------------------------
PORT_PATH = HERE / "_build" / "libasicp_port.so"
_PORT = None


def port_available() -> bool:
    return PORT_PATH.exists()


def desk_trace_file(path, seed: int = 0, n_init: int = 100, n_top: int = 6, k_max: int = 40, k_stein: int = 15,
                    anneal_total: int = 40) -> None:
    """The reference trace file (graspmatch::export_trace, io.cpp:691-710) of
    the desk scenario, written by oracle/ref_trace_cli.py in a subprocess (the
    library's static libstdc++ iostreams cannot share a process with numpy's
    libstdc++)."""
    import subprocess
    import sys

    rc = subprocess.run([sys.executable, str(HERE / "ref_trace_cli.py"), str(seed), str(n_init), str(n_top),
                         str(k_max), str(k_stein), str(anneal_total), str(path)]).returncode
    if rc != 0:
        raise RuntimeError(f"reference export_trace failed ({rc})")


def port_optimize_grasp(problem) -> GraspSolution:
    global _PORT
    if _PORT is None:
        _PORT = C.CDLL(str(PORT_PATH))
        _PORT.port_optimize_grasp.argtypes = [C.POINTER(L.Problem), C.POINTER(L.Solution), C.c_char_p, C.c_size_t]
    cp = problem if hasattr(problem, "ptr") else CProblem(problem)
    bufs = SolutionBuffers(cp.J, cp.k_max, cp.record_trace)
    err = C.create_string_buffer(512)
    rc = _PORT.port_optimize_grasp(cp.ptr(), C.byref(bufs.struct), err, 512)
    if rc == L.ASICP_INVALID_ARGUMENT:
        raise InvalidArgument(err.value.decode())
    if rc != L.ASICP_OK:
        raise RuntimeError(err.value.decode())
    return bufs.solution(cp.k_stein)


# ---------------------------------------------------------------------------
# register_sgd_icp (optim.cpp:274-321): the reference and the C restatement.
# ---------------------------------------------------------------------------
def _reg_call(fn, source, reference, initial, cfg, seed):
    from paper_2412_08346_b200.registration import _cloud, _pose, _result, sgd_config_struct

    src, ref, init = _cloud(source), _cloud(reference), _pose(initial)
    c = sgd_config_struct(cfg)
    out = L.Registration()
    err = C.create_string_buffer(512)
    fn.argtypes = [L.c_double_p, C.c_int64, L.c_double_p, C.c_int64, L.c_double_p, C.POINTER(L.SgdCfg), C.c_uint64,
                   C.POINTER(L.Registration), C.c_char_p, C.c_size_t]
    rc = fn(src.ctypes.data_as(L.c_double_p), len(src), ref.ctypes.data_as(L.c_double_p), len(ref),
            init.ctypes.data_as(L.c_double_p), C.byref(c), C.c_uint64(int(seed)), C.byref(out), err, 512)
    if rc == L.ASICP_INVALID_ARGUMENT:
        raise InvalidArgument(err.value.decode())
    if rc != L.ASICP_OK:
        raise RuntimeError(err.value.decode())
    return _result(out)


def register_sgd_icp(source, reference, initial, cfg, seed):
    """Reference graspmatch::register_sgd_icp (oracle/_ref)."""
    return _reg_call(load().ref_register_sgd_icp, source, reference, initial, cfg, seed)


def port_register_sgd_icp(source, reference, initial, cfg, seed):
    """The plain-C restatement (oracle/port/asicp_port.c)."""
    global _PORT
    if _PORT is None:
        _PORT = C.CDLL(str(PORT_PATH))
        _PORT.port_optimize_grasp.argtypes = [C.POINTER(L.Problem), C.POINTER(L.Solution), C.c_char_p, C.c_size_t]
    return _reg_call(_PORT.port_register_sgd_icp, source, reference, initial, cfg, seed)


def c2_trial(trial: int, n: int = 500):
    """Acceptance C2 inputs from the reference's own generators."""
    lib = load()
    lib.ref_c2_trial.argtypes = [C.c_int, C.c_int, L.c_double_p, L.c_double_p, L.c_double_p]
    src, ref, truth = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(7)
    lib.ref_c2_trial(trial, n, src.ctypes.data_as(L.c_double_p), ref.ctypes.data_as(L.c_double_p),
                     truth.ctypes.data_as(L.c_double_p))
    return src, ref, truth


def blob_cloud(n: int, radius: float, seed: int) -> np.ndarray:
    lib = load()
    lib.ref_blob_cloud.argtypes = [C.c_int, C.c_double, C.c_uint64, L.c_double_p]
    out = np.zeros((n, 3))
    lib.ref_blob_cloud(n, radius, seed, out.ctypes.data_as(L.c_double_p))
    return out


def quaternion_angle(q1, q2) -> float:
    lib = load()
    lib.ref_quaternion_angle.restype = C.c_double
    lib.ref_quaternion_angle.argtypes = [L.c_double_p, L.c_double_p]
    a = np.ascontiguousarray(q1, dtype=np.float64)
    b = np.ascontiguousarray(q2, dtype=np.float64)
    return lib.ref_quaternion_angle(a.ctypes.data_as(L.c_double_p), b.ctypes.data_as(L.c_double_p))


def _icp_call(fn, source, reference, theta):
    from paper_2412_08346_b200.registration import ClosedFormStepResult, _cloud, _pose

    src, ref, th = _cloud(source), _cloud(reference), _pose(theta)
    out = L.IcpStep()
    err = C.create_string_buffer(512)
    fn.argtypes = [L.c_double_p, C.c_int64, L.c_double_p, C.c_int64, L.c_double_p, C.POINTER(L.IcpStep), C.c_char_p,
                   C.c_size_t]
    rc = fn(src.ctypes.data_as(L.c_double_p), len(src), ref.ctypes.data_as(L.c_double_p), len(ref),
            th.ctypes.data_as(L.c_double_p), C.byref(out), err, 512)
    if rc == L.ASICP_INVALID_ARGUMENT:
        raise InvalidArgument(err.value.decode())
    if rc != L.ASICP_OK:
        raise RuntimeError(err.value.decode())
    return ClosedFormStepResult(np.array(out.theta[:]), bool(out.degenerate))


def icp_closed_form_step(source, reference, theta):
    """Reference graspmatch::icp_closed_form_step (oracle/_ref)."""
    return _icp_call(load().ref_icp_closed_form_step, source, reference, theta)


def port_icp_closed_form_step(source, reference, theta):
    """The plain-C restatement (oracle/port/asicp_port.c)."""
    global _PORT
    if _PORT is None:
        _PORT = C.CDLL(str(PORT_PATH))
        _PORT.port_optimize_grasp.argtypes = [C.POINTER(L.Problem), C.POINTER(L.Solution), C.c_char_p, C.c_size_t]
    return _icp_call(_PORT.port_icp_closed_form_step, source, reference, theta)
