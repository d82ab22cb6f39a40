"""Synthetic workloads (include/asicp_fixtures.h) as owned asicp_problem views.

desk(seed)      — graspmatch::synthetic::desk_grasp_problem (synthetic.cpp:179-206)
config(n, ...)  — SURVEY.md §8(d) bench workloads cfg1 / cfg2 (KG3 gripper)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .grasp import GraspProblem, problem_from_c


class Fixture:
    """Owning handle; behaves like grasp.CProblem for Solver.prepare()."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("unknown fixture")
        self.lib = L.load_fixtures()
        self.handle = handle
        self._view = self.lib.asicp_fx_view(handle)

    @property
    def struct(self) -> L.Problem:
        return self._view.contents

    def ptr(self):
        return self._view

    @property
    def J(self) -> int:
        v = self.struct
        return int(sum(v.init_counts[i] for i in range(v.n_init_lists)))

    @property
    def k_max(self) -> int:
        return int(self.struct.k_max)

    @property
    def k_stein(self) -> int:
        return int(self.struct.k_stein)

    @property
    def record_trace(self) -> bool:
        return bool(self.struct.record_trace)

    def set(self, **fields) -> "Fixture":
        for k, v in fields.items():
            setattr(self.struct, k, v)
        return self

    def problem(self) -> GraspProblem:
        return problem_from_c(self.struct)

    def close(self):
        if self.handle:
            self.lib.asicp_fx_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def desk(seed: int = 0, n_init: int = 100, n_top: int = 6) -> Fixture:
    return Fixture(L.load_fixtures().asicp_fx_desk(seed, n_init, n_top))


def config(cfg: int, seed: int = 0, particles_per_preshape: int = 0, n_object: int = 0) -> Fixture:
    return Fixture(L.load_fixtures().asicp_fx_config(cfg, seed, particles_per_preshape, n_object))


def cylinder_cloud(radius: float = 0.03, height: float = 0.12, n: int = 1500, seed: int = 1) -> np.ndarray:
    out = np.zeros((n, 3))
    L.load_fixtures().asicp_fx_cylinder_cloud(radius, height, n, seed, out.ctypes.data_as(L.c_double_p))
    a_side = 2.0 * np.pi * radius * height
    a_cap = np.pi * radius * radius
    n_side = int(n * a_side / (a_side + 2.0 * a_cap))
    return out[: n_side + 2 * ((n - n_side) // 2)]


def build_sdf(cloud: np.ndarray, voxel: float, padding: float = -1.0, band: float = 0.003):
    cloud = np.ascontiguousarray(cloud, dtype=np.float64)
    dims = (C.c_int32 * 3)()
    meta = (C.c_double * 5)()
    lib = L.load_fixtures()
    n = lib.asicp_fx_build_sdf(cloud.ctypes.data_as(L.c_double_p), len(cloud), voxel, padding, band, dims, meta, None)
    vals = np.zeros(n, dtype=np.float32)
    lib.asicp_fx_build_sdf(cloud.ctypes.data_as(L.c_double_p), len(cloud), voxel, padding, band, dims, meta,
                           vals.ctypes.data_as(L.c_float_p))
    return tuple(dims), np.array(meta[:3]), meta[3], meta[4], vals


def c2_trial(trial: int, n: int = 500):
    """Acceptance C2 trial inputs (test_acceptance.cpp:256-282): (source,
    reference, truth pose) — the reference box cloud displaced by the trial's
    seeded rigid transform."""
    lib = L.load_fixtures()
    src = np.zeros((n, 3))
    ref = np.zeros((n, 3))
    truth = np.zeros(7)
    lib.asicp_fx_c2_trial(trial, n, src.ctypes.data_as(L.c_double_p), ref.ctypes.data_as(L.c_double_p),
                          truth.ctypes.data_as(L.c_double_p))
    return src, ref, truth


def blob_cloud(n: int, radius: float, seed: int) -> np.ndarray:
    """synthetic::blob_cloud (synthetic.cpp:69-83)."""
    out = np.zeros((n, 3))
    L.load_fixtures().asicp_fx_blob_cloud(n, radius, seed, out.ctypes.data_as(L.c_double_p))
    return out
