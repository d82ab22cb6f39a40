"""SGD-ICP registration — the drop-in for graspmatch::register_sgd_icp.

Mirrors optim.hpp:163-176 (RegistrationResult, register_sgd_icp) over the
C-ABI of include/asicp.h (asicp_register_sgd_icp / _batch / _prepare / _run);
the work runs in csrc/register.cu, one CTA per problem.  Same names, argument
meaning and errors as the reference: InvalidArgument carries the message the
reference's `require` throws.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import _lib as L
from .grasp import PreconditionerMode, SgdConfig, Solver, _check

__all__ = ["RegistrationResult", "register_sgd_icp", "register_sgd_icp_batch", "RegistrationBatch",
           "sgd_config_struct", "ClosedFormStepResult", "icp_closed_form_step", "icp_closed_form_step_batch"]


@dataclass
class RegistrationResult:
    """graspmatch::RegistrationResult (optim.hpp:163-168); theta = (t, q)."""
    theta: np.ndarray
    iterations: int
    final_loss: float
    converged: bool


def sgd_config_struct(cfg: SgdConfig) -> L.SgdCfg:
    s = L.SgdCfg()
    s.learning_rate = float(cfg.learning_rate)
    s.A[:] = [float(x) for x in np.asarray(cfg.A, dtype=np.float64).reshape(49)]
    s.max_iterations = int(cfg.max_iterations)
    s.convergence_threshold = float(cfg.convergence_threshold)
    s.preconditioner_mode = int(PreconditionerMode(cfg.preconditioner_mode))
    s.gn_damping = float(cfg.gn_damping)
    s.minibatch_size = int(cfg.minibatch_size)
    return s


def _cloud(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.size == 0:
        return np.zeros((0, 3))
    return a.reshape(-1, 3)


def _pose(p) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(7))


def _result(r: L.Registration) -> RegistrationResult:
    return RegistrationResult(np.array(r.theta[:]), int(r.iterations), float(r.final_loss), bool(r.converged))


def _pack(sources: Sequence, references: Sequence, initials, seeds):
    src = [_cloud(s) for s in sources]
    ref = [_cloud(r) for r in references]
    if len(src) != len(ref):
        raise ValueError("register_sgd_icp_batch: sources and references differ in length")
    n = len(src)
    so = np.zeros(n + 1, dtype=np.int64)
    ro = np.zeros(n + 1, dtype=np.int64)
    so[1:] = np.cumsum([len(s) for s in src])
    ro[1:] = np.cumsum([len(r) for r in ref])
    S = np.ascontiguousarray(np.concatenate(src) if n else np.zeros((0, 3)))
    R = np.ascontiguousarray(np.concatenate(ref) if n else np.zeros((0, 3)))
    init = np.ascontiguousarray(np.asarray(initials, dtype=np.float64).reshape(n, 7))
    sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(n))
    return n, S, so, R, ro, init, sd


def _dp(a: np.ndarray):
    return a.ctypes.data_as(L.c_double_p)


def register_sgd_icp(source, reference, initial, cfg: SgdConfig, seed: int, solver: Solver | None = None
                     ) -> RegistrationResult:
    """graspmatch::register_sgd_icp (optim.cpp:274-321) on the GPU."""
    own = solver is None
    s = Solver() if own else solver
    try:
        src, ref, init = _cloud(source), _cloud(reference), _pose(initial)
        c = sgd_config_struct(cfg)
        out = L.Registration()
        err = C.create_string_buffer(512)
        _check(s.lib.asicp_register_sgd_icp(s.ctx, _dp(src), len(src), _dp(ref), len(ref), _dp(init), C.byref(c),
                                            C.c_uint64(int(seed)), C.byref(out), err, 512), err)
        return _result(out)
    finally:
        if own:
            s.close()


class RegistrationBatch:
    """Independent registrations with one SgdConfig, uploaded once and solved
    on the device (one CTA per problem); `run()` may repeat."""

    def __init__(self, solver: Solver, sources: Sequence, references: Sequence, initials, seeds,
                 cfg: SgdConfig):
        self.solver = solver
        self.n, self.S, self.so, self.R, self.ro, self.init, self.seeds = _pack(sources, references, initials, seeds)
        self.cfg = sgd_config_struct(cfg)
        self.out = (L.Registration * max(self.n, 1))()
        err = C.create_string_buffer(512)
        _check(solver.lib.asicp_register_prepare(
            solver.ctx, self.n, _dp(self.S), self.so.ctypes.data_as(L.c_i64_p), _dp(self.R),
            self.ro.ctypes.data_as(L.c_i64_p), _dp(self.init), self.seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            C.byref(self.cfg), err, 512), err)

    def run(self) -> List[RegistrationResult]:
        err = C.create_string_buffer(512)
        _check(self.solver.lib.asicp_register_run(self.solver.ctx, self.out, err, 512), err)
        return [_result(self.out[i]) for i in range(self.n)]

    @property
    def input_bytes(self) -> int:
        return self.S.nbytes + self.R.nbytes + self.so.nbytes + self.ro.nbytes + self.init.nbytes + self.seeds.nbytes

    @property
    def output_bytes(self) -> int:
        return self.n * (7 * 8 + 8 + 8 + 4 + 4)


def register_sgd_icp_batch(sources: Sequence, references: Sequence, initials, cfg: SgdConfig, seeds,
                           solver: Solver | None = None) -> List[RegistrationResult]:
    """register_sgd_icp for every (source, reference, initial, seed) at once."""
    own = solver is None
    s = Solver() if own else solver
    try:
        n, S, so, R, ro, init, sd = _pack(sources, references, initials, seeds)
        c = sgd_config_struct(cfg)
        out = (L.Registration * max(n, 1))()
        err = C.create_string_buffer(512)
        _check(s.lib.asicp_register_sgd_icp_batch(
            s.ctx, n, _dp(S), so.ctypes.data_as(L.c_i64_p), _dp(R), ro.ctypes.data_as(L.c_i64_p), _dp(init),
            sd.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(c), out, err, 512), err)
        return [_result(out[i]) for i in range(n)]
    finally:
        if own:
            s.close()


@dataclass
class ClosedFormStepResult:
    """graspmatch::ClosedFormStepResult (optim.hpp:82-85); theta = (t, q)."""
    theta: np.ndarray
    degenerate: bool


def icp_closed_form_step_batch(sources: Sequence, references: Sequence, thetas, solver: Solver | None = None
                               ) -> List[ClosedFormStepResult]:
    """graspmatch::icp_closed_form_step (optim.cpp:51-90) for every (source,
    reference, theta) at once, one CTA each.  The reference's NnIndex argument
    is its reference cloud here."""
    own = solver is None
    s = Solver() if own else solver
    try:
        n, S, so, R, ro, th, _ = _pack(sources, references, thetas, np.zeros(len(sources), dtype=np.uint64))
        out = (L.IcpStep * max(n, 1))()
        err = C.create_string_buffer(512)
        _check(s.lib.asicp_icp_closed_form_step_batch(s.ctx, n, _dp(S), so.ctypes.data_as(L.c_i64_p), _dp(R),
                                                      ro.ctypes.data_as(L.c_i64_p), _dp(th), out, err, 512), err)
        return [ClosedFormStepResult(np.array(out[i].theta[:]), bool(out[i].degenerate)) for i in range(n)]
    finally:
        if own:
            s.close()


def icp_closed_form_step(source, reference, theta, solver: Solver | None = None) -> ClosedFormStepResult:
    """graspmatch::icp_closed_form_step (optim.cpp:51-90) on the GPU."""
    own = solver is None
    s = Solver() if own else solver
    try:
        src, ref, th = _cloud(source), _cloud(reference), _pose(theta)
        out = L.IcpStep()
        err = C.create_string_buffer(512)
        _check(s.lib.asicp_icp_closed_form_step(s.ctx, _dp(src), len(src), _dp(ref), len(ref), _dp(th), C.byref(out),
                                                err, 512), err)
        return ClosedFormStepResult(np.array(out.theta[:]), bool(out.degenerate))
    finally:
        if own:
            s.close()
