"""Python mirror of the reference optimiser API (proj/include/graspmatch/grasp.hpp).

Same names, field meanings and error behaviour as graspmatch:
  * GraspProblem / Preshape / StackedSdf / SgdConfig / SteinConfig
    (grasp.hpp:16-44, sdf.hpp:23-47, optim.hpp:28-76)
  * optimize_grasp(problem) -> GraspSolution (grasp.hpp:141) — runs on the
    B200 through the C-ABI (include/asicp.h); contract violations raise
    InvalidArgument with the reference's message (types.hpp:65-72).
Point clouds are float64 numpy arrays of shape (n, 3); poses are 7-vectors
(tx, ty, tz, qw, qx, qy, qz) like PoseParams::as_vector (types.hpp:31-35).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


class InvalidArgument(ValueError):
    """graspmatch::InvalidArgument (types.hpp:65-68)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the B200 solver."""


class GraspStatus(enum.IntEnum):
    kFound = 0
    kNoGraspFound = 1


class ParticlePhase(enum.IntEnum):
    kStein = 0
    kSgd = 1


class BandwidthMode(enum.IntEnum):
    kMedianHeuristic = 0
    kFixed = 1


def _cloud(a) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))
    return arr


@dataclass
class SdfGrid:
    """graspmatch::SdfGrid (sdf.hpp:23-39); values x-major float32."""
    origin: np.ndarray
    voxel: float
    dims: tuple
    values: np.ndarray
    boundary_max_abs: float

    def max_corner(self) -> np.ndarray:
        return np.asarray(self.origin, dtype=np.float64) + self.voxel * (np.asarray(self.dims, dtype=np.float64) - 1)


@dataclass
class StackedSdf:
    """graspmatch::StackedSdf (sdf.hpp:43-47)."""
    grids: List[SdfGrid] = field(default_factory=list)
    epsilon: float = 0.0
    offsets: List[np.ndarray] = field(default_factory=list)


@dataclass
class Preshape:
    """graspmatch::Preshape (grasp.hpp:16-24)."""
    id: str
    inner_surface_cloud: np.ndarray
    full_cloud: np.ndarray
    tcp: np.ndarray
    sdf_index: int = 0


@dataclass
class PosePrior:
    t_mean: np.ndarray = field(default_factory=lambda: np.zeros(3))
    t_sigma: np.ndarray = field(default_factory=lambda: np.ones(3))
    q_location: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0, 0.0]))
    q_kappa: np.ndarray = field(default_factory=lambda: np.zeros(4))


@dataclass
class AnnealingSchedule:
    period_total: int = 40
    cycles: int = 5
    exponent: float = 2.0


class PreconditionerMode(enum.IntEnum):
    """graspmatch::PreconditionerMode (optim.hpp:14-27)."""
    kFixed = 0
    kGaussNewtonRotation = 1


@dataclass
class SgdConfig:
    """graspmatch::SgdConfig (optim.hpp:29-43).  optimize_grasp reads the
    first three fields; register_sgd_icp reads all of them."""
    learning_rate: float = 1.0
    A: np.ndarray = field(default_factory=lambda: np.eye(7))
    convergence_threshold: float = 0.0002
    max_iterations: int = 500
    preconditioner_mode: PreconditionerMode = PreconditionerMode.kFixed
    gn_damping: float = 1e-6
    minibatch_size: int = 100


@dataclass
class SteinConfig:
    bandwidth_mode: BandwidthMode = BandwidthMode.kMedianHeuristic
    fixed_bandwidth: float = 1.0
    prior: PosePrior = field(default_factory=PosePrior)
    annealing: AnnealingSchedule = field(default_factory=AnnealingSchedule)
    step_scale: float = 1.0


@dataclass
class GraspProblem:
    """graspmatch::GraspProblem (grasp.hpp:27-44)."""
    object_cloud: np.ndarray
    scene_cloud: np.ndarray
    preshapes: List[Preshape]
    sdf: StackedSdf
    com: np.ndarray
    initializations: List[np.ndarray]  # per preshape: (K, 7)
    sgd: SgdConfig = field(default_factory=SgdConfig)
    stein: SteinConfig = field(default_factory=SteinConfig)
    k_stein: int = 15
    k_max: int = 40
    contact_tolerance: float = 0.0
    seed: int = 0
    workers: int = 0
    record_trace: bool = False

    @property
    def n_particles(self) -> int:
        return int(sum(len(np.asarray(i).reshape(-1, 7)) for i in self.initializations))


@dataclass
class ParticleSummary:
    particle: int
    preshape_id: int
    theta: np.ndarray
    full_cloud_loss: float
    collision_free: bool
    converged: bool


@dataclass
class TraceRecord:
    iteration: int
    particle: int
    preshape_id: int
    loss: float
    in_collision: bool
    phase: ParticlePhase
    theta: np.ndarray


@dataclass
class GraspSolution:
    """graspmatch::GraspSolution (grasp.hpp:78-86), with array views."""
    status: GraspStatus
    theta: np.ndarray
    preshape_id: int
    final_loss: float
    converged: bool
    particle_theta: np.ndarray
    particle_loss: np.ndarray
    particle_collision_free: np.ndarray
    particle_converged: np.ndarray
    particle_preshape: np.ndarray
    trace_theta: Optional[np.ndarray] = None      # (k_max, J, 7)
    trace_loss: Optional[np.ndarray] = None       # (k_max, J)
    trace_in_collision: Optional[np.ndarray] = None
    k_stein: int = 0
    diagnostics: dict = field(default_factory=dict)

    @property
    def particles(self) -> List[ParticleSummary]:
        return [ParticleSummary(j, int(self.particle_preshape[j]), self.particle_theta[j],
                                float(self.particle_loss[j]), bool(self.particle_collision_free[j]),
                                bool(self.particle_converged[j])) for j in range(len(self.particle_loss))]

    @property
    def trace(self) -> List[TraceRecord]:
        if self.trace_theta is None:
            return []
        out = []
        for k in range(self.trace_theta.shape[0]):
            for j in range(self.trace_theta.shape[1]):
                out.append(TraceRecord(k, j, int(self.particle_preshape[j]), float(self.trace_loss[k, j]),
                                       bool(self.trace_in_collision[k, j]),
                                       ParticlePhase.kStein if k < self.k_stein else ParticlePhase.kSgd,
                                       self.trace_theta[k, j]))
        return out


# ---------------------------------------------------------------------------
# Marshalling (problem <-> asicp_problem)
# ---------------------------------------------------------------------------
class CProblem:
    """Owns the numpy buffers behind an asicp_problem struct."""

    def __init__(self, p: GraspProblem):
        keep = []

        def dptr(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a.ctypes.data_as(L.c_double_p), a

        s = L.Problem()
        obj = _cloud(p.object_cloud)
        scene = _cloud(p.scene_cloud)
        s.object_cloud, _ = dptr(obj)
        s.n_object = obj.shape[0]
        s.scene_cloud, _ = dptr(scene)
        s.n_scene = scene.shape[0]
        pres = (L.Preshape * max(1, len(p.preshapes)))()
        for i, ps in enumerate(p.preshapes):
            inner = _cloud(ps.inner_surface_cloud)
            full = _cloud(ps.full_cloud)
            pres[i].inner_surface, _ = dptr(inner)
            pres[i].n_surface = inner.shape[0]
            pres[i].full_cloud, _ = dptr(full)
            pres[i].n_full = full.shape[0]
            pres[i].tcp[:] = [float(x) for x in np.asarray(ps.tcp, dtype=np.float64).reshape(3)]
            pres[i].sdf_index = int(ps.sdf_index)
        keep.append(pres)
        s.preshapes = C.cast(pres, C.POINTER(L.Preshape))
        s.n_preshapes = len(p.preshapes)
        grids = (L.SdfGrid * max(1, len(p.sdf.grids)))()
        for i, g in enumerate(p.sdf.grids):
            vals = np.ascontiguousarray(g.values, dtype=np.float32).reshape(-1)
            keep.append(vals)
            grids[i].dims[:] = [int(x) for x in g.dims]
            grids[i].origin[:] = [float(x) for x in np.asarray(g.origin).reshape(3)]
            grids[i].voxel = float(g.voxel)
            grids[i].boundary_max_abs = float(g.boundary_max_abs)
            off = p.sdf.offsets[i] if i < len(p.sdf.offsets) else np.zeros(3)
            grids[i].offset[:] = [float(x) for x in np.asarray(off).reshape(3)]
            grids[i].values = vals.ctypes.data_as(L.c_float_p)
        keep.append(grids)
        s.sdf_grids = C.cast(grids, C.POINTER(L.SdfGrid))
        s.n_sdf_grids = len(p.sdf.grids)
        s.com[:] = [float(x) for x in np.asarray(p.com, dtype=np.float64).reshape(3)]
        inits = [np.asarray(i, dtype=np.float64).reshape(-1, 7) for i in p.initializations]
        allp = np.ascontiguousarray(np.concatenate(inits, axis=0) if inits else np.zeros((0, 7)))
        s.init_poses, _ = dptr(allp)
        counts = np.ascontiguousarray([len(i) for i in inits] or [0], dtype=np.int64)
        keep.append(counts)
        s.init_counts = counts.ctypes.data_as(L.c_i64_p)
        s.n_init_lists = len(inits)
        s.learning_rate = float(p.sgd.learning_rate)
        s.A[:] = [float(x) for x in np.asarray(p.sgd.A, dtype=np.float64).reshape(49)]
        s.convergence_threshold = float(p.sgd.convergence_threshold)
        s.bandwidth_mode = int(p.stein.bandwidth_mode)
        s.fixed_bandwidth = float(p.stein.fixed_bandwidth)
        s.prior_t_mean[:] = [float(x) for x in p.stein.prior.t_mean]
        s.prior_t_sigma[:] = [float(x) for x in p.stein.prior.t_sigma]
        s.prior_q_location[:] = [float(x) for x in p.stein.prior.q_location]
        s.prior_q_kappa[:] = [float(x) for x in p.stein.prior.q_kappa]
        s.anneal_period_total = int(p.stein.annealing.period_total)
        s.anneal_cycles = int(p.stein.annealing.cycles)
        s.anneal_exponent = float(p.stein.annealing.exponent)
        s.step_scale = float(p.stein.step_scale)
        s.k_stein = int(p.k_stein)
        s.k_max = int(p.k_max)
        s.contact_tolerance = float(p.contact_tolerance)
        s.seed = int(p.seed)
        s.workers = int(p.workers)
        s.record_trace = 1 if p.record_trace else 0
        self.struct = s
        self._keep = keep
        self.J = int(allp.shape[0])
        self.k_max = int(p.k_max)
        self.k_stein = int(p.k_stein)
        self.record_trace = bool(p.record_trace)

    def ptr(self):
        return C.byref(self.struct)


def problem_from_c(v: L.Problem) -> GraspProblem:
    """Copy an asicp_problem view (e.g. a fixture) into a GraspProblem."""
    def arr(ptr, n, cols=3):
        return np.ctypeslib.as_array(ptr, shape=(n * cols,)).reshape(n, cols).copy() if n else np.zeros((0, cols))

    pres, grids = [], []
    offsets = []
    for i in range(v.n_preshapes):
        s = v.preshapes[i]
        pres.append(Preshape(f"preshape-{i}", arr(s.inner_surface, s.n_surface), arr(s.full_cloud, s.n_full),
                             np.array(s.tcp[:]), int(s.sdf_index)))
    for i in range(v.n_sdf_grids):
        g = v.sdf_grids[i]
        n = g.dims[0] * g.dims[1] * g.dims[2]
        vals = np.ctypeslib.as_array(g.values, shape=(n,)).copy()
        grids.append(SdfGrid(np.array(g.origin[:]), g.voxel, tuple(g.dims[:]), vals, g.boundary_max_abs))
        offsets.append(np.array(g.offset[:]))
    counts = [v.init_counts[i] for i in range(v.n_init_lists)]
    allp = arr(v.init_poses, int(sum(counts)), 7)
    inits, o = [], 0
    for c in counts:
        inits.append(allp[o:o + c].copy())
        o += c
    prior = PosePrior(np.array(v.prior_t_mean[:]), np.array(v.prior_t_sigma[:]), np.array(v.prior_q_location[:]),
                      np.array(v.prior_q_kappa[:]))
    stein = SteinConfig(BandwidthMode(v.bandwidth_mode), v.fixed_bandwidth, prior,
                        AnnealingSchedule(v.anneal_period_total, v.anneal_cycles, v.anneal_exponent), v.step_scale)
    sgd = SgdConfig(v.learning_rate, np.array(v.A[:]).reshape(7, 7), v.convergence_threshold)
    return GraspProblem(arr(v.object_cloud, v.n_object), arr(v.scene_cloud, v.n_scene), pres,
                        StackedSdf(grids, 0.0, offsets), np.array(v.com[:]), inits, sgd, stein, int(v.k_stein),
                        int(v.k_max), v.contact_tolerance, int(v.seed), int(v.workers), bool(v.record_trace))


class SolutionBuffers:
    """Caller-allocated output arrays of an asicp_solution."""

    def __init__(self, J: int, k_max: int, record_trace: bool):
        self.J = J
        self.theta = np.zeros((J, 7))
        self.loss = np.zeros(J)
        self.free = np.zeros(J, dtype=np.int32)
        self.conv = np.zeros(J, dtype=np.int32)
        self.pre = np.zeros(J, dtype=np.int64)
        s = L.Solution()
        s.particle_theta = self.theta.ctypes.data_as(L.c_double_p)
        s.particle_loss = self.loss.ctypes.data_as(L.c_double_p)
        s.particle_collision_free = self.free.ctypes.data_as(L.c_i32_p)
        s.particle_converged = self.conv.ctypes.data_as(L.c_i32_p)
        s.particle_preshape = self.pre.ctypes.data_as(L.c_i64_p)
        self.trace = record_trace and k_max > 0
        if self.trace:
            self.tr_theta = np.zeros((k_max, J, 7))
            self.tr_loss = np.zeros((k_max, J))
            self.tr_col = np.zeros((k_max, J), dtype=np.int32)
            s.trace_theta = self.tr_theta.ctypes.data_as(L.c_double_p)
            s.trace_loss = self.tr_loss.ctypes.data_as(L.c_double_p)
            s.trace_in_collision = self.tr_col.ctypes.data_as(L.c_i32_p)
        self.struct = s

    def solution(self, k_stein: int) -> GraspSolution:
        s = self.struct
        diag = dict(nn_queries=s.nn_queries, nn_uncertified=s.nn_uncertified, nn_full_refines=s.nn_full_refines,
                    nn_pool_ties=s.nn_pool_ties, nn_pairs=s.nn_pairs)
        return GraspSolution(GraspStatus(s.status), np.array(s.theta[:]), int(s.preshape_id), float(s.final_loss),
                             bool(s.converged), self.theta.copy(), self.loss.copy(), self.free.astype(bool),
                             self.conv.astype(bool), self.pre.copy(),
                             self.tr_theta.copy() if self.trace else None,
                             self.tr_loss.copy() if self.trace else None,
                             self.tr_col.astype(bool) if self.trace else None, k_stein, diag)


def _check(rc: int, err: C.Array) -> None:
    if rc == L.ASICP_OK:
        return
    msg = err.value.decode(errors="replace")
    if rc == L.ASICP_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    raise DeviceError(msg)


class Solver:
    """A context on one B200: device buffers (and the captured CUDA graph)
    persist across calls.  `stream` may be a torch CUDA stream handle."""

    def __init__(self, device: int = 0, stream: int | None = None, nn_mode: int = 0, use_graph: bool = True,
                 profile: bool = False, window_pool: int = 0, max_chunks: int = 0, throughput: bool = False,
                 nn_tc: bool | None = None):
        self.lib = L.load()
        err = C.create_string_buffer(512)
        self.ctx = self.lib.asicp_create(device, C.c_void_p(stream) if stream else None, err, 512)
        if not self.ctx:
            raise DeviceError(err.value.decode(errors="replace"))
        self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_NN_MODE, nn_mode)
        self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_USE_GRAPH, 1 if use_graph else 0)
        self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_PROFILE, 1 if profile else 0)
        if window_pool:
            self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_WINDOW_POOL, window_pool)
        if max_chunks:
            self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_MAX_CHUNKS, max_chunks)
        if throughput:  # the context shares the GPU with other solves (BatchSolver)
            self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_THROUGHPUT, 1)
        if nn_tc is not None:  # tensor-core NN filter (default: ASICP_NN_TC, else off)
            self.lib.asicp_set_option(self.ctx, L.ASICP_OPT_NN_TC, 1 if nn_tc else 0)
        self._cp: CProblem | None = None
        self._bufs: SolutionBuffers | None = None

    def close(self):
        if self.ctx:
            self.lib.asicp_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, problem: GraspProblem | CProblem) -> None:
        cp = problem if hasattr(problem, "ptr") else CProblem(problem)
        err = C.create_string_buffer(512)
        _check(self.lib.asicp_prepare(self.ctx, cp.ptr(), err, 512), err)
        self._cp = cp
        self._bufs = SolutionBuffers(cp.J, cp.k_max, cp.record_trace)

    def run(self) -> GraspSolution:
        err = C.create_string_buffer(512)
        _check(self.lib.asicp_run(self.ctx, C.byref(self._bufs.struct), err, 512), err)
        return self._bufs.solution(self._cp.k_stein)

    def build_sdf(self, cloud, voxel: float, padding: float = -1.0, surface_band: float = 0.003) -> SdfGrid:
        """graspmatch::build_sdf (sdf.cpp:48-175) on this context's GPU."""
        cloud = np.ascontiguousarray(np.asarray(cloud, dtype=np.float64).reshape(-1, 3))
        dims = (C.c_int32 * 3)()
        meta = (C.c_double * 5)()
        err = C.create_string_buffer(512)
        cp = cloud.ctypes.data_as(L.c_double_p)
        _check(self.lib.asicp_build_sdf(self.ctx, cp, len(cloud), voxel, padding, surface_band, dims, meta, None, err,
                                        512), err)
        values = np.zeros(int(dims[0]) * int(dims[1]) * int(dims[2]), dtype=np.float32)
        _check(self.lib.asicp_build_sdf(self.ctx, cp, len(cloud), voxel, padding, surface_band, dims, meta,
                                        values.ctypes.data_as(L.c_float_p), err, 512), err)
        return SdfGrid(np.array(meta[:3]), float(meta[3]), tuple(int(d) for d in dims), values, float(meta[4]))

    def set_partition_nccl(self, rank: int, world: int, unique_id: bytes) -> None:
        """Shard every population's particles over `world` ranks (one process
        per GPU); collective — every rank calls it with rank 0's id."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        err = C.create_string_buffer(512)
        _check(self.lib.asicp_set_partition_nccl(self.ctx, rank, world, unique_id, err, 512), err)
        self._cp = None

    def set_partition_group(self, group: "Group", rank: int) -> None:
        """Shard with the contexts of this process (one host thread per rank)."""
        err = C.create_string_buffer(512)
        _check(self.lib.asicp_set_partition_group(self.ctx, group.handle, rank, err, 512), err)
        self._cp = None

    def clear_partition(self) -> None:
        self.lib.asicp_clear_partition(self.ctx)
        self._cp = None

    def run_async(self) -> None:
        """Enqueue the prepared solve on this context's stream and return
        (asicp_run_async); collect it with `wait`."""
        err = C.create_string_buffer(512)
        _check(self.lib.asicp_run_async(self.ctx, err, 512), err)

    def wait(self) -> GraspSolution:
        err = C.create_string_buffer(512)
        _check(self.lib.asicp_wait(self.ctx, C.byref(self._bufs.struct), err, 512), err)
        return self._bufs.solution(self._cp.k_stein)

    def optimize(self, problem: GraspProblem | CProblem) -> GraspSolution:
        self.prepare(problem)
        return self.run()

    def stats(self) -> L.Stats:
        st = L.Stats()
        self.lib.asicp_get_stats(self.ctx, C.byref(st))
        return st

    def raw_stats(self) -> list:
        """The last solve's device counters (asicp_dbg_raw_stats, include/asicp_debug.h):
        [0] uncertified NN windows, [1] full FP64 rescans, [2] NN queries, [3] pool ties,
        [4] NN pairs, [12] forward/final filter pairs, [13] active particle evaluations."""
        out = (C.c_uint64 * 256)()
        self.lib.asicp_dbg_raw_stats(self.ctx, out)
        return list(out)


class Group:
    """An in-process exchange group for particle sharding (asicp_group)."""

    def __init__(self, world: int):
        self.lib = L.load()
        self.world = world
        self.handle = self.lib.asicp_group_create(world)
        if not self.handle:
            raise InvalidArgument("asicp_group_create: world must be >= 1")

    def close(self):
        if self.handle:
            self.lib.asicp_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 makes it, the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    err = C.create_string_buffer(512)
    _check(L.load().asicp_nccl_unique_id(buf, err, 512), err)
    return buf.raw


_DEFAULT: Solver | None = None


def optimize_grasp(problem: GraspProblem) -> GraspSolution:
    """graspmatch::optimize_grasp (grasp.hpp:141) on the B200."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Solver()
    return _DEFAULT.optimize(problem)


def export_trace(solution: GraspSolution, path) -> None:
    """graspmatch::export_trace (io.cpp:691-710) of a solution recorded with
    record_trace: the reference's 13-field text format (host only)."""
    lib = L.load()
    if solution.trace_theta is None:
        k_max, J = 0, len(solution.particle_loss)
        th = np.zeros((0, 7))
        loss = np.zeros(0)
        col = np.zeros(0, dtype=np.int32)
    else:
        k_max, J = solution.trace_loss.shape
        th = np.ascontiguousarray(solution.trace_theta, dtype=np.float64)
        loss = np.ascontiguousarray(solution.trace_loss, dtype=np.float64)
        col = np.ascontiguousarray(solution.trace_in_collision, dtype=np.int32)
    pre = np.ascontiguousarray(solution.particle_preshape, dtype=np.int64)
    err = C.create_string_buffer(512)
    _check(lib.asicp_export_trace(str(path).encode(), k_max, J, solution.k_stein, pre.ctypes.data_as(L.c_i64_p),
                                  th.ctypes.data_as(L.c_double_p), loss.ctypes.data_as(L.c_double_p),
                                  col.ctypes.data_as(L.c_i32_p), err, 512), err)


def build_sdf(cloud, voxel: float, padding: float = -1.0, surface_band: float = 0.003) -> SdfGrid:
    """graspmatch::build_sdf (sdf.hpp, sdf.cpp:48-175) on the B200."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Solver()
    return _DEFAULT.build_sdf(cloud, voxel, padding, surface_band)


def minibatch_schedule(k: int, k_max: int, n_ref: int) -> int:
    return int(L.load().asicp_minibatch_schedule(k, k_max, n_ref))


def annealing(t: int, T: int, C_: int, p: float) -> float:
    return float(L.load().asicp_annealing(t, T, C_, p))
