"""ctypes binding of the C-ABI in include/asicp.h and include/asicp_fixtures.h.

The product path is the CUDA library libasicp.so built in-tree by
paper_2412_08346_b200/build.py.  There is no CPU fallback: if the library is
missing, loading fails loudly.  The synthetic-input generators of
include/asicp_fixtures.h (tests and bench inputs, not the product) are a
separate host-only library, libasicp_fixtures.so.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libasicp.so"
FIXTURES_PATH = PKG / "libasicp_fixtures.so"

c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)
c_i32_p = C.POINTER(C.c_int32)
c_i64_p = C.POINTER(C.c_int64)

ASICP_OK = 0
ASICP_INVALID_ARGUMENT = 1
ASICP_DEVICE_ERROR = 2
ASICP_STATUS_FOUND = 0
ASICP_STATUS_NO_GRASP_FOUND = 1
ASICP_BANDWIDTH_MEDIAN = 0
ASICP_BANDWIDTH_FIXED = 1
ASICP_OPT_NN_MODE = 1
ASICP_OPT_USE_GRAPH = 2
ASICP_OPT_PROFILE = 3
ASICP_OPT_MAX_CHUNKS = 4
ASICP_OPT_WINDOW_POOL = 5
ASICP_OPT_THROUGHPUT = 6
ASICP_OPT_NN_TC = 7
ASICP_PRECOND_FIXED = 0
ASICP_PRECOND_GAUSS_NEWTON_ROTATION = 1


class SdfGrid(C.Structure):
    _fields_ = [
        ("dims", C.c_int32 * 3),
        ("origin", C.c_double * 3),
        ("voxel", C.c_double),
        ("boundary_max_abs", C.c_double),
        ("offset", C.c_double * 3),
        ("values", c_float_p),
    ]


class Preshape(C.Structure):
    _fields_ = [
        ("inner_surface", c_double_p),
        ("n_surface", C.c_int64),
        ("full_cloud", c_double_p),
        ("n_full", C.c_int64),
        ("tcp", C.c_double * 3),
        ("sdf_index", C.c_int64),
    ]


class Problem(C.Structure):
    _fields_ = [
        ("object_cloud", c_double_p),
        ("n_object", C.c_int64),
        ("scene_cloud", c_double_p),
        ("n_scene", C.c_int64),
        ("preshapes", C.POINTER(Preshape)),
        ("n_preshapes", C.c_int64),
        ("sdf_grids", C.POINTER(SdfGrid)),
        ("n_sdf_grids", C.c_int64),
        ("com", C.c_double * 3),
        ("init_poses", c_double_p),
        ("init_counts", c_i64_p),
        ("n_init_lists", C.c_int64),
        ("learning_rate", C.c_double),
        ("A", C.c_double * 49),
        ("convergence_threshold", C.c_double),
        ("bandwidth_mode", C.c_int32),
        ("fixed_bandwidth", C.c_double),
        ("prior_t_mean", C.c_double * 3),
        ("prior_t_sigma", C.c_double * 3),
        ("prior_q_location", C.c_double * 4),
        ("prior_q_kappa", C.c_double * 4),
        ("anneal_period_total", C.c_int64),
        ("anneal_cycles", C.c_int64),
        ("anneal_exponent", C.c_double),
        ("step_scale", C.c_double),
        ("k_stein", C.c_int64),
        ("k_max", C.c_int64),
        ("contact_tolerance", C.c_double),
        ("seed", C.c_uint64),
        ("workers", C.c_int32),
        ("record_trace", C.c_int32),
    ]


class Solution(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("theta", C.c_double * 7),
        ("preshape_id", C.c_int64),
        ("final_loss", C.c_double),
        ("converged", C.c_int32),
        ("n_particles", C.c_int64),
        ("particle_theta", c_double_p),
        ("particle_loss", c_double_p),
        ("particle_collision_free", c_i32_p),
        ("particle_converged", c_i32_p),
        ("particle_preshape", c_i64_p),
        ("trace_theta", c_double_p),
        ("trace_loss", c_double_p),
        ("trace_in_collision", c_i32_p),
        ("nn_queries", C.c_int64),
        ("nn_uncertified", C.c_int64),
        ("nn_full_refines", C.c_int64),
        ("nn_pool_ties", C.c_int64),
        ("nn_pairs", C.c_double),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("solve_ms", C.c_double),
        ("nn_ms", C.c_double),
        ("nn_launches", C.c_int64),
        ("nn_pairs", C.c_double),
        ("collide_ms", C.c_double),
        ("minibatch_ms", C.c_double),
        ("cost_ms", C.c_double),
        ("svgd_ms", C.c_double),
        ("kernel_launches", C.c_int64),
    ]


class SgdCfg(C.Structure):
    """asicp_sgd_config (graspmatch::SgdConfig, optim.hpp:29-43)."""
    _fields_ = [
        ("learning_rate", C.c_double),
        ("A", C.c_double * 49),
        ("max_iterations", C.c_int64),
        ("convergence_threshold", C.c_double),
        ("preconditioner_mode", C.c_int32),
        ("gn_damping", C.c_double),
        ("minibatch_size", C.c_int64),
    ]


class Registration(C.Structure):
    """asicp_registration (graspmatch::RegistrationResult, optim.hpp:163-168)."""
    _fields_ = [
        ("theta", C.c_double * 7),
        ("iterations", C.c_int64),
        ("final_loss", C.c_double),
        ("converged", C.c_int32),
    ]


class IcpStep(C.Structure):
    """asicp_icp_step (graspmatch::ClosedFormStepResult, optim.hpp:82-85)."""
    _fields_ = [("theta", C.c_double * 7), ("degenerate", C.c_int32)]


# Every symbol include/asicp.h declares (libasicp.so) ...
EXPORTS = (
    "asicp_abi_version", "asicp_create", "asicp_destroy", "asicp_set_option", "asicp_prepare",
    "asicp_run", "asicp_run_async", "asicp_wait", "asicp_optimize_grasp", "asicp_build_sdf", "asicp_export_trace",
    "asicp_nccl_unique_id", "asicp_set_partition_nccl", "asicp_group_create", "asicp_group_destroy",
    "asicp_set_partition_group", "asicp_clear_partition", "asicp_get_stats", "asicp_minibatch_schedule",
    "asicp_annealing", "asicp_register_sgd_icp", "asicp_register_sgd_icp_batch",
    "asicp_register_prepare", "asicp_register_run",
    "asicp_icp_closed_form_step", "asicp_icp_closed_form_step_batch",
)
# ... and every symbol include/asicp_fixtures.h declares (libasicp_fixtures.so).
FIXTURE_EXPORTS = (
    "asicp_fx_desk", "asicp_fx_config", "asicp_fx_view", "asicp_fx_free", "asicp_fx_cylinder_cloud",
    "asicp_fx_build_sdf", "asicp_fx_c2_trial", "asicp_fx_blob_cloud",
)


def _declare(lib: C.CDLL) -> C.CDLL:
    lib.asicp_abi_version.restype = C.c_int
    lib.asicp_create.restype = C.c_void_p
    lib.asicp_create.argtypes = [C.c_int, C.c_void_p, C.c_char_p, C.c_size_t]
    lib.asicp_destroy.argtypes = [C.c_void_p]
    lib.asicp_set_option.argtypes = [C.c_void_p, C.c_int, C.c_int64]
    lib.asicp_prepare.argtypes = [C.c_void_p, C.POINTER(Problem), C.c_char_p, C.c_size_t]
    lib.asicp_run.argtypes = [C.c_void_p, C.POINTER(Solution), C.c_char_p, C.c_size_t]
    lib.asicp_run_async.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
    lib.asicp_wait.argtypes = [C.c_void_p, C.POINTER(Solution), C.c_char_p, C.c_size_t]
    lib.asicp_build_sdf.argtypes = [C.c_void_p, c_double_p, C.c_int64, C.c_double, C.c_double, C.c_double, c_i32_p,
                                    c_double_p, c_float_p, C.c_char_p, C.c_size_t]
    lib.asicp_export_trace.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, c_i64_p, c_double_p, c_double_p,
                                       c_i32_p, C.c_char_p, C.c_size_t]
    lib.asicp_nccl_unique_id.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
    lib.asicp_set_partition_nccl.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_size_t]
    lib.asicp_group_create.restype = C.c_void_p
    lib.asicp_group_create.argtypes = [C.c_int]
    lib.asicp_group_destroy.argtypes = [C.c_void_p]
    lib.asicp_set_partition_group.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_size_t]
    lib.asicp_clear_partition.argtypes = [C.c_void_p]
    lib.asicp_optimize_grasp.argtypes = [C.c_void_p, C.POINTER(Problem), C.POINTER(Solution), C.c_char_p,
                                         C.c_size_t]
    lib.asicp_get_stats.argtypes = [C.c_void_p, C.POINTER(Stats)]
    lib.asicp_minibatch_schedule.restype = C.c_int64
    lib.asicp_minibatch_schedule.argtypes = [C.c_int64, C.c_int64, C.c_int64]
    lib.asicp_annealing.restype = C.c_double
    lib.asicp_annealing.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double]
    lib.asicp_register_sgd_icp.argtypes = [C.c_void_p, c_double_p, C.c_int64, c_double_p, C.c_int64, c_double_p,
                                           C.POINTER(SgdCfg), C.c_uint64, C.POINTER(Registration), C.c_char_p,
                                           C.c_size_t]
    lib.asicp_register_sgd_icp_batch.argtypes = [C.c_void_p, C.c_int64, c_double_p, c_i64_p, c_double_p, c_i64_p,
                                                 c_double_p, C.POINTER(C.c_uint64), C.POINTER(SgdCfg),
                                                 C.POINTER(Registration), C.c_char_p, C.c_size_t]
    lib.asicp_register_prepare.argtypes = [C.c_void_p, C.c_int64, c_double_p, c_i64_p, c_double_p, c_i64_p,
                                           c_double_p, C.POINTER(C.c_uint64), C.POINTER(SgdCfg), C.c_char_p,
                                           C.c_size_t]
    lib.asicp_register_run.argtypes = [C.c_void_p, C.POINTER(Registration), C.c_char_p, C.c_size_t]
    lib.asicp_icp_closed_form_step.argtypes = [C.c_void_p, c_double_p, C.c_int64, c_double_p, C.c_int64, c_double_p,
                                               C.POINTER(IcpStep), C.c_char_p, C.c_size_t]
    lib.asicp_icp_closed_form_step_batch.argtypes = [C.c_void_p, C.c_int64, c_double_p, c_i64_p, c_double_p, c_i64_p,
                                                     c_double_p, C.POINTER(IcpStep), C.c_char_p, C.c_size_t]
    # include/asicp_debug.h (diagnostics)
    lib.asicp_dbg_raw_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    lib.asicp_dbg_iter_stats.restype = C.c_int64
    lib.asicp_dbg_iter_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]
    lib.asicp_dbg_ffma_tflops.restype = C.c_double
    lib.asicp_dbg_ffma_tflops.argtypes = [C.c_int]
    lib.asicp_dbg_dfma_tflops.restype = C.c_double
    lib.asicp_dbg_dfma_tflops.argtypes = [C.c_int]
    return lib


def declare_fixtures(lib: C.CDLL) -> C.CDLL:
    """Signatures of include/asicp_fixtures.h (any library exporting them)."""
    lib.asicp_fx_desk.restype = C.c_void_p
    lib.asicp_fx_desk.argtypes = [C.c_uint64, C.c_int64, C.c_int64]
    lib.asicp_fx_config.restype = C.c_void_p
    lib.asicp_fx_config.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64]
    lib.asicp_fx_view.restype = C.POINTER(Problem)
    lib.asicp_fx_view.argtypes = [C.c_void_p]
    lib.asicp_fx_free.argtypes = [C.c_void_p]
    lib.asicp_fx_cylinder_cloud.argtypes = [C.c_double, C.c_double, C.c_int, C.c_uint64, c_double_p]
    lib.asicp_fx_build_sdf.restype = C.c_int64
    lib.asicp_fx_build_sdf.argtypes = [c_double_p, C.c_int64, C.c_double, C.c_double, C.c_double, c_i32_p,
                                       c_double_p, c_float_p]
    lib.asicp_fx_c2_trial.argtypes = [C.c_int, C.c_int, c_double_p, c_double_p, c_double_p]
    lib.asicp_fx_blob_cloud.argtypes = [C.c_int, C.c_double, C.c_uint64, c_double_p]
    return lib


_LIB: C.CDLL | None = None
_FX: C.CDLL | None = None


def load() -> C.CDLL:
    """Load libasicp.so (raises if it was not built — there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2412_08346_b200.build`")
        _LIB = _declare(C.CDLL(str(LIB_PATH)))
    return _LIB


def load_fixtures() -> C.CDLL:
    """Load libasicp_fixtures.so (the synthetic-input generators)."""
    global _FX
    if _FX is None:
        if not FIXTURES_PATH.exists():
            raise RuntimeError(f"{FIXTURES_PATH} is missing: build it with `python -m paper_2412_08346_b200.build`")
        _FX = declare_fixtures(C.CDLL(str(FIXTURES_PATH)))
    return _FX
