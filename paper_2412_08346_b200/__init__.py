"""B200-native AS-ICP grasp optimiser (arXiv 2412.08346).

Drop-in for graspmatch::optimize_grasp (proj/include/graspmatch/grasp.hpp:141):
the CUDA library libasicp.so (csrc/, sm_100a) behind the C-ABI of
include/asicp.h, with a Python mirror of the reference API in grasp.py.
"""
from .grasp import (  # noqa: F401
    AnnealingSchedule,
    BandwidthMode,
    DeviceError,
    GraspProblem,
    GraspSolution,
    GraspStatus,
    InvalidArgument,
    ParticlePhase,
    PosePrior,
    PreconditionerMode,
    Preshape,
    SdfGrid,
    SgdConfig,
    Solver,
    StackedSdf,
    SteinConfig,
    annealing,
    build_sdf,
    export_trace,
    minibatch_schedule,
    optimize_grasp,
)
from .registration import (  # noqa: F401
    ClosedFormStepResult,
    RegistrationBatch,
    RegistrationResult,
    register_sgd_icp,
    register_sgd_icp_batch,
    icp_closed_form_step,
    icp_closed_form_step_batch,
)
