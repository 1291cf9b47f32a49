"""B200-native (sm_100a, FP64) MB4 time-stepping core for the 2-D NLS lattice.

Drop-in for the reference's hot path (proj/include/nls2d: mb4_step,
StepDriver::advance, observables) through the C ABI in include/mb4cu.h.
"""
from . import _lib  # noqa: F401
from .nls2d import (  # noqa: F401
    GridModel, GridSpec, Mb4Scheme, NewtonConfig, NonConvergenceError, Observables, Session,
    StepDriver, StepStats, build_delta_potential, eval_phi, initial_condition, mb4_step,
    observables, rhs,
)

__all__ = [
    "GridModel", "GridSpec", "Mb4Scheme", "NewtonConfig", "NonConvergenceError", "Observables",
    "Session", "StepDriver", "StepStats", "build_delta_potential", "eval_phi",
    "initial_condition", "mb4_step", "observables", "rhs",
]
