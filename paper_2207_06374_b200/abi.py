"""ctypes mirror of include/trstmi_b200.h (POD structs and constants).

Shared by the Python host mirror (api.py), bench.py and the tests.  Pure
layout definitions: importing this module loads no native code.
"""
import ctypes

TRSTMI_OK = 0
TRSTMI_ERR_INVALID_ARG = 1
TRSTMI_ERR_DIM_MISMATCH = 2
TRSTMI_ERR_ZERO_COLUMN = 3
TRSTMI_ERR_ALL_FAILED = 4
TRSTMI_ERR_CUDA = 5
TRSTMI_ERR_NCCL = 6
TRSTMI_ERR_UNSUPPORTED = 7
TRSTMI_ERR_NO_DEVICE = 8

COMPLEX = 0
REAL = 1

HVP_CENTRAL, HVP_FORWARD, HVP_BACKWARD, HVP_ZERO_DIR, HVP_FAILED = 0, 1, 2, 3, -1
ST_GRADIENT_TOLERANCE, ST_ITERATION_LIMIT, ST_RADIUS_UNDERFLOW = 0, 1, 2
TRIAL_OK, TRIAL_ZERO_COLUMN, TRIAL_NONFINITE_X0, TRIAL_NEED_RESCUE, TRIAL_INVALID = 0, 1, 2, 3, 4
CG_SMALL_RESIDUAL, CG_NEGATIVE_CURVATURE, CG_BOUNDARY_HIT, CG_ZERO_GRADIENT = 0, 1, 2, 3
MAX_STAGES = 32


class Cfg(ctypes.Structure):
    _fields_ = [
        ("field", ctypes.c_int32), ("d", ctypes.c_int32), ("N", ctypes.c_int32),
        ("n_stages", ctypes.c_int32), ("schedule", ctypes.c_double * MAX_STAGES),
        ("eps_target", ctypes.c_double),
        ("delta0", ctypes.c_double), ("delta_max", ctypes.c_double), ("eta", ctypes.c_double),
        ("shrink", ctypes.c_double), ("grow", ctypes.c_double), ("grad_tol", ctypes.c_double),
        ("max_outer", ctypes.c_int32), ("max_cg", ctypes.c_int32), ("cg_force_c", ctypes.c_double),
        ("record_cap", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


class TrialOut(ctypes.Structure):
    _fields_ = [
        ("coherence", ctypes.c_double), ("argmax_pair", ctypes.c_int64),
        ("status", ctypes.c_int32), ("stages_done", ctypes.c_int32),
        ("zero_col", ctypes.c_int32), ("fail_stage", ctypes.c_int32),
        ("outer_iterations", ctypes.c_int64), ("evals", ctypes.c_int64),
        ("hvps", ctypes.c_int64), ("records", ctypes.c_int64),
    ]


class StageOut(ctypes.Structure):
    _fields_ = [
        ("delta", ctypes.c_double), ("objective", ctypes.c_double), ("coherence", ctypes.c_double),
        ("argmax_pair", ctypes.c_int64), ("outer_iterations", ctypes.c_int32), ("status", ctypes.c_int32),
    ]


class OuterOut(ctypes.Structure):
    _fields_ = [
        ("stage", ctypes.c_int32), ("iteration", ctypes.c_int32), ("cg_exit", ctypes.c_int32),
        ("cg_iterations", ctypes.c_int32), ("accepted", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("value", ctypes.c_double), ("grad_norm", ctypes.c_double), ("radius", ctypes.c_double),
        ("rho", ctypes.c_double), ("step_norm", ctypes.c_double),
    ]


def default_cfg(field, d, N, max_outer=200, eps_target=1e-7):
    """trust_region.hpp:20-30 + solver.hpp:21-29 defaults (trstmi_cfg_defaults)."""
    c = Cfg()
    c.field, c.d, c.N = field, d, N
    c.n_stages = 0
    c.eps_target = eps_target
    c.delta0, c.delta_max, c.eta, c.shrink, c.grow = 0.0, 1e3, 0.05, 0.25, 2.0
    c.grad_tol, c.max_outer, c.max_cg, c.cg_force_c = 1e-9, max_outer, 0, 0.5
    c.record_cap = 0
    return c


def dim_of(field, d, N):
    return (2 if field == COMPLEX else 1) * d * N


def lanes_for(field, d, N):
    """CAS reduction width S — trstmi_lanes() of the built library
    (a pure function; loading the library needs no GPU)."""
    from . import api
    return api.load_library().trstmi_lanes(field, d, N)
