"""ctypes binding of the C ABI in include/stmg_b200.h.

This is the reference-side binding a Python caller would add (see
INTEGRATION.md).  It loads the in-tree ``libstmg_b200.so``; there is no
fallback -- importing without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STMG_LIB") or os.path.join(_HERE, "libstmg_b200.so")

STMG_OK, STMG_EINVAL, STMG_ERUNTIME = 0, 1, 2
PATH_SPECTRAL, PATH_PHYSICAL = 0, 1

D = C.c_double
PD = C.POINTER(C.c_double)
VP = C.c_void_p


class HierarchyParams(C.Structure):
    _fields_ = [("p_t", C.c_int), ("dim", C.c_int), ("space_level", C.c_int),
                ("time_level", C.c_int), ("t_final", D), ("mu_star", D),
                ("policy", C.c_int), ("two_grid", C.c_int), ("device", C.c_int),
                ("shards", C.c_int)]


class CycleConfig(C.Structure):
    _fields_ = [("nu1", C.c_int), ("nu2", C.c_int), ("gamma", C.c_int),
                ("omega_t", D), ("path", C.c_int), ("block_solver", C.c_int),
                ("omega_x", D), ("nu1_x", C.c_int), ("nu2_x", C.c_int), ("gamma_x", C.c_int)]


class SmootherConfig(C.Structure):
    _fields_ = [("omega_t", D), ("nu", C.c_int), ("block_solver", C.c_int), ("omega_x", D),
                ("nu1_x", C.c_int), ("nu2_x", C.c_int), ("gamma_x", C.c_int)]


class SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("wall_time_seconds", D), ("device_time_seconds", D),
                ("r0", D), ("r_final", D), ("seed", C.c_uint64)]


class LevelInfo(C.Structure):
    _fields_ = [("n_t", C.c_int64), ("n_x", C.c_int64), ("n_loc", C.c_int64),
                ("n1", C.c_int64), ("dim", C.c_int), ("space_level", C.c_int),
                ("coarsen_to_next", C.c_int), ("tau", D), ("h", D), ("mu", D)]


class RhoProblem(C.Structure):
    _fields_ = [("p_t", C.c_int), ("dim", C.c_int), ("space_level", C.c_int),
                ("time_level", C.c_int), ("mu", D), ("mode", C.c_int), ("device", C.c_int)]


class RhoMeasurement(C.Structure):
    _fields_ = [("measured_rho", D), ("predicted_rho", D), ("n_iterations_used", C.c_int),
                ("seed_used", C.c_uint64)]


# (name, restype, argtypes) for every symbol declared in include/stmg_b200.h
SIGNATURES = [
    ("stmg_last_error", C.c_char_p, []),
    ("stmg_critical_mu", D, [C.c_int]),
    ("stmg_dg_block", C.c_int, [C.c_int, D, PD, PD, PD]),
    ("stmg_time_transfer", C.c_int, [C.c_int, D, PD, PD]),
    ("stmg_create", C.c_int, [C.POINTER(HierarchyParams), C.POINTER(VP)]),
    ("stmg_destroy", C.c_int, [VP]),
    ("stmg_num_levels", C.c_int, [VP, C.POINTER(C.c_int)]),
    ("stmg_get_level_info", C.c_int, [VP, C.c_int, C.POINTER(LevelInfo)]),
    ("stmg_level_size", C.c_int, [VP, C.c_int, C.POINTER(C.c_int64)]),
    ("stmg_device_alloc", C.c_int, [VP, C.c_size_t, C.POINTER(VP)]),
    ("stmg_device_free", C.c_int, [VP, VP]),
    ("stmg_upload", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("stmg_download", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("stmg_memset_zero", C.c_int, [VP, VP, C.c_size_t]),
    ("stmg_host_alloc", C.c_int, [VP, C.c_size_t, C.POINTER(VP)]),
    ("stmg_host_free", C.c_int, [VP, VP]),
    ("stmg_synchronize", C.c_int, [VP]),
    ("stmg_fill_uniform", C.c_int, [VP, VP, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64]),
    ("stmg_fill_random_host", C.c_int, [VP, C.c_int64, C.c_uint64]),
    ("stmg_fold_u0", C.c_int, [VP, VP, VP]),
    ("stmg_apply", C.c_int, [VP, C.c_int, VP, VP]),
    ("stmg_residual", C.c_int, [VP, C.c_int, VP, VP, VP]),
    ("stmg_norm", C.c_int, [VP, C.c_int, VP, PD]),
    ("stmg_block_solve", C.c_int, [VP, C.c_int, VP, VP]),
    ("stmg_smooth", C.c_int, [VP, C.c_int, VP, VP, D, C.c_int]),
    ("stmg_block_jacobi_step", C.c_int, [VP, C.c_int, VP, VP, C.POINTER(SmootherConfig)]),
    ("stmg_spatial_vcycle", C.c_int, [VP, C.c_int, VP, VP, VP, C.POINTER(SmootherConfig)]),
    ("stmg_cycle_config_init", C.c_int, [C.POINTER(CycleConfig)]),
    ("stmg_smoother_config_init", C.c_int, [C.POINTER(SmootherConfig)]),
    ("stmg_restrict", C.c_int, [VP, C.c_int, C.c_int, VP, VP]),
    ("stmg_prolong", C.c_int, [VP, C.c_int, C.c_int, VP, VP]),
    ("stmg_forward_substitution", C.c_int, [VP, C.c_int, VP, VP]),
    ("stmg_mg_cycle", C.c_int, [VP, C.c_int, VP, VP, C.POINTER(CycleConfig)]),
    ("stmg_solve", C.c_int, [VP, VP, VP, C.POINTER(CycleConfig), D, C.c_int, PD, C.c_int,
                             C.POINTER(SolveReport)]),
    ("stmg_solve_host", C.c_int, [VP, VP, VP, C.POINTER(CycleConfig), D, C.c_int, PD, C.c_int,
                                  C.POINTER(SolveReport)]),
    ("stmg_solve_host_batch", C.c_int, [VP, C.c_int, VP, VP, VP, C.POINTER(CycleConfig), D,
                                        C.c_int, C.POINTER(SolveReport)]),
    ("stmg_nccl_unique_id", C.c_int, [VP, C.c_size_t]),
    ("stmg_create_distributed", C.c_int, [C.POINTER(HierarchyParams), C.c_int, C.c_int, VP,
                                          C.c_size_t, C.POINTER(VP)]),
    ("stmg_shard_plan", C.c_int, [C.POINTER(HierarchyParams), C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int64)]),
    ("stmg_local_steps", C.c_int, [VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("stmg_profile_enable", C.c_int, [VP, C.c_int]),
    ("stmg_profile_read", C.c_int, [VP, C.c_int, PD, C.POINTER(C.c_int64), PD]),
    ("stmg_profile_reset", C.c_int, [VP]),
    ("stmg_launch_count", C.c_int, [VP, C.POINTER(C.c_int64)]),
    ("stmg_lfa_beta", C.c_int, [D, PD]),
    ("stmg_lfa_alpha", C.c_int, [C.c_int, D, D, PD]),
    ("stmg_lfa_smoother_rho", C.c_int, [C.c_int, D, D, D, D, PD, PD]),
    ("stmg_lfa_smoother_symbol", C.c_int, [C.c_int, D, D, D, D, PD, PD]),
    ("stmg_lfa_twogrid_symbol", C.c_int, [C.c_int, D, C.POINTER(CycleConfig), C.c_int, D, D,
                                          PD, PD]),
    ("stmg_lfa_spectral_radius", C.c_int, [C.c_int, PD, PD, PD]),
    ("stmg_lfa_smoothing_factor", C.c_int, [C.c_int, D, D, C.c_int, C.c_int, C.c_int, PD]),
    ("stmg_lfa_twogrid_factor", C.c_int, [C.c_int, D, C.POINTER(CycleConfig), C.c_int, C.c_int,
                                          C.c_int, PD]),
    ("stmg_lfa_twogrid_factor_inexact", C.c_int, [C.c_int, D, C.POINTER(CycleConfig), D, C.c_int,
                                                  C.c_int, C.c_int, C.c_int, C.c_int, PD]),
    ("stmg_measure_convergence_factor", C.c_int, [C.POINTER(RhoProblem), C.POINTER(CycleConfig),
                                                  C.c_uint64, C.c_int, C.c_int,
                                                  C.POINTER(RhoMeasurement)]),
]

_lib = None


def lib():
    """Load libstmg_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1411_0519_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == STMG_OK:
        return
    msg = lib().stmg_last_error().decode()
    if rc == STMG_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)
