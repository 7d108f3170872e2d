"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product library
(``paper_1411_0519_b200``) never calls it.

It wraps ``oracle/_build/libstmg_oracle.so`` (built by ``oracle/Makefile``),
the C++ restatement of the reference solver in ``/root/reference/proj/src``
(see ``stmg_oracle.cpp`` for the file:line map).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libstmg_oracle.so")
_lib = None

P = C.POINTER(C.c_double)


class _Params(C.Structure):
    _fields_ = [("p_t", C.c_int), ("dim", C.c_int), ("space_level", C.c_int),
                ("time_level", C.c_int), ("t_final", C.c_double),
                ("mu_star", C.c_double), ("policy", C.c_int),
                ("two_grid", C.c_int)]


class _Cycle(C.Structure):
    _fields_ = [("nu1", C.c_int), ("nu2", C.c_int), ("gamma", C.c_int),
                ("omega_t", C.c_double), ("block_solver", C.c_int),
                ("omega_x", C.c_double), ("nu1_x", C.c_int), ("nu2_x", C.c_int),
                ("gamma_x", C.c_int)]


class _Smoother(C.Structure):
    _fields_ = [("omega_t", C.c_double), ("nu", C.c_int), ("block_solver", C.c_int),
                ("omega_x", C.c_double), ("nu1_x", C.c_int), ("nu2_x", C.c_int),
                ("gamma_x", C.c_int)]


# SmootherConfig defaults (smoother.hpp:15-24): omega_x = 2/3, nu1_x = nu2_x = 2,
# gamma_x = 1.  block_solver: "exact" (0) or "vcycle" (1, spatial_vcycle).
SPATIAL_DEFAULTS = dict(omega_x=2.0 / 3.0, nu1_x=2, nu2_x=2, gamma_x=1)


def _solver_kind(block_solver) -> int:
    if block_solver in (0, "exact"):
        return 0
    if block_solver in (1, "vcycle", "spatial_vcycle"):
        return 1
    raise ValueError("block_solver must be 'exact' or 'vcycle'")


def _cycle(nu1, nu2, gamma, omega_t, block_solver="exact", **sp):
    x = dict(SPATIAL_DEFAULTS, **sp)
    return _Cycle(nu1, nu2, gamma, omega_t, _solver_kind(block_solver), x["omega_x"],
                  x["nu1_x"], x["nu2_x"], x["gamma_x"])


def _smoother(omega_t=0.5, nu=1, block_solver="exact", **sp):
    x = dict(SPATIAL_DEFAULTS, **sp)
    return _Smoother(omega_t, nu, _solver_kind(block_solver), x["omega_x"], x["nu1_x"],
                     x["nu2_x"], x["gamma_x"])


class _LevelInfo(C.Structure):
    _fields_ = [("n_t", C.c_int64), ("n_x", C.c_int64), ("n_loc", C.c_int64),
                ("n1", C.c_int64), ("dim", C.c_int), ("space_level", C.c_int),
                ("coarsen_to_next", C.c_int), ("tau", C.c_double),
                ("h", C.c_double), ("mu", C.c_double)]


def build() -> str:
    """Compile the oracle with its Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_pade.restype = C.c_double
        L.or_critical_mu.restype = C.c_double
        L.or_norm.restype = C.c_double
        L.or_hier_create.argtypes = [C.POINTER(_Params), C.POINTER(C.c_void_p)]
        L.or_hier_destroy.argtypes = [C.c_void_p]
        L.or_hier_levels.argtypes = [C.c_void_p]
        L.or_level_info_get.argtypes = [C.c_void_p, C.c_int, C.POINTER(_LevelInfo)]
        for name in ("or_apply", "or_block_solve", "or_forward_substitution"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_int, P, P]
        L.or_residual.argtypes = [C.c_void_p, C.c_int, P, P, P]
        L.or_norm.argtypes = [C.c_void_p, C.c_int, P]
        L.or_residual_norm.restype = C.c_double
        L.or_residual_norm.argtypes = [C.c_void_p, C.c_int, P, P]
        L.or_smooth.argtypes = [C.c_void_p, C.c_int, P, P, C.c_double, C.c_int]
        L.or_smooth_ex.argtypes = [C.c_void_p, C.c_int, P, P, C.POINTER(_Smoother)]
        L.or_spatial_vcycle.argtypes = [C.c_void_p, C.c_int, P, P, P, C.POINTER(_Smoother)]
        L.or_restrict.argtypes = [C.c_void_p, C.c_int, C.c_int, P, P]
        L.or_prolong.argtypes = [C.c_void_p, C.c_int, C.c_int, P, P]
        L.or_mg_cycle.argtypes = [C.c_void_p, C.c_int, P, P, C.POINTER(_Cycle)]
        L.or_solve.argtypes = [C.c_void_p, P, P, C.POINTER(_Cycle), C.c_double,
                               C.c_int, P, C.c_int, C.POINTER(C.c_int),
                               C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.or_fill_uniform.argtypes = [P, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64]
        L.or_fold_u0.argtypes = [C.c_void_p, P, P]
        L.or_assemble_dg.argtypes = [C.c_int, C.c_double, P, P, P]
        L.or_time_transfer.argtypes = [C.c_int, C.c_double, P, P]
        L.or_pade.argtypes = [C.c_int, C.c_double]
        L.or_critical_mu.argtypes = [C.c_int]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(P)


def assemble_dg(p_t: int, tau: float):
    n = p_t + 1
    K, M, N = (np.zeros((n, n)) for _ in range(3))
    _check(lib().or_assemble_dg(p_t, tau, _ptr(K), _ptr(M), _ptr(N)))
    return K, M, N


def time_transfer(p_t: int, tau: float):
    n = p_t + 1
    R1, R2 = np.zeros((n, n)), np.zeros((n, n))
    _check(lib().or_time_transfer(p_t, tau, _ptr(R1), _ptr(R2)))
    return R1, R2


def pade(p_t: int, z: float) -> float:
    return lib().or_pade(p_t, z)


def critical_mu(p_t: int) -> float:
    return lib().or_critical_mu(p_t)


def fill_uniform(n: int, seed: int = 42, stream: int = 0, offset: int = 0) -> np.ndarray:
    v = np.empty(n)
    lib().or_fill_uniform(_ptr(v), n, seed, stream, offset)
    return v


@dataclass
class LevelInfo:
    n_t: int
    n_x: int
    n_loc: int
    n1: int
    dim: int
    space_level: int
    coarsen_to_next: int
    tau: float
    h: float
    mu: float

    @property
    def size(self) -> int:
        return self.n_t * self.n_x * self.n_loc


class Hierarchy:
    """Oracle hierarchy (mg.cpp:10-94)."""

    def __init__(self, p_t, dim, space_level, time_level, t_final=1.0,
                 mu_star=0.0, policy=0, two_grid=0):
        self._h = C.c_void_p()
        prm = _Params(p_t, dim, space_level, time_level, t_final, mu_star,
                      policy, two_grid)
        _check(lib().or_hier_create(C.byref(prm), C.byref(self._h)))
        self.levels = []
        for i in range(lib().or_hier_levels(self._h)):
            li = _LevelInfo()
            _check(lib().or_level_info_get(self._h, i, C.byref(li)))
            self.levels.append(LevelInfo(li.n_t, li.n_x, li.n_loc, li.n1, li.dim,
                                         li.space_level, li.coarsen_to_next,
                                         li.tau, li.h, li.mu))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None and _lib is not None:
            _lib.or_hier_destroy(self._h)
            self._h = None

    def zeros(self, level=0):
        return np.zeros(self.levels[level].size)

    def apply(self, level, u):
        y = np.zeros_like(u)
        _check(lib().or_apply(self._h, level, _ptr(u), _ptr(y)))
        return y

    def residual(self, level, u, f):
        r = np.zeros_like(u)
        _check(lib().or_residual(self._h, level, _ptr(u), _ptr(f), _ptr(r)))
        return r

    def norm(self, level, v):
        return lib().or_norm(self._h, level, _ptr(v))

    def residual_norm(self, level, u, f):
        """norm(residual(u, f)) without a residual vector (bitwise the same)."""
        return lib().or_residual_norm(self._h, level, _ptr(u), _ptr(f))

    def mg_cycle_inplace(self, level, u, f, nu1=1, nu2=1, gamma=1, omega_t=0.5,
                         block_solver="exact", **sp):
        """mg_cycle on u in place (no copy; full-size fixture generation)."""
        assert u.dtype == np.float64 and u.flags.c_contiguous
        cfg = _cycle(nu1, nu2, gamma, omega_t, block_solver, **sp)
        _check(lib().or_mg_cycle(self._h, level, _ptr(u), _ptr(f), C.byref(cfg)))
        return u

    def block_solve(self, level, b):
        x = np.zeros_like(b)
        _check(lib().or_block_solve(self._h, level, _ptr(b), _ptr(x)))
        return x

    def forward_substitution(self, level, f):
        u = np.zeros_like(f)
        _check(lib().or_forward_substitution(self._h, level, _ptr(f), _ptr(u)))
        return u

    def smooth(self, level, u, f, omega_t=0.5, nu=1):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        _check(lib().or_smooth(self._h, level, _ptr(u), _ptr(f), omega_t, nu))
        return u

    def block_jacobi_step(self, level, u, f, omega_t=0.5, nu=1, block_solver="exact", **sp):
        """block_jacobi_step with a full SmootherConfig (smoother.cpp:96-106)."""
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        sc = _smoother(omega_t, nu, block_solver, **sp)
        _check(lib().or_smooth_ex(self._h, level, _ptr(u), _ptr(f), C.byref(sc)))
        return u

    def spatial_vcycle(self, level, b, x0=None, **sp):
        """SpatialVCycleSolver::cycle on every time step (smoother.cpp:71-78)."""
        x = np.zeros_like(b)
        sc = _smoother(block_solver="vcycle", **sp)
        x0p = _ptr(np.ascontiguousarray(x0, np.float64)) if x0 is not None else None
        _check(lib().or_spatial_vcycle(self._h, level, _ptr(b), x0p, _ptr(x), C.byref(sc)))
        return x

    def coarse_size(self, level, mode=0):
        L = self.levels[level]
        mode = mode or L.coarsen_to_next
        n1 = L.n1 if mode == 1 else (L.n1 - 1) // 2
        return (L.n_t // 2) * L.n_loc * n1 ** L.dim

    def restrict(self, level, fine, mode=0):
        out = np.zeros(self.coarse_size(level, mode))
        _check(lib().or_restrict(self._h, level, mode, _ptr(fine), _ptr(out)))
        return out

    def prolong(self, level, coarse, mode=0):
        out = self.zeros(level)
        _check(lib().or_prolong(self._h, level, mode, _ptr(coarse), _ptr(out)))
        return out

    def mg_cycle(self, level, u, f, nu1=1, nu2=1, gamma=1, omega_t=0.5,
                 block_solver="exact", **sp):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        cfg = _cycle(nu1, nu2, gamma, omega_t, block_solver, **sp)
        _check(lib().or_mg_cycle(self._h, level, _ptr(u), _ptr(f), C.byref(cfg)))
        return u

    def solve(self, f, u=None, nu1=1, nu2=1, gamma=1, omega_t=0.5, eps=1e-8,
              max_iter=250, block_solver="exact", **sp):
        u = self.zeros(0) if u is None else np.ascontiguousarray(u, np.float64).copy()
        cfg = _cycle(nu1, nu2, gamma, omega_t, block_solver, **sp)
        hist = np.zeros(max_iter + 1)
        it, conv, wall = C.c_int(), C.c_int(), C.c_double()
        _check(lib().or_solve(self._h, _ptr(f), _ptr(u), C.byref(cfg), eps, max_iter,
                              _ptr(hist), len(hist), C.byref(it), C.byref(conv),
                              C.byref(wall)))
        return u, dict(iterations=it.value, converged=bool(conv.value),
                       residual_history=hist[: it.value + 1].tolist(),
                       wall_time_seconds=wall.value)

    def fold_u0(self, f, u0):
        _check(lib().or_fold_u0(self._h, _ptr(f), _ptr(u0)))
        return f


def make_inputs(h: Hierarchy, seed: int = 42, random_u0: bool = False):
    """Seeded synthetic f (stream 0) and optional u0 (stream 1) folded into f."""
    L0 = h.levels[0]
    f = fill_uniform(L0.size, seed, 0)
    if random_u0:
        u0 = fill_uniform(L0.n_x, seed, 1)
        h.fold_u0(f, u0)
    return f
