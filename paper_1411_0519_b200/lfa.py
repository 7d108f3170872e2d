"""Local Fourier analysis and the two-grid factor measurement.

Mirror of the reference's ``stmg::lfa`` (lfa.hpp:15-150) and
``stmg::bench::measure_convergence_factor`` (bench.hpp:31-39) over the C ABI:
the symbols and factors are computed by the library's host code
(``csrc/stmg_lfa.cpp``), the measurement runs two-grid cycles on the GPU.
Frequencies are nondimensionalised like the reference (h = 1, tau = mu).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi as A
from .stmg import CycleConfig, check

SEMI, FULL = 1, 2  # Coarsening::semi / full (mg.hpp:12)


def _out(fn, *args) -> float:
    v = C.c_double()
    check(fn(*args, C.byref(v)))
    return v.value


def beta(theta_x: float) -> float:
    """6 (1 - cos)/(2 + cos) (lfa.hpp:15-17)."""
    return _out(A.lib().stmg_lfa_beta, theta_x)


def alpha(p_t: int, mu: float, theta_x: float) -> float:
    """R(-mu beta(theta_x)) (lfa.hpp:19-20)."""
    return _out(A.lib().stmg_lfa_alpha, p_t, mu, theta_x)


def shift(theta: float) -> float:
    """Aliased harmonic gamma(t) = t -/+ pi (lfa.hpp:22-24)."""
    return theta - np.pi if theta > 0.0 else theta + np.pi


def smoother_rho(p_t: int, mu: float, omega_t: float, theta_x: float, theta_t: float):
    """(spectral radius by eigenvalues, closed form) of the block-Jacobi symbol."""
    a, b = C.c_double(), C.c_double()
    check(A.lib().stmg_lfa_smoother_rho(p_t, mu, omega_t, theta_x, theta_t, C.byref(a),
                                        C.byref(b)))
    return a.value, b.value


def _cmat(n: int, fn, *args) -> np.ndarray:
    re, im = np.zeros(n * n), np.zeros(n * n)
    check(fn(*args, re.ctypes.data_as(A.PD), im.ctypes.data_as(A.PD)))
    return (re + 1j * im).reshape(n, n)


def smoother_symbol(p_t: int, mu: float, omega_t: float, theta_x: float,
                    theta_t: float) -> np.ndarray:
    """(1 - w) I + w e^{-i tt} (K + beta M)^{-1} N (lfa.hpp:75-77)."""
    return _cmat(p_t + 1, A.lib().stmg_lfa_smoother_symbol, p_t, mu, omega_t, theta_x, theta_t)


def twogrid_symbol(p_t: int, mu: float, cfg: CycleConfig, mode: int, theta_x: float,
                   theta_t: float) -> np.ndarray:
    """4 N_t x 4 N_t two-grid symbol on the four harmonics (lfa.hpp:93-99)."""
    c = cfg.c()
    return _cmat(4 * (p_t + 1), A.lib().stmg_lfa_twogrid_symbol, p_t, mu, C.byref(c), mode,
                 theta_x, theta_t)


def spectral_radius(m: np.ndarray) -> float:
    m = np.ascontiguousarray(m, dtype=np.complex128)
    re, im = np.ascontiguousarray(m.real), np.ascontiguousarray(m.imag)
    return _out(A.lib().stmg_lfa_spectral_radius, m.shape[0], re.ctypes.data_as(A.PD),
                im.ctypes.data_as(A.PD))


def smoothing_factor(p_t: int, mu: float, omega_t: float, mode: int, n_theta_x: int = 256,
                     n_theta_t: int = 256) -> float:
    """Sup of the smoother symbol radius over the high frequencies (lfa.hpp:125-132)."""
    return _out(A.lib().stmg_lfa_smoothing_factor, p_t, mu, omega_t, mode, n_theta_x, n_theta_t)


def twogrid_factor(p_t: int, mu: float, cfg: CycleConfig, mode: int, n_theta_x: int = 256,
                   n_theta_t: int = 256) -> float:
    """Asymptotic two-grid factor (lfa.hpp:137-141)."""
    c = cfg.c()
    return _out(A.lib().stmg_lfa_twogrid_factor, p_t, mu, C.byref(c), mode, n_theta_x, n_theta_t)


def twogrid_factor_inexact(p_t: int, mu: float, cfg: CycleConfig, mode: int,
                           omega_x: float = 2.0 / 3.0, nu1_x: int = 2, nu2_x: int = 2,
                           n_theta_x: int = 256, n_theta_t: int = 256) -> float:
    """Two-grid factor with one spatial two-grid iteration per block (lfa.hpp:142-145)."""
    c = cfg.c()
    return _out(A.lib().stmg_lfa_twogrid_factor_inexact, p_t, mu, C.byref(c), omega_x, nu1_x,
                nu2_x, mode, n_theta_x, n_theta_t)


@dataclass
class RhoMeasurement:
    measured_rho: float
    predicted_rho: float
    n_iterations_used: int
    seed_used: int


def measure_convergence_factor(p_t: int, dim: int, space_level: int, time_level: int, mu: float,
                               mode: int, cfg: CycleConfig, seed: int = 42,
                               n_theta_x: int = 256, n_theta_t: int = 256,
                               device: int = 0) -> RhoMeasurement:
    """Two-grid cycles on the GPU from a seeded random guess, f = 0
    (bench.cpp:77-145), next to the LFA prediction."""
    pr = A.RhoProblem(p_t, dim, space_level, time_level, mu, mode, device)
    c = cfg.c()
    out = A.RhoMeasurement()
    check(A.lib().stmg_measure_convergence_factor(C.byref(pr), C.byref(c), seed, n_theta_x,
                                                  n_theta_t, C.byref(out)))
    return RhoMeasurement(out.measured_rho, out.predicted_rho, out.n_iterations_used,
                          int(out.seed_used))
