"""Pins the oracle's inexact block solver (SpatialVCycleSolver, smoother.cpp:8-92)
against the reference's own tests for it (test_smoother.cpp:83-142) and the
independent dense numpy restatement (oracle/dense.py).  CPU only."""
import numpy as np
import pytest

from oracle import dense


def _single_step(oracle, p, tau, dim, level):
    """A context whose level 0 is one time step of size tau (so or_apply = A x)."""
    return oracle.Hierarchy(p, dim, level, 0, t_final=tau)


def test_spatial_vcycle_exact_data_is_fixed_point(oracle):
    # test_smoother.cpp:83-98: dg(p=1, tau=0.05), dim 1, level 4, x0 = x*
    h = _single_step(oracle, 1, 0.05, 1, 4)
    x_star = oracle.fill_uniform(h.levels[0].size, 5, 0)
    b = h.apply(0, x_star)
    got = h.spatial_vcycle(0, b, x0=x_star)
    assert np.abs(got - x_star).max() <= 1e-12 * np.abs(x_star).max()


def test_spatial_vcycle_contracts_4x_per_cycle(oracle):
    # test_smoother.cpp:100-126: level 5, p = 0, tau = h^2 (mu = 1), defaults
    level = 5
    hh = 2.0 ** -(level + 1)
    h = _single_step(oracle, 0, hh * hh, 1, level)
    x_star = oracle.fill_uniform(h.levels[0].size, 7, 0)
    b = h.apply(0, x_star)
    x = np.zeros_like(b)
    err = np.linalg.norm(x - x_star)
    for _ in range(4):
        x = h.spatial_vcycle(0, b, x0=x)
        e = np.linalg.norm(x - x_star)
        assert e <= 0.25 * err
        err = e


def test_vcycle_smoother_keeps_exact_solution_fixed(oracle):
    # test_smoother.cpp:128-142: Setting(1, 0.02, 1, 4, 4)
    h = oracle.Hierarchy(1, 1, 4, 2, t_final=0.08, policy=1, two_grid=1)
    f = oracle.fill_uniform(h.levels[0].size, 31, 0)
    exact = h.forward_substitution(0, f)
    u = h.block_jacobi_step(0, exact, f, 0.5, 1, block_solver="vcycle")
    assert np.abs(u - exact).max() <= 1e-11 * np.abs(exact).max()


@pytest.mark.parametrize("p,dim,level,tau,nu1,nu2,gamma,omega", [
    (1, 1, 4, 0.05, 2, 2, 1, 2 / 3), (0, 1, 3, 0.01, 1, 2, 2, 0.6), (2, 2, 2, 0.1, 2, 2, 1, 2 / 3),
    (1, 2, 3, 0.003, 2, 1, 2, 2 / 3), (1, 3, 1, 0.2, 2, 2, 1, 2 / 3), (1, 1, 0, 0.3, 2, 2, 1, 2 / 3)])
def test_spatial_vcycle_matches_dense(oracle, p, dim, level, tau, nu1, nu2, gamma, omega):
    h = _single_step(oracle, p, tau, dim, level)
    b = oracle.fill_uniform(h.levels[0].size, 11, 0)
    x0 = oracle.fill_uniform(h.levels[0].size, 12, 0)
    sp = dict(omega_x=omega, nu1_x=nu1, nu2_x=nu2, gamma_x=gamma)
    for guess in (None, x0):
        got = h.spatial_vcycle(0, b, x0=guess, **sp)
        ref = dense.spatial_vcycle(p, tau, dim, level, b, guess, **sp)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("p,dim,sl,tl,T", [(1, 1, 3, 4, 0.05), (1, 2, 2, 3, 1.0),
                                            (2, 1, 3, 3, 0.3), (1, 3, 1, 2, 0.5)])
def test_inexact_vcycle_matches_dense_oracle(oracle, p, dim, sl, tl, T):
    """Two space-time V-cycles with spatial-V-cycle block solves equal the dense oracle."""
    mu_star = oracle.critical_mu(p)
    h = oracle.Hierarchy(p, dim, sl, tl, t_final=T)
    d = dense.DenseHierarchy(p, dim, sl, tl, t_final=T, mu_star=mu_star, block_solver="vcycle")
    f = oracle.fill_uniform(h.levels[0].size, 9, 0)
    u = np.zeros_like(f)
    ud = np.zeros_like(f)
    for _ in range(2):
        u = h.mg_cycle(0, u, f, block_solver="vcycle")
        ud = d.cycle(0, ud, f)
        assert np.abs(u - ud).max() <= 1e-11 * np.abs(ud).max()


def test_inexact_solve_converges_c1(oracle):
    """configs[0] with the paper's inexact variant converges to 1e-8 (Table 1 setting)."""
    h = oracle.Hierarchy(1, 1, 5, 6, t_final=1.0)
    f = oracle.make_inputs(h, 42)
    u, rep = h.solve(f, eps=1e-8, block_solver="vcycle")
    ue, repe = h.solve(f, eps=1e-8)
    assert rep["converged"]
    assert rep["iterations"] <= repe["iterations"] + 10
    assert np.abs(u - ue).max() <= 1e-6 * np.abs(ue).max()
