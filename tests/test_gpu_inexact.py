"""GPU parity of the inexact block solver: one spatial V-cycle
per time-step block (SpatialVCycleSolver, smoother.cpp:8-78) behind the
damped block-Jacobi smoother, on both GPU paths, against the CPU oracle
(pinned in tests/test_oracle_inexact.py), through the C ABI.

Tolerances as for the exact variant: operators 1e-12 relative, V-cycle
iterates 1e-10 relative per cycle, identical iteration counts to 1e-8.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_1411_0519_b200 import build
    build.build()
    O.build()
    from paper_1411_0519_b200 import stmg
    return stmg


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


SVC = [  # (p_t, dim, space_level, tau, nu1_x, nu2_x, gamma_x, omega_x)
    (1, 1, 4, 0.05, 2, 2, 1, 2 / 3), (0, 1, 3, 0.01, 1, 2, 2, 0.6), (2, 2, 2, 0.1, 2, 2, 1, 2 / 3),
    (1, 2, 4, 0.003, 2, 1, 2, 2 / 3), (1, 3, 2, 0.2, 2, 2, 1, 2 / 3), (1, 1, 0, 0.3, 2, 2, 1, 2 / 3),
    (3, 2, 3, 0.02, 0, 3, 1, 0.5), (1, 2, 1, 0.1, 2, 2, 3, 2 / 3)]


@pytest.mark.parametrize("case", SVC)
def test_spatial_vcycle_matches_oracle(S, case):
    p, dim, sl, tau, n1, n2, gx, om = case
    g = S.Hierarchy(p, dim, sl, 2, t_final=4 * tau, policy=1, two_grid=1)
    o = O.Hierarchy(p, dim, sl, 2, t_final=4 * tau, policy=1, two_grid=1)
    sp = dict(omega_x=om, nu1_x=n1, nu2_x=n2, gamma_x=gx)
    cfg = S.SmootherConfig(block_solver="vcycle", **sp)
    n = o.levels[0].size
    b = O.fill_uniform(n, 3, 0)
    x0 = O.fill_uniform(n, 4, 0)
    got = g.spatial_vcycle(0, g.upload(b), cfg=cfg).numpy()
    assert rel(got, o.spatial_vcycle(0, b, **sp)) < 1e-12
    got0 = g.spatial_vcycle(0, g.upload(b), x0=g.upload(x0), cfg=cfg).numpy()
    assert rel(got0, o.spatial_vcycle(0, b, x0=x0, **sp)) < 1e-12


def test_spatial_vcycle_exact_data_is_fixed_point(S):
    # test_smoother.cpp:83-98
    g = S.Hierarchy(1, 1, 4, 0, t_final=0.05)
    o = O.Hierarchy(1, 1, 4, 0, t_final=0.05)
    x_star = O.fill_uniform(o.levels[0].size, 5, 0)
    b = o.apply(0, x_star)
    got = g.spatial_vcycle(0, g.upload(b), x0=g.upload(x_star)).numpy()
    assert np.abs(got - x_star).max() <= 1e-12 * np.abs(x_star).max()


def test_spatial_vcycle_contracts_4x_per_cycle(S):
    # test_smoother.cpp:100-126 (level 5, p = 0, mu = 1)
    level = 5
    hh = 2.0 ** -(level + 1)
    g = S.Hierarchy(0, 1, level, 0, t_final=hh * hh)
    o = O.Hierarchy(0, 1, level, 0, t_final=hh * hh)
    x_star = O.fill_uniform(o.levels[0].size, 7, 0)
    b = g.upload(o.apply(0, x_star))
    x = g.vector(0)
    err = np.linalg.norm(x.numpy() - x_star)
    for _ in range(4):
        x = g.spatial_vcycle(0, b, x0=x)
        e = np.linalg.norm(x.numpy() - x_star)
        assert e <= 0.25 * err
        err = e


CASES = [  # (p_t, dim, space_level, time_level, T, policy)
    (0, 1, 3, 3, 1.0, 0), (1, 1, 5, 6, 1.0, 0), (2, 1, 4, 4, 0.5, 0), (1, 2, 3, 4, 1.0, 0),
    (2, 2, 3, 3, 0.25, 0), (1, 3, 2, 3, 1.0, 0), (1, 2, 3, 3, 1.0, 1), (3, 2, 2, 3, 1.0, 2)]


@pytest.mark.parametrize("case", CASES)
def test_inexact_smoother_matches_oracle(S, case):
    p, dim, sl, tl, T, pol = case
    g = S.Hierarchy(p, dim, sl, tl, t_final=T, policy=pol)
    o = O.Hierarchy(p, dim, sl, tl, t_final=T, policy=pol)
    cfg = S.SmootherConfig(omega_t=0.5, nu=2, block_solver="vcycle")
    for lev in range(len(o.levels)):
        n = o.levels[lev].size
        u = O.fill_uniform(n, 100 + lev, 0)
        f = O.fill_uniform(n, 200 + lev, 0)
        got = g.block_jacobi_step(lev, g.upload(u, lev), g.upload(f, lev), cfg=cfg).numpy()
        ref = o.block_jacobi_step(lev, u, f, 0.5, 2, block_solver="vcycle")
        assert rel(got, ref) < 1e-11, lev


@pytest.mark.parametrize("path", ["spectral", "physical"])
@pytest.mark.parametrize("case", CASES)
def test_inexact_vcycles_match_oracle(S, case, path):
    p, dim, sl, tl, T, pol = case
    g = S.Hierarchy(p, dim, sl, tl, t_final=T, policy=pol)
    o = O.Hierarchy(p, dim, sl, tl, t_final=T, policy=pol)
    f = O.make_inputs(o, 42)
    df = g.upload(f)
    cfg = S.CycleConfig(nu1=1, nu2=1, path=path, block_solver="vcycle")
    u_o = o.zeros(0)
    du = g.vector(0)
    for _ in range(3):
        u_o = o.mg_cycle(0, u_o, f, block_solver="vcycle")
        g.mg_cycle(0, du, df, cfg)
        assert rel(du.numpy(), u_o) < 1e-10


def test_inexact_general_cycle_shapes(S):
    """V(2,1) and W(1,2) cycles with gamma_x = 2, nu_x = (1, 3), omega_x = 0.6."""
    g = S.Hierarchy(1, 2, 3, 4)
    o = O.Hierarchy(1, 2, 3, 4)
    f = O.make_inputs(o, 5)
    sp = dict(omega_x=0.6, nu1_x=1, nu2_x=3, gamma_x=2)
    for nu1, nu2, gam in ((2, 1, 1), (1, 2, 2)):
        cfg = S.CycleConfig(nu1=nu1, nu2=nu2, gamma=gam, block_solver="vcycle", **sp)
        du = g.vector(0)
        u_o = o.zeros(0)
        for _ in range(2):
            u_o = o.mg_cycle(0, u_o, f, nu1, nu2, gam, block_solver="vcycle", **sp)
            g.mg_cycle(0, du, g.upload(f), cfg)
            assert rel(du.numpy(), u_o) < 1e-10


@pytest.mark.parametrize("case,random_u0", [((1, 1, 5, 6, 1.0, 0), False),
                                            ((1, 2, 5, 6, 1.0, 0), True),
                                            ((2, 2, 4, 5, 1.0, 0), False),
                                            ((1, 3, 3, 4, 1.0, 0), False)])
def test_inexact_solve_matches_oracle(S, case, random_u0):
    """Full solves to 1e-8: identical iteration count, history and iterate to 1e-10."""
    p, dim, sl, tl, T, pol = case
    g = S.Hierarchy(p, dim, sl, tl, t_final=T, policy=pol)
    o = O.Hierarchy(p, dim, sl, tl, t_final=T, policy=pol)
    f = O.make_inputs(o, 42, random_u0=random_u0)
    u_o, rep_o = o.solve(f, eps=1e-8, block_solver="vcycle")
    for path in ("spectral", "physical"):
        du = g.vector(0)
        cfg = S.CycleConfig(nu1=1, nu2=1, path=path, block_solver="vcycle")
        rep = g.solve(g.upload(f), du, cfg, 1e-8)
        assert rep.iterations == rep_o["iterations"], (path, rep.iterations, rep_o["iterations"])
        h, ho = np.array(rep.residual_history), np.array(rep_o["residual_history"])
        assert np.abs(h - ho).max() <= 1e-10 * ho[0]
        assert rel(du.numpy(), u_o) < 1e-10


def test_inexact_c2_full_size(S):
    """configs[1] (C2) with inexact blocks: 2 cycles vs the oracle, then the full
    solve converges in the physical residual."""
    g = S.Hierarchy(1, 2, 6, 8)
    o = O.Hierarchy(1, 2, 6, 8)
    f = O.make_inputs(o, 42, random_u0=True)
    df = g.upload(f)
    cfg = S.CycleConfig(nu1=1, nu2=1, block_solver="vcycle")
    du = g.vector(0)
    u_o = o.zeros(0)
    for _ in range(2):
        u_o = o.mg_cycle(0, u_o, f, block_solver="vcycle")
        g.mg_cycle(0, du, df, cfg)
        assert rel(du.numpy(), u_o) < 1e-10
    du = g.vector(0)
    rep = g.solve(df, du, cfg, 1e-8)
    assert rep.converged
    r = g.residual(0, du, df)
    assert g.norm(0, r) <= 1e-8 * rep.residual_history[0] * (1 + 1e-6)


def test_inexact_rejected_on_shards(S):
    g = S.Hierarchy(1, 2, 3, 4, shards=2)
    cfg = S.CycleConfig(nu1=1, nu2=1, block_solver="vcycle")
    with pytest.raises(ValueError):
        g.solve(g.vector(0), g.vector(0), cfg, 1e-8)


def test_bad_spatial_config_rejected(S):
    g = S.Hierarchy(1, 1, 3, 3)
    with pytest.raises(ValueError):
        g.solve(g.vector(0), g.vector(0), S.CycleConfig(block_solver="vcycle", gamma_x=0), 1e-8)
    with pytest.raises(ValueError):
        S.CycleConfig(block_solver="lu").c()
