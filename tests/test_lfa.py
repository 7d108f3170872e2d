"""Local Fourier analysis engine, host code of the library.

Mirrors the behaviours the reference's tests pin for lfa.cpp
(test_lfa.cpp:17-230): symbol values and ranges, closed form vs eigenvalues,
the smoothing factors of the paper, mu*, two-grid factor bounds, the
theta_x = 0 rejection, and the inexact-solver factors.  An independent numpy
restatement of the symbols cross-checks the two-grid symbol entry by entry.
CPU only (no GPU call).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

PI = math.pi


@pytest.fixture(scope="module")
def L():
    from paper_1411_0519_b200 import build
    build.build()
    from paper_1411_0519_b200 import lfa
    return lfa


@pytest.fixture(scope="module")
def S():
    from paper_1411_0519_b200 import stmg
    return stmg


def test_beta_values_and_range(L):  # test_lfa.cpp:17-27
    assert L.beta(0.0) == 0.0
    assert abs(L.beta(PI / 2) - 3.0) < 1e-14 * 3
    assert abs(L.beta(PI) - 12.0) < 1e-14 * 12
    for i in range(101):
        b = L.beta(-PI + 2 * PI * i / 100)
        assert -1e-14 <= b <= 12 + 1e-12


def test_alpha_is_pade_of_minus_mu_beta(L):  # test_lfa.cpp:29-42
    for p in (0, 1, 2, 3):
        for mu in (1e-3, 0.3, 1.0, 1e3):
            for i in range(33):
                tx = PI * i / 32
                a = L.alpha(p, mu, tx)
                assert abs(a) <= 1 + 1e-12
                want = O.pade(p, -mu * L.beta(tx))
                assert abs(a - want) <= 1e-14 * max(1.0, abs(want))
            assert abs(L.alpha(p, mu, 0.0) - 1.0) < 1e-14


def test_smoother_symbol_p0_closed_form(L):  # test_lfa.cpp:44-55
    mu, om = 0.8, 0.5
    for tx in (0.3, 1.2, 2.9):
        for tt in (0.0, 0.7, PI):
            got = L.smoother_symbol(0, mu, om, tx, tt)[0, 0]
            want = (1 - om) + om * np.exp(-1j * tt) / (1 + mu * L.beta(tx))
            assert abs(got - want) < 1e-13


def test_smoother_radius_one_at_theta_x_zero(L):  # test_lfa.cpp:57-64
    for p in (0, 1, 3):
        rho, _ = L.smoother_rho(p, 2.5, 1.0, 0.0, 1.1)
        assert abs(rho - 1.0) < 1e-12


def test_closed_form_equals_eigenvalues(L):  # test_lfa.cpp:66-80
    rng = np.random.default_rng(2024)
    for _ in range(300):
        p = int(rng.integers(0, 4))
        mu = 10 ** (-4 + 8 * rng.random())
        om = 0.05 + 0.95 * rng.random()
        tx, tt = -PI + 2 * PI * rng.random(), -PI + 2 * PI * rng.random()
        via_eig, closed = L.smoother_rho(p, mu, om, tx, tt)
        assert abs(via_eig - closed) < 1e-10


def test_spectral_radius_vs_numpy(L):
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 4, 8, 12, 16):
        for _ in range(20):
            m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
            assert abs(L.spectral_radius(m) - np.abs(np.linalg.eigvals(m)).max()) < 1e-10 * n
    # defective / non-normal: Jordan-like block and a nilpotent shift
    j = np.eye(6) * 0.3 + np.diag(np.ones(5), 1)
    assert abs(L.spectral_radius(j) - 0.3) < 1e-2
    assert L.spectral_radius(np.diag(np.ones(5), 1)) < 1e-2


def test_smoothing_factors(L):  # test_lfa.cpp:82-124
    s2 = 1 / math.sqrt(2)
    for p in (0, 2):
        for mu in (1e-3, 1.0, 1e3):
            assert abs(L.smoothing_factor(p, mu, 0.5, L.SEMI, 128, 128) - s2) < 2e-3
            want = 0.5 * (1 + O.pade(p, -3 * mu))
            assert abs(L.smoothing_factor(p, mu, 0.5, L.FULL, 128, 128) - want) < 2e-3
    for p in (1, 3):
        for mu in (1e-2, 1.0, 1e2):
            assert L.smoothing_factor(p, mu, 0.5, L.SEMI, 128, 128) <= s2 + 1e-12
    for p in (0, 1, 2):
        ms = O.critical_mu(p)
        assert abs(L.smoothing_factor(p, ms, 0.5, L.FULL, 128, 128) - s2) < 2e-3


def test_twogrid_factor_bounds(L, S):  # test_lfa.cpp:172-194
    cfg = S.CycleConfig(nu1=1, nu2=1)
    rho = L.twogrid_factor(0, 1.0, cfg, L.SEMI, 64, 64)
    assert 0.05 < rho <= 0.5 + 1e-3
    for mu in (1e-4, 1e2):
        assert L.twogrid_factor(1, mu, cfg, L.SEMI, 64, 64) <= 0.5 + 1e-3
    ms0 = O.critical_mu(0)
    assert L.twogrid_factor(0, 2 * ms0, cfg, L.FULL, 64, 64) <= 0.5 + 1e-3
    assert L.twogrid_factor(0, 1e-3, cfg, L.FULL, 64, 64) > 0.6


def test_twogrid_rejects_theta_x_zero(L, S):  # test_lfa.cpp:196-201
    with pytest.raises(ValueError):
        L.twogrid_symbol(0, 1.0, S.CycleConfig(), L.SEMI, 0.0, 0.3)


def test_semi_factor_decreases_with_mu(L, S):  # test_lfa.cpp:203-217
    cfg = S.CycleConfig(nu1=1, nu2=1)
    r_small = L.twogrid_factor(0, 1e-2, cfg, L.SEMI, 64, 64)
    r_mid = L.twogrid_factor(0, 1.0, cfg, L.SEMI, 64, 64)
    r_large = L.twogrid_factor(0, 1e4, cfg, L.SEMI, 64, 64)
    assert r_large < r_mid and r_large < r_small
    assert abs(r_large - 0.25) < 1e-3 * 0.25  # (1 - omega)^(nu1 + nu2)


def test_inexact_factors(L, S):  # test_lfa.cpp:219-236
    cfg = S.CycleConfig(nu1=1, nu2=1)
    for p in (0, 1):
        for mu in (1e-3, 1e-1, 1.0, 1e2):
            assert L.twogrid_factor_inexact(p, mu, cfg, L.SEMI, n_theta_x=64, n_theta_t=64) \
                <= 0.5 + 1e-3
        ms = O.critical_mu(p)
        for mu in (ms, 2 * ms, 50 * ms):
            ex = L.twogrid_factor(p, mu, cfg, L.FULL, 64, 64)
            inex = L.twogrid_factor_inexact(p, mu, cfg, L.FULL, n_theta_x=64, n_theta_t=64)
            assert abs(ex - inex) <= 0.05


# ---- independent numpy restatement of the two-grid symbol (lfa.cpp:12-200) --
def _np_twogrid(p, mu, om, nu1, nu2, mode, tx, tt):
    n = p + 1
    K, M, N = O.assemble_dg(p, mu)
    Kc, Mc, Nc = O.assemble_dg(p, 2 * mu)
    R1, R2 = O.time_transfer(p, mu)

    def beta(t):
        return 6 * (1 - math.cos(t)) / (2 + math.cos(t))

    def ph(t):
        return np.exp(-1j * t)

    def op(k, m, nn, h, x, t):
        return h / 3 * (2 + math.cos(x)) * (k + beta(x) / h ** 2 * m - ph(t) * nn)

    def sm(x, t):
        return (1 - om) * np.eye(n) + om * ph(t) * np.linalg.solve(K + beta(x) * M, N)

    def g(t):
        return t - PI if t > 0 else t + PI

    hx, ht = (tx, g(tx)), (tt, g(tt))
    opb = np.zeros((4 * n, 4 * n), complex)
    S1 = np.zeros_like(opb)
    S2 = np.zeros_like(opb)
    for j in range(4):
        sl = slice(j * n, (j + 1) * n)
        opb[sl, sl] = op(K, M, N, 1.0, hx[j % 2], ht[j // 2])
        s = sm(hx[j % 2], ht[j // 2])
        S1[sl, sl] = np.linalg.matrix_power(s, nu1)
        S2[sl, sl] = np.linalg.matrix_power(s, nu2)
    rt = lambda t: ph(t) * R1 + R2  # noqa: E731
    pt = lambda t: 0.5 * (ph(-t) * R1.T + R2.T)  # noqa: E731
    r0, rg, p0, pg = rt(tt), rt(g(tt)), pt(tt), pt(g(tt))
    if mode == 1:
        R = np.zeros((2 * n, 4 * n), complex)
        P = np.zeros((4 * n, 2 * n), complex)
        Cm = np.zeros((2 * n, 2 * n), complex)
        R[:n, :n], R[:n, 2 * n:3 * n], R[n:, n:2 * n], R[n:, 3 * n:] = r0, rg, r0, rg
        P[:n, :n], P[n:2 * n, n:], P[2 * n:3 * n, :n], P[3 * n:, n:] = p0, p0, pg, pg
        Cm[:n, :n] = op(Kc, Mc, Nc, 1.0, tx, 2 * tt)
        Cm[n:, n:] = op(Kc, Mc, Nc, 1.0, g(tx), 2 * tt)
    else:
        sx, sg = 1 + math.cos(tx), 1 + math.cos(g(tx))
        R = np.hstack([sx * r0, sg * r0, sx * rg, sg * rg])
        P = 0.5 * np.vstack([sx * p0, sg * p0, sx * pg, sg * pg])
        Cm = op(Kc, Mc, Nc, 2.0, 2 * tx, 2 * tt)
    cgc = np.eye(4 * n) - P @ np.linalg.solve(Cm, R @ opb)
    return S2 @ cgc @ S1


@pytest.mark.parametrize("p", [0, 1, 2])
@pytest.mark.parametrize("mode", [1, 2])
def test_twogrid_symbol_vs_numpy(L, S, p, mode):
    rng = np.random.default_rng(11 + p + 10 * mode)
    for _ in range(6):
        mu = 10 ** (-2 + 3 * rng.random())
        tx, tt = 0.05 + 1.5 * rng.random(), -PI + 2 * PI * rng.random()
        cfg = S.CycleConfig(nu1=1, nu2=2, omega_t=0.6)
        got = L.twogrid_symbol(p, mu, cfg, mode, tx, tt)
        want = _np_twogrid(p, mu, 0.6, 1, 2, mode, tx, tt)
        assert np.abs(got - want).max() < 1e-11 * max(1.0, np.abs(want).max())
        assert abs(L.spectral_radius(got) - np.abs(np.linalg.eigvals(want)).max()) < 1e-9


def test_lfa_bad_arguments(L, S):
    with pytest.raises(ValueError):
        L.smoothing_factor(1, -1.0, 0.5, L.SEMI)
    with pytest.raises(ValueError):
        L.smoothing_factor(1, 1.0, 0.5, 0)
    with pytest.raises(ValueError):
        L.twogrid_factor(1, 1.0, S.CycleConfig(), 3)
