"""Pins the CPU oracle against the reference's known-answer tests, scipy's
sparse LU (the reference's Eigen SparseLU boundary) and the independent dense
numpy oracle.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import dense

HERE = os.path.dirname(os.path.abspath(__file__))
KATS = json.load(open(os.path.join(HERE, "golden", "kats.json")))


def test_dg_blocks_match_reference_kats(oracle):
    k = KATS["dg_p0"]
    K, M, N = oracle.assemble_dg(0, k["tau"])
    assert abs(K[0, 0] - 1.0) < 1e-14 and abs(M[0, 0] - k["tau"]) < 1e-14 and abs(N[0, 0] - 1.0) < 1e-14
    k = KATS["dg_p1"]
    K, M, N = oracle.assemble_dg(1, k["tau"])
    assert np.abs(K - np.array(k["K"])).max() < 1e-14
    assert np.abs(N - np.array(k["N"])).max() < 1e-14
    assert abs(M[0, 0] - k["M_diag"][0]) < 1e-14 * k["tau"] * 10
    assert abs(M[1, 1] - k["M_diag"][1]) < 1e-14
    assert abs(M[0, 1]) < 1e-15
    k = KATS["dg_p2"]
    K, M, N = oracle.assemble_dg(2, k["tau"])
    assert np.abs(K - np.array(k["K"])).max() < 1e-13
    assert abs(M[2, 2] - k["M22"]) < 1e-13


@pytest.mark.parametrize("p,tau", [tuple(c) for c in KATS["dg_bad_args"]["cases"]])
def test_dg_rejects_bad_arguments(oracle, p, tau):
    with pytest.raises(ValueError):
        oracle.assemble_dg(p, tau)


def test_dg_blocks_match_dense_numpy(oracle):
    for p in range(0, 6):
        K, M, N = oracle.assemble_dg(p, 0.3)
        Kd, Md, Nd = dense.dg_block(p, 0.3)
        assert np.abs(K - Kd).max() < 1e-12
        assert np.abs(M - Md).max() < 1e-13
        assert np.abs(N - Nd).max() < 1e-13


def test_pade_closed_forms(oracle):
    z = -1.3
    assert abs(oracle.pade(0, z) - 1.0 / (1.0 - z)) < 1e-14
    r1 = (1 + z / 3) / (1 - 2 * z / 3 + z * z / 6)
    assert abs(oracle.pade(1, z) - r1) < 1e-14
    assert abs(oracle.pade(1, -3.0)) < 1e-15
    for p in range(11):
        assert abs(oracle.pade(p, 0.0) - 1.0) < 1e-15


def test_time_transfer_kats(oracle):
    R1, R2 = oracle.time_transfer(0, 0.4)
    assert abs(R1[0, 0] - 1) < 1e-14 and abs(R2[0, 0] - 1) < 1e-14
    k = KATS["transfer_p1"]
    R1, R2 = oracle.time_transfer(1, 1.0)
    assert np.abs(R1.T - np.array(k["R1T"])).max() < 1e-13
    assert np.abs(R2.T - np.array(k["R2T"])).max() < 1e-13
    k = KATS["transfer_p2"]
    R1, _ = oracle.time_transfer(2, 0.25)
    assert np.abs(R1.T - np.array(k["R1T"])).max() < 1e-12
    for p in range(5):
        a1, a2 = oracle.time_transfer(p, 0.6)
        d1, d2 = dense.time_transfer(p, 0.6)
        assert np.abs(a1 - d1).max() < 1e-12 and np.abs(a2 - d2).max() < 1e-12


def test_prolongation_reproduces_coarse_polynomials(oracle):
    # test_transfer.cpp:47-66
    tau = 0.6
    for p in range(6):
        R1, R2 = oracle.time_transfer(p, tau)
        for mode in range(p + 1):
            c = np.zeros(p + 1)
            c[mode] = 1.0
            f1, f2 = R1.T @ c, R2.T @ c
            for s in (0.05 * tau, 0.33 * tau, 0.92 * tau):
                w1 = dense.leg(mode, 2 * s / (2 * tau) - 1)
                w2 = dense.leg(mode, 2 * (s + tau) / (2 * tau) - 1)
                e1 = sum(f1[l] * dense.leg(l, 2 * s / tau - 1) for l in range(p + 1))
                e2 = sum(f2[l] * dense.leg(l, 2 * s / tau - 1) for l in range(p + 1))
                assert abs(e1 - w1) <= 1e-12 * max(1, abs(w1))
                assert abs(e2 - w2) <= 1e-12 * max(1, abs(w2))


def test_critical_mu_kats(oracle):
    for p, v in KATS["critical_mu"]["values"].items():
        assert abs(oracle.critical_mu(int(p)) - v) < 1e-8
    assert abs(oracle.critical_mu(0) - math.sqrt(2) / 3) < 1e-10
    for p in range(11):
        mu = oracle.critical_mu(p)
        assert abs(oracle.pade(p, -3 * mu) - (math.sqrt(2) - 1)) < 1e-10


def test_hand_example_1x1(oracle):
    k = KATS["hand_1x1"]
    h = oracle.Hierarchy(0, 1, 0, 1, t_final=2.0, policy=1, two_grid=1)
    # level 0: p_t=0, tau=1, h=1/2, n_t=2 -> A = 13/3, B = -1/3
    y = h.apply(0, np.array(k["u"]))
    assert np.allclose(y, k["Lu"], rtol=1e-14, atol=0)
    sol = h.forward_substitution(0, np.array(k["f"]))
    assert np.allclose(sol, k["sol"], rtol=1e-13, atol=0)


def test_restrict_semi_p0_pair(oracle):
    h = oracle.Hierarchy(0, 1, 0, 1, t_final=1.0, policy=1)
    c = h.restrict(0, np.array([3.0, 5.0]))
    assert c[0] == 8.0


def test_space_restriction_unit_weights(oracle):
    # test_transfer.cpp:157-174 via a p_t=0 full step (R1 = R2 = 1)
    h = oracle.Hierarchy(0, 1, 3, 1, policy=2)
    assert h.levels[0].coarsen_to_next == 2
    for node, want in KATS["restrict_space_unit"]["cases"]:
        u = np.zeros(h.levels[0].size)
        u[node] = 1.0  # step 0 only
        c = h.restrict(0, u)
        expect = np.zeros(7)
        for j, v in want.items():
            expect[int(j)] = v
        assert np.array_equal(c, expect)


@pytest.mark.parametrize("dim,level", [(1, 2), (2, 1), (2, 2), (3, 1)])
def test_apply_matches_dense_kronecker(oracle, dim, level):
    p, tau, n_t = 1, 0.3, 4
    h = oracle.Hierarchy(p, dim, level, 2, t_final=tau * n_t, policy=1)
    u = oracle.fill_uniform(h.levels[0].size, 7, 0)
    K, M, N = dense.dg_block(p, tau)
    Mh, Kh = dense.space_mats(dim, level)
    L = dense.dense_space_time(K, M, N, Mh, Kh, n_t)
    want = L @ u
    got = h.apply(0, u)
    assert np.abs(got - want).max() < 1e-12 * np.abs(want).max()
    f = oracle.fill_uniform(u.size, 3, 0)
    r = h.residual(0, u, f)
    assert np.abs(r - (f - want)).max() < 1e-12 * np.abs(f).max() * 10


def _sparse_block(p, tau, dim, level):
    K, M, _ = dense.dg_block(p, tau)
    Mh, Kh = dense.space_mats(dim, level)
    return sp.csc_matrix(np.kron(K, Mh) + np.kron(M, Kh))


@pytest.mark.parametrize("p,dim,level", [(0, 1, 3), (1, 1, 4), (2, 2, 2), (1, 2, 3), (1, 3, 1), (3, 2, 1)])
def test_block_solve_matches_sparse_lu(oracle, p, dim, level):
    """The exact DST block solve equals SparseLU (st_system.cpp:103-116)."""
    n_t = 4
    tau = 0.05
    h = oracle.Hierarchy(p, dim, level, 2, t_final=tau * n_t, policy=1)
    b = oracle.fill_uniform(h.levels[0].size, 11, 0)
    x = h.block_solve(0, b)
    lu = spla.splu(_sparse_block(p, tau, dim, level))
    slab = h.levels[0].n_x * (p + 1)
    for n in range(n_t):
        want = lu.solve(b[n * slab:(n + 1) * slab])
        assert np.abs(x[n * slab:(n + 1) * slab] - want).max() < 1e-12 * np.abs(want).max()


def test_forward_substitution_residual_contract(oracle):
    # test_st_system.cpp:121-135
    h = oracle.Hierarchy(2, 1, 4, 3, t_final=1.0, policy=1, two_grid=1)
    f = oracle.fill_uniform(h.levels[0].size, 5, 0)
    assert np.all(h.forward_substitution(0, np.zeros_like(f)) == 0.0)
    u = h.forward_substitution(0, f)
    r = h.residual(0, u, f)
    assert h.norm(0, r) <= 1e-12 * h.norm(0, f)


def test_smoother_fixed_point_and_single_step(oracle):
    # test_smoother.cpp:32-62
    h = oracle.Hierarchy(1, 1, 3, 2, t_final=0.4, policy=1, two_grid=1)
    f = oracle.fill_uniform(h.levels[0].size, 17, 0)
    exact = h.forward_substitution(0, f)
    for om in (0.3, 0.5, 1.0):
        u = h.smooth(0, exact, f, om, 2)
        assert np.abs(u - exact).max() <= 1e-12 * np.abs(exact).max()
    h1 = oracle.Hierarchy(2, 1, 3, 0, t_final=0.4)
    f1 = oracle.fill_uniform(h1.levels[0].size, 23, 0)
    ex1 = h1.forward_substitution(0, f1)
    u1 = h1.smooth(0, np.zeros_like(f1), f1, 1.0, 1)
    assert np.abs(u1 - ex1).max() <= 1e-11 * np.abs(ex1).max()


@pytest.mark.parametrize("dim,level,mode", [(1, 2, 1), (1, 2, 2), (2, 2, 2), (2, 1, 1), (3, 2, 2)])
def test_transfers_are_adjoint(oracle, dim, level, mode):
    # test_transfer.cpp:113-145 (+3D)
    h = oracle.Hierarchy(1, dim, level, 3, t_final=1.6, policy=mode)
    u = oracle.fill_uniform(h.levels[0].size, 101, 0)
    w = oracle.fill_uniform(h.coarse_size(0, mode), 103, 0)
    ru = h.restrict(0, u, mode)
    pw = h.prolong(0, w, mode)
    assert abs(ru @ w - u @ pw) <= 1e-12 * abs(u @ pw)


@pytest.mark.parametrize("p,dim,sl,tl,T", [(1, 1, 2, 3, 1.0), (1, 1, 3, 4, 0.05), (2, 2, 1, 3, 1.0),
                                            (0, 2, 2, 3, 0.1), (1, 3, 1, 2, 0.5)])
def test_vcycle_matches_dense_oracle(oracle, p, dim, sl, tl, T):
    """Two V-cycles of the C++ oracle equal the dense numpy oracle."""
    mu_star = oracle.critical_mu(p)
    h = oracle.Hierarchy(p, dim, sl, tl, t_final=T)
    d = dense.DenseHierarchy(p, dim, sl, tl, t_final=T, mu_star=mu_star)
    assert [L.coarsen_to_next for L in h.levels] == [L["coarsen"] for L in d.levels]
    f = oracle.fill_uniform(h.levels[0].size, 9, 0)
    u = np.zeros_like(f)
    ud = np.zeros_like(f)
    for _ in range(2):
        u = h.mg_cycle(0, u, f)
        ud = d.cycle(0, ud, f)
        assert np.abs(u - ud).max() <= 1e-11 * np.abs(ud).max()


def test_c1_solve_converges_and_matches_forward_substitution(oracle):
    # solve at eps=1e-10 vs forward substitution <= 1e-6
    h = oracle.Hierarchy(1, 1, 5, 6, t_final=1.0)
    assert [L.coarsen_to_next for L in h.levels] == [2, 2, 2, 2, 2, 1, 0]
    f = oracle.make_inputs(h, 42)
    u, rep = h.solve(f, eps=1e-10)
    assert rep["converged"] and rep["iterations"] <= 20
    h2 = oracle.Hierarchy(1, 1, 5, 6, t_final=1.0, policy=1, two_grid=1)
    ref = h2.forward_substitution(0, f)
    assert np.abs(u - ref).max() <= 1e-6 * np.abs(ref).max()
    u8, rep8 = h.solve(f, eps=1e-8)
    assert rep8["residual_history"][-1] <= 1e-8 * rep8["residual_history"][0]


def test_hierarchy_patterns_match_survey(oracle):
    """level ladders of the BASELINE configs (setup only)."""
    pats = {
        (1, 1, 5, 6, 1.0): "FFFFFS",
        (1, 2, 6, 8, 1.0): "FFFFFFSS",
        (2, 2, 7, 12, 1.0): "FFFFFFSFSSSS",
        (1, 3, 5, 10, 1.0): "FFFFSFSSSS",
        (1, 2, 8, 11, 1.0): "FFFFFFFFSSS",
    }
    import ctypes  # noqa: F401  (hierarchy setup allocates nothing large)
    for (p, dim, sl, tl, T), pat in pats.items():
        h = oracle.Hierarchy(p, dim, sl, tl, t_final=T)
        got = "".join("SF"[L.coarsen_to_next - 1] for L in h.levels[:-1])
        assert got == pat, (p, dim, sl, tl, got)
        assert h.levels[-1].n_t == 1 and h.levels[-1].n_x == 1


def test_generator_is_counter_based(oracle):
    a = oracle.fill_uniform(1000, 42, 0)
    b = oracle.fill_uniform(500, 42, 0, offset=500)
    assert np.array_equal(a[500:], b)
    assert a.min() >= -1.0 and a.max() < 1.0
    c = oracle.fill_uniform(1000, 42, 1)
    assert not np.array_equal(a, c)


def test_full_c2_fixture_reproduces(oracle):
    """tests/golden/full_C2.npz (tools/make_golden.py) is what the oracle
    computes: its first two cycles and residual history entries."""
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "full_C2.npz"))
    m = json.loads(str(z["meta"]))
    assert m["iterations"] == len(z["history"]) - 1 and m["converged"]
    h = oracle.Hierarchy(m["p_t"], m["dim"], m["space_level"], m["time_level"], m["t_final"])
    f = oracle.make_inputs(h, m["seed"], random_u0=m["random_u0"])
    u = np.zeros_like(f)
    assert h.residual_norm(0, u, f) == z["history"][0]
    for k in (1, 2):
        h.mg_cycle_inplace(0, u, f, 1, 1, 1, 0.5)
        assert np.array_equal(u[z["idx"]], z[f"u{k}"])
        assert h.residual_norm(0, u, f) == z["history"][k]
