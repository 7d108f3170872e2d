"""GPU parity: every C-ABI entry point against the CPU oracle on the same
seeded inputs (oracle = C++ restatement of the reference, pinned in
tests/test_oracle.py).

Tolerances: operators 1e-12 relative (the reference's matrix-free vs dense
bar, test_st_system.cpp:83-84); V-cycle iterates 1e-10 relative per cycle and
identical iteration counts to 1e-8 (BASELINE.json north_star).
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def S():
    from paper_1411_0519_b200 import build
    build.build()
    O.build()
    from paper_1411_0519_b200 import stmg
    return stmg


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


CASES = [  # (p_t, dim, space_level, time_level, T, policy)
    (0, 1, 3, 3, 1.0, 0),
    (1, 1, 5, 6, 1.0, 0),
    (2, 1, 4, 4, 0.5, 0),
    (3, 1, 3, 3, 1.0, 0),
    (1, 2, 3, 4, 1.0, 0),
    (2, 2, 3, 3, 0.25, 0),
    (1, 3, 2, 3, 1.0, 0),
    (1, 2, 3, 3, 1.0, 1),
    (1, 2, 3, 3, 1.0, 2),
]


def pair(S, p, dim, sl, tl, T, policy=0, two_grid=0):
    g = S.Hierarchy(p, dim, sl, tl, t_final=T, policy=policy, two_grid=two_grid)
    o = O.Hierarchy(p, dim, sl, tl, t_final=T, policy=policy, two_grid=two_grid)
    assert [L["coarsen_to_next"] for L in g.levels] == [L.coarsen_to_next for L in o.levels]
    assert [L["n_t"] for L in g.levels] == [L.n_t for L in o.levels]
    return g, o


@pytest.mark.parametrize("case", CASES)
def test_operators_match_oracle(S, case):
    p, dim, sl, tl, T, pol = case
    g, o = pair(S, p, dim, sl, tl, T, pol)
    for lev in range(len(o.levels)):
        n = o.levels[lev].size
        u = O.fill_uniform(n, 100 + lev, 0)
        f = O.fill_uniform(n, 200 + lev, 0)
        du, df = g.upload(u, lev), g.upload(f, lev)
        # apply / residual (st_system.cpp:44-67)
        assert rel(g.apply(lev, du).numpy(), o.apply(lev, u)) < 1e-12
        r_o = o.residual(lev, u, f)
        assert rel(g.residual(lev, du, df).numpy(), r_o) < 1e-12
        # norm (st_system.cpp:8-16)
        assert abs(g.norm(lev, df) - o.norm(lev, f)) <= 1e-13 * o.norm(lev, f)
        # exact block solves (st_system.cpp:103-116)
        assert rel(g.block_solve(lev, df).numpy(), o.block_solve(lev, f)) < 1e-12
        # block Jacobi (smoother.cpp:96-106)
        us = g.block_jacobi_step(lev, g.upload(u, lev), df, 0.5, 2).numpy()
        assert rel(us, o.smooth(lev, u, f, 0.5, 2)) < 1e-11
        # forward substitution (st_system.cpp:118-130)
        assert rel(g.forward_substitution_solve(lev, df).numpy(), o.forward_substitution(lev, f)) < 1e-11
        # transfers (transfer.cpp)
        if o.levels[lev].coarsen_to_next:
            for mode in (1, 2):
                if mode == 2 and o.levels[lev].n1 == 1:
                    continue
                rc = g.restrict(lev, du, mode).numpy()
                assert rel(rc, o.restrict(lev, u, mode)) < 1e-13
                c = O.fill_uniform(rc.size, 300 + lev, 0)
                dc = g.coarse_vector(lev, mode).copy_from(c)
                assert rel(g.prolong(lev, dc, mode).numpy(), o.prolong(lev, c, mode)) < 1e-13


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("path", ["spectral", "physical"])
def test_vcycle_iterates_match_oracle(S, case, path):
    p, dim, sl, tl, T, pol = case
    g, o = pair(S, p, dim, sl, tl, T, pol)
    f = O.fill_uniform(o.levels[0].size, 7, 0)
    df = g.upload(f)
    u = np.zeros_like(f)
    du = g.upload(u)
    cfg = S.CycleConfig(nu1=1, nu2=1, gamma=1, omega_t=0.5, path=path)
    for k in range(4):
        u = o.mg_cycle(0, u, f, 1, 1, 1, 0.5)
        g.mg_cycle(0, du, df, cfg)
        assert rel(du.numpy(), u) < 1e-10, (k, path)


@pytest.mark.parametrize("nu", [(2, 2), (1, 0), (0, 1), (2, 1)])
def test_vcycle_general_nu_and_gamma(S, nu):
    g, o = pair(S, 1, 2, 3, 4, 1.0)
    f = O.fill_uniform(o.levels[0].size, 8, 0)
    df = g.upload(f)
    for gamma in (1, 2):
        u = np.zeros_like(f)
        du = g.upload(u)
        cfg = S.CycleConfig(nu1=nu[0], nu2=nu[1], gamma=gamma, omega_t=0.5)
        for _ in range(2):
            u = o.mg_cycle(0, u, f, nu[0], nu[1], gamma, 0.5)
            g.mg_cycle(0, du, df, cfg)
        assert rel(du.numpy(), u) < 1e-10


@pytest.mark.parametrize("path", ["spectral", "physical"])
def test_c1_solve_matches_oracle(S, path):
    """configs[0]: iteration count identical, iterate and history within 1e-10."""
    g, o = pair(S, 1, 1, 5, 6, 1.0)
    f = O.make_inputs(o, 42)
    u_o, rep_o = o.solve(f, eps=1e-8)
    du = g.vector(0)
    rep = g.solve(g.upload(f), du, S.CycleConfig(nu1=1, nu2=1, path=path), 1e-8)
    assert rep.converged and rep.iterations == rep_o["iterations"]
    h_o = np.array(rep_o["residual_history"])
    assert rel(np.array(rep.residual_history), h_o) < 1e-10
    assert rel(du.numpy(), u_o) < 1e-10
    margin = abs(h_o[-1] / h_o[0] - 1e-8) / 1e-8
    print(json.dumps({"path": path, "iterations": rep.iterations, "stop_margin": margin}))


def test_two_grid_matches_oracle(S):
    for mode in (1, 2):
        g, o = pair(S, 1, 2, 3, 3, 1.0, two_grid=mode)
        f = O.fill_uniform(o.levels[0].size, 12, 0)
        df = g.upload(f)
        u = np.zeros_like(f)
        du = g.upload(u)
        for _ in range(3):
            u = o.mg_cycle(0, u, f, 2, 2, 1, 0.5)
            g.mg_cycle(0, du, df, S.CycleConfig(nu1=2, nu2=2))
        assert rel(du.numpy(), u) < 1e-10


def test_c2_reduced_solve_matches_oracle(S):
    """configs[1] shape family (2D, random u0) at 63^2 x 64 steps."""
    g, o = pair(S, 1, 2, 5, 6, 1.0)
    f = O.make_inputs(o, 42, random_u0=True)
    u_o, rep_o = o.solve(f, eps=1e-8)
    du = g.vector(0)
    rep = g.solve(g.upload(f), du, S.CycleConfig(nu1=1, nu2=1), 1e-8)
    assert rep.iterations == rep_o["iterations"]
    assert rel(du.numpy(), u_o) < 1e-10


@pytest.mark.slow
def test_c2_full_solve_matches_oracle(S):
    """configs[1] exactly: 127^2, N_t = 256, p_t = 1, random u0."""
    g, o = pair(S, 1, 2, 6, 8, 1.0)
    f = O.make_inputs(o, 42, random_u0=True)
    u = np.zeros_like(f)
    for _ in range(2):
        u = o.mg_cycle(0, u, f, 1, 1, 1, 0.5)
    du = g.vector(0)
    df = g.upload(f)
    cfg = S.CycleConfig(nu1=1, nu2=1)
    for _ in range(2):
        g.mg_cycle(0, du, df, cfg)
    assert rel(du.numpy(), u) < 1e-10
    rep = g.solve(df, g.vector(0), cfg, 1e-8)
    assert rep.converged
    print(json.dumps({"c2_iterations": rep.iterations}))


def test_device_generator_matches_host(S):
    g = S.Hierarchy(1, 2, 3, 3)
    v = g.vector(0)
    g.fill_uniform(v, 42, 0, 1000)
    assert np.array_equal(v.numpy(), O.fill_uniform(v.n, 42, 0, 1000))
    o = O.Hierarchy(1, 2, 3, 3)
    f = O.fill_uniform(v.n, 42, 0)
    u0 = O.fill_uniform(o.levels[0].n_x, 42, 1)
    want = o.fold_u0(f.copy(), u0)
    df = g.upload(f)
    du0 = S.BlockVector(g, u0.size, (u0.size,)).copy_from(u0)
    assert rel(g.fold_u0(df, du0).numpy(), want) < 1e-14


def test_full_size_linearity_c2(S):
    """configs[1] at full size: a V-cycle from zero is linear in f."""
    g = S.Hierarchy(1, 2, 6, 8, 1.0)
    f1, f2 = g.vector(0), g.vector(0)
    g.fill_uniform(f1, 42, 0)
    g.fill_uniform(f2, 43, 0)
    cfg = S.CycleConfig(nu1=1, nu2=1)
    u1, u2, u12 = g.vector(0), g.vector(0), g.vector(0)
    g.mg_cycle(0, u1, f1, cfg)
    g.mg_cycle(0, u2, f2, cfg)
    f12 = g.upload(f1.numpy() + f2.numpy())
    g.mg_cycle(0, u12, f12, cfg)
    assert rel(u12.numpy(), u1.numpy() + u2.numpy()) < 1e-12


@pytest.mark.parametrize("cfgname,params", [
    ("C3", (2, 2, 7, 12, 1.0)),
    ("C4", (1, 3, 5, 10, 1.0)),
    ("C5_G1", (1, 2, 8, 11, 1.0)),
])
def test_full_size_solves(S, cfgname, params):
    """configs[2..4] at full size: converges to 1e-8 in the physical residual
    (stmg_residual + stmg_norm), deterministically (bitwise equal reruns)."""
    g = S.Hierarchy(*params)
    f = g.vector(0)
    g.fill_uniform(f, 42, 0)
    cfg = S.CycleConfig(nu1=1, nu2=1)
    u = g.vector(0)
    ra = g.solve(f, u, cfg, 1e-8)
    assert ra.converged
    r = g.residual(0, u, f)
    assert g.norm(0, r) <= 1.0001e-8 * g.norm(0, f)
    # the residual of the zero vector is f itself, entry by entry (f - 0): equal
    # norms to the last bit, at the BASELINE size of the row-band kernels
    z = g.vector(0)
    g.residual(0, z, f, r)
    assert g.norm(0, r) == g.norm(0, f)
    del r, z
    u2 = g.vector(0)
    rb = g.solve(f, u2, cfg, 1e-8)
    assert ra.iterations == rb.iterations and ra.residual_history == rb.residual_history
    print(json.dumps({"config": cfgname, "iterations": ra.iterations,
                      "solve_s": ra.device_time_seconds, "dofs": g.size(0)}))


def test_error_behaviour(S):
    g = S.Hierarchy(1, 1, 2, 2)
    v = g.vector(0)
    with pytest.raises(ValueError):
        g.residual(9, v, v)
    last = len(g.levels) - 1
    with pytest.raises(ValueError):
        g.restrict(last, g.vector(last), 1)  # n_t = 1: no coarser level
    with pytest.raises(ValueError):
        g.solve(v, g.vector(0), S.CycleConfig(), 0.0)


def test_cpp_shim_solves_c1(S):
    exe = os.path.join(ROOT, "tests", "cpp", "_shim_smoke")
    from paper_1411_0519_b200 import _capi
    r = subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "shim_smoke.cpp"), _capi.LIB_PATH,
                        "-Wl,-rpath," + os.path.dirname(_capi.LIB_PATH), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    rep = json.loads(out.stdout.strip().splitlines()[-1])
    o = O.Hierarchy(1, 1, 5, 6)
    _, rep_o = o.solve(O.make_inputs(o, 42))
    assert rep["iterations"] == rep_o["iterations"]
    _, rep_i = o.solve(O.make_inputs(o, 42), block_solver="vcycle")
    assert rep["inexact_iterations"] == rep_i["iterations"]
    assert rep["vcycle_size"] == o.levels[0].size


@pytest.mark.parametrize("case", [
    (1, 1, 3, 0, 1.0, 0),   # single time step: the hierarchy is one level (n_t = 1)
    (1, 2, 0, 5, 1.0, 0),   # one spatial node, 32 steps (semi coarsening only)
    (0, 1, 4, 4, 1.0, 1),   # p_t = 0, always_semi
    (3, 1, 3, 3, 1.0, 2),   # p_t = 3, prefer_full
    (1, 3, 2, 4, 0.25, 0),  # 3D
])
def test_solve_edge_cases_match_oracle(S, case):
    p, dim, sl, tl, T, pol = case
    g, o = pair(S, p, dim, sl, tl, T, pol)
    f = O.fill_uniform(o.levels[0].size, 77, 0)
    u0 = O.fill_uniform(o.levels[0].size, 78, 0)
    u_o, rep_o = o.solve(f, u0, eps=1e-9)
    du = g.upload(u0)
    rep = g.solve(g.upload(f), du, S.CycleConfig(nu1=1, nu2=1), 1e-9)
    assert rep.converged and rep.iterations == rep_o["iterations"]
    assert rel(du.numpy(), u_o) < 1e-10


def test_solve_zero_rhs_and_iteration_cap(S):
    g = S.Hierarchy(1, 2, 3, 4)
    f = g.vector(0)  # zero rhs and zero guess: r0 = 0 -> converged, no cycles (mg.cpp:146-149)
    u = g.vector(0)
    rep = g.solve(f, u, S.CycleConfig(nu1=1, nu2=1), 1e-8)
    assert rep.converged and rep.iterations == 0 and rep.residual_history == [0.0]
    g.fill_uniform(f, 5, 0)
    rep = g.solve(f, u, S.CycleConfig(nu1=1, nu2=1), 1e-14, max_iter=3)
    assert not rep.converged and rep.iterations == 3 and len(rep.residual_history) == 4
    o = O.Hierarchy(1, 2, 3, 4)
    _, rep_o = o.solve(O.fill_uniform(o.levels[0].size, 5, 0), eps=1e-14, max_iter=3)
    assert not rep_o["converged"]
    assert rel(np.array(rep.residual_history), np.array(rep_o["residual_history"])) < 1e-10


def test_distributed_api_single_rank(S):
    """stmg_create_distributed with world = 1 is the plain context (the
    multi-rank path needs one GPU per rank)."""
    uid = S.Hierarchy.unique_id()
    g = S.Hierarchy(1, 2, 4, 5, rank=0, world=1, nccl_id=uid)
    assert g.local_steps() == (0, 32)
    o = O.Hierarchy(1, 2, 4, 5)
    f = O.make_inputs(o, 42)
    _, rep_o = o.solve(f)
    rep = g.solve(g.upload(f), g.vector(0), S.CycleConfig(nu1=1, nu2=1), 1e-8)
    assert rep.iterations == rep_o["iterations"]


@pytest.mark.parametrize("p,dim,tl", [(1, 1, 3), (1, 2, 2), (2, 2, 1), (1, 3, 1)])
def test_n63_transforms_match_oracle(S, p, dim, tl):
    """63-node axes (C4's grid) use the dense tensor-core DST-I: the exact block
    solve (forward + inverse transforms on every axis), the physical smoother
    and a solve against the oracle."""
    g, o = pair(S, p, dim, 5, tl, 0.05, 1, 1)
    n = o.levels[0].size
    b = O.fill_uniform(n, 31, 0)
    u = O.fill_uniform(n, 32, 0)
    assert rel(g.block_solve(0, g.upload(b)).numpy(), o.block_solve(0, b)) < 1e-12
    us = g.block_jacobi_step(0, g.upload(u), g.upload(b), 0.5, 1).numpy()
    assert rel(us, o.smooth(0, u, b, 0.5, 1)) < 1e-11
    du = g.upload(u)
    g.mg_cycle(0, du, g.upload(b), S.CycleConfig(nu1=1, nu2=1))
    assert rel(du.numpy(), o.mg_cycle(0, u, b)) < 1e-10


def test_host_solves_match_device_solve(S):
    """stmg_solve_host and the pipelined stmg_solve_host_batch give the device
    solve's iterate bit for bit, for distinct problems in one batch (in place
    and from separate initial guesses), and the oracle's within 1e-10."""
    g, o = pair(S, 1, 2, 4, 5, 1.0)
    cfg = S.CycleConfig(nu1=1, nu2=1)
    fs = [O.make_inputs(o, 40 + i, random_u0=True) for i in range(5)]
    u0s = [O.fill_uniform(o.levels[0].size, 70 + i, 1) for i in range(5)]
    ref, iters = [], []
    for f, u0 in zip(fs, u0s):
        du = g.upload(u0)
        rep = g.solve(g.upload(f), du, cfg, 1e-8)
        ref.append(du.numpy())
        iters.append(rep.iterations)
    u_o, rep_o = o.solve(fs[0], u=u0s[0], eps=1e-8)
    assert rep_o["iterations"] == iters[0] and rel(ref[0], u_o) < 1e-10
    uh = u0s[0].copy()
    rep = g.solve_host(fs[0], uh, cfg, 1e-8)
    assert rep.iterations == iters[0] and np.array_equal(uh, ref[0])
    # in place
    us = [u.copy() for u in u0s]
    reps = g.solve_host_batch(fs, us, cfg, 1e-8)
    assert [r.iterations for r in reps] == iters and all(r.converged for r in reps)
    for u, r in zip(us, ref):
        assert np.array_equal(u, r)
    # separate initial guesses (inputs untouched), outputs reused round-robin
    outs = [np.empty_like(u0s[0]) for _ in range(5)]
    keep = [u.copy() for u in u0s]
    reps = g.solve_host_batch(fs, outs, cfg, 1e-8, u0s=u0s)
    for u, r in zip(outs, ref):
        assert np.array_equal(u, r)
    assert all(np.array_equal(a, b) for a, b in zip(u0s, keep))
    assert g.solve_host_batch([], [], cfg, 1e-8) == []
    with pytest.raises(ValueError):
        g.solve_host_batch(fs, us[:2], cfg, 1e-8)
    with pytest.raises(Exception):
        g.solve_host_batch(fs[:1], us[:1], cfg, -1.0)
    # zero initial guesses (None: nothing uploaded) = solves from a zero vector
    zref = []
    for f in fs[:3]:
        du = g.vector(0)
        g.solve(g.upload(f), du, cfg, 1e-8)
        zref.append(du.numpy())
    outs = [np.full_like(u0s[0], 7.0) for _ in range(3)]
    g.solve_host_batch(fs[:3], outs, cfg, 1e-8, u0s=[None] * 3)
    for u, r in zip(outs, zref):
        assert np.array_equal(u, r)
    # inputs of problem j may not alias the outputs of the two problems before it
    g.solve_host_batch(fs[:3], [outs[0], outs[1], outs[0]], cfg, 1e-8, u0s=[None] * 3)
    assert np.array_equal(outs[0], zref[2])  # outputs may repeat: D2Hs are ordered
    with pytest.raises(ValueError):  # in place: problem 2 uploads the buffer problem 0 downloads into
        g.solve_host_batch(fs[:3], [outs[0], outs[1], outs[0]], cfg, 1e-8)
    with pytest.raises(ValueError):
        g.solve_host_batch(fs[:2], [outs[0], outs[1]], cfg, 1e-8, u0s=[None, outs[0]])


def test_cached_fused_loop_after_other_cycle_shapes(S):
    """A cached fused V(1,1) device loop replayed after cycles that move the
    coarse buffer indices (mg_cycle, a V(2,1) solve) still returns the right
    iterate: the suffix reads the coarse correction the graph wrote."""
    g, o = pair(S, 1, 2, 4, 5, 1.0)
    f = O.make_inputs(o, 42, random_u0=True)
    u_o, rep_o = o.solve(f, eps=1e-8)
    df = g.upload(f)
    v11 = S.CycleConfig(nu1=1, nu2=1)
    for _ in range(2):
        du = g.vector(0)
        rep = g.solve(df, du, v11, 1e-8)
        assert rep.iterations == rep_o["iterations"] and rel(du.numpy(), u_o) < 1e-10
        g.mg_cycle(0, g.vector(0), df, S.CycleConfig(nu1=2, nu2=1))
        g.solve(df, g.vector(0), S.CycleConfig(nu1=2, nu2=1), 1e-8)


@pytest.mark.parametrize("shards", [0, 2])
def test_history_buffer_regrowth(S, shards):
    """A solve with max_iter >= 1024 regrows the device history; later solves
    with a smaller max_iter must not replay graphs that captured the old
    buffer (fused bodies and device loops)."""
    g = S.Hierarchy(1, 2, 4, 5, shards=shards)
    o = O.Hierarchy(1, 2, 4, 5)
    f = O.make_inputs(o, 42)
    u_o, rep_o = o.solve(f, eps=1e-8)
    df = g.upload(f)
    cfg = S.CycleConfig(nu1=1, nu2=1)
    for mi in (50, 1500, 50):
        du = g.vector(0)
        rep = g.solve(df, du, cfg, 1e-8, max_iter=mi)
        assert rep.converged and rep.iterations == rep_o["iterations"]
        assert rel(np.array(rep.residual_history), np.array(rep_o["residual_history"])) < 1e-10
        assert rel(du.numpy(), u_o) < 1e-10


@pytest.mark.parametrize("sl", [6, 7])
def test_one_pass_2d_transform_matches_oracle(S, sl):
    """127^2 and 255^2 slabs use the one-pass cluster DST (k_dst2d): the exact
    block solve (forward + inverse 2D transforms) and the physical smoother
    against the oracle, the accumulate mode, and in-place use."""
    g, o = pair(S, 1, 2, sl, 2, 0.1, 1, 1)
    n = o.levels[0].size
    b = O.fill_uniform(n, 41, 0)
    u = O.fill_uniform(n, 42, 0)
    assert rel(g.block_solve(0, g.upload(b)).numpy(), o.block_solve(0, b)) < 1e-12
    us = g.block_jacobi_step(0, g.upload(u), g.upload(b), 0.5, 2).numpy()
    assert rel(us, o.smooth(0, u, b, 0.5, 2)) < 1e-11
    fs = g.forward_substitution_solve(0, g.upload(b)).numpy()
    assert rel(fs, o.forward_substitution(0, b)) < 1e-11


@pytest.mark.parametrize("case", [
    (4, 1, 4, 3, 1.0, 0), (5, 2, 3, 3, 0.5, 0), (7, 1, 3, 2, 1.0, 2), (10, 1, 3, 2, 1.0, 0),
    (4, 3, 2, 2, 1.0, 0),
])
def test_high_degree_matches_oracle(S, case):
    """p_t 4..10 (dg_time.hpp:10; SPEC acceptance p_t 0..5): every operator
    and a full solve against the oracle (runtime-NL physical kernels)."""
    p, dim, sl, tl, T, pol = case
    g, o = pair(S, p, dim, sl, tl, T, pol)
    for lev in range(len(o.levels)):
        n = o.levels[lev].size
        u = O.fill_uniform(n, 100 + lev, 0)
        f = O.fill_uniform(n, 200 + lev, 0)
        du, df = g.upload(u, lev), g.upload(f, lev)
        assert rel(g.apply(lev, du).numpy(), o.apply(lev, u)) < 1e-12
        assert rel(g.residual(lev, du, df).numpy(), o.residual(lev, u, f)) < 1e-12
        assert rel(g.block_solve(lev, df).numpy(), o.block_solve(lev, f)) < 1e-11
        us = g.block_jacobi_step(lev, g.upload(u, lev), df, 0.5, 1).numpy()
        assert rel(us, o.smooth(lev, u, f, 0.5, 1)) < 1e-11
        assert rel(g.forward_substitution_solve(lev, df).numpy(),
                   o.forward_substitution(lev, f)) < 1e-10
        if o.levels[lev].coarsen_to_next:
            mode = o.levels[lev].coarsen_to_next
            rc = g.restrict(lev, du, mode).numpy()
            assert rel(rc, o.restrict(lev, u, mode)) < 1e-13
            dc = g.coarse_vector(lev, mode).copy_from(rc)
            assert rel(g.prolong(lev, dc, mode).numpy(), o.prolong(lev, rc, mode)) < 1e-13
    f = O.fill_uniform(o.levels[0].size, 7, 0)
    u_o, rep_o = o.solve(f, eps=1e-8)
    du = g.vector(0)
    rep = g.solve(g.upload(f), du, S.CycleConfig(nu1=1, nu2=1), 1e-8)  # spectral request -> physical
    assert rep.converged and rep.iterations == rep_o["iterations"]
    assert rel(du.numpy(), u_o) < 1e-9
    with pytest.raises(ValueError):
        g.solve(g.upload(f), g.vector(0), S.CycleConfig(nu1=1, nu2=1, block_solver="vcycle"), 1e-8)


@pytest.mark.parametrize("case", [
    (0, 2, 6, 3), (1, 2, 6, 6), (2, 2, 6, 4), (3, 2, 6, 2), (2, 2, 7, 3), (1, 2, 8, 2),
    (1, 3, 5, 4), (2, 3, 5, 2), (0, 3, 5, 3), (3, 3, 5, 1), (1, 3, 6, 1),
])
def test_row_band_residual_matches_oracle(S, case):
    """apply / residual on grids wide enough for the row-band kernels
    (csrc/stmg_apply.cu: 127 .. 511 nodes per axis in 2D, 63 / 127 in 3D),
    several time chunks per CTA column, partial last band."""
    p, dim, sl, tl = case
    g, o = pair(S, p, dim, sl, tl, 1.0)
    n = o.levels[0].size
    u = O.fill_uniform(n, 300 + sl, 0)
    f = O.fill_uniform(n, 400 + sl, 0)
    du, df = g.upload(u, 0), g.upload(f, 0)
    assert rel(g.apply(0, du).numpy(), o.apply(0, u)) < 1e-12
    assert rel(g.residual(0, du, df).numpy(), o.residual(0, u, f)) < 1e-12
    # transfers at the same sizes (k_restrict / the round-2 k_prolong)
    if o.levels[0].coarsen_to_next:
        for mode in (1, 2):
            rc = g.restrict(0, du, mode).numpy()
            assert rel(rc, o.restrict(0, u, mode)) < 1e-13
            c = O.fill_uniform(rc.size, 500 + sl, 0)
            dc = g.coarse_vector(0, mode).copy_from(c)
            assert rel(g.prolong(0, dc, mode).numpy(), o.prolong(0, c, mode)) < 1e-13


@pytest.mark.parametrize("case", [(1, 2, 6, 3), (2, 2, 6, 2), (1, 3, 5, 2)])
def test_physical_path_cycle_on_row_band_sizes(S, case):
    """Two V-cycles through the reference call structure (physical path:
    residual, exact block solves, transfers as separate operators) on grids
    where level 0 runs the row-band residual and the one-pass / dense
    transforms; 1e-10 per cycle against the oracle."""
    p, dim, sl, tl = case
    g, o = pair(S, p, dim, sl, tl, 1.0)
    f = O.fill_uniform(o.levels[0].size, 11, 0)
    df = g.upload(f)
    u = np.zeros_like(f)
    du = g.upload(u)
    cfg = S.CycleConfig(nu1=1, nu2=1, gamma=1, omega_t=0.5, path="physical")
    for k in range(2):
        u = o.mg_cycle(0, u, f, 1, 1, 1, 0.5)
        g.mg_cycle(0, du, df, cfg)
        assert rel(du.numpy(), u) < 1e-10, k
    us = g.block_jacobi_step(0, g.upload(u), df, 0.5, 1).numpy()
    assert rel(us, o.smooth(0, u, f, 0.5, 1)) < 1e-11
