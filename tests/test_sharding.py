"""Time-slab sharding.

CPU: the host-side plan, and a world_size-2 gloo run of the decomposition the
multi-GPU driver uses -- contiguous time slabs, a one-slab trace halo sent to
rank g+1, per-step norm partials all-gathered and summed in global order --
checked against the undecomposed operator (dense oracle).
GPU: virtual shards on one device run the exact multi-GPU code path (halo /
gather / scatter / partial all-gather with D2D copies instead of NCCL); their
iterates and residual histories must be BITWISE equal to the 1-shard solve,
for the per-level and the fused level-0 schedule alike.
"""
import os
import socket

import numpy as np
import pytest

from oracle import dense


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_plan_levels():
    from paper_1411_0519_b200 import build, stmg
    build.build()
    for cfg in [(1, 1, 5, 6), (1, 2, 6, 8), (2, 2, 7, 12), (1, 3, 5, 10), (1, 2, 8, 11)]:
        for S in (1, 2, 4, 8):
            lg, n = stmg.shard_plan(*cfg, S)
            assert n * S == 2 ** cfg[3]
            assert lg >= 1
            # every sharded level keeps >= 2 (even) steps per shard
            assert (2 ** cfg[3]) // 2 ** (lg - 1) >= 2 * S
    with pytest.raises(ValueError):
        stmg.shard_plan(1, 1, 3, 2, 4)  # 4 steps cannot feed 4 shards x 2


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    p, lev, tl = 1, 3, 3
    n_t, tau = 2 ** tl, 0.05
    K, M, N = dense.dg_block(p, tau)
    Mh, Kh = dense.space_mats(1, lev)
    nx, nl = Mh.shape[0], p + 1
    slab = nx * nl
    rng = np.random.default_rng(7)
    u = rng.uniform(-1, 1, n_t * slab)
    f = rng.uniform(-1, 1, n_t * slab)
    # slab split from the library's own host-side plan (stmg_shard_plan, the
    # function stmg_create_distributed uses), not re-derived here
    from paper_1411_0519_b200 import stmg
    gather_level, n_loc = stmg.shard_plan(p, 1, lev, tl, world)
    assert n_loc * world == n_t and gather_level >= 1
    lo, hi = rank * n_loc * slab, (rank + 1) * n_loc * slab
    u_loc, f_loc = u[lo:hi].copy(), f[lo:hi].copy()
    # trace halo: last slab of rank g goes to rank g+1
    halo = torch.zeros(slab, dtype=torch.float64)
    reqs = []
    if rank + 1 < world:
        reqs.append(dist.isend(torch.from_numpy(u_loc[-slab:].copy()), rank + 1))
    if rank > 0:
        reqs.append(dist.irecv(halo, rank - 1))
    for r in reqs:
        r.wait()
    ext_n = n_loc + (1 if rank > 0 else 0)
    L = dense.dense_space_time(K, M, N, Mh, Kh, ext_n)
    ext_u = np.concatenate([halo.numpy(), u_loc]) if rank > 0 else u_loc
    r_loc = (np.concatenate([np.zeros(slab), f_loc]) if rank > 0 else f_loc) - L @ ext_u
    r_loc = r_loc[slab:] if rank > 0 else r_loc
    # per-step partial sums, gathered and summed in global step order
    part = torch.tensor([float(np.sum(r_loc[k * slab:(k + 1) * slab] ** 2)) for k in range(n_loc)],
                        dtype=torch.float64)
    allp = [torch.zeros_like(part) for _ in range(world)]
    dist.all_gather(allp, part)
    total = 0.0
    for t in allp:
        for v in t.tolist():
            total += v
    rs = [torch.zeros(n_loc * slab, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(rs, torch.from_numpy(r_loc))
    if rank == 0:
        Lg = dense.dense_space_time(K, M, N, Mh, Kh, n_t)
        r_glob = f - Lg @ u
        parts = [float(np.sum(r_glob[k * slab:(k + 1) * slab] ** 2)) for k in range(n_t)]
        ref = 0.0
        for v in parts:
            ref += v
        got = np.concatenate([t.numpy() for t in rs])
        out.put((float(np.abs(got - r_glob).max() / np.abs(r_glob).max()), total == ref))
    dist.destroy_process_group()


def test_gloo_two_ranks_time_slab_residual_and_norm():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, bitwise = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-14
    assert bitwise


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(1, 1, 5, 6, 1.0), (1, 2, 4, 6, 1.0), (2, 2, 4, 5, 0.5),
                                 (1, 3, 3, 5, 1.0), (1, 2, 6, 8, 1.0)])
@pytest.mark.parametrize("S", [2, 4])
def test_virtual_shards_bitwise(cfg, S):
    from oracle import oracle as O
    from paper_1411_0519_b200 import build, stmg
    build.build()
    p, dim, sl, tl, T = cfg
    o = O.Hierarchy(p, dim, sl, tl, t_final=T)
    f = O.make_inputs(o, 42, random_u0=(dim == 2))
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    # both schedules -- per-level (STMG_FUSED=0) and fused level-0 (default)
    # -- on S shards against the same schedule on one shard
    for fused in ("0", "1"):
        os.environ["STMG_FUSED"] = fused
        try:
            g1 = stmg.Hierarchy(p, dim, sl, tl, t_final=T)
            gs = stmg.Hierarchy(p, dim, sl, tl, t_final=T, shards=S)
        finally:
            os.environ.pop("STMG_FUSED", None)
        u1 = g1.vector(0)
        r1 = g1.solve(g1.upload(f), u1, cc, 1e-8)
        us = gs.vector(0)
        rs = gs.solve(gs.upload(f), us, cc, 1e-8)
        assert rs.iterations == r1.iterations, fused
        assert rs.residual_history == r1.residual_history, fused
        assert np.array_equal(us.numpy(), u1.numpy()), fused
        del g1, gs


@pytest.mark.gpu
def test_virtual_shards_general_cycle_and_initial_guess():
    from oracle import oracle as O
    from paper_1411_0519_b200 import build, stmg
    build.build()
    p, dim, sl, tl = 1, 2, 4, 6
    o = O.Hierarchy(p, dim, sl, tl)
    f = O.fill_uniform(o.levels[0].size, 3, 0)
    u0 = O.fill_uniform(o.levels[0].size, 4, 0)
    cc = stmg.CycleConfig(nu1=2, nu2=2)
    g1 = stmg.Hierarchy(p, dim, sl, tl)
    u1 = g1.upload(u0)
    r1 = g1.solve(g1.upload(f), u1, cc, 1e-9)
    g2 = stmg.Hierarchy(p, dim, sl, tl, shards=4)
    u2 = g2.upload(u0)
    r2 = g2.solve(g2.upload(f), u2, cc, 1e-9)
    assert r2.iterations == r1.iterations and r2.residual_history == r1.residual_history
    assert np.array_equal(u2.numpy(), u1.numpy())
    # and against the CPU oracle
    u_o, rep_o = o.solve(f, u0, nu1=2, nu2=2, eps=1e-9)
    assert rep_o["iterations"] == r2.iterations
    assert np.abs(u2.numpy() - u_o).max() <= 1e-10 * np.abs(u_o).max()


@pytest.mark.gpu
@pytest.mark.parametrize("S", [2, 4, 8])
def test_virtual_shards_fused_nonzero_guess_vs_oracle(S):
    """Fused sharded schedule from a nonzero initial guess (prefix k_down with
    a 2-slab halo), checked bitwise against one shard and against the oracle."""
    from oracle import oracle as O
    from paper_1411_0519_b200 import build, stmg
    build.build()
    p, dim, sl, tl = 2, 1, 6, 7
    o = O.Hierarchy(p, dim, sl, tl)
    f = O.fill_uniform(o.levels[0].size, 11, 0)
    u0 = O.fill_uniform(o.levels[0].size, 12, 0)
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    g1 = stmg.Hierarchy(p, dim, sl, tl)
    u1 = g1.upload(u0)
    r1 = g1.solve(g1.upload(f), u1, cc, 1e-9)
    gs = stmg.Hierarchy(p, dim, sl, tl, shards=S)
    us = gs.upload(u0)
    rs = gs.solve(gs.upload(f), us, cc, 1e-9)
    assert rs.iterations == r1.iterations and rs.residual_history == r1.residual_history
    assert np.array_equal(us.numpy(), u1.numpy())
    u_o, rep_o = o.solve(f, u0, nu1=1, nu2=1, eps=1e-9)
    assert rep_o["iterations"] == rs.iterations
    assert np.abs(us.numpy() - u_o).max() <= 1e-10 * np.abs(u_o).max()


def _solve_with_env(env, p, dim, sl, tl, f):
    from paper_1411_0519_b200 import stmg
    for k, v in env.items():
        os.environ[k] = v
    try:
        g = stmg.Hierarchy(p, dim, sl, tl)
    finally:
        for k in env:
            os.environ.pop(k, None)
    u = g.vector(0)
    r = g.solve(g.upload(f), u, stmg.CycleConfig(nu1=1, nu2=1), 1e-8)
    return r, u.numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(1, 1, 5, 6), (1, 2, 6, 8), (2, 2, 4, 6), (1, 3, 3, 5)])
def test_schedule_switches_agree(cfg):
    """The coarse operator (tail as a precomputed matrix, STMG_COARSE_OP) agrees
    with the tail kernel to rounding."""
    from oracle import oracle as O
    from paper_1411_0519_b200 import build
    build.build()
    p, dim, sl, tl = cfg
    o = O.Hierarchy(p, dim, sl, tl)
    f = O.make_inputs(o, 42, random_u0=(dim == 2))
    r_ref, u_ref = _solve_with_env({"STMG_COARSE_OP": "0"}, p, dim, sl, tl, f)
    r_op, u_op = _solve_with_env({}, p, dim, sl, tl, f)
    assert r_op.iterations == r_ref.iterations
    assert np.abs(u_op - u_ref).max() <= 1e-12 * np.abs(u_ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(1, 2, 6, 8), (2, 2, 6, 7), (1, 3, 4, 6), (1, 2, 7, 6)])
@pytest.mark.parametrize("depth", ["1", "3"])
def test_fused_coarse_trees_bitwise(cfg, depth):
    """The alias-group-tree kernels for the coarse levels (STMG_CSUB=1,
    k_csub_down/up) run the per-level kernels' arithmetic: bitwise equal
    iterates and histories."""
    from oracle import oracle as O
    from paper_1411_0519_b200 import build
    build.build()
    p, dim, sl, tl = cfg
    o = O.Hierarchy(p, dim, sl, tl)
    f = O.make_inputs(o, 42, random_u0=(dim == 2))
    r_ref, u_ref = _solve_with_env({"STMG_CSUB": "0"}, p, dim, sl, tl, f)
    r_cs, u_cs = _solve_with_env({"STMG_CSUB": "1", "STMG_CSUB_DEPTH": depth}, p, dim, sl, tl, f)
    assert r_cs.iterations == r_ref.iterations
    assert r_cs.residual_history == r_ref.residual_history
    assert np.array_equal(u_cs, u_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("cyc", [(1, 1), (2, 2)])
def test_virtual_shards_host_batch(cyc):
    """stmg_solve_host_batch on a 4-shard context (fused and general cycles):
    bitwise the one-shard device solve of every problem."""
    from oracle import oracle as O
    from paper_1411_0519_b200 import build, stmg
    build.build()
    p, dim, sl, tl = 1, 2, 4, 6
    o = O.Hierarchy(p, dim, sl, tl)
    n = o.levels[0].size
    fs = [O.fill_uniform(n, 20 + i, 0) for i in range(4)]
    u0s = [O.fill_uniform(n, 30 + i, 0) for i in range(4)]
    cc = stmg.CycleConfig(nu1=cyc[0], nu2=cyc[1])
    g1 = stmg.Hierarchy(p, dim, sl, tl)
    ref, iters = [], []
    for f, u0 in zip(fs, u0s):
        u = g1.upload(u0)
        iters.append(g1.solve(g1.upload(f), u, cc, 1e-9).iterations)
        ref.append(u.numpy())
    gs = stmg.Hierarchy(p, dim, sl, tl, shards=4)
    outs = [np.empty(n) for _ in range(4)]
    reps = gs.solve_host_batch(fs, outs, cc, 1e-9, u0s=u0s)
    assert [r.iterations for r in reps] == iters
    for a, b in zip(outs, ref):
        assert np.array_equal(a, b)
