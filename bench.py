#!/usr/bin/env python3
"""bench.py -- space-time multigrid V-cycle throughput on B200.

Workload (BASELINE.json configs[1], the single-B200 case the metric is quoted
on): 2D heat equation on the unit square, Q1 on a uniform 128x128 grid (127^2
interior nodes), T = 1, N_t = 256, DG p_t = 1, FP64; f i.i.d. uniform[-1,1]
per space-time dof and u0 i.i.d. uniform[-1,1] per interior node (seed 42,
counter-based generator); zero initial guess; V(1,1) cycles
with damped block Jacobi (omega_t = 1/2, exact block solves), mu-driven
coarsening; stop at ||r_k|| <= 1e-8 ||r_0||.

One step = one full solve to 1e-8 (basis transforms included) on inputs
resident in HBM.  value = fine DoF x V-cycles / s, summed over ranks.
e2e = the same K solves through stmg_solve_host_batch with pinned HOST buffers
(H2D of f, D2H of u inside the timed region for every step, zero initial
guess; step i+1's upload and step i-1's download overlap solve i);
e2e.single_call is the unpipelined reference-shaped stmg_solve_host per step
(f and the initial guess uploaded, u downloaded).  --impl reference times the
CPU oracle (the reference algorithm restated in C++/OpenMP; the reference
itself cannot be built here) on all host cores.

Multi-GPU (--gpus N > 1): bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU) unless it already runs under
torchrun (WORLD_SIZE set, which must equal N); it exits non-zero when fewer
than N GPUs are visible or any rank fails -- there is no replica fallback.
The main line is configs[1] scaled weakly in time (N_t = 256 N, tau fixed:
per-GPU work constant, time slabs over the ranks, NCCL halo exchange inside
the library).  Every run (N = 1 included) adds "scaling" sub-records:
configs[2] C3 and configs[3] C4 strong scaling (N_t fixed) and configs[4] C5
weak scaling (N_t = 2048 N), each with ms per solve and per V-cycle, iterations
and the per-rank k_updown HBM GB/s, so the driver's per-N runs give the curves.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": dict(p_t=1, dim=1, space_level=5, time_level=6, t_final=1.0, random_u0=False,
               desc="configs[0]: 1D heat, Q1 h=1/64 (63 nodes), N_t=64, p_t=1"),
    "C2": dict(p_t=1, dim=2, space_level=6, time_level=8, t_final=1.0, random_u0=True,
               desc="configs[1]: 2D heat, Q1 128x128 grid (127^2 interior), N_t=256, p_t=1, random u0"),
    "C3": dict(p_t=2, dim=2, space_level=7, time_level=12, t_final=1.0, random_u0=False,
               desc="configs[2]: 2D heat, Q1 256x256 grid (255^2 interior), N_t=4096, p_t=2"),
    "C4": dict(p_t=1, dim=3, space_level=5, time_level=10, t_final=1.0, random_u0=False,
               desc="configs[3]: 3D heat, Q1 64^3 grid (63^3 interior), N_t=1024, p_t=1"),
    "C5": dict(p_t=1, dim=2, space_level=8, time_level=11, t_final=1.0, random_u0=False,
               desc="configs[4] G=1: 2D heat, Q1 512x512 grid (511^2 interior), N_t=2048, p_t=1"),
}
METRIC = "space-time DoF*V-cycles/s (full solve to 1e-8 residual reduction)"
UNIT = "DoF*V-cycles/s"
EPS = 1e-8
SEED = 42
L2_FLUSH_BYTES = 512 << 20


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(expect_world: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != expect_world:
        raise SystemExit(f"[bench] WORLD_SIZE={world} but --gpus {expect_world}: refusing to run")
    dist = None
    if world > 1:
        # watchdog: the NCCL transport has only ever run on virtual shards (one
        # GPU per box here); a rank that deadlocks must not hang the node
        limit = float(os.environ.get("STMG_BENCH_TIMEOUT", "900"))

        def _abort():
            print(f"[bench] rank {rank}: no result after {limit:.0f} s -- aborting (exit 3)",
                  file=sys.stderr, flush=True)
            os._exit(3)

        wd = threading.Timer(limit, _abort)
        wd.daemon = True
        wd.start()
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        if local >= ndev:
            raise SystemExit(f"[bench] rank {rank}: LOCAL_RANK {local} but only {ndev} GPU(s) visible")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"[bench] rank {rank}/{world} on cuda:{local} "
              f"({torch.cuda.get_device_name(local)}): NCCL process group up", file=sys.stderr,
              flush=True)
    return world, rank, local, dist


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_command(argv, n: int, port: int):
    """torchrun command that re-runs this script with n ranks on one node."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__)] + list(argv)


def spawn(args, argv) -> int:
    """--gpus N > 1 without torchrun: start N ranks, fail loudly on fewer GPUs."""
    try:
        import torch
        ndev = torch.cuda.device_count()
    except Exception as exc:  # pragma: no cover
        print(f"[bench] cannot query GPUs: {exc}", file=sys.stderr)
        return 2
    if ndev < args.gpus:
        print(f"[bench] --gpus {args.gpus} needs {args.gpus} GPUs on this node, found {ndev}; "
              "not running (no replica fallback)", file=sys.stderr, flush=True)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines: one per rank
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = launch_command(argv, args.gpus, free_port())
    print("[bench] launching: " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env).returncode


def allreduce_max(dist, local, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(dist, local, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist, local):
    if dist is not None:
        import torch
        torch.cuda.synchronize(local)
        dist.barrier()


def oracle_inputs(cfg):
    from oracle import oracle as O
    h = O.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    return h, O.make_inputs(h, SEED, random_u0=cfg["random_u0"])


def cpu_reference_cycles(cfg, cycles: int, warm: int = 0):
    """Time `cycles` V(1,1) cycles of the oracle (+ stop-test residual and norm
    each cycle, mg.cpp:150-160) on all host cores.  Returns (s_per_cycle, n0)."""
    from oracle import oracle as O
    h, f = oracle_inputs(cfg)
    u = np.zeros_like(f)
    n0 = f.size
    times = []
    for k in range(warm + cycles):
        t0 = time.perf_counter()
        h.mg_cycle_inplace(0, u, f, 1, 1, 1, 0.5)
        h.residual_norm(0, u, f)  # stop-test residual + norm (mg.cpp:150-160)
        dt = time.perf_counter() - t0
        if k >= warm:
            times.append(dt)
    return times, n0


def run_reference(args, cfgname):
    # under torchrun rank 0 alone runs the CPU reference; no process group needed
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    cfg = scaled(cfgname, args.gpus, weak=True)  # the workload of our arm at this N
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    times, n0 = cpu_reference_cycles(cfg, args.steps, args.warmup)
    per = sum(times) / len(times)
    value = n0 / per
    sample = (f"{args.steps} V(1,1) cycles (+ stop-test residual/norm each) of {cfgname} from a "
              f"zero guess, {args.warmup} untimed; one step = one cycle; value = dofs / mean "
              f"cycle time")
    workload = cfg["desc"] + (f"; weak in time over {args.gpus} GPUs: N_t = "
                              f"{2 ** cfg['time_level']}, T = {cfg['t_final']:g}"
                              if args.gpus > 1 else "")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "weak" if args.gpus > 1 else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 uniform[-1,1], f and u0)",
        "config": {"workload": workload, "dofs": n0,
                   "cycle": "V(1,1), omega_t=0.5, exact DG block solves, mu-driven coarsening",
                   "eps": EPS, "parallelism": f"CPU oracle, {cores} host threads (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference (Eigen3) cannot be built here; CPU oracle = C++/OpenMP restatement "
                "of the reference algorithm (oracle/)",
    }
    print(json.dumps(line), flush=True)
    return 0


def traffic_from_profiles(kernel_tag: str):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(kernel_tag)
    except Exception:
        return None


def make_hierarchy(stmg, cfg, world, rank, local, dist):
    """One context: plain on one GPU, time slabs over the ranks otherwise.
    Any failure propagates (no replica fallback)."""
    if world == 1:
        return stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"],
                              cfg["t_final"], device=local)
    uid = [stmg.Hierarchy.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"],
                       cfg["t_final"], device=local, rank=rank, world=world, nccl_id=uid[0])
    first, n = h.local_steps()
    print(f"[bench] rank {rank}/{world}: time-slab context up (steps [{first}, {first + n}) of "
          f"{h.levels[0]['n_t']}, own NCCL communicator)", file=sys.stderr, flush=True)
    return h


def scaled(cfgname, world, weak):
    """configs entry for N ranks: weak = N_t x N with tau fixed (T = N)."""
    cfg = dict(CONFIGS[cfgname])
    if weak and world > 1:
        cfg["time_level"] += int(round(math.log2(world)))
        cfg["t_final"] = float(world)
    return cfg


def local_inputs(stmg, h, cfg):
    """This rank's slabs of the seeded f (u0 folded into f on rank 0)."""
    first, _ = h.local_steps()
    L0 = h.levels[0]
    slab = L0["n_loc"] * L0["n_x"]
    f = h.local_vector()
    h.fill_uniform(f, SEED, 0, first * slab)
    if cfg["random_u0"] and first == 0:
        u0 = stmg.BlockVector(h, L0["n_x"], (L0["n_x"],))
        h.fill_uniform(u0, SEED, 1)
        h.fold_u0(f, u0)
        del u0
    return f


def gather_obj(dist, x):
    if dist is None:
        return [x]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, x)
    return out


def updown_profile(h, step):
    """k_updown (or k_down/k_up) per-launch ms and algorithmic bytes from CUDA
    events around every level-0 launch during one profiled replay of `step`."""
    h.profile(True)
    h.profile_reset()
    dev = step().device_time_seconds
    prof = {k: h.profile_read(k) for k in (0, 1, 2)}
    h.profile(False)
    return prof, dev


def operator_record(h, f, u, reps=6):
    """Reference-API operators on level 0 of an open single-GPU context:
    the physical Q1 residual (stmg_residual, 24 B per dof) and one damped
    block-Jacobi sweep through stmg_smooth (exact blocks).  Residual: CUDA
    events on the library stream around each launch (profile slot 3), L2
    evicted before every launch when the vectors are smaller than L2;
    smoother: events around each whole sweep (profile slot 5: residual +
    transforms + modal solve + update launches)."""
    import ctypes as C
    from paper_1411_0519_b200 import _capi as A
    peak, kind = peaks()
    n0 = h.size(0)
    r = h.vector(0)
    flush = None
    if 3 * n0 * 8 < (512 << 20):
        flush = C.c_void_p()
        A.check(A.lib().stmg_device_alloc(h._ctx, L2_FLUSH_BYTES, C.byref(flush)))

    def evict():
        if flush is not None:
            A.check(A.lib().stmg_memset_zero(h._ctx, flush, L2_FLUSH_BYTES))

    h.residual(0, u, f, r)  # warm-up
    h.synchronize()
    h.profile(True)
    h.profile_reset()
    for _ in range(reps):
        evict()
        h.residual(0, u, f, r)
    ms, n, b = h.profile_read(3)
    h.profile(False)
    res = b / ((ms / n) * 1e-3) / 1e9
    h.block_jacobi_step(0, r, f, 0.5, 1)  # warm-up (r as the iterate: u stays intact)
    h.synchronize()
    h.profile(True)
    h.profile_reset()
    for _ in range(reps):
        evict()
        h.block_jacobi_step(0, r, f, 0.5, 1)
    sms, sn, _ = h.profile_read(5)
    h.profile(False)
    sm = sms / sn
    if flush is not None:
        A.lib().stmg_device_free(h._ctx, flush)
    del r
    return {
        "residual": {"kernel": "k_apply_rows (stmg_residual)", "ms_per_launch": ms / n,
                     "achieved": res, "unit": "GB/s", "peak": peak, "peak_kind": kind,
                     "frac": res / peak, "algorithmic_bytes_per_dof": 24},
        "smoother_reference_api": {
            "api": "stmg_smooth, one sweep: residual + forward sine transform + modal block "
                   "solve + inverse transform with u += omega x",
            "ms_per_sweep": sm, "achieved": 24.0 * n0 / (sm * 1e-3) / 1e9, "unit": "GB/s",
            "frac": 24.0 * n0 / (sm * 1e-3) / 1e9 / peak, "algorithmic_bytes_per_dof": 24,
            "bound": "shared-memory pipe of the FFT passes, not HBM (DESIGN.md 5)"},
    }


def concurrent_record(stmg, cfg, local, steps, contexts=3):
    """Aggregate throughput of the same solves when `contexts` independent
    problems are in flight (one context, host thread and library stream each;
    device-resident inputs).  A single C2 solve leaves the GPU partly idle
    during its latency-bound coarse levels; independent problems fill it.
    Extra information: `value` stays the one-problem-at-a-time figure."""
    import threading
    from paper_1411_0519_b200 import _capi as A
    ccfg = stmg.CycleConfig(nu1=1, nu2=1, gamma=1, omega_t=0.5)
    ctxs = []
    for _ in range(contexts):
        h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"],
                           cfg["t_final"], device=local)
        f, u = h.vector(0), h.vector(0)
        h.fill_uniform(f, SEED, 0)
        if cfg["random_u0"]:
            L0 = h.levels[0]
            u0 = stmg.BlockVector(h, L0["n_x"], (L0["n_x"],))
            h.fill_uniform(u0, SEED, 1)
            h.fold_u0(f, u0)
        ctxs.append((h, f, u))
    its = []

    def work(c, k):
        h, f, u = c
        for _ in range(k):
            A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, u.n * 8))
            its.append(h.solve(f, u, ccfg, EPS).iterations)
        h.synchronize()

    per = max(steps // contexts, 1)
    for c in ctxs:
        work(c, 2)
    its.clear()
    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(c, per)) for c in ctxs]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    n0 = ctxs[0][1].n
    rec = {"contexts": contexts, "solves": per * contexts, "ms_per_solve": 1e3 * dt / (per * contexts),
           "value": float(n0) * sum(its) / dt, "unit": UNIT,
           "timing": "host wall clock around the worker threads (each ends with a stream "
                     "synchronisation); no L2 flush (the contexts' working sets exceed L2)"}
    for h, f, u in ctxs:
        del f, u
        h.close()
    return rec


def scaling_record(stmg, name, base, weak, world, rank, local, dist, steps, warmup):
    """Sub-record of one scaling curve at this N (the driver's per-N runs give
    the curve; efficiencies are computed by the reader, not here)."""
    import gc
    cfg = scaled(base, world, weak)
    h = make_hierarchy(stmg, cfg, world, rank, local, dist)
    f = local_inputs(stmg, h, cfg)
    u = h.local_vector()
    ccfg = stmg.CycleConfig(nu1=1, nu2=1, gamma=1, omega_t=0.5)
    n0 = f.n

    def step():
        from paper_1411_0519_b200 import _capi as A
        A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, n0 * 8))
        return h.solve(f, u, ccfg, EPS)

    for _ in range(warmup):
        step()
    barrier(dist, local)
    dev, its = [], []
    for _ in range(steps):
        r = step()
        if not r.converged:
            raise RuntimeError(f"{name}: solve did not converge")
        dev.append(r.device_time_seconds)
        its.append(r.iterations)
    barrier(dist, local)
    prof, _ = updown_profile(h, step)
    ms, nl, b = prof[0]
    gbs = (b / ((ms / nl) * 1e-3) / 1e9) if nl else None
    t = allreduce_max(dist, local, sum(dev))
    work = allreduce_sum(dist, local, float(n0 * sum(its)))
    rec = {
        "workload": CONFIGS[base]["desc"] + (f"; weak in time: N_t = {h.levels[0]['n_t']}, "
                                             f"T = {cfg['t_final']:g}" if weak else ""),
        "scaling": "weak" if weak else "strong", "n_gpus": world, "n_t": h.levels[0]["n_t"],
        "dofs": h.size(0), "dofs_per_gpu": n0, "iterations": its[0],
        "ms_per_solve": 1e3 * t / steps, "ms_per_vcycle": 1e3 * t / sum(its),
        "value": work / t, "unit": UNIT, "steps": steps, "warmup": warmup,
        "updown_gbs_per_rank": gather_obj(dist, gbs),
        "updown_ms_per_launch_rank0": (ms / nl) if nl else None,
    }
    if world == 1:
        h.fill_uniform(u, SEED + 1, 0)
        rec["operators"] = operator_record(h, f, u, reps=3)
    del f, u, h
    gc.collect()
    return rec


def run_ours(args, cfgname):
    import gc
    world, rank, local, dist = dist_setup(args.gpus)
    from paper_1411_0519_b200 import stmg
    from paper_1411_0519_b200 import _capi as A
    import ctypes as C
    # main line: configs[1] at N = 1; weak in time over N ranks (tau fixed)
    cfg = scaled(cfgname, world, weak=True)
    scaling = "weak" if world > 1 else "strong"
    parallelism = ("single GPU" if world == 1 else
                   f"time slabs x{world} (NCCL halo send/recv, coarse levels gathered on rank 0)")
    t_setup0 = time.perf_counter()
    h = make_hierarchy(stmg, cfg, world, rank, local, dist)
    t_created = time.perf_counter()
    L0 = h.levels[0]
    nlev = len(h.levels)
    f = local_inputs(stmg, h, cfg)
    n0 = f.n
    u = h.local_vector()
    ccfg = stmg.CycleConfig(nu1=1, nu2=1, gamma=1, omega_t=0.5)
    flush = C.c_void_p()
    A.check(A.lib().stmg_device_alloc(h._ctx, L2_FLUSH_BYTES, C.byref(flush)))

    def one_step():
        A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, n0 * 8))
        A.check(A.lib().stmg_memset_zero(h._ctx, flush, L2_FLUSH_BYTES))  # evict L2
        h.synchronize()
        return h.solve(f, u, ccfg, EPS)

    t_first0 = time.perf_counter()
    first = one_step()  # context setup: coarse operator, graph capture
    h.synchronize()
    setup = {"create_context_ms": 1e3 * (t_created - t_setup0),
             "first_solve_wall_ms": 1e3 * (time.perf_counter() - t_first0),
             "first_solve_device_ms": 1e3 * first.device_time_seconds,
             "note": "context creation includes the process's first CUDA module load; the "
                     "first solve builds the coarse operator (one launch) and captures the "
                     "solve graph"}
    for _ in range(max(args.warmup - 1, 0)):
        one_step()
    launches0 = h.launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    barrier(dist, local)
    h.synchronize()
    t_wall0 = time.perf_counter()
    dev_s, iters = [], []
    for _ in range(args.steps):
        rep = one_step()
        if not rep.converged:
            raise RuntimeError("solve did not converge")
        dev_s.append(rep.device_time_seconds)
        iters.append(rep.iterations)
    h.synchronize()
    barrier(dist, local)
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    launches = h.launch_count() - launches0
    # per-kernel durations: CUDA events on the library stream around the
    # level-0 fused kernels, in a replay of the same K steps (event nodes in
    # the cycle graph replace the device-side while loop, so they are kept out
    # of the timed region above)
    h.profile(True)
    h.profile_reset()
    prof_dev = []
    for _ in range(args.steps):
        prof_dev.append(one_step().device_time_seconds)
    prof = {k: h.profile_read(k) for k in (0, 1, 2)}
    h.profile(False)

    total_dev = allreduce_max(dist, local, sum(dev_s))
    work = allreduce_sum(dist, local, float(n0 * sum(iters)))
    value = work / total_dev
    ms_per_step = 1e3 * total_dev / args.steps

    # end to end through the C ABI with pinned host buffers
    hf, hu, hu2 = C.c_void_p(), C.c_void_p(), C.c_void_p()
    for p_ in (hf, hu, hu2):
        A.check(A.lib().stmg_host_alloc(h._ctx, n0 * 8, C.byref(p_)))
    arr = lambda p_: np.ctypeslib.as_array((C.c_double * n0).from_address(p_.value))  # noqa: E731
    hf_np, hu_np, hu2_np = arr(hf), arr(hu), arr(hu2)
    A.check(A.lib().stmg_download(h._ctx, hf.value, f.ptr, n0 * 8))
    # reference-shaped single call: solve(f, u) with u (the zero initial guess)
    # uploaded and the result downloaded, copies serialised with the solve
    e2e_s, e2e_it = [], []
    for k in range(args.warmup + args.steps):
        hu_np[:] = 0.0
        A.check(A.lib().stmg_memset_zero(h._ctx, flush, L2_FLUSH_BYTES))
        h.synchronize()
        barrier(dist, local)
        rep = h.solve_host(hf_np, hu_np, ccfg, EPS)
        if k >= args.warmup:
            e2e_s.append(rep.wall_time_seconds)
            e2e_it.append(rep.iterations)
    e2e1_total = allreduce_max(dist, local, sum(e2e_s))
    e2e1_work = allreduce_sum(dist, local, float(n0 * sum(e2e_it)))
    # the same solves streamed through stmg_solve_host_batch: step i+1's H2D
    # and step i-1's D2H run on the copy engines during solve i; zero initial
    # guess (nothing uploaded for it), so every step moves f in and u out
    outs = [hu_np, hu2_np]

    def batch(k):
        return h.solve_host_batch([hf_np] * k, [outs[i % 2] for i in range(k)], ccfg, EPS,
                                  u0s=[None] * k)

    batch(args.warmup)
    h.synchronize()
    barrier(dist, local)
    tb0 = time.perf_counter()
    breps = batch(args.steps)
    h.synchronize()
    tb = time.perf_counter() - tb0
    if not all(r.converged for r in breps):
        raise RuntimeError("batched solve did not converge")
    if [r.iterations for r in breps] != iters:
        raise RuntimeError("batched solves disagree with the device-resident solves")
    e2e_total = allreduce_max(dist, local, tb)
    e2e_work = allreduce_sum(dist, local, float(n0 * sum(r.iterations for r in breps)))
    for p_ in (hf, hu, hu2):
        A.lib().stmg_host_free(h._ctx, p_)

    peak, peak_kind = peaks()
    fused = prof[1][1] == 0  # fused schedule: slot 0 = k_updown, no standalone k_up
    names = ({0: "k_updown (level 0: post-smooth of cycle k + stop-test residual + pre-smooth "
                 "and restriction of cycle k+1, one pass)"} if fused else
             {0: "k_down (level 0: pre-smooth + residual + restrict)",
              1: "k_up (level 0: prolong + correct + post-smooth + residual norm)"})
    cands = [k for k in names if prof[k][1]]
    dom = max(cands, key=lambda k: prof[k][0])
    ms, nl, b = prof[dom]
    avg_s = (ms / nl) * 1e-3
    achieved = b / avg_s / 1e9
    tag = {0: "k_updown" if fused else "k_down", 1: "k_up"}[dom]
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic_from_profiles(tag),
            "kernel": names[dom], "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": b, "avg_launch_ms": avg_s * 1e3,
            "launches_per_step": nl / max(len(prof_dev), 1),
            # share of the TIMED (unprofiled) device time per step
            "step_share": (ms / max(len(prof_dev), 1)) / ms_per_step,
            "measured": "CUDA events on the library stream around every launch, in a replay of "
                        "the K timed steps right after the timed region",
            "transform_ms_per_solve": prof[2][0] / max(len(prof_dev), 1)}
    ops = None
    if world == 1:
        h.fill_uniform(u, SEED + 1, 0)
        ops = {cfgname: operator_record(h, f, u)}
    del f, u
    A.lib().stmg_device_free(h._ctx, flush)
    h.close()
    del h
    gc.collect()

    conc = None
    if world == 1 and not args.no_scaling:
        conc = concurrent_record(stmg, cfg, local, max(args.steps, 12))
        gc.collect()
    subs = {}
    if not args.no_scaling:
        subs["C3_strong"] = scaling_record(stmg, "C3_strong", "C3", False, world, rank, local,
                                           dist, args.scaling_steps, 1)
        subs["C4_strong"] = scaling_record(stmg, "C4_strong", "C4", False, world, rank, local,
                                           dist, args.scaling_steps, 1)
        subs["C5_weak"] = scaling_record(stmg, "C5_weak", "C5", True, world, rank, local, dist,
                                         args.scaling_steps, 1)
        if world == 1:
            for k_ in ("C3_strong", "C4_strong", "C5_weak"):
                ops[k_[:2]] = subs[k_].pop("operators")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 uniform[-1,1], f and u0)",
        "config": {"workload": cfg["desc"] + (f"; weak in time over {world} GPUs: N_t = "
                                              f"{L0['n_t']}, T = {cfg['t_final']:g}"
                                              if world > 1 else ""),
                   "dofs": sum(gather_obj(dist, n0)), "dofs_per_gpu": n0,
                   "n_t": L0["n_t"], "levels": nlev,
                   "cycle": "V(1,1), omega_t=0.5, exact DG block solves, mu-driven coarsening",
                   "eps": EPS, "step": "one full solve to 1e-8 incl. sine-basis transforms",
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB memset); vector {n0 * 8 / 1e6:.0f} MB",
                   "parallelism": parallelism,
                   "path": "spectral fused V-cycle; all cycles in one CUDA graph (conditional "
                           "while node, device-side stop test)"},
        "iterations": iters[0], "time_to_1e-8_ms": ms_per_step,
        "wall_ms_per_step_incl_flush": 1e3 * t_wall / args.steps,
        "setup": setup,
        "e2e": {"value": e2e_work / e2e_total, "unit": UNIT,
                "h2d_bytes_per_step": n0 * 8, "d2h_bytes_per_step": n0 * 8,
                "ms_per_step": 1e3 * e2e_total / args.steps,
                "api": "stmg_solve_host_batch (pinned host f in, u out, zero initial guess; H2D "
                       "of step i+1 and D2H of step i-1 overlap solve i; wall clock around the "
                       "K-step batch)",
                "single_call": {"value": e2e1_work / e2e1_total,
                                "unit": UNIT, "ms_per_step": 1e3 * e2e1_total / args.steps,
                                "h2d_bytes_per_step": 2 * n0 * 8, "d2h_bytes_per_step": n0 * 8,
                                "api": "stmg_solve_host (reference-shaped solve(f, u)), one call "
                                       "per step, f and u uploaded, u downloaded, copies "
                                       "serialised with the solve"}},
        "gpu_launches": int(launches),
        "roofline": roof,
        "operators": ops,
        "concurrent_problems": conc,
        "clocks": clk,
        "scaling_runs": subs,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        times, n0c = cpu_reference_cycles(CONFIGS[cfgname], args.cpu_cycles, 1)
        per = sum(times) / len(times)
        line["cpu_baseline"] = {
            "value": n0c / per, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{args.cpu_cycles} V(1,1) cycles (+ stop-test residual/norm each) of "
                      f"{cfgname} from a zero guess on the CPU oracle, 1 untimed, OpenMP over "
                      f"time steps; value = dofs / mean cycle time (same definition as "
                      f"--impl reference)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-cycles", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling-steps", type=int, default=3,
                    help="timed solves per scaling sub-record (C3 strong, C5 weak)")
    ap.add_argument("--no-scaling", action="store_true")
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args, argv)
    return run_ours(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
