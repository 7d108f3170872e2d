"""Host-side mirror of the reference ``stmg::`` API over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/stmg/*.hpp): invalid arguments raise
``ValueError`` (the reference's ``std::invalid_argument``), CUDA/runtime
failures raise ``RuntimeError``.  Vectors live on the GPU (``BlockVector``
wraps a device allocation in the reference layout, block_vector.hpp:12-29).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as A
from ._capi import check

COARSEN_NONE, COARSEN_SEMI, COARSEN_FULL = 0, 1, 2
POLICY_MU_DRIVEN, POLICY_ALWAYS_SEMI, POLICY_PREFER_FULL = 0, 1, 2


def _pd(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(A.PD)


def critical_mu(p_t: int) -> float:
    """lfa::critical_mu (lfa.cpp:317-328)."""
    v = A.lib().stmg_critical_mu(p_t)
    if v != v:
        check(A.STMG_EINVAL)
    return v


def fill_random_host(n: int, seed: int) -> np.ndarray:
    """fill_random (mg.cpp:168-173), reference-exact: std::mt19937_64(seed),
    v[i] = (gen() >> 11) * 2^-53 in [0, 1); host only."""
    v = np.empty(int(n))
    check(A.lib().stmg_fill_random_host(v.ctypes.data, int(n), int(seed)))
    return v


def assemble_dg_block(p_t: int, tau: float):
    """assemble_dg_block (dg_time.cpp:125-166) -> (K, M, N)."""
    n = max(p_t + 1, 1)
    K, M, N = np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n))
    check(A.lib().stmg_dg_block(p_t, tau, _pd(K), _pd(M), _pd(N)))
    return K, M, N


def build_time_transfer(p_t: int, tau: float):
    """build_time_transfer (transfer.cpp:50-73) -> (R1, R2)."""
    n = max(p_t + 1, 1)
    R1, R2 = np.zeros((n, n)), np.zeros((n, n))
    check(A.lib().stmg_time_transfer(p_t, tau, _pd(R1), _pd(R2)))
    return R1, R2


def shard_plan(p_t: int, dim: int, space_level: int, time_level: int, shards: int,
               t_final: float = 1.0, mu_star: float = 0.0, policy: int = POLICY_MU_DRIVEN):
    """(gather level, finest steps per shard) of the time-slab decomposition."""
    prm = A.HierarchyParams(p_t, dim, space_level, time_level, t_final, mu_star, policy, 0, 0, 0)
    lg, n = C.c_int(), C.c_int64()
    check(A.lib().stmg_shard_plan(C.byref(prm), shards, C.byref(lg), C.byref(n)))
    return lg.value, n.value


@dataclass
class CycleConfig:
    """CycleConfig + SmootherConfig (mg.hpp:66-71, smoother.hpp:15-24)."""
    nu1: int = 2
    nu2: int = 2
    gamma: int = 1
    omega_t: float = 0.5
    path: str = "spectral"  # or "physical"
    block_solver: str = "exact"  # or "vcycle" (BlockSolverKind::spatial_vcycle)
    omega_x: float = 2.0 / 3.0
    nu1_x: int = 2
    nu2_x: int = 2
    gamma_x: int = 1

    def c(self) -> A.CycleConfig:
        if self.path not in ("spectral", "physical"):
            raise ValueError("unknown cycle path")
        return A.CycleConfig(self.nu1, self.nu2, self.gamma, self.omega_t,
                             A.PATH_SPECTRAL if self.path == "spectral" else A.PATH_PHYSICAL,
                             block_solver_kind(self.block_solver), self.omega_x, self.nu1_x,
                             self.nu2_x, self.gamma_x)


def block_solver_kind(name) -> int:
    """'exact' -> 0, 'vcycle' -> 1 (config.cpp:64-70 spellings)."""
    if name in ("exact", 0):
        return BLOCK_EXACT
    if name in ("vcycle", "spatial_vcycle", 1):
        return BLOCK_VCYCLE
    raise ValueError("block_solver must be 'exact' or 'vcycle'")


BLOCK_EXACT = 0
BLOCK_VCYCLE = 1


@dataclass
class SmootherConfig:
    """SmootherConfig (smoother.hpp:15-24)."""
    omega_t: float = 0.5
    nu: int = 1
    block_solver: str = "exact"
    omega_x: float = 2.0 / 3.0
    nu1_x: int = 2
    nu2_x: int = 2
    gamma_x: int = 1

    def c(self) -> A.SmootherConfig:
        return A.SmootherConfig(self.omega_t, self.nu, block_solver_kind(self.block_solver),
                                self.omega_x, self.nu1_x, self.nu2_x, self.gamma_x)


@dataclass
class SolveReport:
    """SolveReport (mg.hpp:83-89)."""
    iterations: int = 0
    converged: bool = False
    residual_history: List[float] = field(default_factory=list)
    wall_time_seconds: float = 0.0
    device_time_seconds: float = 0.0
    seed: int = 0


class BlockVector:
    """Device-resident space-time vector (n_t, n_loc, n_x), reference layout."""

    def __init__(self, hier: "Hierarchy", n: int, shape):
        self.hier = hier
        self.n = int(n)
        self.shape = tuple(shape)
        p = C.c_void_p()
        check(A.lib().stmg_device_alloc(hier._ctx, self.n * 8, C.byref(p)))
        self.ptr = p.value
        check(A.lib().stmg_memset_zero(hier._ctx, self.ptr, self.n * 8))

    def __del__(self):
        if getattr(self, "ptr", None) and self.hier._ctx:
            A.lib().stmg_device_free(self.hier._ctx, self.ptr)
            self.ptr = None

    def numpy(self) -> np.ndarray:
        out = np.empty(self.n)
        check(A.lib().stmg_download(self.hier._ctx, out.ctypes.data, self.ptr, self.n * 8))
        return out

    def copy_from(self, a: np.ndarray) -> "BlockVector":
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        if a.size != self.n:
            raise ValueError("space-time vector shape mismatch")
        check(A.lib().stmg_upload(self.hier._ctx, self.ptr, a.ctypes.data, self.n * 8))
        check(A.lib().stmg_synchronize(self.hier._ctx))
        return self


class Hierarchy:
    """STHierarchy (mg.hpp:38-45) + device context; build_hierarchy when
    two_grid == 0, build_two_grid(mode) otherwise (mg.cpp:10-94)."""

    def __init__(self, p_t: int, dim: int, space_level: int, time_level: int,
                 t_final: float = 1.0, mu_star: float = 0.0, policy: int = POLICY_MU_DRIVEN,
                 two_grid: int = 0, device: int = 0, shards: int = 0,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        """shards > 1: time-slab sharding emulated on one device; world > 1:
        one rank per GPU over NCCL (nccl_id from unique_id() on rank 0)."""
        self._ctx = None
        prm = A.HierarchyParams(p_t, dim, space_level, time_level, t_final, mu_star, policy,
                                two_grid, device, shards)
        ctx = C.c_void_p()
        if world > 1 or nccl_id is not None:
            if nccl_id is None:
                raise ValueError("world > 1 needs the NCCL id of rank 0")
            check(A.lib().stmg_create_distributed(C.byref(prm), rank, world, nccl_id,
                                                  len(nccl_id), C.byref(ctx)))
        else:
            check(A.lib().stmg_create(C.byref(prm), C.byref(ctx)))
        self._ctx = ctx
        self.rank, self.world = rank, world
        n = C.c_int()
        check(A.lib().stmg_num_levels(ctx, C.byref(n)))
        self.levels = []
        for i in range(n.value):
            li = A.LevelInfo()
            check(A.lib().stmg_get_level_info(ctx, i, C.byref(li)))
            self.levels.append({k: getattr(li, k) for k, _ in A.LevelInfo._fields_})
        self.p_t, self.dim = p_t, dim

    def close(self):
        if self._ctx:
            A.lib().stmg_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def unique_id() -> bytes:
        """NCCL unique id for stmg_create_distributed (call on rank 0)."""
        buf = C.create_string_buffer(128)
        check(A.lib().stmg_nccl_unique_id(buf, 128))
        return buf.raw

    def local_steps(self):
        a, b = C.c_int64(), C.c_int64()
        check(A.lib().stmg_local_steps(self._ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def local_vector(self) -> "BlockVector":
        """This rank's finest-level time slabs (whole vector if not distributed)."""
        L = self.levels[0]
        _, n = self.local_steps()
        return BlockVector(self, n * L["n_loc"] * L["n_x"], (n, L["n_loc"], L["n_x"]))

    # ---- vectors ----------------------------------------------------------
    def _lev(self, level: int) -> dict:
        if not 0 <= level < len(self.levels):
            raise ValueError("level index out of range")
        return self.levels[level]

    def size(self, level: int = 0) -> int:
        L = self._lev(level)
        return L["n_t"] * L["n_loc"] * L["n_x"]

    def vector(self, level: int = 0) -> BlockVector:
        L = self._lev(level)
        return BlockVector(self, self.size(level), (L["n_t"], L["n_loc"], L["n_x"]))

    def coarse_vector(self, level: int, mode: int = 0) -> BlockVector:
        L = self._lev(level)
        mode = mode or L["coarsen_to_next"]
        n1 = L["n1"] if mode == COARSEN_SEMI else (L["n1"] - 1) // 2
        nx = n1 ** L["dim"]
        return BlockVector(self, (L["n_t"] // 2) * L["n_loc"] * nx, (L["n_t"] // 2, L["n_loc"], nx))

    def upload(self, a: np.ndarray, level: int = 0) -> BlockVector:
        return self.vector(level).copy_from(a)

    # ---- operators (reference entry points) --------------------------------
    def apply(self, level: int, u: BlockVector, y: Optional[BlockVector] = None) -> BlockVector:
        y = y or self.vector(level)
        check(A.lib().stmg_apply(self._ctx, level, u.ptr, y.ptr))
        return y

    def residual(self, level: int, u: BlockVector, f: BlockVector,
                 r: Optional[BlockVector] = None) -> BlockVector:
        r = r or self.vector(level)
        check(A.lib().stmg_residual(self._ctx, level, u.ptr, f.ptr, r.ptr))
        return r

    def norm(self, level: int, v: BlockVector) -> float:
        out = C.c_double()
        check(A.lib().stmg_norm(self._ctx, level, v.ptr, C.byref(out)))
        return out.value

    def block_solve(self, level: int, b: BlockVector, x: Optional[BlockVector] = None) -> BlockVector:
        x = x or self.vector(level)
        check(A.lib().stmg_block_solve(self._ctx, level, b.ptr, x.ptr))
        return x

    def block_jacobi_step(self, level: int, u: BlockVector, f: BlockVector,
                          omega_t: float = 0.5, nu: int = 1,
                          cfg: Optional[SmootherConfig] = None) -> BlockVector:
        """block_jacobi_step (smoother.cpp:96-106); cfg selects the block solver."""
        if cfg is None:
            check(A.lib().stmg_smooth(self._ctx, level, u.ptr, f.ptr, omega_t, nu))
        else:
            sc = cfg.c()
            check(A.lib().stmg_block_jacobi_step(self._ctx, level, u.ptr, f.ptr, C.byref(sc)))
        return u

    def spatial_vcycle(self, level: int, b: BlockVector, x0: Optional[BlockVector] = None,
                       x: Optional[BlockVector] = None,
                       cfg: Optional[SmootherConfig] = None) -> BlockVector:
        """SpatialVCycleSolver::cycle on every time step (smoother.cpp:71-78)."""
        x = x or self.vector(level)
        sc = (cfg or SmootherConfig(block_solver="vcycle")).c()
        check(A.lib().stmg_spatial_vcycle(self._ctx, level, b.ptr, x0.ptr if x0 else None,
                                          x.ptr, C.byref(sc)))
        return x

    def restrict(self, level: int, fine: BlockVector, mode: int = 0) -> BlockVector:
        out = self.coarse_vector(level, mode)
        check(A.lib().stmg_restrict(self._ctx, level, mode, fine.ptr, out.ptr))
        return out

    def prolong(self, level: int, coarse: BlockVector, mode: int = 0) -> BlockVector:
        out = self.vector(level)
        check(A.lib().stmg_prolong(self._ctx, level, mode, coarse.ptr, out.ptr))
        return out

    def forward_substitution_solve(self, level: int, f: BlockVector) -> BlockVector:
        u = self.vector(level)
        check(A.lib().stmg_forward_substitution(self._ctx, level, f.ptr, u.ptr))
        return u

    def mg_cycle(self, level: int, u: BlockVector, f: BlockVector, cfg: CycleConfig) -> BlockVector:
        c = cfg.c()
        check(A.lib().stmg_mg_cycle(self._ctx, level, u.ptr, f.ptr, C.byref(c)))
        return u

    def solve(self, f: BlockVector, u: BlockVector, cfg: CycleConfig, eps_mg: float,
              max_iter: int = 250) -> SolveReport:
        c = cfg.c()
        hist = np.zeros(max_iter + 1)
        rep = A.SolveReport()
        check(A.lib().stmg_solve(self._ctx, f.ptr, u.ptr, C.byref(c), eps_mg, max_iter,
                                 _pd(hist), len(hist), C.byref(rep)))
        return SolveReport(rep.iterations, bool(rep.converged),
                           hist[: rep.iterations + 1].tolist(), rep.wall_time_seconds,
                           rep.device_time_seconds, rep.seed)

    def solve_host(self, f: np.ndarray, u: np.ndarray, cfg: CycleConfig, eps_mg: float,
                   max_iter: int = 250) -> SolveReport:
        """solve() on HOST arrays (u updated in place); H2D/D2H inside."""
        assert f.dtype == np.float64 and u.dtype == np.float64
        _, n = self.local_steps()
        local = n * self.levels[0]["n_loc"] * self.levels[0]["n_x"]
        if f.size != local or u.size != local:
            raise ValueError("space-time vector shape mismatch")
        c = cfg.c()
        hist = np.zeros(max_iter + 1)
        rep = A.SolveReport()
        check(A.lib().stmg_solve_host(self._ctx, f.ctypes.data, u.ctypes.data, C.byref(c), eps_mg,
                                      max_iter, _pd(hist), len(hist), C.byref(rep)))
        return SolveReport(rep.iterations, bool(rep.converged),
                           hist[: rep.iterations + 1].tolist(), rep.wall_time_seconds,
                           rep.device_time_seconds, rep.seed)

    def solve_host_batch(self, fs, us, cfg: CycleConfig, eps_mg: float, max_iter: int = 250,
                         u0s=None) -> List[SolveReport]:
        """Independent solves of HOST arrays streamed through the context
        (stmg_solve_host_batch): problem i+1's upload and problem i-1's download
        overlap solve i.  us[i] is updated in place, or written from u0s[i]
        (None: zero initial guess, no upload)."""
        _, n = self.local_steps()
        local = n * self.levels[0]["n_loc"] * self.levels[0]["n_x"]
        k = len(fs)
        if len(us) != k or (u0s is not None and len(u0s) != k):
            raise ValueError("batch length mismatch")
        for a in list(fs) + list(us) + [a for a in (u0s or []) if a is not None]:
            if a.dtype != np.float64 or a.size != local or not a.flags.c_contiguous:
                raise ValueError("space-time vector shape mismatch")
        P = C.c_void_p * max(k, 1)
        pf = P(*[a.ctypes.data for a in fs])
        pu = P(*[a.ctypes.data for a in us])
        # a None entry of u0s: zero initial guess (nothing uploaded)
        p0 = P(*[a.ctypes.data if a is not None else None for a in u0s]) if u0s is not None else None
        reps = (A.SolveReport * max(k, 1))()
        c = cfg.c()
        check(A.lib().stmg_solve_host_batch(self._ctx, k, pf, p0, pu, C.byref(c), eps_mg, max_iter,
                                            reps))
        return [SolveReport(r.iterations, bool(r.converged), [r.r0, r.r_final][: r.iterations + 1],
                            r.wall_time_seconds, r.device_time_seconds, r.seed)
                for r in reps[:k]]

    # ---- inputs ----------------------------------------------------------------
    def fill_random(self, v: BlockVector, seed: int) -> BlockVector:
        """fill_random(v, seed) of the reference (mg.cpp:168-173), bit-exact."""
        return v.copy_from(fill_random_host(v.n, seed))

    def fill_uniform(self, v: BlockVector, seed: int, stream: int, offset: int = 0) -> BlockVector:
        check(A.lib().stmg_fill_uniform(self._ctx, v.ptr, v.n, seed, stream, offset))
        return v

    def fold_u0(self, f: BlockVector, u0: BlockVector) -> BlockVector:
        check(A.lib().stmg_fold_u0(self._ctx, f.ptr, u0.ptr))
        return f

    # ---- profiling --------------------------------------------------------------
    def profile(self, on: bool = True) -> None:
        check(A.lib().stmg_profile_enable(self._ctx, int(on)))

    def profile_read(self, kernel_id: int):
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        check(A.lib().stmg_profile_read(self._ctx, kernel_id, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def profile_reset(self) -> None:
        check(A.lib().stmg_profile_reset(self._ctx))

    def launch_count(self) -> int:
        n = C.c_int64()
        check(A.lib().stmg_launch_count(self._ctx, C.byref(n)))
        return n.value

    def synchronize(self) -> None:
        check(A.lib().stmg_synchronize(self._ctx))
