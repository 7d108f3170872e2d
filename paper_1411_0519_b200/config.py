"""Run configuration and report I/O (reference config.hpp:12-44, config.cpp:38-193,
io.cpp:9-46): one JSON document per run, validated field by field with the
reference's field names and messages; JSON / CSV reports.

Differences from the reference, by design of this library: ``dim`` may also be 3
(the GPU path has 3D Q1).  ``block_solver = "vcycle"`` selects the inexact
spatial-V-cycle block solver: on the B200 path it is a field
of the cycle configuration (no per-level setup), so ``cycle_config`` carries it
together with ``omega_x``, ``nu1_x`` and ``nu2_x``.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from typing import List, Sequence

from .stmg import CycleConfig, SolveReport

K_MAX_TIME_DEGREE = 10  # dg_time.hpp:11
_POLICY = {"auto": 0, "semi": 1, "full": 2}  # CoarseningPolicy (mg.hpp:47)


@dataclass
class RunConfig:
    p_t: int = 0
    dim: int = 1
    space_levels: int = 4
    time_levels: int = 4
    t_final: float = 1.0
    omega_t: float = 0.5
    omega_x: float = 2.0 / 3.0
    nu1: int = 2
    nu2: int = 2
    nu1_x: int = 2
    nu2_x: int = 2
    gamma: int = 1
    eps_mg: float = 1e-8
    max_iter: int = 250
    seed: int = 0
    block_solver: str = "exact"  # "exact" | "vcycle"
    coarsening: str = "auto"     # "auto" | "semi" | "full"


def _bad(field: str, why: str):
    raise ValueError(f"config field '{field}': {why}")


def _get(j: dict, field: str, kind, default=None, required=True):
    if field not in j:
        if required:
            _bad(field, "missing")
        return default
    v = j[field]
    ok = {
        int: isinstance(v, int) and not isinstance(v, bool),
        float: isinstance(v, (int, float)) and not isinstance(v, bool),
        str: isinstance(v, str),
    }[kind]
    if not ok:
        _bad(field, "wrong type")
    return kind(v)


def parse_config(json_text: str) -> RunConfig:
    """Parse + validate (config.cpp:38-103); ValueError names the field."""
    try:
        j = json.loads(json_text)
    except json.JSONDecodeError as e:
        raise ValueError(f"config is not valid JSON: {e}") from None
    if not isinstance(j, dict):
        raise ValueError("config is not valid JSON: top level must be an object")
    c = RunConfig()
    c.p_t = _get(j, "p_t", int)
    c.dim = _get(j, "dim", int)
    c.space_levels = _get(j, "space_levels", int)
    c.time_levels = _get(j, "time_levels", int)
    c.t_final = _get(j, "T", float)
    c.omega_t = _get(j, "omega_t", float, 0.5, required=False)
    c.omega_x = _get(j, "omega_x", float)
    c.nu1 = _get(j, "nu1", int)
    c.nu2 = _get(j, "nu2", int)
    c.nu1_x = _get(j, "nu1_x", int)
    c.nu2_x = _get(j, "nu2_x", int)
    c.gamma = _get(j, "gamma", int, 1, required=False)
    c.eps_mg = _get(j, "eps_mg", float)
    c.max_iter = _get(j, "max_iter", int, 250, required=False)
    c.seed = _get(j, "seed", int)
    if c.seed < 0 or c.seed >= 2 ** 64:
        _bad("seed", "wrong type")
    c.block_solver = _get(j, "block_solver", str)
    if c.block_solver not in ("exact", "vcycle"):
        _bad("block_solver", "must be 'exact' or 'vcycle'")
    c.coarsening = _get(j, "coarsening", str)
    if c.coarsening not in _POLICY:
        _bad("coarsening", "must be 'auto', 'semi' or 'full'")
    if c.p_t < 0 or c.p_t > K_MAX_TIME_DEGREE:
        _bad("p_t", f"must be in [0, {K_MAX_TIME_DEGREE}]")
    if c.dim not in (1, 2, 3):
        _bad("dim", "must be 1, 2 or 3")
    if c.space_levels < 0:
        _bad("space_levels", "must be >= 0")
    if c.time_levels < 0:
        _bad("time_levels", "must be >= 0")
    if not c.t_final > 0.0:
        _bad("T", "must be > 0")
    if not 0.0 < c.omega_t <= 1.0:
        _bad("omega_t", "must be in (0, 1]")
    if not 0.0 < c.omega_x <= 1.0:
        _bad("omega_x", "must be in (0, 1]")
    if c.nu1 < 0:
        _bad("nu1", "must be >= 0")
    if c.nu2 < 0:
        _bad("nu2", "must be >= 0")
    if c.nu1 + c.nu2 == 0:
        _bad("nu1", "nu1 + nu2 must be >= 1")
    if c.nu1_x < 0:
        _bad("nu1_x", "must be >= 0")
    if c.nu2_x < 0:
        _bad("nu2_x", "must be >= 0")
    if c.gamma < 1:
        _bad("gamma", "must be >= 1")
    if not c.eps_mg > 0.0:
        _bad("eps_mg", "must be > 0")
    if c.max_iter < 1:
        _bad("max_iter", "must be >= 1")
    return c


def _as_dict(c: RunConfig) -> dict:
    return {"p_t": c.p_t, "dim": c.dim, "space_levels": c.space_levels,
            "time_levels": c.time_levels, "T": c.t_final, "omega_t": c.omega_t,
            "omega_x": c.omega_x, "nu1": c.nu1, "nu2": c.nu2, "nu1_x": c.nu1_x,
            "nu2_x": c.nu2_x, "gamma": c.gamma, "eps_mg": c.eps_mg, "max_iter": c.max_iter,
            "seed": c.seed, "block_solver": c.block_solver, "coarsening": c.coarsening}


def dump_config(c: RunConfig) -> str:
    """config.cpp:105-130: every field, two-space indent, trailing newline."""
    return json.dumps(_as_dict(c), indent=2) + "\n"


def hierarchy_params(c: RunConfig) -> dict:
    """Keyword arguments of stmg.Hierarchy (config.cpp:132-143; mu* = critical_mu)."""
    return {"p_t": c.p_t, "dim": c.dim, "space_level": c.space_levels,
            "time_level": c.time_levels, "t_final": c.t_final, "mu_star": 0.0,
            "policy": _POLICY[c.coarsening]}


def cycle_config(c: RunConfig) -> CycleConfig:
    """config.cpp:145-156."""
    return CycleConfig(nu1=c.nu1, nu2=c.nu2, gamma=c.gamma, omega_t=c.omega_t,
                       block_solver=c.block_solver, omega_x=c.omega_x, nu1_x=c.nu1_x,
                       nu2_x=c.nu2_x)


def solve_report_json(c: RunConfig, r: SolveReport) -> str:
    """config.cpp:158-168."""
    j = {"config": _as_dict(c), "iterations": r.iterations, "converged": bool(r.converged),
         "wall_time_seconds": r.wall_time_seconds, "seed": r.seed,
         "residual_history": list(r.residual_history)}
    return json.dumps(j, indent=2) + "\n"


def format_double(v: float) -> str:
    """Shortest round-trip decimal (io.cpp:9-13, std::to_chars)."""
    return repr(float(v))


class CsvWriter:
    """io.cpp:15-40: header + rows with a fixed column count."""

    def __init__(self, header: Sequence[str]):
        self._cols = len(header)
        self._out = ",".join(header) + "\n"
        self._row: List[str] = []

    def cell(self, v) -> "CsvWriter":
        if isinstance(v, float):
            v = format_double(v)
        self._row.append(str(v))
        return self

    def end_row(self) -> None:
        if len(self._row) != self._cols:
            raise RuntimeError("csv row has wrong number of cells")
        self._out += ",".join(self._row) + "\n"
        self._row = []

    def str(self) -> str:
        return self._out


def residual_history_csv(r: SolveReport) -> str:
    """config.cpp:170-178."""
    w = CsvWriter(["iteration", "residual_l2"])
    for k, v in enumerate(r.residual_history):
        w.cell(k).cell(float(v)).end_row()
    return w.str()


@dataclass
class ScalingRecord:
    """bench.hpp:52-60 (threads -> GPUs here)."""
    threads: int
    n_t: int
    n_x: int
    p_t: int
    iterations: int
    wall_time_seconds: float
    fwd_sub_seconds: float = 0.0


def scaling_csv(records: Sequence[ScalingRecord], with_forward_substitution_column: bool) -> str:
    """config.cpp:180-193."""
    header = ["threads", "n_t", "n_x", "p_t", "iterations", "wall_time_seconds"]
    if with_forward_substitution_column:
        header.append("fwd_sub_seconds")
    w = CsvWriter(header)
    for r in records:
        w.cell(r.threads).cell(r.n_t).cell(r.n_x).cell(r.p_t).cell(r.iterations)
        w.cell(float(r.wall_time_seconds))
        if with_forward_substitution_column:
            w.cell(float(r.fwd_sub_seconds))
        w.end_row()
    return w.str()
