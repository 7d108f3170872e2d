"""Run configuration / report I/O (reference config.cpp:38-193, io.cpp:9-46;
SURVEY.md 8(f)3).  CPU, except the last test (one solve from a config)."""
import json

import numpy as np
import pytest

GOOD = {"p_t": 1, "dim": 2, "space_levels": 4, "time_levels": 5, "T": 1.0, "omega_x": 0.6667,
        "nu1": 1, "nu2": 1, "nu1_x": 2, "nu2_x": 2, "eps_mg": 1e-8, "seed": 7,
        "block_solver": "exact", "coarsening": "auto"}


@pytest.fixture(scope="module")
def Cfg():
    from paper_1411_0519_b200 import build
    build.build()
    from paper_1411_0519_b200 import config
    return config


def test_parse_defaults_and_roundtrip(Cfg):
    c = Cfg.parse_config(json.dumps(GOOD))
    assert (c.omega_t, c.gamma, c.max_iter) == (0.5, 1, 250)  # documented defaults
    assert c.t_final == 1.0 and c.seed == 7
    again = Cfg.parse_config(Cfg.dump_config(c))
    assert again == c
    assert Cfg.dump_config(c).endswith("\n")


@pytest.mark.parametrize("field,value,msg", [
    ("p_t", 11, "must be in [0, 10]"), ("dim", 4, "must be 1, 2 or 3"),
    ("space_levels", -1, "must be >= 0"), ("T", 0.0, "must be > 0"),
    ("omega_x", 1.5, "must be in (0, 1]"), ("nu1", -1, "must be >= 0"),
    ("eps_mg", 0.0, "must be > 0"), ("block_solver", "lu", "must be 'exact' or 'vcycle'"),
    ("coarsening", "x", "must be 'auto', 'semi' or 'full'"), ("p_t", "1", "wrong type"),
    ("omega_t", 0.0, "must be in (0, 1]"), ("gamma", 0, "must be >= 1"),
    ("max_iter", 0, "must be >= 1")])
def test_validation_names_the_field(Cfg, field, value, msg):
    j = dict(GOOD)
    j[field] = value
    with pytest.raises(ValueError) as e:
        Cfg.parse_config(json.dumps(j))
    assert f"config field '{field}'" in str(e.value) and msg in str(e.value)


def test_missing_field_and_bad_json(Cfg):
    j = dict(GOOD)
    del j["seed"]
    with pytest.raises(ValueError, match="config field 'seed': missing"):
        Cfg.parse_config(json.dumps(j))
    with pytest.raises(ValueError, match="not valid JSON"):
        Cfg.parse_config("{p_t: 1")
    j = dict(GOOD, nu1=0, nu2=0)
    with pytest.raises(ValueError, match="nu1 \\+ nu2 must be >= 1"):
        Cfg.parse_config(json.dumps(j))


def test_mapping_to_library_params(Cfg):
    c = Cfg.parse_config(json.dumps(dict(GOOD, coarsening="semi", nu1=2, gamma=2)))
    hp = Cfg.hierarchy_params(c)
    assert hp["policy"] == 1 and hp["space_level"] == 4 and hp["time_level"] == 5
    cc = Cfg.cycle_config(c)
    assert (cc.nu1, cc.nu2, cc.gamma, cc.omega_t) == (2, 1, 2, 0.5)
    ci = Cfg.cycle_config(Cfg.parse_config(json.dumps(dict(GOOD, block_solver="vcycle",
                                                          omega_x=0.6, nu1_x=1, nu2_x=3))))
    assert (ci.block_solver, ci.omega_x, ci.nu1_x, ci.nu2_x) == ("vcycle", 0.6, 1, 3)
    assert ci.c().block_solver == 1 and cc.c().block_solver == 0


def test_reports_and_csv(Cfg):
    from paper_1411_0519_b200.stmg import SolveReport
    c = Cfg.parse_config(json.dumps(GOOD))
    r = SolveReport(iterations=2, converged=True, residual_history=[1.0, 0.1, 0.01],
                    wall_time_seconds=0.5, seed=7)
    j = json.loads(Cfg.solve_report_json(c, r))
    assert j["iterations"] == 2 and j["converged"] is True and j["config"]["seed"] == 7
    assert j["residual_history"] == [1.0, 0.1, 0.01]
    csv = Cfg.residual_history_csv(r).splitlines()
    assert csv[0] == "iteration,residual_l2" and csv[2] == "1,0.1"
    recs = [Cfg.ScalingRecord(1, 64, 63, 1, 10, 0.25, 0.125)]
    s = Cfg.scaling_csv(recs, True).splitlines()
    assert s[0].endswith(",fwd_sub_seconds") and s[1] == "1,64,63,1,10,0.25,0.125"
    w = Cfg.CsvWriter(["a", "b"])
    w.cell(1)
    with pytest.raises(RuntimeError):
        w.end_row()


@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["exact", "vcycle"])
def test_solve_from_config_matches_oracle(Cfg, solver):
    from oracle import oracle as O
    from paper_1411_0519_b200 import stmg
    c = Cfg.parse_config(json.dumps(dict(GOOD, dim=1, space_levels=5, time_levels=6,
                                         block_solver=solver)))
    h = stmg.Hierarchy(**Cfg.hierarchy_params(c))
    o = O.Hierarchy(c.p_t, c.dim, c.space_levels, c.time_levels, t_final=c.t_final)
    f = O.fill_uniform(o.levels[0].size, c.seed, 0)
    u = h.vector(0)
    r = h.solve(h.upload(f), u, Cfg.cycle_config(c), c.eps_mg, c.max_iter)
    u_o, rep_o = o.solve(f, nu1=c.nu1, nu2=c.nu2, eps=c.eps_mg, block_solver=solver,
                         omega_x=c.omega_x, nu1_x=c.nu1_x, nu2_x=c.nu2_x)
    assert r.iterations == rep_o["iterations"]
    assert np.abs(u.numpy() - u_o).max() <= 1e-10 * np.abs(u_o).max()
    j = json.loads(Cfg.solve_report_json(c, r))
    assert j["iterations"] == r.iterations
