"""Two-grid convergence factor measured on the GPU vs the LFA prediction
(the reference's measure_convergence_factor, bench.cpp:77-145,
and its acceptance |measured - predicted| <= 0.05)."""
import pytest


@pytest.mark.gpu
@pytest.mark.parametrize("p_t,mu,mode", [(0, 1.0, 1), (1, 0.5, 1), (1, 10.0, 1), (0, 2.0, 2),
                                         (1, 1.0, 2), (2, 0.8, 2)])
def test_measured_twogrid_factor_matches_lfa(p_t, mu, mode):
    from paper_1411_0519_b200 import build, lfa, stmg
    build.build()
    cfg = stmg.CycleConfig(nu1=1, nu2=1)
    m = lfa.measure_convergence_factor(p_t, 1, 7, 6, mu, mode, cfg, seed=42,
                                       n_theta_x=128, n_theta_t=128)
    assert m.n_iterations_used >= 3
    assert 0.0 < m.measured_rho < 1.0
    assert abs(m.measured_rho - m.predicted_rho) <= 0.05, (m.measured_rho, m.predicted_rho)


@pytest.mark.gpu
@pytest.mark.parametrize("p_t,mu,mode", [(0, 1.0, 1), (1, 10.0, 1), (1, 1.0, 2), (1, 4.0, 2)])
def test_measured_inexact_twogrid_factor(p_t, mu, mode):
    """Two-grid cycles with spatial-V-cycle block solves (f2) vs the LFA
    inexact-block factor (lfa.cpp twogrid_factor_inexact; its spatial part is a
    two-grid model of the V-cycle; measured within 0.01 on B200)."""
    from paper_1411_0519_b200 import build, lfa, stmg
    build.build()
    cfg = stmg.CycleConfig(nu1=1, nu2=1, block_solver="vcycle")
    m = lfa.measure_convergence_factor(p_t, 1, 7, 6, mu, mode, cfg, seed=42,
                                       n_theta_x=128, n_theta_t=128)
    exact = lfa.measure_convergence_factor(p_t, 1, 7, 6, mu, mode, stmg.CycleConfig(nu1=1, nu2=1),
                                           seed=42, n_theta_x=128, n_theta_t=128)
    assert 0.0 < m.measured_rho < 1.0
    assert abs(m.measured_rho - m.predicted_rho) <= 0.05, (m.measured_rho, m.predicted_rho)
    assert m.measured_rho >= exact.measured_rho - 0.02


@pytest.mark.gpu
def test_measurement_bad_arguments():
    from paper_1411_0519_b200 import build, lfa, stmg
    build.build()
    with pytest.raises(ValueError):
        lfa.measure_convergence_factor(1, 1, 5, 4, -1.0, 1, stmg.CycleConfig())
    with pytest.raises(ValueError):
        lfa.measure_convergence_factor(1, 1, 5, 4, 1.0, 0, stmg.CycleConfig())
