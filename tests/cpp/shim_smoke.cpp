// Uses the C++ shim exactly like a caller of the reference stmg:: API would
// (mg.hpp / st_system.hpp / smoother.hpp / transfer.hpp) and prints a JSON
// line; run on a GPU by tests/test_gpu_parity.py::test_cpp_shim_solves_c1.
#include <cmath>
#include <cstdio>

#include "stmg_b200.hpp"

int main() {
  using namespace stmg;
  HierarchyParams p;
  p.p_t = 1;
  p.dim = 1;
  p.space_level = 5;
  p.time_level = 6;
  p.t_final = 1.0;
  p.mu_star = lfa::critical_mu(1);
  const STHierarchy h = build_hierarchy(p);
  const STOperator op = h.finest().op();
  BlockVector f = make_vector(op), u = make_vector(op), r = make_vector(op);
  fill_uniform(f, 42, 0);
  CycleConfig cfg;
  cfg.nu1 = cfg.nu2 = 1;
  const SolveReport rep = solve(h, f, u, cfg, 1e-8);
  residual(op, u, f, r);
  const double rel = norm(op, r) / norm(op, f);
  // the paper's inexact variant: one spatial V-cycle per block (smoother.hpp:15-24)
  CycleConfig icfg = cfg;
  icfg.smoother.block_solver = BlockSolverKind::spatial_vcycle;
  BlockVector ui = make_vector(op);
  const SolveReport irep = solve(h, f, ui, icfg, 1e-8);
  const SpatialVCycleSolver vc(op);
  const BlockVector x = vc.cycle(f, nullptr, icfg.smoother);
  // reference-signature overloads (smoother.hpp:68-70, st_system.hpp:70-72, transfer.hpp:27-44)
  const BlockSolver lu(op);
  const SpatialVCycleSolver svc(op);
  BlockSolveContext bctx;
  bctx.exact = &lu;
  bctx.vcycle = &svc;
  BlockVector us = make_vector(op);
  fill_random(us, 7);  // mt19937_64, [0, 1) (mg.cpp:168-173)
  block_jacobi_step(op, bctx, us, f, cfg.smoother);
  const BlockVector fs = forward_substitution_solve(op, lu, f);
  const TimeTransfer tt = build_time_transfer(p.p_t, 1.0);
  const SpaceGrid g0 = build_space_grid(1, p.space_level), g1 = build_space_grid(1, p.space_level - 1);
  const BlockVector rf = restrict_full(tt, g0, g1, us);
  const BlockVector pf = prolong_full(tt, g1, g0, rf);
  const bool overloads_ok = rf.n_t() == us.n_t() / 2 && rf.n_x() == g1.n_nodes &&
                            pf.size() == us.size() && fs.size() == f.size();
  bool threw = false;
  try {
    BlockVector odd(op.ctx, 3, 63, 2);
    (void)restrict_semi(STOperator{op.ctx, int(h.levels.size()) - 1}, odd);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  std::printf("{\"iterations\": %d, \"converged\": %d, \"rel_residual\": %.17g, \"levels\": %zu, \"threw\": %d, \"inexact_iterations\": %d, \"inexact_converged\": %d, \"vcycle_size\": %lld, \"overloads_ok\": %d}\n",
              rep.iterations, int(rep.converged), rel, h.levels.size(), int(threw),
              irep.iterations, int(irep.converged), (long long)x.size(), int(overloads_ok));
  return rep.converged && rel <= 1e-8 && threw && irep.converged && overloads_ok ? 0 : 1;
}
