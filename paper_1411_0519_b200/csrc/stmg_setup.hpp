// stmg_setup.hpp -- host-side discretisation setup of the B200 library:
// DG(p_t) time blocks, Pade stability / critical mu, time transfer blocks and
// the mu-driven level ladder.  Tiny, runs once per context.
#pragma once

#include <cstdint>
#include <vector>

namespace stmg {

constexpr int kMaxTimeDegree = 10;  // reference dg_time.hpp:11

// Row-major (p_t+1)^2 blocks of one DG time step on (0, tau), Legendre basis
// (dg_time.hpp:14-26): K[k,l] = -int psi_l psi_k' + psi_l(tau) psi_k(tau),
// M[k,l] = int psi_l psi_k, N[k,l] = psi_l(tau) psi_k(0).
struct DGBlock {
  int p = 0;
  double tau = 1.0;
  std::vector<double> K, M, N;
};

DGBlock dg_block(int p_t, double tau);
// (p_t, p_t+1) Pade approximant of e^z at real z (dg_time.cpp:168-198).
double pade_stability(int p_t, double z);
// R(-3 mu*) = sqrt(2) - 1 by bisection (lfa.cpp:317-328).
double critical_mu(int p_t);
// R1, R2 row-major: coarse step n <- R1 fine_2n + R2 fine_2n+1 (transfer.cpp:50-73).
void time_transfer(int p_t, double tau, std::vector<double>& R1, std::vector<double>& R2);
double legendre(int n, double x);

struct LevelSpec {
  int64_t n_t = 1;
  int space_level = 0;
  int dim = 1;
  int p_t = 0;
  double tau = 1.0, h = 0.5, mu = 0.0;
  int coarsen = 0;  // 0 none, 1 semi, 2 full
  int64_t n1() const { return (int64_t(1) << (space_level + 1)) - 1; }
  int64_t nx() const {
    int64_t v = 1;
    for (int a = 0; a < dim; ++a) v *= n1();
    return v;
  }
  int64_t size() const { return n_t * int64_t(p_t + 1) * nx(); }
};

// build_hierarchy / build_two_grid ladder (mg.cpp:10-94); throws
// std::invalid_argument like the reference.
std::vector<LevelSpec> build_ladder(int p_t, int dim, int space_level, int time_level,
                                    double t_final, double mu_star, int policy, int two_grid);

}  // namespace stmg
