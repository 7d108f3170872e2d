// stmg_lfa.hpp -- local Fourier analysis of the space-time two-grid method
// (reference lfa.hpp:15-150).  Host only.
#pragma once

namespace stmg::lfa {

// beta(tx) = 6 (1 - cos tx)/(2 + cos tx) (lfa.hpp:15-17).
double beta(double theta_x);
// alpha = R(-mu beta(tx)), the Pade stability function (lfa.hpp:19-20).
double alpha(int p_t, double mu, double theta_x);
// aliased harmonic g(t) = t -/+ pi (lfa.hpp:22-24).
double shift(double theta);
// spectral radius of an n x n complex matrix (row-major re/im; im may be null).
double spectral_radius(int n, const double* re, const double* im);

// Symbols for one (p_t, mu) (SymbolBuilder, lfa.hpp:54-123); mode 1 = semi,
// 2 = full coarsening.
class Symbols {
 public:
  Symbols(int p_t, double mu);
  ~Symbols();
  Symbols(const Symbols&) = delete;
  Symbols& operator=(const Symbols&) = delete;
  int n_loc() const;
  double smoother_rho(double omega_t, double tx, double tt) const;
  double smoother_rho_closed_form(double omega_t, double tx, double tt) const;
  void smoother_symbol(double omega_t, double tx, double tt, double* re, double* im) const;
  // (4 n_loc)^2 two-grid symbol; throws std::domain_error at tx = 0
  void twogrid_symbol(double omega_t, int nu1, int nu2, int mode, double tx, double tt,
                      double* re, double* im) const;
  double twogrid_rho(double omega_t, int nu1, int nu2, int mode, double tx, double tt) const;
  double twogrid_rho_inexact(double omega_t, int nu1, int nu2, double omega_x, int nu1x,
                             int nu2x, int mode, double tx, double tt) const;

 private:
  struct Impl;
  Impl* impl_;
};

// lfa.hpp:125-150
double smoothing_factor(int p_t, double mu, double omega_t, int mode, int n_theta_x,
                        int n_theta_t);
double twogrid_factor(int p_t, double mu, double omega_t, int nu1, int nu2, int mode,
                      int n_theta_x, int n_theta_t);
double twogrid_factor_inexact(int p_t, double mu, double omega_t, int nu1, int nu2,
                              double omega_x, int nu1x, int nu2x, int mode, int n_theta_x,
                              int n_theta_t);

}  // namespace stmg::lfa
