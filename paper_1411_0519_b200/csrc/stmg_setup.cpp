// stmg_setup.cpp -- host setup numerics (see stmg_setup.hpp).
//
// The DG blocks use the closed forms of the Legendre basis on (0, tau):
// psi_l(tau) = 1, psi_k(0) = (-1)^k, int psi_l psi_k = tau/(2k+1) delta_kl and
// -int psi_l psi_k' + 1 = 1 - 2 [k > l, k + l odd]; the reference assembles
// the same matrices by Gauss quadrature (dg_time.cpp:125-166).  tests/ check
// the two agree to rounding.
#include "stmg_setup.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

namespace stmg {
namespace {

constexpr double kPi = 3.14159265358979323846;

void check_degree(int p) {
  if (p < 0 || p > kMaxTimeDegree)
    throw std::invalid_argument("time degree p_t out of supported range [0," +
                                std::to_string(kMaxTimeDegree) + "]: " + std::to_string(p));
}

double legendre_d(int n, double x) {
  if (n == 0) return 0.0;
  if (std::abs(x) == 1.0) return ((x > 0 || n % 2 == 1) ? 1.0 : -1.0) * 0.5 * n * (n + 1);
  return n * (x * legendre(n, x) - legendre(n - 1, x)) / (x * x - 1.0);
}

// Gauss-Legendre nodes/weights on (-1, 1), Newton from a Chebyshev guess.
void gauss(int np, std::vector<double>& x, std::vector<double>& w) {
  x.resize(np);
  w.resize(np);
  for (int i = 0; i < np; ++i) {
    double t = std::cos(kPi * (i + 0.75) / (np + 0.5));
    for (int it = 0; it < 100; ++it) {
      const double d = legendre(np, t) / legendre_d(np, t);
      t -= d;
      if (std::abs(d) < 1e-15) break;
    }
    const double dp = legendre_d(np, t);
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}

}  // namespace

double legendre(int n, double x) {
  double a = 1.0, b = x;
  if (n == 0) return a;
  for (int l = 1; l < n; ++l) {
    const double c = ((2 * l + 1) * x * b - l * a) / (l + 1);
    a = b;
    b = c;
  }
  return b;
}

DGBlock dg_block(int p, double tau) {
  check_degree(p);
  if (!(tau > 0.0)) throw std::invalid_argument("tau must be positive");
  const int nl = p + 1;
  DGBlock b;
  b.p = p;
  b.tau = tau;
  b.K.assign(nl * nl, 0.0);
  b.M.assign(nl * nl, 0.0);
  b.N.assign(nl * nl, 0.0);
  for (int k = 0; k < nl; ++k) {
    const double start_k = (k % 2 == 0) ? 1.0 : -1.0;  // psi_k(0) = P_k(-1)
    for (int l = 0; l < nl; ++l) {
      b.K[k * nl + l] = (k > l && (k + l) % 2 == 1) ? -1.0 : 1.0;
      b.N[k * nl + l] = start_k;  // psi_l(tau) = P_l(1) = 1
    }
    b.M[k * nl + k] = tau / double(2 * k + 1);
  }
  return b;
}

double pade_stability(int p, double z) {
  check_degree(p);
  const int m = p, n = p + 1;
  // numerator sum_j a_j z^j, denominator sum_j b_j (-z)^j, Horner form
  std::vector<double> a(m + 1), bq(n + 1);
  a[0] = 1.0;
  for (int j = 0; j < m; ++j) a[j + 1] = a[j] * double(m - j) / (double(m + n - j) * double(j + 1));
  bq[0] = 1.0;
  for (int j = 0; j < n; ++j) bq[j + 1] = bq[j] * double(n - j) / (double(m + n - j) * double(j + 1));
  double num = 0.0, den = 0.0;
  for (int j = m; j >= 0; --j) num = num * z + a[j];
  for (int j = n; j >= 0; --j) den = den * (-z) + bq[j];
  if (den == 0.0) throw std::domain_error("pade_stability: z is a pole of the denominator");
  return num / den;
}

double critical_mu(int p) {
  const double target = std::sqrt(2.0) - 1.0;
  auto f = [&](double mu) { return pade_stability(p, -3.0 * mu) - target; };
  double lo = 1e-12, hi = 10.0;
  if (f(lo) < 0.0 || f(hi) > 0.0) throw std::runtime_error("critical_mu: no sign change on (0, 10]");
  while (hi - lo > 1e-12) {
    const double mid = 0.5 * (lo + hi);
    if (f(mid) >= 0.0) lo = mid;
    else hi = mid;
  }
  return 0.5 * (lo + hi);
}

void time_transfer(int p, double tau, std::vector<double>& R1, std::vector<double>& R2) {
  check_degree(p);
  if (!(tau > 0.0)) throw std::invalid_argument("tau must be positive");
  const int nl = p + 1;
  std::vector<double> x, w;
  gauss(nl + 1, x, w);
  R1.assign(nl * nl, 0.0);
  R2.assign(nl * nl, 0.0);
  // R1[k,l] = (2l+1)/tau int_0^tau phi^{2tau}_k(s) psi_l(s) ds (M diagonal):
  // the L2 projection of coarse basis k onto fine basis l, transposed.
  for (int k = 0; k < nl; ++k)
    for (int l = 0; l < nl; ++l) {
      double s1 = 0.0, s2 = 0.0;
      for (size_t q = 0; q < x.size(); ++q) {
        const double s = 0.5 * tau * (x[q] + 1.0);  // local time in (0, tau)
        const double wq = 0.5 * tau * w[q];
        const double fl = legendre(l, 2.0 * s / tau - 1.0);
        s1 += wq * legendre(k, s / tau - 1.0) * fl;          // coarse on (0, 2tau), first half
        s2 += wq * legendre(k, (s + tau) / tau - 1.0) * fl;  // second half
      }
      const double inv_m = double(2 * l + 1) / tau;
      R1[k * nl + l] = inv_m * s1;
      R2[k * nl + l] = inv_m * s2;
    }
}

std::vector<LevelSpec> build_ladder(int p_t, int dim, int space_level, int time_level,
                                    double t_final, double mu_star, int policy, int two_grid) {
  if (time_level < 0 || space_level < 0) throw std::invalid_argument("hierarchy levels must be >= 0");
  check_degree(p_t);
  if (dim < 1 || dim > 3) throw std::invalid_argument("dim must be 1, 2 or 3");
  if (!(t_final > 0.0)) throw std::invalid_argument("tau must be positive");
  if (time_level > 40 || space_level > 20) throw std::invalid_argument("hierarchy levels too large");
  if (two_grid) {
    if (time_level < 1) throw std::invalid_argument("two-grid cycle needs at least 2 time steps");
    if (two_grid == 2 && space_level == 0) throw std::invalid_argument("full coarsening needs space level > 0");
    policy = two_grid == 2 ? 2 : 1;
  }
  if (policy < 0 || policy > 2) throw std::invalid_argument("unknown coarsening policy");
  const double ms = mu_star > 0.0 ? mu_star : critical_mu(p_t);
  std::vector<LevelSpec> out;
  int64_t n_t = int64_t(1) << time_level;
  double tau = t_final / double(n_t);
  int s = space_level;
  while (true) {
    LevelSpec L;
    L.n_t = n_t;
    L.space_level = s;
    L.dim = dim;
    L.p_t = p_t;
    L.tau = tau;
    L.h = std::ldexp(1.0, -(s + 1));
    L.mu = tau / (L.h * L.h);
    out.push_back(L);
    if (n_t == 1) break;
    bool full = false;
    if (policy == 0) full = out.back().mu >= ms && s > 0;
    else if (policy == 2) full = s > 0;
    out.back().coarsen = full ? 2 : 1;
    n_t /= 2;
    tau *= 2.0;
    if (full) --s;
  }
  if (two_grid) {
    out.resize(2);
    out[1].coarsen = 0;
  }
  return out;
}

}  // namespace stmg
