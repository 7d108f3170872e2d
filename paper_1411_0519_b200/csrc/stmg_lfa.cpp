// stmg_lfa.cpp -- host-side local Fourier analysis (LFA) engine: Fourier
// symbols of the space-time operator, the damped block-Jacobi smoother and
// the two-grid cycle, smoothing and two-grid convergence factors.  Restates
// the reference's lfa.cpp (lfa.hpp:15-150) on this library's DG/transfer
// setup (stmg_setup.cpp).  Not a hot path: it predicts the
// convergence factors that tools/harness.py and the tests measure on the GPU.
//
// Nondimensionalised like the reference: h = 1, tau = mu on the fine level
// (lfa.hpp:44-45); 1D space symbols; harmonics {(tx,tt), (g tx,tt), (tx,g tt),
// (g tx,g tt)} with g(t) = t -/+ pi.
#include <algorithm>
#include <cmath>
#include <complex>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "stmg_lfa.hpp"
#include "stmg_setup.hpp"

namespace stmg::lfa {

namespace {

constexpr double kPi = 3.14159265358979323846;
using cd = std::complex<double>;

// Dense complex matrix, row-major.
struct CMat {
  int r = 0, c = 0;
  std::vector<cd> a;
  CMat() = default;
  CMat(int rows, int cols) : r(rows), c(cols), a(size_t(rows) * cols, cd(0.0, 0.0)) {}
  cd& operator()(int i, int j) { return a[size_t(i) * c + j]; }
  cd operator()(int i, int j) const { return a[size_t(i) * c + j]; }
  static CMat eye(int n) {
    CMat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  static CMat real(int n, const std::vector<double>& v) {  // n x n row-major
    CMat m(n, n);
    for (int i = 0; i < n * n; ++i) m.a[i] = v[i];
    return m;
  }
};

CMat operator*(const CMat& x, const CMat& y) {
  if (x.c != y.r) throw std::logic_error("lfa: shape mismatch in product");
  CMat z(x.r, y.c);
  for (int i = 0; i < x.r; ++i)
    for (int k = 0; k < x.c; ++k) {
      const cd v = x(i, k);
      if (v == cd(0.0, 0.0)) continue;
      for (int j = 0; j < y.c; ++j) z(i, j) += v * y(k, j);
    }
  return z;
}
CMat operator+(CMat x, const CMat& y) {
  for (size_t i = 0; i < x.a.size(); ++i) x.a[i] += y.a[i];
  return x;
}
CMat operator-(CMat x, const CMat& y) {
  for (size_t i = 0; i < x.a.size(); ++i) x.a[i] -= y.a[i];
  return x;
}
CMat operator*(cd s, CMat x) {
  for (auto& v : x.a) v *= s;
  return x;
}
CMat transpose(const CMat& x) {
  CMat z(x.c, x.r);
  for (int i = 0; i < x.r; ++i)
    for (int j = 0; j < x.c; ++j) z(j, i) = x(i, j);
  return z;
}
void put(CMat& dst, int i0, int j0, const CMat& b) {
  for (int i = 0; i < b.r; ++i)
    for (int j = 0; j < b.c; ++j) dst(i0 + i, j0 + j) = b(i, j);
}

// Solve A X = B by LU with partial pivoting (Eigen partialPivLu in the
// reference).
CMat solve(CMat A, CMat B) {
  const int n = A.r;
  if (A.c != n || B.r != n) throw std::logic_error("lfa: shape mismatch in solve");
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(p, k))) p = i;
    if (std::abs(A(p, k)) == 0.0) throw std::runtime_error("lfa: singular symbol");
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      for (int j = 0; j < B.c; ++j) std::swap(B(k, j), B(p, j));
    }
    for (int i = k + 1; i < n; ++i) {
      const cd f = A(i, k) / A(k, k);
      if (f == cd(0.0, 0.0)) continue;
      for (int j = k; j < n; ++j) A(i, j) -= f * A(k, j);
      for (int j = 0; j < B.c; ++j) B(i, j) -= f * B(k, j);
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < B.c; ++j) {
      cd s = B(k, j);
      for (int i = k + 1; i < n; ++i) s -= A(k, i) * B(i, j);
      B(k, j) = s / A(k, k);
    }
  return B;
}

CMat power(const CMat& m, int nu) {
  CMat out = CMat::eye(m.r);
  for (int i = 0; i < nu; ++i) out = out * m;
  return out;
}

cd phase(double theta) { return cd(std::cos(theta), -std::sin(theta)); }

// Eigenvalues of a small complex matrix: Householder reduction to upper
// Hessenberg form, then single-shift QR with Wilkinson shifts and deflation.
std::vector<cd> eigenvalues(CMat A) {
  const int n = A.r;
  std::vector<cd> ev(n);
  if (n == 0) return ev;
  for (int k = 0; k + 2 < n; ++k) {  // Hessenberg
    double norm = 0.0;
    for (int i = k + 1; i < n; ++i) norm += std::norm(A(i, k));
    norm = std::sqrt(norm);
    if (norm == 0.0) continue;
    const cd x0 = A(k + 1, k);
    const cd alpha = (std::abs(x0) > 0.0 ? -x0 / std::abs(x0) : cd(-1.0, 0.0)) * norm;
    std::vector<cd> v(n, 0.0);
    for (int i = k + 1; i < n; ++i) v[i] = A(i, k);
    v[k + 1] -= alpha;
    double vn = 0.0;
    for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
    if (vn == 0.0) continue;
    // A <- H A H with H = I - 2 v v^H / (v^H v)
    for (int j = 0; j < n; ++j) {
      cd s = 0.0;
      for (int i = k + 1; i < n; ++i) s += std::conj(v[i]) * A(i, j);
      s *= 2.0 / vn;
      for (int i = k + 1; i < n; ++i) A(i, j) -= v[i] * s;
    }
    for (int i = 0; i < n; ++i) {
      cd s = 0.0;
      for (int j = k + 1; j < n; ++j) s += A(i, j) * v[j];
      s *= 2.0 / vn;
      for (int j = k + 1; j < n; ++j) A(i, j) -= s * std::conj(v[j]);
    }
  }
  double anorm = 0.0;  // Frobenius norm: absolute deflation floor
  for (const cd& v : A.a) anorm += std::norm(v);
  anorm = std::sqrt(anorm);
  int hi = n - 1, iter = 0;
  std::vector<double> cs(n);
  std::vector<cd> sn(n);
  while (hi >= 0) {
    if (hi == 0) {
      ev[0] = A(0, 0);
      break;
    }
    int l = hi;
    while (l > 0) {
      const double scale = std::abs(A(l, l)) + std::abs(A(l - 1, l - 1));
      const double sub = std::abs(A(l, l - 1));
      if (sub <= 1e-16 * scale || sub <= 1e-15 * anorm) break;
      --l;
    }
    if (l == hi) {
      ev[hi] = A(hi, hi);
      --hi;
      iter = 0;
      continue;
    }
    if (++iter > 500) throw std::runtime_error("lfa: QR iteration did not converge");
    // Wilkinson shift from the trailing 2x2 block (exceptional shift every 11th)
    const cd a = A(hi - 1, hi - 1), b = A(hi - 1, hi), c = A(hi, hi - 1), d = A(hi, hi);
    cd shift;
    if (iter % 11 == 0) {
      shift = d + cd(std::abs(c), 0.0);
    } else {
      const cd half = 0.5 * (a - d);
      const cd disc = std::sqrt(half * half + b * c);
      const cd m1 = 0.5 * (a + d) + disc, m2 = 0.5 * (a + d) - disc;
      shift = std::abs(m1 - d) < std::abs(m2 - d) ? m1 : m2;
    }
    for (int k = l; k <= hi; ++k) A(k, k) -= shift;
    for (int k = l; k < hi; ++k) {  // R = G_{hi-1} ... G_l (A - shift I)
      const cd x = A(k, k), y = A(k + 1, k);
      const double r = std::sqrt(std::norm(x) + std::norm(y));
      double cc;
      cd ss;
      if (r == 0.0) {
        cc = 1.0;
        ss = 0.0;
      } else if (std::abs(x) == 0.0) {
        cc = 0.0;
        ss = std::conj(y) / std::abs(y);
      } else {
        cc = std::abs(x) / r;
        ss = (x / std::abs(x)) * std::conj(y) / r;
      }
      cs[k] = cc;
      sn[k] = ss;
      for (int j = k; j <= hi; ++j) {
        const cd t1 = A(k, j), t2 = A(k + 1, j);
        A(k, j) = cc * t1 + ss * t2;
        A(k + 1, j) = -std::conj(ss) * t1 + cc * t2;
      }
    }
    for (int k = l; k < hi; ++k) {  // R Q
      const double cc = cs[k];
      const cd ss = sn[k];
      for (int i = l; i <= std::min(k + 2, hi); ++i) {
        const cd t1 = A(i, k), t2 = A(i, k + 1);
        A(i, k) = t1 * cc + t2 * std::conj(ss);
        A(i, k + 1) = -t1 * ss + t2 * cc;
      }
    }
    for (int k = l; k <= hi; ++k) A(k, k) += shift;
  }
  return ev;
}

double radius(const CMat& m) {
  double r = 0.0;
  for (const cd& e : eigenvalues(m)) r = std::max(r, std::abs(e));
  return r;
}

double space_restriction_symbol(double theta_x) { return 1.0 + std::cos(theta_x); }

// max over i in [lo, hi] of f(i) on the host cores (the reference uses an
// OpenMP max-reduction); the first exception is rethrown on the caller.
template <class F>
double parallel_max(int lo, int hi, F&& f) {
  const int n = hi - lo + 1;
  if (n <= 0) return 0.0;
  const int nth = std::max(1, std::min<int>(n, int(std::thread::hardware_concurrency())));
  std::vector<double> part(nth, 0.0);
  std::vector<std::exception_ptr> errs(nth);
  std::vector<std::thread> pool;
  for (int t = 0; t < nth; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int i = lo + t; i <= hi; i += nth) part[t] = std::max(part[t], f(i));
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  return *std::max_element(part.begin(), part.end());
}

}  // namespace

double beta(double theta_x) {
  const double c = std::cos(theta_x);
  return 6.0 * (1.0 - c) / (2.0 + c);
}

double alpha(int p_t, double mu, double theta_x) { return pade_stability(p_t, -mu * beta(theta_x)); }

double shift(double theta) { return theta > 0.0 ? theta - kPi : theta + kPi; }

struct Symbols::Impl {
  int p = 0, n = 1;
  double mu = 1.0;
  CMat K, M, N, Kc, Mc, Nc, R1, R2;
  // L_{tau,h} symbol (Lemma form): (h/3)(2 + cos tx)[K + h^-2 beta(tx) M - e^{-i tt} N]
  CMat op(const CMat& k, const CMat& m, const CMat& nn, double h, double tx, double tt) const {
    const double scale = h / 3.0 * (2.0 + std::cos(tx));
    return cd(scale, 0.0) * (k + cd(beta(tx) / (h * h), 0.0) * m - phase(tt) * nn);
  }
  CMat op_fine(double tx, double tt) const { return op(K, M, N, 1.0, tx, tt); }
  CMat op_semi(double tx, double tt) const { return op(Kc, Mc, Nc, 1.0, tx, 2.0 * tt); }
  CMat op_full(double tx, double tt) const { return op(Kc, Mc, Nc, 2.0, 2.0 * tx, 2.0 * tt); }
  // Jacobi block A(tx) = (h/3)(2 + cos tx) K + (2/h)(1 - cos tx) M
  CMat diag(double h, double tx, const CMat& k, const CMat& m) const {
    return cd(h / 3.0 * (2.0 + std::cos(tx)), 0.0) * k +
           cd(2.0 / h * (1.0 - std::cos(tx)), 0.0) * m;
  }
  CMat smoother(double omega, double tx, double tt) const {
    const CMat shifted = K + cd(beta(tx), 0.0) * M;
    const CMat prop = solve(shifted, N);
    return cd(1.0 - omega, 0.0) * CMat::eye(n) + (omega * phase(tt)) * prop;
  }
  CMat rt(double tt) const { return phase(tt) * R1 + R2; }
  CMat pt(double tt) const {
    return cd(0.5, 0.0) * (phase(-tt) * transpose(R1) + transpose(R2));
  }
  CMat harmonic_smoother(double omega, int nu, double tx, double tt) const {
    const double hx[2] = {tx, shift(tx)}, ht[2] = {tt, shift(tt)};
    CMat s(4 * n, 4 * n);
    for (int j = 0; j < 4; ++j) put(s, j * n, j * n, power(smoother(omega, hx[j % 2], ht[j / 2]), nu));
    return s;
  }
  CMat coarse_correction(int mode, double tx, double tt) const {
    const double gx = shift(tx), gt = shift(tt);
    const double hx[2] = {tx, gx}, ht[2] = {tt, gt};
    CMat opb(4 * n, 4 * n);
    for (int j = 0; j < 4; ++j) put(opb, j * n, j * n, op_fine(hx[j % 2], ht[j / 2]));
    const CMat r0 = rt(tt), rg = rt(gt), p0 = pt(tt), pg = pt(gt);
    CMat cgc;
    if (mode == 1) {  // semi: pairs (tx, .) and (gx, .) stay separate in space
      CMat R(2 * n, 4 * n), P(4 * n, 2 * n), C(2 * n, 2 * n);
      put(R, 0, 0, r0);
      put(R, 0, 2 * n, rg);
      put(R, n, n, r0);
      put(R, n, 3 * n, rg);
      put(P, 0, 0, p0);
      put(P, n, n, p0);
      put(P, 2 * n, 0, pg);
      put(P, 3 * n, n, pg);
      put(C, 0, 0, op_semi(tx, tt));
      put(C, n, n, op_semi(gx, tt));
      cgc = P * solve(C, R * opb);
    } else {  // full: space restriction symbol 1 + cos
      const double sx = space_restriction_symbol(tx), sg = space_restriction_symbol(gx);
      CMat R(n, 4 * n), P(4 * n, n);
      put(R, 0, 0, cd(sx, 0.0) * r0);
      put(R, 0, n, cd(sg, 0.0) * r0);
      put(R, 0, 2 * n, cd(sx, 0.0) * rg);
      put(R, 0, 3 * n, cd(sg, 0.0) * rg);
      put(P, 0, 0, cd(0.5 * sx, 0.0) * p0);
      put(P, n, 0, cd(0.5 * sg, 0.0) * p0);
      put(P, 2 * n, 0, cd(0.5 * sx, 0.0) * pg);
      put(P, 3 * n, 0, cd(0.5 * sg, 0.0) * pg);
      cgc = P * solve(op_full(tx, tt), R * opb);
    }
    return CMat::eye(4 * n) - cgc;
  }
  CMat twogrid(double omega, int nu1, int nu2, int mode, double tx, double tt) const {
    if (tx == 0.0)
      throw std::domain_error(
          "twogrid_symbol: theta_x = 0 is the singular frequency of the Laplacian symbol and "
          "is excluded");
    return harmonic_smoother(omega, nu2, tx, tt) * coarse_correction(mode, tx, tt) *
           harmonic_smoother(omega, nu1, tx, tt);
  }
  // spatial two-grid iteration of the inexact block solver on (tx, g tx)
  CMat spatial_twogrid(double omega_x, int nu1x, int nu2x, double tx) const {
    const double gx = shift(tx);
    const CMat a_tx = diag(1.0, tx, K, M), a_gx = diag(1.0, gx, K, M), a_c = diag(2.0, 2.0 * tx, K, M);
    const CMat dx = cd(2.0 / 3.0, 0.0) * K + cd(2.0, 0.0) * M;  // space Jacobi block (h = 1)
    auto jac = [&](const CMat& a, int nu) {
      return power(CMat::eye(n) - cd(omega_x, 0.0) * solve(dx, a), nu);
    };
    CMat pre(2 * n, 2 * n), post(2 * n, 2 * n), af(2 * n, 2 * n), R(n, 2 * n);
    put(pre, 0, 0, jac(a_tx, nu1x));
    put(pre, n, n, jac(a_gx, nu1x));
    put(post, 0, 0, jac(a_tx, nu2x));
    put(post, n, n, jac(a_gx, nu2x));
    put(af, 0, 0, a_tx);
    put(af, n, n, a_gx);
    put(R, 0, 0, cd(space_restriction_symbol(tx), 0.0) * CMat::eye(n));
    put(R, 0, n, cd(space_restriction_symbol(gx), 0.0) * CMat::eye(n));
    const CMat P = cd(0.5, 0.0) * transpose(R);
    const CMat cgc = CMat::eye(2 * n) - P * solve(a_c, R * af);
    return post * cgc * pre;
  }
  CMat approx_smoother(double omega, const CMat& spatial, double tx, double tt) const {
    const double hx[2] = {tx, shift(tx)}, ht[2] = {tt, shift(tt)};
    CMat opb(4 * n, 4 * n), db(4 * n, 4 * n), sp(4 * n, 4 * n);
    for (int j = 0; j < 4; ++j) {
      put(opb, j * n, j * n, op_fine(hx[j % 2], ht[j / 2]));
      put(db, j * n, j * n, diag(1.0, hx[j % 2], K, M));
    }
    put(sp, 0, 0, spatial);
    put(sp, 2 * n, 2 * n, spatial);
    return CMat::eye(4 * n) - cd(omega, 0.0) * ((CMat::eye(4 * n) - sp) * solve(db, opb));
  }
};

Symbols::Symbols(int p_t, double mu) : impl_(new Impl) {
  if (!(mu > 0.0)) throw std::invalid_argument("mu must be positive");
  Impl& s = *impl_;
  s.p = p_t;
  s.n = p_t + 1;
  s.mu = mu;
  const DGBlock f = dg_block(p_t, mu), c = dg_block(p_t, 2.0 * mu);
  s.K = CMat::real(s.n, f.K);
  s.M = CMat::real(s.n, f.M);
  s.N = CMat::real(s.n, f.N);
  s.Kc = CMat::real(s.n, c.K);
  s.Mc = CMat::real(s.n, c.M);
  s.Nc = CMat::real(s.n, c.N);
  std::vector<double> r1, r2;
  time_transfer(p_t, mu, r1, r2);
  s.R1 = CMat::real(s.n, r1);
  s.R2 = CMat::real(s.n, r2);
}
Symbols::~Symbols() { delete impl_; }

int Symbols::n_loc() const { return impl_->n; }

double Symbols::smoother_rho(double omega_t, double tx, double tt) const {
  return radius(impl_->smoother(omega_t, tx, tt));
}

double Symbols::smoother_rho_closed_form(double omega_t, double tx, double tt) const {
  const double a = alpha(impl_->p, impl_->mu, tx);
  const double s2 = (1.0 - omega_t) * (1.0 - omega_t) +
                    2.0 * omega_t * (1.0 - omega_t) * a * std::cos(tt) + a * a * omega_t * omega_t;
  const double moving = std::sqrt(std::max(s2, 0.0));
  if (impl_->p == 0) return moving;  // scalar symbol: only the moving eigenvalue
  return std::max(std::abs(1.0 - omega_t), moving);
}

void Symbols::smoother_symbol(double omega_t, double tx, double tt, double* re, double* im) const {
  const CMat s = impl_->smoother(omega_t, tx, tt);
  for (size_t i = 0; i < s.a.size(); ++i) {
    re[i] = s.a[i].real();
    im[i] = s.a[i].imag();
  }
}

void Symbols::twogrid_symbol(double omega_t, int nu1, int nu2, int mode, double tx, double tt,
                             double* re, double* im) const {
  const CMat s = impl_->twogrid(omega_t, nu1, nu2, mode, tx, tt);
  for (size_t i = 0; i < s.a.size(); ++i) {
    re[i] = s.a[i].real();
    im[i] = s.a[i].imag();
  }
}

double Symbols::twogrid_rho(double omega_t, int nu1, int nu2, int mode, double tx,
                            double tt) const {
  return radius(impl_->twogrid(omega_t, nu1, nu2, mode, tx, tt));
}

double Symbols::twogrid_rho_inexact(double omega_t, int nu1, int nu2, double omega_x, int nu1x,
                                    int nu2x, int mode, double tx, double tt) const {
  if (tx == 0.0) throw std::domain_error("twogrid_symbol_inexact: theta_x = 0 is excluded");
  const CMat sp = impl_->spatial_twogrid(omega_x, nu1x, nu2x, tx);
  const CMat sm = impl_->approx_smoother(omega_t, sp, tx, tt);
  const CMat t = power(sm, nu2) * impl_->coarse_correction(mode, tx, tt) * power(sm, nu1);
  return radius(t);
}

double spectral_radius(int n, const double* re, const double* im) {
  CMat m(n, n);
  for (int i = 0; i < n * n; ++i) m.a[i] = cd(re[i], im ? im[i] : 0.0);
  return radius(m);
}

double smoothing_factor(int p_t, double mu, double omega_t, int mode, int n_theta_x,
                        int n_theta_t) {
  if (mode != 1 && mode != 2) throw std::invalid_argument("smoothing factor needs semi or full mode");
  const int nx = std::max(n_theta_x, 64), nt = std::max(n_theta_t, 64);
  const Symbols s(p_t, mu);
  // closed high-frequency regions (the supremum sits on the included boundary)
  const double tx_lo = mode == 1 ? 0.0 : kPi / 2.0;
  const double tt_lo = mode == 1 ? kPi / 2.0 : 0.0;
  return parallel_max(0, nx, [&](int i) {
    const double tx = tx_lo + (kPi - tx_lo) * double(i) / double(nx);
    double rho = 0.0;
    for (int j = 0; j <= nt; ++j) {
      const double tt = tt_lo + (kPi - tt_lo) * double(j) / double(nt);
      rho = std::max(rho, s.smoother_rho(omega_t, tx, tt));
    }
    return rho;
  });
}

namespace {
// max over theta = 2 pi k / n on the low quarter (0, pi/2] x [0, pi/2]
// (symmetries rho(-tx, tt) = rho(tx, tt) = rho(tx, -tt); theta_x = 0 excluded)
template <class F>
double max_over_low_quarter(int nx, int nt, F&& rho_at) {
  return parallel_max(1, nx / 4, [&](int k) {
    const double tx = 2.0 * kPi * k / nx;
    double rho = 0.0;
    for (int l = 0; l <= nt / 4; ++l) rho = std::max(rho, rho_at(tx, 2.0 * kPi * l / nt));
    return rho;
  });
}
}  // namespace

double twogrid_factor(int p_t, double mu, double omega_t, int nu1, int nu2, int mode,
                      int n_theta_x, int n_theta_t) {
  if (mode != 1 && mode != 2) throw std::invalid_argument("two-grid factor needs semi or full mode");
  if (n_theta_x < 4 || n_theta_t < 4) throw std::invalid_argument("frequency grid too small");
  const Symbols s(p_t, mu);
  return max_over_low_quarter(n_theta_x, n_theta_t, [&](double tx, double tt) {
    return s.twogrid_rho(omega_t, nu1, nu2, mode, tx, tt);
  });
}

double twogrid_factor_inexact(int p_t, double mu, double omega_t, int nu1, int nu2,
                              double omega_x, int nu1x, int nu2x, int mode, int n_theta_x,
                              int n_theta_t) {
  if (mode != 1 && mode != 2) throw std::invalid_argument("two-grid factor needs semi or full mode");
  if (n_theta_x < 4 || n_theta_t < 4) throw std::invalid_argument("frequency grid too small");
  const Symbols s(p_t, mu);
  return max_over_low_quarter(n_theta_x, n_theta_t, [&](double tx, double tt) {
    return s.twogrid_rho_inexact(omega_t, nu1, nu2, omega_x, nu1x, nu2x, mode, tx, tt);
  });
}

}  // namespace stmg::lfa
