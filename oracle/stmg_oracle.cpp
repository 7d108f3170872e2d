// stmg_oracle.cpp -- CPU oracle for the space-time multigrid V-cycle.
//
// TEST INFRASTRUCTURE ONLY: a plain C++17/OpenMP restatement of the reference
// algorithm (/root/reference/proj/src) that the B200 library is checked
// against.  It keeps the reference's call structure and operation order
// (static per-time-step decomposition, per-step norm partials summed in step
// order, frozen-residual Jacobi, zero coarse guess, stop rule rk <= eps*r0).
//
// The one substitution: Eigen SparseLU (st_system.cpp:103-116) is replaced by
// an exact direct block solve -- orthonormal DST-I along every axis (dense
// sine matrices) diagonalises M_h and K_h, leaving one (p_t+1)^2 system per
// spatial mode, solved by Gaussian elimination with partial pivoting.  This is
// pinned against scipy.sparse.linalg.splu in tests/test_oracle.py.
//
// Parity pinning: reference KATs (tests/golden/kats.json), scipy splu, and the
// independent dense-Kronecker numpy oracle (oracle/dense.py).

#include "stmg_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using i64 = int64_t;
constexpr int kMaxTimeDegree = 10;  // dg_time.hpp:11
constexpr double kPi = 3.14159265358979323846;

thread_local std::string g_err;

// ---------------------------------------------------------------- dg_time --
// Legendre recurrences (dg_time.cpp:104-123).
double leg_val(int n, double x) {
  if (n == 0) return 1.0;
  double a = 1.0, b = x;
  for (int l = 1; l < n; ++l) {
    const double c = ((2 * l + 1) * x * b - l * a) / (l + 1);
    a = b;
    b = c;
  }
  return b;
}

double leg_der(int n, double x) {
  if (n == 0) return 0.0;
  if (std::abs(x) == 1.0) {
    const double s = (x > 0 || n % 2 == 1) ? 1.0 : -1.0;
    return s * 0.5 * n * (n + 1);
  }
  return n * (x * leg_val(n, x) - leg_val(n - 1, x)) / (x * x - 1.0);
}

// Gauss-Legendre on (-1,1) by Newton from a Chebyshev guess (dg_time.cpp:83-102).
void gauss_legendre(int np, std::vector<double>& x, std::vector<double>& w) {
  x.assign(np, 0.0);
  w.assign(np, 0.0);
  for (int i = 0; i < np; ++i) {
    double t = std::cos(kPi * (i + 0.75) / (np + 0.5));
    for (int it = 0; it < 100; ++it) {
      const double d = leg_val(np, t) / leg_der(np, t);
      t -= d;
      if (std::abs(d) < 1e-15) break;
    }
    const double dp = leg_der(np, t);
    x[np - 1 - i] = t;
    w[np - 1 - i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}

// Recursive pairwise summation (dg_time.cpp:12-20).
double psum(const double* v, size_t n) {
  if (n <= 2) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += v[i];
    return s;
  }
  const size_t h = n / 2;
  return psum(v, h) + psum(v + h, n - h);
}

void check_degree(int p) {
  if (p < 0 || p > kMaxTimeDegree)
    throw std::invalid_argument("time degree p_t out of supported range [0," +
                                std::to_string(kMaxTimeDegree) +
                                "]: " + std::to_string(p));
}

// Row-major n_loc x n_loc blocks; K[k*nl+l] = K(k,l).
struct DG {
  int p = 0;
  double tau = 1.0;
  std::vector<double> K, M, N;
  int nl() const { return p + 1; }
};

// Local Legendre basis psi_l on (0,tau) (dg_time.cpp:61-79).
double basis(int l, double t, double tau) { return leg_val(l, 2.0 * t / tau - 1.0); }
double basis_der(int l, double t, double tau) {
  return leg_der(l, 2.0 * t / tau - 1.0) * 2.0 / tau;
}

// dg_time.cpp:125-166 (Legendre basis).
DG assemble_dg(int p, double tau) {
  check_degree(p);
  if (!(tau > 0.0)) throw std::invalid_argument("tau must be positive");
  const int nl = p + 1;
  DG b;
  b.p = p;
  b.tau = tau;
  b.K.assign(nl * nl, 0.0);
  b.M.assign(nl * nl, 0.0);
  b.N.assign(nl * nl, 0.0);
  std::vector<double> qx, qw;
  gauss_legendre(nl, qx, qw);
  std::vector<double> val(nl * nl), der(nl * nl), w(nl), terms(nl);
  for (int q = 0; q < nl; ++q) {
    const double t = 0.5 * tau * (qx[q] + 1.0);
    w[q] = 0.5 * tau * qw[q];
    for (int l = 0; l < nl; ++l) {
      val[l * nl + q] = basis(l, t, tau);
      der[l * nl + q] = basis_der(l, t, tau);
    }
  }
  for (int k = 0; k < nl; ++k) {
    const double end_k = basis(k, tau, tau), start_k = basis(k, 0.0, tau);
    for (int l = 0; l < nl; ++l) {
      const double end_l = basis(l, tau, tau);
      for (int q = 0; q < nl; ++q) terms[q] = -w[q] * val[l * nl + q] * der[k * nl + q];
      b.K[k * nl + l] = psum(terms.data(), nl) + end_l * end_k;
      for (int q = 0; q < nl; ++q) terms[q] = w[q] * val[l * nl + q] * val[k * nl + q];
      b.M[k * nl + l] = psum(terms.data(), nl);
      b.N[k * nl + l] = end_l * start_k;
    }
  }
  return b;
}

// (p, p+1) Pade approximant of e^z, real argument (dg_time.cpp:46-58,168-198).
double pade(int p, double z) {
  check_degree(p);
  const int m = p, n = p + 1;
  std::vector<double> pc(m + 1), qc(n + 1);
  pc[0] = 1.0;
  for (int j = 0; j < m; ++j) pc[j + 1] = pc[j] * double(m - j) / (double(m + n - j) * double(j + 1));
  qc[0] = 1.0;
  for (int j = 0; j < n; ++j) qc[j + 1] = qc[j] * double(n - j) / (double(m + n - j) * double(j + 1));
  std::vector<double> t;
  double zj = 1.0;
  for (double c : pc) { t.push_back(c * zj); zj *= z; }
  const double num = psum(t.data(), t.size());
  t.clear();
  zj = 1.0;
  for (double c : qc) { t.push_back(c * zj); zj *= -z; }
  const double den = psum(t.data(), t.size());
  if (den == 0.0) throw std::domain_error("pade_stability: z is a pole of the denominator");
  return num / den;
}

// lfa.cpp:317-328: R(-3 mu*) = sqrt(2) - 1 by bisection on (1e-12, 10].
double critical_mu(int p) {
  const double target = std::sqrt(2.0) - 1.0;
  auto f = [&](double mu) { return pade(p, -3.0 * mu) - target; };
  double lo = 1e-12, hi = 10.0;
  if (f(lo) < 0.0 || f(hi) > 0.0) throw std::runtime_error("critical_mu: no sign change on (0, 10]");
  while (hi - lo > 1e-12) {
    const double mid = 0.5 * (lo + hi);
    (f(mid) >= 0.0 ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}

// Small dense solve A X = B (n x n, n x m; row-major) with partial pivoting.
void dense_solve(int n, std::vector<double> A, double* B, int m) {
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::abs(A[r * n + c]) > std::abs(A[piv * n + c])) piv = r;
    if (A[piv * n + c] == 0.0) throw std::runtime_error("time-step block factorization failed");
    if (piv != c) {
      for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[piv * n + k]);
      for (int k = 0; k < m; ++k) std::swap(B[c * m + k], B[piv * m + k]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = A[r * n + c] / A[c * n + c];
      if (f == 0.0) continue;
      for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
      for (int k = 0; k < m; ++k) B[r * m + k] -= f * B[c * m + k];
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    for (int k = 0; k < m; ++k) {
      double s = B[c * m + k];
      for (int j = c + 1; j < n; ++j) s -= A[c * n + j] * B[j * m + k];
      B[c * m + k] = s / A[c * n + c];
    }
  }
}

// transfer.cpp:50-73: R1^T = M^-1 Mt1, R2^T = M^-1 Mt2 (row-major R1[k*nl+l]).
struct TT {
  std::vector<double> R1, R2;
};

TT time_transfer(int p, double tau) {
  const DG fine = assemble_dg(p, tau);
  const int nl = p + 1;
  std::vector<double> qx, qw;
  gauss_legendre(nl, qx, qw);
  std::vector<double> Mt1(nl * nl, 0.0), Mt2(nl * nl, 0.0);
  for (int q = 0; q < nl; ++q) {
    const double s = 0.5 * tau * (qx[q] + 1.0);
    const double w = 0.5 * tau * qw[q];
    for (int k = 0; k < nl; ++k) {
      const double fk = basis(k, s, tau);
      for (int l = 0; l < nl; ++l) {
        Mt1[k * nl + l] += w * basis(l, s, 2.0 * tau) * fk;
        Mt2[k * nl + l] += w * basis(l, s + tau, 2.0 * tau) * fk;
      }
    }
  }
  dense_solve(nl, fine.M, Mt1.data(), nl);  // Mt1 <- M^-1 Mt1 = R1^T
  dense_solve(nl, fine.M, Mt2.data(), nl);
  TT t;
  t.R1.resize(nl * nl);
  t.R2.resize(nl * nl);
  for (int k = 0; k < nl; ++k)
    for (int l = 0; l < nl; ++l) {
      t.R1[k * nl + l] = Mt1[l * nl + k];
      t.R2[k * nl + l] = Mt2[l * nl + k];
    }
  return t;
}

// -------------------------------------------------------------- fem_space --
// fem_space.cpp:28-58 (+ the 3D Kronecker extension M1(x)M1(x)M1,
// K = K1(x)M1(x)M1 + M1(x)K1(x)M1 + M1(x)M1(x)K1).
struct Grid {
  int dim = 1, level = 0;
  double h = 0.5;
  i64 n1 = 1, nx = 1;
};

Grid make_grid(int dim, int level) {
  if (dim < 1 || dim > 3) throw std::invalid_argument("dim must be 1, 2 or 3");
  if (level < 0) throw std::invalid_argument("level must be >= 0");
  Grid g;
  g.dim = dim;
  g.level = level;
  g.h = std::ldexp(1.0, -(level + 1));
  g.n1 = (i64(1) << (level + 1)) - 1;
  g.nx = g.n1;
  for (int a = 1; a < dim; ++a) g.nx *= g.n1;
  return g;
}

i64 axis_stride(const Grid& g, int axis) {
  i64 s = 1;
  for (int a = 0; a < axis; ++a) s *= g.n1;
  return s;
}

// out = T_axis in for the 1D tridiagonal {off, diag, off} along one axis.
void tri_axis(const Grid& g, int axis, double off, double diag, const double* in, double* out) {
  const i64 s = axis_stride(g, axis), n1 = g.n1;
  for (i64 r = 0; r < g.nx; ++r) {
    const i64 i = (r / s) % n1;
    double v = diag * in[r];
    if (i > 0) v += off * in[r - s];
    if (i + 1 < n1) v += off * in[r + s];
    out[r] = v;
  }
}

// Apply the spatial mass (which_k = false) or stiffness (true) matrix.
void space_apply(const Grid& g, bool stiff, const double* in, double* out) {
  const double mo = g.h / 6.0, md = 4.0 * g.h / 6.0;
  const double ko = -1.0 / g.h, kd = 2.0 / g.h;
  std::vector<double> a(g.nx), b(g.nx);
  if (!stiff) {
    const double* src = in;
    for (int ax = 0; ax < g.dim; ++ax) {
      double* dst = (ax + 1 == g.dim) ? out : (ax % 2 == 0 ? a.data() : b.data());
      tri_axis(g, ax, mo, md, src, dst);
      src = dst;
    }
    return;
  }
  std::fill(out, out + g.nx, 0.0);
  for (int term = 0; term < g.dim; ++term) {  // K1 on axis `term`, M1 elsewhere
    const double* src = in;
    for (int ax = 0; ax < g.dim; ++ax) {
      double* dst = ax % 2 == 0 ? a.data() : b.data();
      if (ax == term) tri_axis(g, ax, ko, kd, src, dst);
      else tri_axis(g, ax, mo, md, src, dst);
      src = dst;
    }
    for (i64 r = 0; r < g.nx; ++r) out[r] += src[r];
  }
}

// -------------------------------------------------------------- hierarchy --
struct Level {
  DG dg;
  Grid grid;
  i64 n_t = 1;
  double mu = 0.0;
  int coarsen = 0;  // 0 none, 1 semi, 2 full
  TT tt;
  // exact block solve data: orthonormal DST-I matrix, per-axis eigenvalues
  std::vector<double> S, mval, kval;
  // SpatialVCycleSolver stack (smoother.cpp:8-27): grids finest..1-node, the
  // point-block Jacobi block diag(M) K + diag(K) M per grid, and the 1-node
  // block matrix of the coarsest grid (row-major nl x nl).
  std::vector<Grid> sgrid;
  std::vector<std::vector<double>> sjac;
  std::vector<double> scoarse;
  i64 nl() const { return dg.nl(); }
  i64 slab() const { return grid.nx * dg.nl(); }
  i64 size() const { return n_t * slab(); }
};

void init_block_solver(Level& L) {
  const i64 n1 = L.grid.n1;
  const double N = double(n1 + 1), h = L.grid.h;
  L.S.resize(n1 * n1);
  const double sc = std::sqrt(2.0 / N);
  for (i64 i = 0; i < n1; ++i)
    for (i64 k = 0; k < n1; ++k) L.S[i * n1 + k] = sc * std::sin(kPi * double((i + 1) * (k + 1)) / N);
  L.mval.resize(n1);
  L.kval.resize(n1);
  for (i64 k = 0; k < n1; ++k) {
    const double th = kPi * double(k + 1) * h;
    const double s = std::sin(0.5 * th);
    L.mval[k] = h / 3.0 * (2.0 + std::cos(th));  // M1 -> (h/3)(2 + c)
    L.kval[k] = 4.0 / h * s * s;                  // K1 -> (2/h)(1 - c)
  }
  // smoother.cpp:8-27: one level per grid L..0; uniform grid, so one
  // diagonal value of M and K per level (M(0,0), K(0,0) of the Kronecker
  // products: md^dim and dim * kd * md^(dim-1)).
  const int nl = L.dg.nl();
  L.sgrid.clear();
  L.sjac.clear();
  for (int g = L.grid.level; g >= 0; --g) {
    const Grid G = make_grid(L.grid.dim, g);
    const double md = 4.0 * G.h / 6.0, kd = 2.0 / G.h;
    const double mdiag = std::pow(md, G.dim), kdiag = G.dim * kd * std::pow(md, G.dim - 1);
    std::vector<double> D(nl * nl);
    for (int i = 0; i < nl * nl; ++i) D[i] = mdiag * L.dg.K[i] + kdiag * L.dg.M[i];
    L.sgrid.push_back(G);
    L.sjac.push_back(std::move(D));
  }
  // coarsest (1-node) grid: assemble_block_matrix = K (x) M_h + M (x) K_h
  L.scoarse = L.sjac.back();
}

struct Hier {
  std::vector<Level> levels;
  int p_t = 0, dim = 1;
};

// mg.cpp:10-75 (build_hierarchy) and 77-94 (build_two_grid).
Hier build_hierarchy(const or_params& p) {
  if (p.time_level < 0 || p.space_level < 0) throw std::invalid_argument("hierarchy levels must be >= 0");
  check_degree(p.p_t);
  if (p.dim < 1 || p.dim > 3) throw std::invalid_argument("dim must be 1, 2 or 3");
  if (p.two_grid) {
    if (p.time_level < 1) throw std::invalid_argument("two-grid cycle needs at least 2 time steps");
    if (p.two_grid == 2 && p.space_level == 0) throw std::invalid_argument("full coarsening needs space level > 0");
  }
  const int policy = p.two_grid == 1 ? 1 : p.two_grid == 2 ? 2 : p.policy;
  const double mu_star = p.mu_star > 0.0 ? p.mu_star : critical_mu(p.p_t);
  Hier h;
  h.p_t = p.p_t;
  h.dim = p.dim;
  i64 n_t = i64(1) << p.time_level;
  double tau = p.t_final / double(n_t);
  int s = p.space_level;
  while (true) {
    Level L;
    L.dg = assemble_dg(p.p_t, tau);
    L.grid = make_grid(p.dim, s);
    L.n_t = n_t;
    L.mu = tau / (L.grid.h * L.grid.h);
    L.tt = time_transfer(p.p_t, tau);
    h.levels.push_back(std::move(L));
    if (n_t == 1) break;
    bool full = false;
    if (policy == 0) full = h.levels.back().mu >= mu_star && s > 0;
    else if (policy == 2) full = s > 0;
    h.levels.back().coarsen = full ? 2 : 1;
    n_t /= 2;
    tau *= 2.0;
    if (full) --s;
  }
  if (p.two_grid) {
    h.levels.resize(2);
    h.levels[1].coarsen = 0;
  }
  for (auto& L : h.levels) init_block_solver(L);
  return h;
}

// -------------------------------------------------------------- st_system --
// Orthonormal DST-I of one component vector along one axis (out may != in).
void dst_axis(const Level& L, int axis, const double* in, double* out) {
  const Grid& g = L.grid;
  const i64 s = axis_stride(g, axis), n1 = g.n1, blk = s * n1;
  const double* S = L.S.data();
  if (s == 1) {
    // x axis: lines are contiguous.  Transpose kB lines into a tile so the
    // sum over i (ascending, the same order as below) runs on kB independent
    // accumulators instead of one dependent FMA chain.
    constexpr i64 kB = 8;
    std::vector<double> tile(n1 * kB), acc(kB);
    const i64 nlines = g.nx / n1;
    for (i64 l0 = 0; l0 < nlines; l0 += kB) {
      const i64 nb = std::min(kB, nlines - l0);
      for (i64 l = 0; l < nb; ++l)
        for (i64 i = 0; i < n1; ++i) tile[i * kB + l] = in[(l0 + l) * n1 + i];
      for (i64 k = 0; k < n1; ++k) {
        for (i64 l = 0; l < kB; ++l) acc[l] = 0.0;
        const double* Sk = S + k * n1;
        for (i64 i = 0; i < n1; ++i) {
          const double c = Sk[i];
          const double* t = tile.data() + i * kB;
          for (i64 l = 0; l < kB; ++l) acc[l] += c * t[l];
        }
        for (i64 l = 0; l < nb; ++l) out[(l0 + l) * n1 + k] = acc[l];
      }
    }
    return;
  }
  for (i64 base = 0; base < g.nx; base += blk)
    for (i64 k = 0; k < n1; ++k) {
      double* o = out + base + k * s;
      for (i64 t = 0; t < s; ++t) o[t] = 0.0;
      for (i64 i = 0; i < n1; ++i) {
        const double c = S[k * n1 + i];
        const double* src = in + base + i * s;
        for (i64 t = 0; t < s; ++t) o[t] += c * src[t];
      }
    }
}

void dst_all(const Level& L, const double* in, double* out) {
  std::vector<double> tmp(L.grid.nx);
  const double* src = in;
  for (int ax = 0; ax < L.grid.dim; ++ax) {
    double* dst = ((L.grid.dim - 1 - ax) % 2 == 0) ? out : tmp.data();
    dst_axis(L, ax, src, dst);
    src = dst;
  }
}

// Mode eigenvalues of M_h, K_h for flat mode index r.
void mode_eig(const Level& L, i64 r, double& Mj, double& Kj) {
  const i64 n1 = L.grid.n1;
  double mv[3], kv[3];
  for (int a = 0; a < L.grid.dim; ++a) {
    const i64 k = r % n1;
    r /= n1;
    mv[a] = L.mval[k];
    kv[a] = L.kval[k];
  }
  Mj = 1.0;
  for (int a = 0; a < L.grid.dim; ++a) Mj *= mv[a];
  Kj = 0.0;
  for (int a = 0; a < L.grid.dim; ++a) {
    double t = kv[a];
    for (int b = 0; b < L.grid.dim; ++b)
      if (b != a) t *= mv[b];
    Kj += t;
  }
}

// Exact solve A x = b for one slab, A = K_tau (x) M_h + M_tau (x) K_h
// (replaces BlockSolver::solve, st_system.cpp:103-116).
void block_solve(const Level& L, const double* b, double* x) {
  const i64 nx = L.grid.nx;
  const int nl = L.dg.nl();
  std::vector<double> bh(nx * nl);
  for (int l = 0; l < nl; ++l) dst_all(L, b + l * nx, bh.data() + l * nx);
  std::vector<double> A(nl * nl), rhs(nl);
  for (i64 r = 0; r < nx; ++r) {
    double Mj, Kj;
    mode_eig(L, r, Mj, Kj);
    for (int i = 0; i < nl * nl; ++i) A[i] = Mj * L.dg.K[i] + Kj * L.dg.M[i];
    for (int l = 0; l < nl; ++l) rhs[l] = bh[l * nx + r];
    dense_solve(nl, A, rhs.data(), 1);
    for (int l = 0; l < nl; ++l) bh[l * nx + r] = rhs[l];
  }
  for (int l = 0; l < nl; ++l) dst_all(L, bh.data() + l * nx, x + l * nx);
}

// st_system.cpp:25-33: y_n = (M U_n) K^T + (K U_n) M^T - (M U_{n-1}) N^T.
// un = step n's slab, up = step n-1's slab (nullptr for n = 0), y = output slab.
void apply_slab(const Level& L, const double* un, const double* up, double* y) {
  const i64 nx = L.grid.nx;
  const int nl = L.dg.nl();
  std::vector<double> MU(nl * nx), KU(nl * nx), out(nl * nx, 0.0);
  for (int l = 0; l < nl; ++l) {
    space_apply(L.grid, false, un + l * nx, MU.data() + l * nx);
    space_apply(L.grid, true, un + l * nx, KU.data() + l * nx);
  }
  for (int k = 0; k < nl; ++k)
    for (int l = 0; l < nl; ++l) {
      const double a = L.dg.K[k * nl + l];
      for (i64 r = 0; r < nx; ++r) out[k * nx + r] += MU[l * nx + r] * a;
    }
  for (int k = 0; k < nl; ++k)
    for (int l = 0; l < nl; ++l) {
      const double a = L.dg.M[k * nl + l];
      for (i64 r = 0; r < nx; ++r) out[k * nx + r] += KU[l * nx + r] * a;
    }
  if (up) {
    for (int l = 0; l < nl; ++l) space_apply(L.grid, false, up + l * nx, MU.data() + l * nx);
    for (int k = 0; k < nl; ++k)
      for (int l = 0; l < nl; ++l) {
        const double a = L.dg.N[k * nl + l];
        for (i64 r = 0; r < nx; ++r) out[k * nx + r] -= MU[l * nx + r] * a;
      }
  }
  std::copy(out.begin(), out.end(), y);
}

void apply_block_row(const Level& L, const double* u, i64 n, double* y) {
  const i64 sl = L.slab();
  apply_slab(L, u + n * sl, n > 0 ? u + (n - 1) * sl : nullptr, y + n * sl);
}

void apply(const Level& L, const double* u, double* y) {
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < L.n_t; ++n) apply_block_row(L, u, n, y);
}

// st_system.cpp:57-67.
void residual(const Level& L, const double* u, const double* f, double* r) {
  const i64 sl = L.slab();
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < L.n_t; ++n) {
    apply_block_row(L, u, n, r);
    for (i64 i = 0; i < sl; ++i) r[n * sl + i] = f[n * sl + i] - r[n * sl + i];
  }
}

// st_system.cpp:8-16: one partial per time step, summed in step order.
double norm(const Level& L, const double* v) {
  const i64 sl = L.slab();
  std::vector<double> part(L.n_t);
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < L.n_t; ++n) {
    double s = 0.0;
    for (i64 i = 0; i < sl; ++i) s += v[n * sl + i] * v[n * sl + i];
    part[n] = s;
  }
  double sum = 0.0;
  for (double p : part) sum += p;
  return std::sqrt(sum);
}

// norm(residual(u, f)) without materialising r: the same per-step partials
// (slab order) summed in step order, so the value is bitwise norm(r).
double residual_norm(const Level& L, const double* u, const double* f) {
  const i64 sl = L.slab();
  std::vector<double> part(L.n_t);
#pragma omp parallel
  {
    std::vector<double> y(sl);
#pragma omp for schedule(static)
    for (i64 n = 0; n < L.n_t; ++n) {
      apply_slab(L, u + n * sl, n > 0 ? u + (n - 1) * sl : nullptr, y.data());
      double s = 0.0;
      for (i64 i = 0; i < sl; ++i) {
        const double r = f[n * sl + i] - y[i];
        s += r * r;
      }
      part[n] = s;
    }
  }
  double sum = 0.0;
  for (double p : part) sum += p;
  return std::sqrt(sum);
}

// st_system.cpp:118-130.
void forward_substitution(const Level& L, const double* f, double* u) {
  const i64 nx = L.grid.nx, sl = L.slab();
  const int nl = L.dg.nl();
  std::vector<double> rhs(sl), MU(nl * nx);
  for (i64 n = 0; n < L.n_t; ++n) {
    std::copy(f + n * sl, f + (n + 1) * sl, rhs.begin());
    if (n > 0) {
      const double* up = u + (n - 1) * sl;
      for (int l = 0; l < nl; ++l) space_apply(L.grid, false, up + l * nx, MU.data() + l * nx);
      for (int k = 0; k < nl; ++k)
        for (int l = 0; l < nl; ++l) {
          const double a = L.dg.N[k * nl + l];
          for (i64 r = 0; r < nx; ++r) rhs[k * nx + r] += MU[l * nx + r] * a;
        }
    }
    block_solve(L, rhs.data(), u + n * sl);
  }
}

// smoother.cpp:96-106 (exact block solves).  Frozen-residual Jacobi,
// u_n += omega A^-1 (f_n - A_nn u_n - B u_{n-1}) with the OLD iterate, done in
// place without a full residual vector: the steps are split into chunks, each
// chunk's left-neighbour slab is saved first, and a chunk is swept from its
// last step down so every step still sees the old u_{n-1}.  The arithmetic is
// exactly residual() + block_solve() per step.
void smooth(const Level& L, double* u, const double* f, double omega, int nu) {
  const i64 sl = L.slab(), nt = L.n_t;
  const i64 nchunk = std::min<i64>(nt, 256);
  std::vector<i64> start(nchunk + 1);
  for (i64 c = 0; c <= nchunk; ++c) start[c] = c * nt / nchunk;
  std::vector<double> left(nchunk * sl);
  for (int s = 0; s < nu; ++s) {
#pragma omp parallel for schedule(static)
    for (i64 c = 1; c < nchunk; ++c)
      std::copy(u + (start[c] - 1) * sl, u + start[c] * sl, left.data() + c * sl);
#pragma omp parallel
    {
      std::vector<double> r(sl), x(sl);
#pragma omp for schedule(static)
      for (i64 c = 0; c < nchunk; ++c)
        for (i64 n = start[c + 1] - 1; n >= start[c]; --n) {
          const double* up = n == 0 ? nullptr
                             : n == start[c] ? left.data() + c * sl
                                             : u + (n - 1) * sl;
          apply_slab(L, u + n * sl, up, r.data());
          for (i64 i = 0; i < sl; ++i) r[i] = f[n * sl + i] - r[i];
          block_solve(L, r.data(), x.data());
          for (i64 i = 0; i < sl; ++i) u[n * sl + i] += omega * x[i];
        }
    }
  }
}

// --------------------------------------------------------------- transfer --
// transfer.cpp:22-46 (full weighting and its transpose on a strided line).
void restrict_line(const double* u, i64 su, i64 m, double* out, i64 so) {
  for (i64 j = 0; j < m; ++j) {
    const double* c = u + 2 * j * su;
    out[j * so] = 0.5 * (c[0] + 2.0 * c[su] + c[2 * su]);
  }
}

void prolong_line(const double* c, i64 sc, i64 m, double* out, i64 so) {
  const i64 n = 2 * m + 1;
  for (i64 i = 0; i < n; ++i) {
    double v;
    if (i % 2 == 1) {
      v = c[(i / 2) * sc];
    } else {
      const i64 j = i / 2;
      v = 0.0;
      if (j > 0) v += 0.5 * c[(j - 1) * sc];
      if (j < m) v += 0.5 * c[j * sc];
    }
    out[i * so] = v;
  }
}

// Separable space restriction of one component (transfer.cpp:98-116; axes
// x, then y, then z through temporaries).
void restrict_space(const Grid& fg, const Grid& cg, const double* u, double* out) {
  const i64 n1 = fg.n1, m1 = cg.n1;
  // current array shape: per-axis extents ext[0..dim)
  i64 ext[3] = {n1, n1, n1};
  std::vector<double> cur(u, u + fg.nx), nxt;
  for (int ax = 0; ax < fg.dim; ++ax) {
    i64 total_in = 1, total_out = 1, stride = 1;
    for (int a = 0; a < fg.dim; ++a) total_in *= ext[a];
    for (int a = 0; a < ax; ++a) stride *= ext[a];
    i64 ext2[3] = {ext[0], ext[1], ext[2]};
    ext2[ax] = m1;
    for (int a = 0; a < fg.dim; ++a) total_out *= ext2[a];
    nxt.assign(total_out, 0.0);
    const i64 outer = total_in / (stride * ext[ax]);
    for (i64 o = 0; o < outer; ++o)
      for (i64 t = 0; t < stride; ++t)
        restrict_line(cur.data() + o * stride * ext[ax] + t, stride, m1,
                      nxt.data() + o * stride * m1 + t, stride);
    cur.swap(nxt);
    ext[ax] = m1;
  }
  std::copy(cur.begin(), cur.end(), out);
}

// transfer.cpp:118-136.
void prolong_space(const Grid& cg, const Grid& fg, const double* c, double* out) {
  const i64 n1 = fg.n1, m1 = cg.n1;
  i64 ext[3] = {m1, m1, m1};
  std::vector<double> cur(c, c + cg.nx), nxt;
  for (int ax = 0; ax < fg.dim; ++ax) {
    i64 total_in = 1, total_out = 1, stride = 1;
    for (int a = 0; a < fg.dim; ++a) total_in *= ext[a];
    for (int a = 0; a < ax; ++a) stride *= ext[a];
    i64 ext2[3] = {ext[0], ext[1], ext[2]};
    ext2[ax] = n1;
    for (int a = 0; a < fg.dim; ++a) total_out *= ext2[a];
    nxt.assign(total_out, 0.0);
    const i64 outer = total_in / (stride * ext[ax]);
    for (i64 o = 0; o < outer; ++o)
      for (i64 t = 0; t < stride; ++t)
        prolong_line(cur.data() + o * stride * m1 + t, stride, m1,
                     nxt.data() + o * stride * n1 + t, stride);
    cur.swap(nxt);
    ext[ax] = n1;
  }
  std::copy(cur.begin(), cur.end(), out);
}

// ------------------------------------------------ smoother.cpp:8-92 --
// SpatialVCycleSolver: one geometric multigrid cycle in space for one
// time-step block A = K_tau (x) M_h + M_tau (x) K_h (damped point-block
// Jacobi on every grid, full weighting / linear interpolation per DG
// component, direct solve on the 1-node grid).  x, b: one slab (nl
// components of nx values, component-major as BlockVector::step).
struct SvcCfg {
  double omega_x = 2.0 / 3.0;
  int nu1_x = 2, nu2_x = 2, gamma_x = 1;
};

// st_system.cpp:18-23: y = (M_h X) K^T + (K_h X) M^T.
void apply_diag_block(const DG& dg, const Grid& g, const double* x, double* y) {
  const int nl = dg.nl();
  const i64 nx = g.nx;
  std::vector<double> MX(nl * nx), KX(nl * nx);
  for (int l = 0; l < nl; ++l) {
    space_apply(g, false, x + l * nx, MX.data() + l * nx);
    space_apply(g, true, x + l * nx, KX.data() + l * nx);
  }
  for (int k = 0; k < nl; ++k) {
    double* yk = y + k * nx;
    for (i64 r = 0; r < nx; ++r) yk[r] = 0.0;
    for (int l = 0; l < nl; ++l) {
      const double a = dg.K[k * nl + l];
      for (i64 r = 0; r < nx; ++r) yk[r] += MX[l * nx + r] * a;
    }
    for (int l = 0; l < nl; ++l) {
      const double a = dg.M[k * nl + l];
      for (i64 r = 0; r < nx; ++r) yk[r] += KX[l * nx + r] * a;
    }
  }
}

// smoother.cpp:29-38: count sweeps x += omega D^-1 (b - A x), D per node.
void svc_jacobi(const Level& L, size_t lev, int count, double omega, double* x, const double* b) {
  const Grid& g = L.sgrid[lev];
  const int nl = L.dg.nl();
  const i64 nx = g.nx;
  std::vector<double> r(nl * nx), node(nl);
  for (int s = 0; s < count; ++s) {
    apply_diag_block(L.dg, g, x, r.data());
    for (i64 i = 0; i < nl * nx; ++i) r[i] = b[i] - r[i];
    for (i64 q = 0; q < nx; ++q) {
      for (int l = 0; l < nl; ++l) node[l] = r[l * nx + q];
      dense_solve(nl, L.sjac[lev], node.data(), 1);
      for (int l = 0; l < nl; ++l) x[l * nx + q] += omega * node[l];
    }
  }
}

// smoother.cpp:40-69.
void svc_recurse(const Level& L, size_t lev, double* x, const double* b, const SvcCfg& cfg) {
  const Grid& g = L.sgrid[lev];
  const int nl = L.dg.nl();
  const i64 nx = g.nx;
  if (lev + 1 == L.sgrid.size()) {  // 1-node grid: direct solve
    std::copy(b, b + nl * nx, x);
    dense_solve(nl, L.scoarse, x, 1);
    return;
  }
  svc_jacobi(L, lev, cfg.nu1_x, cfg.omega_x, x, b);
  std::vector<double> r(nl * nx);
  apply_diag_block(L.dg, g, x, r.data());
  for (i64 i = 0; i < nl * nx; ++i) r[i] = b[i] - r[i];
  const Grid& cg = L.sgrid[lev + 1];
  std::vector<double> rc(nl * cg.nx), ec(nl * cg.nx, 0.0), corr(nl * nx);
  for (int l = 0; l < nl; ++l) restrict_space(g, cg, r.data() + l * nx, rc.data() + l * cg.nx);
  for (int k = 0; k < cfg.gamma_x; ++k) svc_recurse(L, lev + 1, ec.data(), rc.data(), cfg);
  for (int l = 0; l < nl; ++l) prolong_space(cg, g, ec.data() + l * cg.nx, corr.data() + l * nx);
  for (i64 i = 0; i < nl * nx; ++i) x[i] += corr[i];
  svc_jacobi(L, lev, cfg.nu2_x, cfg.omega_x, x, b);
}

// SpatialVCycleSolver::cycle (smoother.cpp:71-78): x = cycle from x0.
void svc_cycle(const Level& L, const double* b, const double* x0, double* x, const SvcCfg& cfg) {
  const i64 sl = L.slab();
  if (x0) std::copy(x0, x0 + sl, x);
  else std::fill(x, x + sl, 0.0);
  svc_recurse(L, 0, x, b, cfg);
}

// block_jacobi_step (smoother.cpp:96-106) with block_solver = spatial_vcycle:
// u_n += omega_t * cycle(r_n, 0) on the frozen residual.
void smooth_inexact(const Level& L, double* u, const double* f, double omega, int nu,
                    const SvcCfg& cfg) {
  const i64 sl = L.slab();
  std::vector<double> r(L.size());
  for (int s = 0; s < nu; ++s) {
    residual(L, u, f, r.data());
#pragma omp parallel for schedule(static)
    for (i64 n = 0; n < L.n_t; ++n) {
      std::vector<double> x(sl);
      svc_cycle(L, r.data() + n * sl, nullptr, x.data(), cfg);
      for (i64 i = 0; i < sl; ++i) u[n * sl + i] += omega * x[i];
    }
  }
}

// transfer.cpp:75-85: c_n = U_2n R1^T + U_2n+1 R2^T.
void restrict_semi(const Level& F, i64 nx, const double* fine, double* coarse) {
  if (F.n_t % 2 != 0) throw std::invalid_argument("restrict_semi requires an even step count");
  const int nl = F.dg.nl();
  const i64 nc = F.n_t / 2, sl = nx * nl;
  const double* R1 = F.tt.R1.data();
  const double* R2 = F.tt.R2.data();
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < nc; ++n) {
    const double* a = fine + 2 * n * sl;
    const double* b = a + sl;
    double* c = coarse + n * sl;
    for (int k = 0; k < nl; ++k)
      for (i64 r = 0; r < nx; ++r) {
        double s = 0.0;
        for (int l = 0; l < nl; ++l) s += a[l * nx + r] * R1[k * nl + l];
        double t = 0.0;
        for (int l = 0; l < nl; ++l) t += b[l * nx + r] * R2[k * nl + l];
        c[k * nx + r] = s + t;
      }
  }
}

// transfer.cpp:87-96: U_2n = C_n R1, U_2n+1 = C_n R2.
void prolong_semi(const Level& F, i64 nx, const double* coarse, double* fine) {
  const int nl = F.dg.nl();
  const i64 nc = F.n_t / 2, sl = nx * nl;
  const double* R1 = F.tt.R1.data();
  const double* R2 = F.tt.R2.data();
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < nc; ++n) {
    const double* c = coarse + n * sl;
    double* a = fine + 2 * n * sl;
    double* b = a + sl;
    for (int l = 0; l < nl; ++l)
      for (i64 r = 0; r < nx; ++r) {
        double s = 0.0, t = 0.0;
        for (int k = 0; k < nl; ++k) {
          s += c[k * nx + r] * R1[k * nl + l];
          t += c[k * nx + r] * R2[k * nl + l];
        }
        a[l * nx + r] = s;
        b[l * nx + r] = t;
      }
  }
}

void restrict_level(const Hier& H, int lev, int mode, const double* fine, double* coarse) {
  const Level& F = H.levels[lev];
  if (mode == 0) mode = F.coarsen;
  if (mode == 0) throw std::invalid_argument("level has no coarser level");
  if (mode == 1) {
    restrict_semi(F, F.grid.nx, fine, coarse);
    return;
  }
  if (F.grid.level == 0) throw std::invalid_argument("cannot coarsen the level-0 space grid");
  const Grid cg = make_grid(F.grid.dim, F.grid.level - 1);
  const int nl = F.dg.nl();
  std::vector<double> tmp((F.n_t / 2) * F.grid.nx * nl);
  restrict_semi(F, F.grid.nx, fine, tmp.data());
  const i64 nc = F.n_t / 2;
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < nc; ++n)
    for (int l = 0; l < nl; ++l)
      restrict_space(F.grid, cg, tmp.data() + (n * nl + l) * F.grid.nx, coarse + (n * nl + l) * cg.nx);
}

void prolong_level(const Hier& H, int lev, int mode, const double* coarse, double* fine) {
  const Level& F = H.levels[lev];
  if (mode == 0) mode = F.coarsen;
  if (mode == 0) throw std::invalid_argument("level has no coarser level");
  if (mode == 1) {
    prolong_semi(F, F.grid.nx, coarse, fine);
    return;
  }
  if (F.grid.level == 0) throw std::invalid_argument("cannot coarsen the level-0 space grid");
  const Grid cg = make_grid(F.grid.dim, F.grid.level - 1);
  const int nl = F.dg.nl();
  const i64 nc = F.n_t / 2;
  std::vector<double> tmp(nc * F.grid.nx * nl);
#pragma omp parallel for schedule(static)
  for (i64 n = 0; n < nc; ++n)
    for (int l = 0; l < nl; ++l)
      prolong_space(cg, F.grid, coarse + (n * nl + l) * cg.nx, tmp.data() + (n * nl + l) * F.grid.nx);
  prolong_semi(F, F.grid.nx, tmp.data(), fine);
}

// --------------------------------------------------------------------- mg --
SvcCfg svc_of(double omega_x, int nu1_x, int nu2_x, int gamma_x) {
  SvcCfg c;
  c.omega_x = omega_x;
  c.nu1_x = nu1_x;
  c.nu2_x = nu2_x;
  c.gamma_x = gamma_x;
  if (nu1_x < 0 || nu2_x < 0 || gamma_x < 1)
    throw std::invalid_argument("spatial smoothing counts must be >= 0 and gamma_x >= 1");
  return c;
}

// block_jacobi_step dispatch on SmootherConfig::block_solver (smoother.cpp:82-92).
void smooth_cfg(const Level& L, double* u, const double* f, const or_cycle& cfg, int nu) {
  if (cfg.block_solver == 1)
    smooth_inexact(L, u, f, cfg.omega_t, nu,
                   svc_of(cfg.omega_x, cfg.nu1_x, cfg.nu2_x, cfg.gamma_x));
  else
    smooth(L, u, f, cfg.omega_t, nu);
}

// mg.cpp:96-132.
void mg_cycle(const Hier& H, size_t lev, double* u, const double* f, const or_cycle& cfg) {
  const Level& L = H.levels[lev];
  if (lev + 1 == H.levels.size()) {
    forward_substitution(L, f, u);
    return;
  }
  smooth_cfg(L, u, f, cfg, cfg.nu1);
  const Level& C = H.levels[lev + 1];
  // Temporaries are scoped so at most one fine-level vector is alive besides
  // u and f (full-size fixtures of C3/C5 run on the CPU box).
  std::vector<double> ec(C.size(), 0.0);
  {
    std::vector<double> rc(C.size());
    {
      std::vector<double> r(L.size());
      residual(L, u, f, r.data());
      restrict_level(H, int(lev), 0, r.data(), rc.data());
    }
    for (int g = 0; g < cfg.gamma; ++g) mg_cycle(H, lev + 1, ec.data(), rc.data(), cfg);
  }
  {
    std::vector<double> corr(L.size());
    prolong_level(H, int(lev), 0, ec.data(), corr.data());
    const i64 sz = L.size();
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < sz; ++i) u[i] += corr[i];
  }
  smooth_cfg(L, u, f, cfg, cfg.nu2);
}

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

const Level& level_of(const or_hier* h, int level);

}  // namespace

struct or_hier {
  Hier H;
};

namespace {
const Level& level_of(const or_hier* h, int level) {
  if (!h) throw std::invalid_argument("null hierarchy");
  if (level < 0 || level >= int(h->H.levels.size())) throw std::invalid_argument("level index out of range");
  return h->H.levels[level];
}
}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }

int or_assemble_dg(int p_t, double tau, double* K, double* M, double* N) {
  return guard([&] {
    const DG b = assemble_dg(p_t, tau);
    std::copy(b.K.begin(), b.K.end(), K);
    std::copy(b.M.begin(), b.M.end(), M);
    std::copy(b.N.begin(), b.N.end(), N);
  });
}

int or_time_transfer(int p_t, double tau, double* R1, double* R2) {
  return guard([&] {
    const TT t = time_transfer(p_t, tau);
    std::copy(t.R1.begin(), t.R1.end(), R1);
    std::copy(t.R2.begin(), t.R2.end(), R2);
  });
}

double or_pade(int p_t, double z) {
  double v = NAN;
  guard([&] { v = pade(p_t, z); });
  return v;
}

double or_critical_mu(int p_t) {
  double v = NAN;
  guard([&] { v = critical_mu(p_t); });
  return v;
}

int or_hier_create(const or_params* p, or_hier** out) {
  return guard([&] {
    if (!p || !out) throw std::invalid_argument("null argument");
    auto h = std::make_unique<or_hier>();
    h->H = build_hierarchy(*p);
    *out = h.release();
  });
}

void or_hier_destroy(or_hier* h) { delete h; }

int or_hier_levels(const or_hier* h) { return h ? int(h->H.levels.size()) : 0; }

int or_level_info_get(const or_hier* h, int level, or_level_info* o) {
  return guard([&] {
    const Level& L = level_of(h, level);
    o->n_t = L.n_t;
    o->n_x = L.grid.nx;
    o->n_loc = L.nl();
    o->n1 = L.grid.n1;
    o->dim = L.grid.dim;
    o->space_level = L.grid.level;
    o->coarsen_to_next = L.coarsen;
    o->tau = L.dg.tau;
    o->h = L.grid.h;
    o->mu = L.mu;
  });
}

int or_apply(const or_hier* h, int level, const double* u, double* y) {
  return guard([&] { apply(level_of(h, level), u, y); });
}

int or_residual(const or_hier* h, int level, const double* u, const double* f, double* r) {
  return guard([&] { residual(level_of(h, level), u, f, r); });
}

double or_residual_norm(const or_hier* h, int level, const double* u, const double* f) {
  double out = NAN;
  guard([&] { out = residual_norm(level_of(h, level), u, f); });
  return out;
}

double or_norm(const or_hier* h, int level, const double* v) {
  double out = NAN;
  guard([&] { out = norm(level_of(h, level), v); });
  return out;
}

int or_block_solve(const or_hier* h, int level, const double* b, double* x) {
  return guard([&] {
    const Level& L = level_of(h, level);
    const i64 sl = L.slab();
#pragma omp parallel for schedule(static)
    for (i64 n = 0; n < L.n_t; ++n) block_solve(L, b + n * sl, x + n * sl);
  });
}

int or_forward_substitution(const or_hier* h, int level, const double* f, double* u) {
  return guard([&] { forward_substitution(level_of(h, level), f, u); });
}

int or_smooth(const or_hier* h, int level, double* u, const double* f, double omega_t, int nu) {
  return guard([&] { smooth(level_of(h, level), u, f, omega_t, nu); });
}

int or_smooth_ex(const or_hier* h, int level, double* u, const double* f, const or_smoother* sc) {
  return guard([&] {
    if (!sc) throw std::invalid_argument("null smoother config");
    const Level& L = level_of(h, level);
    if (sc->block_solver == 1)
      smooth_inexact(L, u, f, sc->omega_t, sc->nu,
                     svc_of(sc->omega_x, sc->nu1_x, sc->nu2_x, sc->gamma_x));
    else
      smooth(L, u, f, sc->omega_t, sc->nu);
  });
}

int or_spatial_vcycle(const or_hier* h, int level, const double* b, const double* x0, double* x,
                      const or_smoother* sc) {
  return guard([&] {
    if (!sc) throw std::invalid_argument("null smoother config");
    const Level& L = level_of(h, level);
    const SvcCfg cfg = svc_of(sc->omega_x, sc->nu1_x, sc->nu2_x, sc->gamma_x);
    const i64 sl = L.slab();
#pragma omp parallel for schedule(static)
    for (i64 n = 0; n < L.n_t; ++n)
      svc_cycle(L, b + n * sl, x0 ? x0 + n * sl : nullptr, x + n * sl, cfg);
  });
}

int or_restrict(const or_hier* h, int level, int mode, const double* fine, double* coarse) {
  return guard([&] {
    level_of(h, level);
    restrict_level(h->H, level, mode, fine, coarse);
  });
}

int or_prolong(const or_hier* h, int level, int mode, const double* coarse, double* fine) {
  return guard([&] {
    level_of(h, level);
    prolong_level(h->H, level, mode, coarse, fine);
  });
}

int or_mg_cycle(const or_hier* h, int level, double* u, const double* f, const or_cycle* cfg) {
  return guard([&] {
    level_of(h, level);
    mg_cycle(h->H, size_t(level), u, f, *cfg);
  });
}

// mg.cpp:134-166.
int or_solve(const or_hier* h, const double* f, double* u, const or_cycle* cfg, double eps,
             int max_iter, double* history, int history_cap, int* iterations, int* converged,
             double* wall_seconds) {
  return guard([&] {
    if (!(eps > 0.0)) throw std::invalid_argument("eps_mg must be positive");
    const Level& L = level_of(h, 0);
    const auto t0 = std::chrono::steady_clock::now();
    const double r0 = residual_norm(L, u, f);
    int it = 0, conv = 0, nh = 0;
    if (history && nh < history_cap) history[nh++] = r0;
    if (r0 == 0.0) {
      conv = 1;
    } else {
      for (int k = 0; k < max_iter; ++k) {
        mg_cycle(h->H, 0, u, f, *cfg);
        const double rk = residual_norm(L, u, f);
        if (history && nh < history_cap) history[nh++] = rk;
        ++it;
        if (rk <= eps * r0) {
          conv = 1;
          break;
        }
      }
    }
    *iterations = it;
    *converged = conv;
    *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

void or_fill_uniform(double* v, int64_t n, uint64_t seed, uint64_t stream, int64_t offset) {
  const uint64_t gamma = 0x9E3779B97F4A7C15ULL;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t ctr = (stream << 56) + uint64_t(offset + i);
    const uint64_t x = mix64(seed + gamma * ctr);
    v[i] = 2.0 * (double(x >> 11) * 0x1.0p-53) - 1.0;
  }
}

int or_fold_u0(const or_hier* h, double* f, const double* u0) {
  return guard([&] {
    const Level& L = level_of(h, 0);
    const i64 nx = L.grid.nx;
    std::vector<double> mu0(nx);
    space_apply(L.grid, false, u0, mu0.data());
    for (int k = 0; k < L.nl(); ++k) {
      const double a = basis(k, 0.0, L.dg.tau);  // psi_k(0) = (-1)^k
      for (i64 r = 0; r < nx; ++r) f[k * nx + r] += a * mu0[r];
    }
  });
}

}  // extern "C"
