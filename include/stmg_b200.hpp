// stmg_b200.hpp -- C++ shim that re-exposes the reference's stmg:: API
// (/root/reference/proj/include/stmg/*.hpp) on top of the C ABI in
// stmg_b200.h.  Header-only; link against libstmg_b200.so.
//
// Differences a caller of the reference sees:
//  * vectors are device-resident (BlockVector owns a GPU allocation); use
//    from_host()/to_host() to move data (the reference's Eigen storage has no
//    equivalent here, so no Eigen dependency);
//  * an STOperator is (hierarchy, level) instead of raw dg/space pointers;
//  * errors map to the same exception types: std::invalid_argument for bad
//    arguments, std::runtime_error for CUDA/runtime failures.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "stmg_b200.h"

namespace stmg {

inline void check(int rc) {
  if (rc == STMG_OK) return;
  if (rc == STMG_EINVAL) throw std::invalid_argument(stmg_last_error());
  throw std::runtime_error(stmg_last_error());
}

enum class Coarsening { none = STMG_COARSEN_NONE, semi = STMG_COARSEN_SEMI, full = STMG_COARSEN_FULL };
enum class CoarseningPolicy {
  mu_driven = STMG_POLICY_MU_DRIVEN,
  always_semi = STMG_POLICY_ALWAYS_SEMI,
  prefer_full = STMG_POLICY_PREFER_FULL
};
enum class BlockSolverKind { exact, spatial_vcycle };

// dg_time.hpp:19-26 (row-major blocks instead of Eigen matrices)
struct DGTimeBlock {
  int p_t = 0;
  double tau = 1.0;
  std::vector<double> K, M, N;
  int n_loc() const { return p_t + 1; }
};

inline DGTimeBlock assemble_dg_block(int p_t, double tau) {
  DGTimeBlock b;
  b.p_t = p_t;
  b.tau = tau;
  const int n = p_t + 1 > 0 ? p_t + 1 : 1;
  b.K.resize(n * n);
  b.M.resize(n * n);
  b.N.resize(n * n);
  check(stmg_dg_block(p_t, tau, b.K.data(), b.M.data(), b.N.data()));
  return b;
}

// transfer.hpp:17-20
struct TimeTransfer {
  std::vector<double> R1, R2;
};

inline TimeTransfer build_time_transfer(int p_t, double tau) {
  TimeTransfer t;
  const int n = p_t + 1 > 0 ? p_t + 1 : 1;
  t.R1.resize(n * n);
  t.R2.resize(n * n);
  check(stmg_time_transfer(p_t, tau, t.R1.data(), t.R2.data()));
  return t;
}

namespace lfa {
inline double critical_mu(int p_t) {
  const double v = stmg_critical_mu(p_t);
  if (v != v) throw std::invalid_argument(stmg_last_error());
  return v;
}
// lfa.hpp:15-47 (host-side analysis; no GPU needed)
inline double beta(double theta_x) {
  double v = 0.0;
  check(stmg_lfa_beta(theta_x, &v));
  return v;
}
inline double alpha(int p_t, double mu, double theta_x) {
  double v = 0.0;
  check(stmg_lfa_alpha(p_t, mu, theta_x, &v));
  return v;
}
struct FrequencyGrid {
  int n_theta_x = 256;
  int n_theta_t = 256;
};
struct TwoGridConfig {
  double omega_t = 0.5;
  int nu1 = 1;
  int nu2 = 1;
};
struct SpatialSmootherConfig {
  double omega_x = 2.0 / 3.0;
  int nu1_x = 2;
  int nu2_x = 2;
};
inline stmg_cycle_config to_c(const TwoGridConfig& c) {
  return stmg_cycle_config{c.nu1, c.nu2, 1, c.omega_t, STMG_PATH_SPECTRAL, STMG_BLOCK_EXACT,
                           2.0 / 3.0, 2, 2, 1};
}
// lfa.hpp:125-150
inline double smoothing_factor(int p_t, double mu, double omega_t, Coarsening mode,
                               const FrequencyGrid& grid = {}) {
  double v = 0.0;
  check(stmg_lfa_smoothing_factor(p_t, mu, omega_t, int(mode), grid.n_theta_x, grid.n_theta_t,
                                  &v));
  return v;
}
inline double twogrid_factor(int p_t, double mu, const TwoGridConfig& cfg, Coarsening mode,
                             const FrequencyGrid& grid = {}) {
  const stmg_cycle_config c = to_c(cfg);
  double v = 0.0;
  check(stmg_lfa_twogrid_factor(p_t, mu, &c, int(mode), grid.n_theta_x, grid.n_theta_t, &v));
  return v;
}
inline double twogrid_factor_inexact(int p_t, double mu, const TwoGridConfig& cfg,
                                     const SpatialSmootherConfig& sp, Coarsening mode,
                                     const FrequencyGrid& grid = {}) {
  const stmg_cycle_config c = to_c(cfg);
  double v = 0.0;
  check(stmg_lfa_twogrid_factor_inexact(p_t, mu, &c, sp.omega_x, sp.nu1_x, sp.nu2_x, int(mode),
                                        grid.n_theta_x, grid.n_theta_t, &v));
  return v;
}
}  // namespace lfa

// mg.hpp:49-58
struct HierarchyParams {
  int p_t = 0;
  int dim = 1;
  int space_level = 4;
  int time_level = 4;
  double t_final = 1.0;
  double mu_star = 0.3;
  CoarseningPolicy policy = CoarseningPolicy::mu_driven;
  BlockSolverKind block_solver = BlockSolverKind::exact;
  int device = 0;
  int shards = 0;  // >1: time-slab sharding emulated on one device
};

// smoother.hpp:15-24
struct SmootherConfig {
  double omega_t = 0.5;
  int nu = 1;
  BlockSolverKind block_solver = BlockSolverKind::exact;
  // spatial multigrid used when block_solver == spatial_vcycle
  double omega_x = 2.0 / 3.0;
  int nu1_x = 2;
  int nu2_x = 2;
  int gamma_x = 1;
};
inline stmg_smoother_config to_c(const SmootherConfig& c) {
  return stmg_smoother_config{c.omega_t, c.nu, int(c.block_solver), c.omega_x,
                              c.nu1_x,   c.nu2_x, c.gamma_x};
}

// mg.hpp:66-71
struct CycleConfig {
  int nu1 = 2;
  int nu2 = 2;
  int gamma = 1;
  SmootherConfig smoother;
  int path = STMG_PATH_SPECTRAL;
};

// mg.hpp:83-89
struct SolveReport {
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  double wall_time_seconds = 0.0;
  double device_time_seconds = 0.0;
  std::uint64_t seed = 0;
};

class STHierarchy;

// st_system.hpp:18-26: a level of a hierarchy.
struct STOperator {
  stmg_ctx* ctx = nullptr;
  int level = 0;
};

struct STLevel {
  stmg_level_info info{};
  STOperator op_{};
  STOperator op() const { return op_; }
  Coarsening coarsen_to_next() const { return Coarsening(info.coarsen_to_next); }
};

class STHierarchy {
 public:
  STHierarchy() = default;
  explicit STHierarchy(const stmg_hierarchy_params& p) {
    stmg_ctx* c = nullptr;
    check(stmg_create(&p, &c));
    ctx_.reset(c, [](stmg_ctx* x) { stmg_destroy(x); });
    int n = 0;
    check(stmg_num_levels(c, &n));
    levels.resize(n);
    for (int i = 0; i < n; ++i) {
      check(stmg_get_level_info(c, i, &levels[i].info));
      levels[i].op_ = {c, i};
    }
  }
  std::vector<STLevel> levels;  // [0] = finest
  stmg_ctx* ctx() const { return ctx_.get(); }
  const STLevel& finest() const { return levels.front(); }

 private:
  std::shared_ptr<stmg_ctx> ctx_;
};

inline stmg_hierarchy_params to_c(const HierarchyParams& p, int two_grid) {
  // block_solver needs no setup on the B200 path (no factorisations; the
  // spatial cycle's constants are built on first use): the cycle config selects it.
  stmg_hierarchy_params c{};
  c.p_t = p.p_t;
  c.dim = p.dim;
  c.space_level = p.space_level;
  c.time_level = p.time_level;
  c.t_final = p.t_final;
  c.mu_star = p.mu_star;
  c.policy = int(p.policy);
  c.two_grid = two_grid;
  c.device = p.device;
  c.shards = p.shards;
  return c;
}

// mg.hpp:64 / mg.hpp:81
inline STHierarchy build_hierarchy(const HierarchyParams& p) { return STHierarchy(to_c(p, 0)); }
inline STHierarchy build_two_grid(const HierarchyParams& p, Coarsening mode) {
  if (mode == Coarsening::none) throw std::invalid_argument("two-grid needs semi or full mode");
  return STHierarchy(to_c(p, int(mode)));
}

// block_vector.hpp:12-57, device-resident.
class BlockVector {
 public:
  BlockVector() = default;
  BlockVector(stmg_ctx* ctx, std::int64_t n_t, std::int64_t n_x, std::int64_t n_loc)
      : ctx_(ctx), n_t_(n_t), n_x_(n_x), n_loc_(n_loc) {
    void* p = nullptr;
    check(stmg_device_alloc(ctx, size_t(size()) * sizeof(double), &p));
    check(stmg_memset_zero(ctx, p, size_t(size()) * sizeof(double)));
    data_.reset(static_cast<double*>(p), [ctx](double* q) { stmg_device_free(ctx, q); });
  }
  static BlockVector for_level(const STOperator& op) {
    stmg_level_info li{};
    check(stmg_get_level_info(op.ctx, op.level, &li));
    return BlockVector(op.ctx, li.n_t, li.n_x, li.n_loc);
  }
  std::int64_t n_t() const { return n_t_; }
  std::int64_t n_x() const { return n_x_; }
  std::int64_t n_loc() const { return n_loc_; }
  std::int64_t size() const { return n_t_ * n_x_ * n_loc_; }
  double* data() { return data_.get(); }
  const double* data() const { return data_.get(); }
  stmg_ctx* ctx() const { return ctx_; }
  void from_host(const std::vector<double>& v) {
    if (std::int64_t(v.size()) != size()) throw std::invalid_argument("space-time vector shape mismatch");
    check(stmg_upload(ctx_, data(), v.data(), v.size() * sizeof(double)));
    check(stmg_synchronize(ctx_));
  }
  std::vector<double> to_host() const {
    std::vector<double> v(static_cast<size_t>(size()));
    check(stmg_download(ctx_, v.data(), data(), v.size() * sizeof(double)));
    return v;
  }
  void setZero() { check(stmg_memset_zero(ctx_, data(), size_t(size()) * sizeof(double))); }

 private:
  stmg_ctx* ctx_ = nullptr;
  std::int64_t n_t_ = 0, n_x_ = 0, n_loc_ = 0;
  std::shared_ptr<double> data_;
};

inline BlockVector make_vector(const STOperator& op) { return BlockVector::for_level(op); }

// st_system.hpp:31-47
inline void apply(const STOperator& op, const BlockVector& u, BlockVector& y) {
  check(stmg_apply(op.ctx, op.level, u.data(), y.data()));
}
inline void residual(const STOperator& op, const BlockVector& u, const BlockVector& f, BlockVector& r) {
  check(stmg_residual(op.ctx, op.level, u.data(), f.data(), r.data()));
}
inline double norm(const STOperator& op, const BlockVector& v) {
  double out = 0.0;
  check(stmg_norm(op.ctx, op.level, v.data(), &out));
  return out;
}
// smoother.hpp:29-58: SpatialVCycleSolver.  On the B200 path it is bound to a
// level's operator (its DG block and finest grid) and cycles every time step
// of a level vector at once; x0 == nullptr is the smoother's zero guess.
class SpatialVCycleSolver {
 public:
  explicit SpatialVCycleSolver(const STOperator& op) : op_(op) {}
  BlockVector cycle(const BlockVector& b, const BlockVector* x0, const SmootherConfig& cfg) const {
    BlockVector x = BlockVector::for_level(op_);
    const stmg_smoother_config c = to_c(cfg);
    check(stmg_spatial_vcycle(op_.ctx, op_.level, b.data(), x0 ? x0->data() : nullptr, x.data(),
                              &c));
    return x;
  }

 private:
  STOperator op_;
};

// st_system.hpp:70-72
inline BlockVector forward_substitution_solve(const STOperator& op, const BlockVector& f) {
  BlockVector u = make_vector(op);
  check(stmg_forward_substitution(op.ctx, op.level, f.data(), u.data()));
  return u;
}
// smoother.hpp:68-70 (exact block solves or one spatial V-cycle per block)
inline void block_jacobi_step(const STOperator& op, BlockVector& u, const BlockVector& f,
                              const SmootherConfig& cfg) {
  const stmg_smoother_config c = to_c(cfg);
  check(stmg_block_jacobi_step(op.ctx, op.level, u.data(), f.data(), &c));
}

namespace detail {
inline BlockVector coarse_like(const STOperator& op, int mode) {
  stmg_level_info li{};
  check(stmg_get_level_info(op.ctx, op.level, &li));
  std::int64_t n1 = mode == STMG_COARSEN_SEMI ? li.n1 : (li.n1 - 1) / 2;
  std::int64_t nx = 1;
  for (int a = 0; a < li.dim; ++a) nx *= n1;
  return BlockVector(op.ctx, li.n_t / 2, nx, li.n_loc);
}
}  // namespace detail

// transfer.hpp:27-44
inline BlockVector restrict_semi(const STOperator& op, const BlockVector& fine) {
  BlockVector c = detail::coarse_like(op, STMG_COARSEN_SEMI);
  check(stmg_restrict(op.ctx, op.level, STMG_COARSEN_SEMI, fine.data(), c.data()));
  return c;
}
inline BlockVector restrict_full(const STOperator& op, const BlockVector& fine) {
  BlockVector c = detail::coarse_like(op, STMG_COARSEN_FULL);
  check(stmg_restrict(op.ctx, op.level, STMG_COARSEN_FULL, fine.data(), c.data()));
  return c;
}
inline BlockVector prolong_semi(const STOperator& op, const BlockVector& coarse) {
  BlockVector f = make_vector(op);
  check(stmg_prolong(op.ctx, op.level, STMG_COARSEN_SEMI, coarse.data(), f.data()));
  return f;
}
inline BlockVector prolong_full(const STOperator& op, const BlockVector& coarse) {
  BlockVector f = make_vector(op);
  check(stmg_prolong(op.ctx, op.level, STMG_COARSEN_FULL, coarse.data(), f.data()));
  return f;
}

inline stmg_cycle_config to_c(const CycleConfig& c) {
  const SmootherConfig& s = c.smoother;
  return stmg_cycle_config{c.nu1,    c.nu2,   c.gamma,   s.omega_t, c.path, int(s.block_solver),
                           s.omega_x, s.nu1_x, s.nu2_x, s.gamma_x};
}

// mg.hpp:75-76
inline void mg_cycle(const STHierarchy& h, std::size_t level, BlockVector& u, const BlockVector& f,
                     const CycleConfig& cfg) {
  const stmg_cycle_config c = to_c(cfg);
  check(stmg_mg_cycle(h.ctx(), int(level), u.data(), f.data(), &c));
}

// mg.hpp:92-94
inline SolveReport solve(const STHierarchy& h, const BlockVector& f, BlockVector& u,
                         const CycleConfig& cfg, double eps_mg, int max_iter = 250) {
  const stmg_cycle_config c = to_c(cfg);
  std::vector<double> hist(size_t(max_iter > 0 ? max_iter : 0) + 1);
  stmg_solve_report r{};
  check(stmg_solve(h.ctx(), f.data(), u.data(), &c, eps_mg, max_iter, hist.data(), int(hist.size()), &r));
  SolveReport out;
  out.iterations = r.iterations;
  out.converged = r.converged != 0;
  out.residual_history.assign(hist.begin(), hist.begin() + r.iterations + 1);
  out.wall_time_seconds = r.wall_time_seconds;
  out.device_time_seconds = r.device_time_seconds;
  out.seed = r.seed;
  return out;
}

// mg.hpp:98 / mg.cpp:168-173, reference-exact: std::mt19937_64(seed),
// v[i] = (gen() >> 11) * 2^-53 in [0, 1) over the flat BlockVector order
// (generated on the host -- the stream is sequential -- then uploaded).
inline void fill_random(BlockVector& v, std::uint64_t seed) {
  std::vector<double> h(static_cast<size_t>(v.size()));
  check(stmg_fill_random_host(h.data(), v.size(), seed));
  v.from_host(h);
}

// The benchmarks' counter-based generator: uniform [-1, 1),
// splitmix64 of (seed, stream, index), generated on the device.
inline void fill_uniform(BlockVector& v, std::uint64_t seed, std::uint64_t stream = 0) {
  check(stmg_fill_uniform(v.ctx(), v.data(), v.size(), seed, stream, 0));
}

// ---- reference-signature overloads ---------------------------------------
// fem_space.hpp:11-17 / fem_space.cpp (host only)
struct SpaceGrid {
  int dim = 1;
  int level = 0;
  double h = 0.5;
  std::int64_t n_per_dim = 1;
  std::int64_t n_nodes = 1;
};
inline SpaceGrid build_space_grid(int dim, int level) {
  if (dim < 1 || dim > 3) throw std::invalid_argument("dim must be 1, 2 or 3");
  if (level < 0) throw std::invalid_argument("level must be >= 0");
  SpaceGrid g;
  g.dim = dim;
  g.level = level;
  g.n_per_dim = (std::int64_t(1) << (level + 1)) - 1;
  g.h = 1.0 / double(g.n_per_dim + 1);
  g.n_nodes = 1;
  for (int a = 0; a < dim; ++a) g.n_nodes *= g.n_per_dim;
  return g;
}

// st_system.hpp:50-63: the exact block solver of a level (sine-basis direct
// solve on the B200 path; there is no factorisation to cache).
class BlockSolver {
 public:
  explicit BlockSolver(const STOperator& op) : op_(op) {}
  // A x = b on every time step of a level vector (the reference solves one slice)
  BlockVector solve(const BlockVector& b) const {
    BlockVector x = BlockVector::for_level(op_);
    check(stmg_block_solve(op_.ctx, op_.level, b.data(), x.data()));
    return x;
  }
  const STOperator& op() const { return op_; }

 private:
  STOperator op_;
};

// smoother.hpp:60-63
struct BlockSolveContext {
  const BlockSolver* exact = nullptr;
  const SpatialVCycleSolver* vcycle = nullptr;
};

// smoother.hpp:68-70: cfg.block_solver picks the solver (smoother.cpp:82-92);
// the context must carry it.
inline void block_jacobi_step(const STOperator& op, const BlockSolveContext& ctx, BlockVector& u,
                              const BlockVector& f, const SmootherConfig& cfg) {
  if (cfg.block_solver == BlockSolverKind::exact ? ctx.exact == nullptr : ctx.vcycle == nullptr)
    throw std::invalid_argument("block_jacobi_step: the context lacks the configured block solver");
  block_jacobi_step(op, u, f, cfg);
}

// st_system.hpp:70-72
inline BlockVector forward_substitution_solve(const STOperator& op, const BlockSolver& block_lu,
                                              const BlockVector& f) {
  (void)block_lu;  // the level's direct solve is part of the context
  return forward_substitution_solve(op, f);
}

namespace detail {
// The hierarchy level a vector belongs to, from its shape (n_t halves every
// level, so (n_t, n_x) is unique); grid_level >= 0 also checks the space level.
inline STOperator level_of(const BlockVector& v, int grid_level = -1) {
  int n = 0;
  check(stmg_num_levels(v.ctx(), &n));
  for (int l = 0; l < n; ++l) {
    stmg_level_info li{};
    check(stmg_get_level_info(v.ctx(), l, &li));
    if (li.n_t == v.n_t() && li.n_x == v.n_x() && li.n_loc == v.n_loc() &&
        (grid_level < 0 || li.space_level == grid_level))
      return STOperator{v.ctx(), l};
  }
  throw std::invalid_argument("vector does not match a level of its hierarchy");
}
inline void check_transfer(const TimeTransfer& t, const BlockVector& v) {
  if (std::int64_t(t.R1.size()) != v.n_loc() * v.n_loc() || t.R1.size() != t.R2.size())
    throw std::invalid_argument("time transfer does not match the vector's DG degree");
}
}  // namespace detail

// transfer.hpp:27-28
inline BlockVector restrict_semi(const TimeTransfer& t, const BlockVector& fine) {
  detail::check_transfer(t, fine);
  if (fine.n_t() % 2 != 0) throw std::invalid_argument("restrict_semi requires an even step count");
  return restrict_semi(detail::level_of(fine), fine);
}
inline BlockVector prolong_semi(const TimeTransfer& t, const BlockVector& coarse) {
  detail::check_transfer(t, coarse);
  // the fine level: twice the steps, same nodes
  int n = 0;
  check(stmg_num_levels(coarse.ctx(), &n));
  for (int l = 0; l < n; ++l) {
    stmg_level_info li{};
    check(stmg_get_level_info(coarse.ctx(), l, &li));
    if (li.n_t == 2 * coarse.n_t() && li.n_x == coarse.n_x() && li.n_loc == coarse.n_loc())
      return prolong_semi(STOperator{coarse.ctx(), l}, coarse);
  }
  throw std::invalid_argument("vector does not match a level of its hierarchy");
}
// transfer.hpp:41-44
inline BlockVector restrict_full(const TimeTransfer& t, const SpaceGrid& fine_grid,
                                 const SpaceGrid& coarse_grid, const BlockVector& fine) {
  detail::check_transfer(t, fine);
  if (coarse_grid.level + 1 != fine_grid.level || fine.n_x() != fine_grid.n_nodes)
    throw std::invalid_argument("restrict_full: grids do not match the vector");
  return restrict_full(detail::level_of(fine, fine_grid.level), fine);
}
inline BlockVector prolong_full(const TimeTransfer& t, const SpaceGrid& coarse_grid,
                                const SpaceGrid& fine_grid, const BlockVector& coarse) {
  detail::check_transfer(t, coarse);
  if (coarse_grid.level + 1 != fine_grid.level || coarse.n_x() != coarse_grid.n_nodes)
    throw std::invalid_argument("prolong_full: grids do not match the vector");
  int n = 0;
  check(stmg_num_levels(coarse.ctx(), &n));
  for (int l = 0; l < n; ++l) {
    stmg_level_info li{};
    check(stmg_get_level_info(coarse.ctx(), l, &li));
    if (li.n_t == 2 * coarse.n_t() && li.space_level == fine_grid.level &&
        li.n_loc == coarse.n_loc())
      return prolong_full(STOperator{coarse.ctx(), l}, coarse);
  }
  throw std::invalid_argument("vector does not match a level of its hierarchy");
}

}  // namespace stmg
