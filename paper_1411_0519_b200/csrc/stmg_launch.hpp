// stmg_launch.hpp -- internal interface between the host driver
// (stmg_capi.cu) and the sm_100a kernels (stmg_kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace stmg {

constexpr int kMaxNL = 11;  // p_t <= kMaxTimeDegree = 10 (dg_time.hpp:10)
constexpr int kFastNL = 4;  // the fused spectral kernels: p_t <= 3

// DG time-step blocks and transfer blocks, row-major with row stride kMaxNL.
struct TimeConsts {
  int nl = 1;
  double K[kMaxNL * kMaxNL] = {};
  double M[kMaxNL * kMaxNL] = {};
  double N[kMaxNL * kMaxNL] = {};
  double R1[kMaxNL * kMaxNL] = {};
  double R2[kMaxNL * kMaxNL] = {};
  double psi0[kMaxNL] = {};  // psi_k(0), for folding u0
};

// Uniform Dirichlet grid of one level and its device-side sine tables.
struct SpaceConsts {
  int dim = 1;
  int64_t n1 = 1;  // interior nodes per axis
  int64_t nx = 1;  // n1^dim
  double h = 0.5;
  const double* mval = nullptr;  // [n1] eigenvalues of M1 in the sine basis
  const double* kval = nullptr;  // [n1] eigenvalues of K1
  const double* rfac = nullptr;  // [n1] full-weighting factor per fine mode
};

// One level as the kernels see it.  first_global: local step 0 is global
// step 0 (no previous slab); otherwise step -1/-2 live in halo slabs in
// front of every level buffer.
struct LevelView {
  int64_t n_t = 1;  // local time steps
  bool first_global = true;
  TimeConsts tc;
  SpaceConsts sp;
  int64_t slab() const { return int64_t(tc.nl) * sp.nx; }
  int64_t size() const { return n_t * slab(); }
};

// ---- physical-space operators (nodal values) ------------------------------
// ab: device array [a_0..a_{kMaxNL}), [b_0..) with N_tau = a b^T.
cudaError_t launch_apply(const LevelView& L, const double* u, const double* f,
                         double* y, bool residual, const double* ab, cudaStream_t st);
// Row-band variant (stmg_apply.cu); cudaErrorNotSupported when the level's
// shape has no such kernel (launch_apply falls through to the tile kernels).
cudaError_t launch_apply_rows(const LevelView& L, const double* u, const double* f,
                              double* y, bool residual, const double* ab, cudaStream_t st);
cudaError_t launch_restrict(const LevelView& F, int mode, int64_t n1c,
                            const double* fine, double* coarse, cudaStream_t st);
cudaError_t launch_prolong(const LevelView& F, int mode, int64_t n1c,
                           const double* coarse, double* fine, cudaStream_t st);
cudaError_t launch_fold_u0(const LevelView& L, double* f, const double* u0,
                           cudaStream_t st);
// Orthonormal DST-I along `axis` of every line of a level vector (in may be
// == out).  accumulate: out += alpha * DST(in), else out = DST(in).
cudaError_t launch_dst_axis(const LevelView& L, int axis, const double* in,
                            double* out, bool accumulate, double alpha,
                            const void* twiddles, cudaStream_t st);
// Both axes of every slab of a 2D level in one pass (thread-block cluster per
// slab); cudaErrorNotSupported when the shape has no one-pass kernel.
cudaError_t launch_dst2d(const LevelView& L, const double* in, double* out,
                         bool accumulate, double alpha, const void* twiddles,
                         cudaStream_t st);
// Constant tables of the kernels (dense DST-I matrix); once per process/device.
cudaError_t init_kernel_tables();
// Per-mode exact block solve in the sine basis, in place.
cudaError_t launch_modal_solve(const LevelView& L, double* x, cudaStream_t st);
// Per-mode sequential forward substitution in the sine basis.
cudaError_t launch_modal_fwdsub(const LevelView& L, const double* f, double* u,
                                cudaStream_t st);
// Per-step sum of squares: partial[n] = sum over slab n of v^2.
cudaError_t launch_step_sumsq(const LevelView& L, const double* v,
                              double* partial, cudaStream_t st);
// out[0] = sqrt(sum partial[0..n)) in a fixed order; hist[hidx] too if hist.
cudaError_t launch_norm_final(const double* partial, int64_t n, double* out,
                              double* hist, int hidx, cudaStream_t st);
cudaError_t launch_fill_uniform(double* v, int64_t n, uint64_t seed,
                                uint64_t stream, int64_t offset, cudaStream_t st);
cudaError_t launch_axpy(double* y, const double* x, double a, int64_t n,
                        cudaStream_t st);
// Device-side stop test: hist[++iter] = norm; loop while norm > eps*r0 and
// iter < max_iter (sets the conditional handle of the solve graph).
cudaError_t launch_decide(cudaGraphConditionalHandle h, const double* norm, const double* r0,
                          double* hist, int* iter, double eps, int max_iter, int* parity,
                          cudaStream_t st);
// launch_norm_final(partial, n, out) + launch_decide(h, out, ...) in one kernel.
cudaError_t launch_norm_decide(const double* partial, int64_t n, double* out,
                               cudaGraphConditionalHandle h, const double* r0, double* hist,
                               int* iter, double eps, int max_iter, int* parity,
                               cudaStream_t st);

// ---- fused spectral V-cycle kernels (sine coefficients) -------------------
struct ModalArgs {
  double omega = 0.5;
  int chunk = 2;         // time steps per thread (even)
  int64_t n1c = 0;       // coarse nodes per axis (full coarsening)
  int mode = 1;          // 1 semi, 2 full (coarsening to the next level)
  int64_t n_partials = 0;  // out: number of partial sums written
  int block = 128;         // threads per CTA of launch_updown (pick_updown_block)
};
// Pre-smooth (one damped block-Jacobi sweep) + residual + restriction.
// zero_guess: u_in == 0 (coarse levels).  Writes u_out and fc.
cudaError_t launch_down(const LevelView& L, ModalArgs& a, bool zero_guess,
                        const double* f, const double* u_in, double* u_out,
                        double* fc, cudaStream_t st);
// Prolong + correct + post-smooth (+ residual sum of squares if partials).
cudaError_t launch_up(const LevelView& L, ModalArgs& a, const double* ec,
                      const double* u_in, const double* f, double* u_out,
                      double* partials, cudaStream_t st);
// Plain damped block-Jacobi sweep u_out = S(u_in).
cudaError_t launch_smooth(const LevelView& L, ModalArgs& a, bool zero_guess,
                          const double* f, const double* u_in, double* u_out,
                          cudaStream_t st);
// Fused level-0 kernel: post-smooth of cycle k + pre-smooth/residual/restriction of
// cycle k+1 (+ stop-test partials).  Buffers: A = tbl[*par] (in), B = tbl[1 - *par] (out).
// s0: global index of local step 0 (time-slab shards read steps -3..-1 from halos).
cudaError_t launch_updown(const LevelView& L, ModalArgs& a, const double* ec,
                          double* const* tbl, const int* par, const double* f, double* fc,
                          double* partials, cudaStream_t st, int64_t s0 = 0);
// Residual sum-of-squares partials of f - L u.
// u_zero: the iterate is known to be zero (u is not read; same partials).
cudaError_t launch_resnorm(const LevelView& L, ModalArgs& a, const double* u,
                           const double* f, double* partials, cudaStream_t st,
                           bool u_zero = false);

// Chunk length heuristic for the modal kernels at a level.
int pick_chunk(const LevelView& L, bool grouped);
// Number of partial sums written by launch_up (grouped) / launch_resnorm
// (block = 128) or launch_updown (block = pick_updown_block).
int64_t partial_count(const LevelView& L, int chunk, bool grouped, int block = 128);
// Threads per CTA of launch_updown for the GLOBAL level G (128 or 256).
int pick_updown_block(const LevelView& G, int chunk, int mode);

// Single-CTA coarse tail (levels[0..nlev) = the small levels down to the
// coarsest).  The device table is built once (outside graph capture).
struct TailSpec {
  LevelView view;
  int64_t n1c = 0;
  int mode = 0;
  double* F = nullptr;
  double* U0 = nullptr;
  double* U1 = nullptr;
};
// host_table: malloc'd host copy (free with std::free).
cudaError_t build_tail_table(const TailSpec* levels, int nlev, void** dev_table,
                             void** host_table);
// cop != nullptr: build the coarse operator instead, cop_n CTAs, CTA i runs
// the tail on e_i and writes column i of cop (row-major cop_n x cop_n).
cudaError_t launch_tail(int dim, int nl, const void* dev_table, const void* host_table, int nlev,
                        double omega, size_t smem_bytes, cudaStream_t st,
                        double* cop = nullptr, int64_t cop_n = 0);
// ---- fused coarse levels (alias-group trees, one launch per pass) ----------
// levels[0..nlev) = coarse levels a..b+1 of a V(1,1) cycle with zero initial
// guess, all coarsened fully down to b + 1.  down: levels a..b (writes U1 and
// the rhs F of a+1..b+1); up: levels b..a (reads U0 of b + 1, writes U0).
struct CsubSpec {
  LevelView view;
  int64_t n1c = 0;
  double* F = nullptr;
  double* U0 = nullptr;
  double* U1 = nullptr;
};
struct CsubPlan {
  void* ctas = nullptr;    // device CsubCta[n_ctas]
  void* roots = nullptr;   // device root group per tree
  void* params = nullptr;  // host copy of the level table (malloc'd)
  int n_ctas = 0, trees = 0, dim = 1, nl = 1, threads = 256;
};
// lanes_target: level-a lanes per CTA when packing small trees.
cudaError_t build_csub(const CsubSpec* levels, int nlev, int lanes_target, CsubPlan* plan);
cudaError_t launch_csub(const CsubPlan& plan, bool up, double omega, cudaStream_t st);
void free_csub(CsubPlan* plan);

// ---- inexact block solver: spatial V-cycle in the sine basis --------------
// (SpatialVCycleSolver, smoother.cpp:8-78; kernels in stmg_spatial.cu.)  The
// LevelView supplies n_t and the DG blocks of the space-time level; SvcArgs
// one spatial sub-level of its cycle.
struct SvcArgs {
  SpaceConsts sp;          // the sub-level's grid and sine tables
  int64_t n1c = 1;         // nodes per axis of the next (coarser) sub-level
  double md = 0.0, kd = 0.0;  // diagonals of M_h, K_h: Jacobi block D = md K + kd M
  double mc = 0.0, kc = 0.0;  // 1-node grid eigenvalues (its direct solve)
  double omega_x = 2.0 / 3.0;
  int nu = 2;              // sweeps (nu1_x down, nu2_x up)
};
// first: B = f - L u (space-time residual of u in the sine basis) instead of
// reading B.  zero: start from x = 0.  to_coarsest: C receives the next
// sub-level's direct solution (the 1-node grid) instead of its rhs.
cudaError_t launch_svc_down(const LevelView& L, const SvcArgs& a, bool first, bool zero,
                            bool to_coarsest, const double* f, const double* u, double* B,
                            double* X, double* C, cudaStream_t st);
// X += P E, nu sweeps; u != null: u += omega_t x instead of writing X.
cudaError_t launch_svc_up(const LevelView& L, const SvcArgs& a, const double* E, const double* B,
                          double* X, double* u, double omega_t, cudaStream_t st);
// Level grid of one node: x = A^-1 b; u_final != null: u_final += omega_t x.
cudaError_t launch_svc_direct(const LevelView& L, const SvcArgs& a, bool first, const double* f,
                              const double* u, double* B, double* X, double* u_final,
                              double omega_t, cudaStream_t st);

// Coarse operator of the tail: y = B x, B row-major n x n (n <= 3200).
cudaError_t launch_cop_gemv(const double* B, const double* x, double* y, int n,
                            cudaStream_t st);

// flag[0] = 1 if any v[i] != 0 (flag must be zeroed before).
cudaError_t launch_nonzero(const double* v, int64_t n, int* flag, cudaStream_t st);

}  // namespace stmg
