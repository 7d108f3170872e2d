// stmg_spatial.cu -- sm_100a kernels of the inexact block solver: one spatial
// V-cycle per time-step block (SpatialVCycleSolver, smoother.cpp:8-78) for
// all time steps of a level at once, in the orthonormal sine basis.
//
// On the uniform Dirichlet grid every operator of the spatial cycle is
// diagonal in the sine modes or couples only the 2^dim alias modes of full
// weighting:
//  * the block A = M_h (x) K_tau + K_h (x) M_tau acts per mode as the
//    (p_t+1)^2 block A_j = M_j K_tau + K_j M_tau;
//  * the damped point-block Jacobi smoother x += w D^-1 (b - A x) has a
//    constant node block D = diag(M_h) K_tau + diag(K_h) M_tau (uniform
//    grid, smoother.cpp:16-20), so D is the same (p_t+1)^2 block per mode;
//  * restrict_space_slice / prolong_space_slice (transfer.cpp:98-136) map the
//    alias group {k, N-k}^dim onto coarse mode k with the per-axis factors
//    (1 + cos)/sqrt(2) (the same tables as the space-time full coarsening);
//  * the 1-node grid's direct solve (smoother.cpp:43-50) is one mode.
// So the cycle is the reference's cycle in an orthonormal basis.  One
// thread owns one alias-group member of one time step; a down kernel does
// nu1_x sweeps + residual + restriction of one sub-level (the group sum is a
// masked warp shuffle), an up kernel prolongation + correction + nu2_x
// sweeps; the finest up kernel also applies the smoother update
// u += omega_t x (block_jacobi_step, smoother.cpp:96-106).
//
// All arithmetic is FP64.  Indexing is 64-bit.

#include "stmg_modal.cuh"

namespace stmg {
namespace {

template <int NL>
__device__ __forceinline__ void ld_nl(const double* p, i64 nx, double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) v[l] = p[l * nx];
}
template <int NL>
__device__ __forceinline__ void st_nl(double* p, i64 nx, const double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) p[l * nx] = v[l];
}

// nu damped point-block Jacobi sweeps of one mode: x += w D^-1 (b - A_j x).
template <int NL>
__device__ __forceinline__ void jacobi_mode(const TM<NL>& t, const ModeLU<NL>& dlu, double Mj,
                                            double Kj, double omega, int nu,
                                            const double (&b)[NL], double (&x)[NL]) {
  for (int s = 0; s < nu; ++s) {
    double ax[NL], r[NL], d[NL];
    apply_mode<NL>(t, Mj, Kj, x, ax);
#pragma unroll
    for (int l = 0; l < NL; ++l) r[l] = b[l] - ax[l];
    dlu.solve(r, d);
#pragma unroll
    for (int l = 0; l < NL; ++l) x[l] += omega * d[l];
  }
}

// b = f_n - A_j u_n + M_j N u_{n-1} (space-time residual of one mode, sine basis).
template <int NL>
__device__ __forceinline__ void st_residual(const TM<NL>& t, double Mj, double Kj,
                                            const double* f, const double* u, i64 n, i64 slab,
                                            i64 nx, bool has_prev, double (&b)[NL]) {
  double fv[NL], un[NL], ax[NL];
  ld_nl<NL>(f + n * slab, nx, fv);
  ld_nl<NL>(u + n * slab, nx, un);
  apply_mode<NL>(t, Mj, Kj, un, ax);
  double nv[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) nv[l] = 0.0;
  if (has_prev) {
    double up[NL];
    ld_nl<NL>(u + (n - 1) * slab, nx, up);
    matvec<NL>(t.N, up, nv);
  }
#pragma unroll
  for (int l = 0; l < NL; ++l) b[l] = fv[l] - ax[l] + Mj * nv[l];
}

// Down: [b = residual of u (first)] -> nu1_x sweeps from x (0 if zero) ->
// residual -> restriction onto the next sub-level (or, when that is the
// 1-node grid, its direct solve).  Threads: x = alias-group member lane,
// y = time steps (grid-stride).
template <int DIM, int NL>
__global__ void __launch_bounds__(128) k_svc_down(
    const double* __restrict__ f, const double* __restrict__ u, double* __restrict__ B,
    double* __restrict__ X, double* __restrict__ C, const TM<NL> t, const SP s, const i64 n1c,
    const double md, const double kd, const double mc, const double kc, const double omega,
    const int nu, const i64 n_t, const bool first, const bool zero, const bool to_coarsest) {
  const i64 tid = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const Member me = make_member<DIM>(s, tid, n1c, true);
  const ModeLU<NL> dlu(t, md, kd);
  const ModeLU<NL> clu(t, mc, kc);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = ipow(n1c, DIM), cslab = NL * nxc;
  const bool leader = (threadIdx.x & ((1 << DIM) - 1)) == 0;
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    double b[NL], x[NL], rr[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) b[l] = x[l] = rr[l] = 0.0;
    if (me.ok) {
      if (first) {
        st_residual<NL>(t, me.Mj, me.Kj, f + me.idx, u + me.idx, n, slab, nx, n > 0, b);
        st_nl<NL>(B + n * slab + me.idx, nx, b);
      } else {
        ld_nl<NL>(B + n * slab + me.idx, nx, b);
      }
      if (!zero) ld_nl<NL>(X + n * slab + me.idx, nx, x);
      jacobi_mode<NL>(t, dlu, me.Mj, me.Kj, omega, nu, b, x);
      st_nl<NL>(X + n * slab + me.idx, nx, x);
      double ax[NL];
      apply_mode<NL>(t, me.Mj, me.Kj, x, ax);
#pragma unroll
      for (int l = 0; l < NL; ++l) rr[l] = me.cok ? me.fac * (b[l] - ax[l]) : 0.0;
    }
    double c[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) c[l] = group_sum<DIM>(rr[l]);
    if (leader && me.cok) {
      if (to_coarsest) {
        double xc[NL];
        clu.solve(c, xc);
        st_nl<NL>(C + n * cslab + me.cidx, nxc, xc);
      } else {
        st_nl<NL>(C + n * cslab + me.cidx, nxc, c);
      }
    }
  }
}

// Up: x = X + P e (e = next sub-level's iterate) -> nu2_x sweeps -> X, or on
// the finest sub-level of the smoother u += omega_t x.
template <int DIM, int NL>
__global__ void __launch_bounds__(128) k_svc_up(
    const double* __restrict__ E, const double* __restrict__ B, double* __restrict__ X,
    double* __restrict__ u, const TM<NL> t, const SP s, const i64 n1c, const double md,
    const double kd, const double omega, const int nu, const double omega_t, const i64 n_t) {
  const i64 tid = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const Member me = make_member<DIM>(s, tid, n1c, true);
  if (!me.ok) return;  // no shuffles below
  const ModeLU<NL> dlu(t, md, kd);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = ipow(n1c, DIM), cslab = NL * nxc;
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    double b[NL], x[NL];
    ld_nl<NL>(B + n * slab + me.idx, nx, b);
    ld_nl<NL>(X + n * slab + me.idx, nx, x);
    if (me.cok) {
      double e[NL];
      ld_nl<NL>(E + n * cslab + me.cidx, nxc, e);
#pragma unroll
      for (int l = 0; l < NL; ++l) x[l] += me.fac * e[l];
    }
    jacobi_mode<NL>(t, dlu, me.Mj, me.Kj, omega, nu, b, x);
    if (u) {
      double* p = u + n * slab + me.idx;
#pragma unroll
      for (int l = 0; l < NL; ++l) p[l * nx] += omega_t * x[l];
    } else {
      st_nl<NL>(X + n * slab + me.idx, nx, x);
    }
  }
}

// 1-node grid (no coarser sub-level): x = A^-1 b directly (smoother.cpp:43-50);
// [b = residual of u (first)]; u += omega_t x when u_final, else X = x.
template <int DIM, int NL>
__global__ void __launch_bounds__(128) k_svc_direct(
    const double* __restrict__ f, const double* __restrict__ u, double* __restrict__ B,
    double* __restrict__ X, double* __restrict__ u_final, const TM<NL> t, const SP s,
    const double omega_t, const i64 n_t, const bool first) {
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.nx) return;
  double Mj, Kj;
  mode_eig<DIM>(s, r, Mj, Kj);
  const ModeLU<NL> lu(t, Mj, Kj);
  const i64 nx = s.nx, slab = NL * nx;
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    double b[NL], x[NL];
    if (first) st_residual<NL>(t, Mj, Kj, f + r, u + r, n, slab, nx, n > 0, b);
    else ld_nl<NL>(B + n * slab + r, nx, b);
    lu.solve(b, x);
    if (u_final) {
      double* p = u_final + n * slab + r;
#pragma unroll
      for (int l = 0; l < NL; ++l) p[l * nx] += omega_t * x[l];
    } else {
      st_nl<NL>(X + n * slab + r, nx, x);
    }
  }
}

}  // namespace

cudaError_t launch_svc_down(const LevelView& L, const SvcArgs& a, bool first, bool zero,
                            bool to_coarsest, const double* f, const double* u, double* B,
                            double* X, double* C, cudaStream_t st) {
  if (L.n_t == 0) return cudaSuccess;
  const SP s = make_sp(a.sp);
  i64 lanes = int64_t(1) << a.sp.dim;
  for (int d = 0; d < a.sp.dim; ++d) lanes *= s.G;
  STMG_DISPATCH(a.sp.dim, L.tc.nl, {
    k_svc_down<DIM, NL><<<grid2(lanes, L.n_t, 128), 128, 0, st>>>(
        f, u, B, X, C, make_tm<NL>(L.tc), s, a.n1c, a.md, a.kd, a.mc, a.kc, a.omega_x, a.nu,
        L.n_t, first, zero, to_coarsest);
  });
  return cudaGetLastError();
}

cudaError_t launch_svc_up(const LevelView& L, const SvcArgs& a, const double* E, const double* B,
                          double* X, double* u, double omega_t, cudaStream_t st) {
  if (L.n_t == 0) return cudaSuccess;
  const SP s = make_sp(a.sp);
  i64 lanes = int64_t(1) << a.sp.dim;
  for (int d = 0; d < a.sp.dim; ++d) lanes *= s.G;
  STMG_DISPATCH(a.sp.dim, L.tc.nl, {
    k_svc_up<DIM, NL><<<grid2(lanes, L.n_t, 128), 128, 0, st>>>(
        E, B, X, u, make_tm<NL>(L.tc), s, a.n1c, a.md, a.kd, a.omega_x, a.nu, omega_t, L.n_t);
  });
  return cudaGetLastError();
}

cudaError_t launch_svc_direct(const LevelView& L, const SvcArgs& a, bool first, const double* f,
                              const double* u, double* B, double* X, double* u_final,
                              double omega_t, cudaStream_t st) {
  if (L.n_t == 0) return cudaSuccess;
  const SP s = make_sp(a.sp);
  STMG_DISPATCH(a.sp.dim, L.tc.nl, {
    k_svc_direct<DIM, NL><<<grid2(s.nx, L.n_t, 128), 128, 0, st>>>(
        f, u, B, X, u_final, make_tm<NL>(L.tc), s, omega_t, L.n_t, first);
  });
  return cudaGetLastError();
}

}  // namespace stmg
