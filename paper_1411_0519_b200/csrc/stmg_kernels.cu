// stmg_kernels.cu -- sm_100a kernels of the space-time multigrid V-cycle.
//
// Two families:
//  * physical-space operators on nodal values, one per reference entry point
//    (apply/residual st_system.cpp:44-67, transfers transfer.cpp:75-158,
//    block solves st_system.cpp:103-130 via orthonormal DST-I line kernels);
//  * the fused spectral V-cycle: on a uniform Dirichlet grid the orthonormal
//    sine basis diagonalises M_h and K_h, so the damped block-Jacobi smoother
//    (smoother.cpp:96-106), the residual and the jump coupling act per mode,
//    and full weighting couples only the 2^dim "alias" modes {k, N-k} per
//    axis.  One thread owns a mode (the 2^dim members of an alias group sit in
//    adjacent lanes) and marches through a chunk of time steps, keeping the
//    previous slab in registers, so one HBM pass does
//    pre-smooth + residual + restriction (k_down) or prolongation + correction
//    + post-smooth + residual norm (k_up).
//
// All arithmetic is FP64.  Indexing is 64-bit (level vectors exceed 2^31).

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <vector>

#include <cooperative_groups.h>

#include "stmg_modal.cuh"

namespace stmg {
namespace {

// cudaFuncSetAttribute is per device: a launcher sets a kernel's attributes on
// the first launch on each device (bit d of the mask = done on device d).
struct PerDevice {
  std::atomic<unsigned long long> mask{0};
  bool first_use() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    return (mask.fetch_or(b) & b) == 0;
  }
};

// ==================================================== fused spectral kernels
// Loads: the standalone kernels read through the read-only / streaming paths;
// the single-CTA tail kernel reads data written earlier in the same launch
// (in shared memory), so it uses plain generic loads (COH).
template <bool COH, int NL>
__device__ __forceinline__ void ld_ro(const double* p, i64 nx, double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) v[l] = COH ? p[l * nx] : __ldg(p + l * nx);
}
template <bool COH, int NL>
__device__ __forceinline__ void ld_st(const double* p, i64 nx, double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) v[l] = COH ? p[l * nx] : __ldcs(p + l * nx);
}

// down: one damped block-Jacobi sweep, the residual of the smoothed iterate
// and its restriction, for steps [n0, nend) of one mode (lane `tid`).  The
// Jacobi sweep uses the frozen old iterate of step n-1 (smoother.cpp:101-104):
//   u'_n = (1-w) u_n + w A_j^-1 (f_n + M_j N u_{n-1}),
// the residual r_n = f_n - A_j u'_n + M_j N u'_{n-1}, and the restriction
// c_{n/2} += fac * R_{1|2} r_n summed over the alias group (transfer.cpp:75-85,
// 138-149 in the sine basis).  has_prev: step n0-1 exists (warm-up).
// WAIT: the body issues the PDL wait itself, after the per-mode setup (sine
// tables, block factors), which only reads constants and so overlaps the
// previous kernel's tail; every read of data a previous kernel wrote follows.
template <int DIM, int NL, bool ZERO, int CO, bool COH, bool ASYNC = false, bool WAIT = false>
__device__ __forceinline__ void down_body(const i64 tid, const i64 n0, const i64 nend,
                                          const double* f, const double* uin, double* uout,
                                          double* fc, const TM<NL>& t, const SP& s,
                                          const i64 n1c, const double omega, const bool has_prev,
                                          const bool has_prev2, double* ring = nullptr) {
  const Member me = make_member<DIM, COH>(s, tid, n1c, CO == 2);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = (CO == 2) ? ipow(n1c, DIM) : nx, cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const ModeOps<NL> mo(t, me.Mj, me.Kj, omega);
  if (WAIT) pdl_wait();
  const double* fp = f + me.idx;
  const double* up = uin + me.idx;
  double* op = uout + me.idx;

  double so = 0.0, sn = 0.0;  // traces of step n-1: old iterate, smoothed

  // (issued before the warm-up, whose loads and solve overlap their latency)
  // ASYNC: the loads of the next kRing-1 step pairs sit in a per-thread
  // cp.async ring in shared memory (no registers held); otherwise a register
  // prefetch of the next pair (memory-level parallelism; latency bound).
  constexpr int Q = (ZERO ? 2 : 4) * NL;  // doubles per pair
  const int T = blockDim.x;
  auto issue = [&](i64 n, int st) {  // step pair n, n+1 -> ring stage st
    double* r = ring + i64(st) * Q * T + threadIdx.x;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cp_async8(r + (e * NL + l) * T, fp + (n + e) * slab + l * nx, me.ok);
        if (!ZERO) cp_async8(r + ((2 + e) * NL + l) * T, up + (n + e) * slab + l * nx, me.ok);
      }
  };
  double f2[2][NL], u2[2][NL];
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int l = 0; l < NL; ++l) f2[e][l] = u2[e][l] = 0.0;
  if (ASYNC) {
#pragma unroll
    for (int q = 0; q < kRing - 1; ++q) {
      if (n0 + 2 * q < nend) issue(n0 + 2 * q, q);
      cp_async_commit();
    }
  } else if (me.ok && n0 < nend) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      ld_st<COH, NL>(fp + (n0 + e) * slab, nx, f2[e]);
      if (!ZERO) ld_st<COH, NL>(up + (n0 + e) * slab, nx, u2[e]);
    }
  }
  if (me.ok && has_prev) {  // warm-up: smoothed step n0-1
    double fv[NL], g[NL], w[NL];
    ld_ro<COH, NL>(fp + (n0 - 1) * slab, nx, fv);
    mo.solve_w(fv, g);
    if (ZERO) {
      sn = trace_sum<NL>(g);
    } else {
      double u1[NL], u2[NL];
      ld_ro<COH, NL>(up + (n0 - 1) * slab, nx, u1);
#pragma unroll
      for (int l = 0; l < NL; ++l) u2[l] = 0.0;
      if (has_prev2) ld_ro<COH, NL>(up + (n0 - 2) * slab, nx, u2);
      mo.sweep(u1, g, trace_sum<NL>(u2), om1, w);
      sn = trace_sum<NL>(w);
      so = trace_sum<NL>(u1);
    }
  }

  int pair = 0;
  for (i64 n = n0; n < nend; n += 2, ++pair) {
    double acc[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = 0.0;
    double fn[2][NL], un2[2][NL];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) fn[e][l] = un2[e][l] = 0.0;
    if (ASYNC) {
      cp_async_wait<kRing - 2>();  // this pair's stage has landed
      const double* r = ring + i64(pair % kRing) * Q * T + threadIdx.x;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          f2[e][l] = r[(e * NL + l) * T];
          if (!ZERO) u2[e][l] = r[((2 + e) * NL + l) * T];
        }
      if (n + 2 * (kRing - 1) < nend) issue(n + 2 * (kRing - 1), (pair + kRing - 1) % kRing);
      cp_async_commit();
    } else if (me.ok && n + 2 < nend) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ld_st<COH, NL>(fp + (n + 2 + e) * slab, nx, fn[e]);
        if (!ZERO) ld_st<COH, NL>(up + (n + 2 + e) * slab, nx, un2[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const i64 m = n + e;
      double g[NL], w[NL];
      mo.solve_w(f2[e], g);
      if (ZERO) {
#pragma unroll
        for (int l = 0; l < NL; ++l) w[l] = g[l];
      } else {
        mo.sweep(u2[e], g, so, om1, w);
      }
      if (me.ok) store_nl<NL>(op + m * slab, nx, w);
      double res[NL], rt[NL];
      mo.residual(f2[e], w, sn, res);
      if (e == 0) matvec<NL>(t.R1, res, rt);
      else matvec<NL>(t.R2, res, rt);
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] += (CO == 2) ? me.fac * rt[l] : rt[l];
      if (!ZERO) so = trace_sum<NL>(u2[e]);
      sn = trace_sum<NL>(w);
    }
    if (!ASYNC) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          f2[e][l] = fn[e][l];
          u2[e][l] = un2[e][l];
        }
    }
    const i64 nc = n >> 1;
    if (CO == 2) {
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] = group_sum<DIM>(me.ok ? acc[l] : 0.0);
      if (me.cok && (tid & ((1 << DIM) - 1)) == 0) store_nl<NL>(fc + nc * cslab + me.cidx, nxc, acc);
    } else if (me.ok) {
      store_nl<NL>(fc + nc * cslab + me.idx, nxc, acc);
    }
  }
}

// up: u <- u + P e_c (mg.cpp:123-127), then one damped block-Jacobi sweep
// (mg.cpp:129-131); with RESID also the residual of the result, returning its
// sum of squares (stop test, mg.cpp:152-153).
template <int DIM, int NL, int CO, bool RESID, bool COH, bool ASYNC = false, bool WAIT = false>
__device__ __forceinline__ double up_body(const i64 tid, const i64 n0, const i64 nend,
                                          const double* ec, const double* uin, const double* f,
                                          double* uout, const TM<NL>& t, const SP& s,
                                          const i64 n1c, const double omega, const bool has_prev,
                                          const bool has_prev2, double* ring = nullptr) {
  const Member me = make_member<DIM, COH>(s, tid, n1c, CO == 2);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = (CO == 2) ? ipow(n1c, DIM) : nx, cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const ModeOps<NL> mo(t, me.Mj, me.Kj, omega);
  if (WAIT) pdl_wait();
  const double fac = (CO == 2) ? me.fac : 1.0;
  const bool has_c = (CO == 2) ? me.cok : me.ok;
  const double* ep = ec + ((CO == 2) ? me.cidx : me.idx);
  const double* fp = f + me.idx;
  const double* up = uin + me.idx;
  double* op = uout + me.idx;
  double sumsq = 0.0;
  if (!me.ok) return 0.0;

  double so = 0.0, sw = 0.0;  // traces of step n-1: corrected, smoothed
  double ev[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) ev[l] = 0.0;

  // software pipeline (see down_body; issued before the warm-up); the
  // register prefetch is off for
  // NL > 2, where the extra registers cost more occupancy than it gains
  constexpr bool PF = !ASYNC && NL <= 2;
  constexpr int Q = 5 * NL;  // u, f of two steps + e of the coarse step
  const int T = blockDim.x;
  auto issue = [&](i64 n, int st) {
    double* r = ring + i64(st) * Q * T + threadIdx.x;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cp_async8(r + (e * NL + l) * T, up + (n + e) * slab + l * nx, true);
        cp_async8(r + ((2 + e) * NL + l) * T, fp + (n + e) * slab + l * nx, true);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l)
      cp_async8(r + (4 * NL + l) * T, has_c ? ep + (n >> 1) * cslab + l * nxc : fp, has_c);
  };
  double u2[2][NL], f2[2][NL], en[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) en[l] = 0.0;
  if (ASYNC) {
#pragma unroll
    for (int q = 0; q < kRing - 1; ++q) {
      if (n0 + 2 * q < nend) issue(n0 + 2 * q, q);
      cp_async_commit();
    }
  } else if (n0 < nend) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      ld_st<COH, NL>(up + (n0 + e) * slab, nx, u2[e]);
      ld_st<COH, NL>(fp + (n0 + e) * slab, nx, f2[e]);
    }
    if (has_c) ld_ro<COH, NL>(ep + (n0 >> 1) * cslab, nxc, en);
  }
  if (has_prev) {
    if (has_c) ld_ro<COH, NL>(ep + ((n0 >> 1) - 1) * cslab, nxc, ev);  // coarse step of n0-2, n0-1
    double u1[NL], c1[NL], vo[NL];
    ld_ro<COH, NL>(up + (n0 - 1) * slab, nx, u1);
    matvec_t<NL>(t.R2, ev, c1);
#pragma unroll
    for (int l = 0; l < NL; ++l) vo[l] = u1[l] + fac * c1[l];
    so = trace_sum<NL>(vo);
    if (RESID) {
      double v2[NL], fv[NL], g[NL], w[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) v2[l] = 0.0;
      if (has_prev2) {
        double uu2[NL], c2[NL];
        ld_ro<COH, NL>(up + (n0 - 2) * slab, nx, uu2);
        matvec_t<NL>(t.R1, ev, c2);
#pragma unroll
        for (int l = 0; l < NL; ++l) v2[l] = uu2[l] + fac * c2[l];
      }
      ld_ro<COH, NL>(fp + (n0 - 1) * slab, nx, fv);
      mo.solve_w(fv, g);
      mo.sweep(vo, g, trace_sum<NL>(v2), om1, w);
      sw = trace_sum<NL>(w);
    }
  }

  int pair = 0;
  for (i64 n = n0; n < nend; n += 2, ++pair) {
#pragma unroll
    for (int l = 0; l < NL; ++l) ev[l] = en[l];
    double un2[2][NL], fn[2][NL];
    if (ASYNC) {
      cp_async_wait<kRing - 2>();
      const double* r = ring + i64(pair % kRing) * Q * T + threadIdx.x;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          u2[e][l] = r[(e * NL + l) * T];
          f2[e][l] = r[((2 + e) * NL + l) * T];
        }
#pragma unroll
      for (int l = 0; l < NL; ++l) ev[l] = r[(4 * NL + l) * T];
      if (n + 2 * (kRing - 1) < nend) issue(n + 2 * (kRing - 1), (pair + kRing - 1) % kRing);
      cp_async_commit();
    }
    if (PF && n + 2 < nend) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ld_st<COH, NL>(up + (n + 2 + e) * slab, nx, un2[e]);
        ld_st<COH, NL>(fp + (n + 2 + e) * slab, nx, fn[e]);
      }
      if (has_c) ld_ro<COH, NL>(ep + ((n + 2) >> 1) * cslab, nxc, en);
    }
    if (!PF && !ASYNC && n > n0) {  // plain: load this pair now
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ld_st<COH, NL>(up + (n + e) * slab, nx, u2[e]);
        ld_st<COH, NL>(fp + (n + e) * slab, nx, f2[e]);
      }
      if (has_c) ld_ro<COH, NL>(ep + (n >> 1) * cslab, nxc, ev);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const i64 m = n + e;
      double c[NL], v[NL], g[NL], w[NL];
      if (e == 0) matvec_t<NL>(t.R1, ev, c);
      else matvec_t<NL>(t.R2, ev, c);
#pragma unroll
      for (int l = 0; l < NL; ++l) v[l] = u2[e][l] + fac * c[l];
      mo.solve_w(f2[e], g);
      mo.sweep(v, g, so, om1, w);
      store_nl<NL>(op + m * slab, nx, w);
      if (RESID) {
        double r[NL];
        mo.residual(f2[e], w, sw, r);
#pragma unroll
        for (int l = 0; l < NL; ++l) sumsq = fma(r[l], r[l], sumsq);
      }
      so = trace_sum<NL>(v);
      sw = trace_sum<NL>(w);
    }
    if (PF && n + 2 < nend) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          u2[e][l] = un2[e][l];
          f2[e][l] = fn[e][l];
        }
    }
  }
  return sumsq;
}

// Ping-pong level-0 buffers selected on the device (the solve graph is
// replayed unchanged while the buffers alternate): A = tbl[*par] holds the
// pre-smoothed iterate of cycle k, B = tbl[1 - *par] receives cycle k+1's.
struct PingPong {
  double* const* tbl;
  const int* par;
};

// updown: the post-smooth of cycle k (prolongation + correction + damped
// Jacobi, mg.cpp:123-131) fused with the pre-smooth, residual and restriction
// of cycle k+1 (mg.cpp:106-117) in ONE pass over a level, plus the residual
// sum of squares of the post-smoothed iterate (the stop test of cycle k,
// mg.cpp:152-153).  Per step n (chains kept in registers):
//   v = u + P e                         corrected iterate of cycle k
//   w = (1-w) v + w A^-1 (f + M N v_{n-1})     post-smoothed (cycle k result)
//   r = f - A w + M N w_{n-1}           stop-test residual
//   x = (1-w) w + w A^-1 (f + M N w_{n-1})     pre-smoothed (cycle k+1)
//   c_{n/2} += fac R (f - A x + M N x_{n-1})   restricted residual (cycle k+1)
// A three-step warm-up rebuilds v, w, x of step n0-1.  Non-sharded only.
template <int DIM, int NL, int CO>
__device__ __forceinline__ double updown_body(const i64 tid, const i64 n0, const i64 nend,
                                              const double* ec, const PingPong pp,
                                              const double* f, double* fc,
                                              const TM<NL>& t, const SP& s, const i64 n1c,
                                              const double omega, double* ring, const i64 s0) {
  const Member me = make_member<DIM>(s, tid, n1c, CO == 2);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = (CO == 2) ? ipow(n1c, DIM) : nx, cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const double Mj = me.Mj, Kj = me.Kj;
  const ModeLU<NL> lu(t, Mj, Kj);
  const double fac = (CO == 2) ? me.fac : 1.0;
  const bool has_c = (CO == 2) ? me.cok : me.ok;
  const double* ep = ec + ((CO == 2) ? me.cidx : me.idx);
  const double* fp = f + me.idx;
  pdl_wait();  // after the constant-only setup above (see down_body)
  const int par = *pp.par;
  const double* up = pp.tbl[par] + me.idx;
  double* op = pp.tbl[1 - par] + me.idx;
  double sumsq = 0.0;

  // corrected iterate v of step m (m >= 0)
  auto vstep = [&](i64 m, double (&v)[NL]) {
    double u[NL], e[NL], c[NL];
    load_nl<NL>(up + m * slab, nx, u);
#pragma unroll
    for (int l = 0; l < NL; ++l) e[l] = 0.0;
    if (has_c) load_nl<NL>(ep + (m >> 1) * cslab, nxc, e);
    if (m & 1) matvec_t<NL>(t.R2, e, c);
    else matvec_t<NL>(t.R1, e, c);
#pragma unroll
    for (int l = 0; l < NL; ++l) v[l] = u[l] + fac * c[l];
  };
  // damped Jacobi sweep of one step: out = (1-w) cur + w A^-1 (fv + M N prev)
  auto sweep = [&](const double (&cur)[NL], const double (&prev)[NL], const double (&fv)[NL],
                   double (&out)[NL]) {
    double nv[NL], rhs[NL], x[NL];
    matvec<NL>(t.N, prev, nv);
#pragma unroll
    for (int l = 0; l < NL; ++l) rhs[l] = fv[l] + Mj * nv[l];
    lu.solve(rhs, x);
#pragma unroll
    for (int l = 0; l < NL; ++l) out[l] = om1 * cur[l] + omega * x[l];
  };

  double vp[NL], wp[NL], xp[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) vp[l] = wp[l] = xp[l] = 0.0;
  // ring prologue first: the warm-up below overlaps its latency
  constexpr int Q = 5 * NL;  // u, f of two steps + e of the coarse step
  const int T = blockDim.x;
  auto issue = [&](i64 n, int st) {
    double* r = ring + i64(st) * Q * T + threadIdx.x;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cp_async8(r + (e * NL + l) * T, up + (n + e) * slab + l * nx, me.ok);
        cp_async8(r + ((2 + e) * NL + l) * T, fp + (n + e) * slab + l * nx, me.ok);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l)
      cp_async8(r + (4 * NL + l) * T, has_c ? ep + (n >> 1) * cslab + l * nxc : fp, has_c);
  };
#pragma unroll
  for (int q = 0; q < kRing - 1; ++q) {
    if (n0 + 2 * q < nend) issue(n0 + 2 * q, q);
    cp_async_commit();
  }
  // s0: global index of local step 0 (sharded: steps -1..-3 are halo slabs)
  if (me.ok && s0 + n0 > 0) {  // warm-up: steps n0-3 .. n0-1
    double v3[NL], v2[NL], w2[NL], f2v[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) v3[l] = w2[l] = 0.0;
    if (s0 + n0 - 3 >= 0) vstep(n0 - 3, v3);
    vstep(n0 - 2, v2);
    load_nl<NL>(fp + (n0 - 2) * slab, nx, f2v);
    sweep(v2, v3, f2v, w2);
    double v1[NL], w1[NL], x1[NL], f1v[NL];
    vstep(n0 - 1, v1);
    load_nl<NL>(fp + (n0 - 1) * slab, nx, f1v);
    sweep(v1, v2, f1v, w1);
    sweep(w1, w2, f1v, x1);
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      vp[l] = v1[l];
      wp[l] = w1[l];
      xp[l] = x1[l];
    }
  }

  int pair = 0;
  for (i64 n = n0; n < nend; n += 2, ++pair) {
    double u2[2][NL], f2[2][NL], ev[NL];
    cp_async_wait<kRing - 2>();
    {
      const double* r = ring + i64(pair % kRing) * Q * T + threadIdx.x;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          u2[e][l] = r[(e * NL + l) * T];
          f2[e][l] = r[((2 + e) * NL + l) * T];
        }
#pragma unroll
      for (int l = 0; l < NL; ++l) ev[l] = r[(4 * NL + l) * T];
    }
    if (n + 2 * (kRing - 1) < nend) issue(n + 2 * (kRing - 1), (pair + kRing - 1) % kRing);
    cp_async_commit();
    double acc[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const i64 m = n + e;
      double c[NL], v[NL], w[NL], x[NL], aw[NL], np[NL], rt[NL], res[NL];
      if (e == 0) matvec_t<NL>(t.R1, ev, c);
      else matvec_t<NL>(t.R2, ev, c);
#pragma unroll
      for (int l = 0; l < NL; ++l) v[l] = u2[e][l] + fac * c[l];
      sweep(v, vp, f2[e], w);
      // stop-test residual of the post-smoothed iterate
      apply_mode<NL>(t, Mj, Kj, w, aw);
      matvec<NL>(t.N, wp, np);
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const double r = f2[e][l] - aw[l] + Mj * np[l];
        sumsq += me.ok ? r * r : 0.0;
      }
      // next cycle's pre-smoothing, residual and restriction
      sweep(w, wp, f2[e], x);
      if (me.ok) store_nl<NL>(op + m * slab, nx, x);
      apply_mode<NL>(t, Mj, Kj, x, aw);
      matvec<NL>(t.N, xp, np);
#pragma unroll
      for (int l = 0; l < NL; ++l) res[l] = f2[e][l] - aw[l] + Mj * np[l];
      if (e == 0) matvec<NL>(t.R1, res, rt);
      else matvec<NL>(t.R2, res, rt);
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        acc[l] += (CO == 2) ? me.fac * rt[l] : rt[l];
        vp[l] = v[l];
        wp[l] = w[l];
        xp[l] = x[l];
      }
    }
    const i64 nc = n >> 1;
    if (CO == 2) {
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] = group_sum<DIM>(me.ok ? acc[l] : 0.0);
      if (me.cok && (tid & ((1 << DIM) - 1)) == 0) store_nl<NL>(fc + nc * cslab + me.cidx, nxc, acc);
    } else if (me.ok) {
      store_nl<NL>(fc + nc * cslab + me.idx, nxc, acc);
    }
  }
  return sumsq;
}

#ifndef STMG_UPDOWN_PTR
#define STMG_UPDOWN_PTR 1
#endif

// The same pass with the explicit per-mode operators (ModeOps): one
// g = w A^-1 f per step serves both sweeps, and the residual of the
// pre-smoothed iterate follows from the stop-test residual without another
// block apply:
//   res = f - A x + ma S(x_{n-1}) = (1-w) r + ma (S(x_{n-1}) - S(w_{n-1}))
// (substitute x = (1-w) w + g + h S(w_{n-1}) and A g = w f, A h = w ma).
// 45 instead of 82 FP64 operations per mode and step for p_t = 1, and
// shorter dependent chains (no substitutions).
template <int DIM, int NL, int CO>
__device__ __forceinline__ double updown_body_ops(const i64 tid, const i64 n0, const i64 nend,
                                                  const double* ec, const PingPong pp,
                                                  const double* f, double* fc,
                                                  const TM<NL>& t, const SP& s, const i64 n1c,
                                                  const double omega, double* ring,
                                                  const i64 s0) {
  const Member me = make_member<DIM>(s, tid, n1c, CO == 2);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = (CO == 2) ? ipow(n1c, DIM) : nx, cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const ModeOps<NL> op_(t, me.Mj, me.Kj, omega);
  const double fac = (CO == 2) ? me.fac : 1.0;
  const bool has_c = (CO == 2) ? me.cok : me.ok;
  const double* ep = ec + ((CO == 2) ? me.cidx : me.idx);
  const double* fp = f + me.idx;
  pdl_wait();  // after the constant-only setup above (see down_body)
  const int par = *pp.par;
  const double* up = pp.tbl[par] + me.idx;
  double* op = pp.tbl[1 - par] + me.idx;
  double sumsq = 0.0;

  // one step: corrected v, post-smoothed w, its residual r, pre-smoothed x
  // (the previous step's traces sv, sw, sx in, this step's out)
  auto step = [&](const double (&u)[NL], const double (&fv)[NL], const double (&c)[NL],
                  double& sv, double& sw, double& sx, double (&r)[NL], double (&x)[NL]) {
    double v[NL], g[NL], w[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) v[l] = fma(fac, c[l], u[l]);
    op_.solve_w(fv, g);
    op_.sweep(v, g, sv, om1, w);
    op_.residual(fv, w, sw, r);
    op_.sweep(w, g, sw, om1, x);
    sv = trace_sum<NL>(v);
    sw = trace_sum<NL>(w);
    sx = trace_sum<NL>(x);
  };

  double svp = 0.0, swp = 0.0, sxp = 0.0;  // traces of step n-1
  constexpr int Q = 5 * NL;  // u, f of two steps + e of the coarse step
  constexpr int T = 128;     // launch_updown's block (immediate ring offsets)
#if STMG_UPDOWN_PTR
  // running offsets of the next pair to issue (strength-reduced addressing)
  const unsigned rs = static_cast<unsigned>(__cvta_generic_to_shared(ring + threadIdx.x));
  i64 uoff = n0 * slab, eoff = (n0 >> 1) * cslab;
  const double* eb = has_c ? ep : fp;
  const i64 estep = has_c ? cslab : 0;
  auto issue = [&](int st) {
    const unsigned r = rs + unsigned(st * Q * T) * 8u;
    const double* ub = up + uoff;
    const double* fb = fp + uoff;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cp_async8s(r + unsigned((e * NL + l) * T) * 8u, ub + e * slab + l * nx, me.ok);
        cp_async8s(r + unsigned(((2 + e) * NL + l) * T) * 8u, fb + e * slab + l * nx, me.ok);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l)
      cp_async8s(r + unsigned((4 * NL + l) * T) * 8u, eb + eoff + l * nxc, has_c);
    uoff += 2 * slab;
    eoff += estep;
  };
#pragma unroll
  for (int q = 0; q < kRing - 1; ++q) {
    if (n0 + 2 * q < nend) issue(q);
    cp_async_commit();
  }
#else
  auto issue = [&](i64 n, int st) {
    double* r = ring + i64(st) * Q * T + threadIdx.x;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cp_async8(r + (e * NL + l) * T, up + (n + e) * slab + l * nx, me.ok);
        cp_async8(r + ((2 + e) * NL + l) * T, fp + (n + e) * slab + l * nx, me.ok);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l)
      cp_async8(r + (4 * NL + l) * T, has_c ? ep + (n >> 1) * cslab + l * nxc : fp, has_c);
  };
#pragma unroll
  for (int q = 0; q < kRing - 1; ++q) {
    if (n0 + 2 * q < nend) issue(n0 + 2 * q, q);
    cp_async_commit();
  }
#endif
  // warm-up: steps n0-3 .. n0-1 (s0: global index of local step 0; sharded:
  // steps -1..-3 are halo slabs).  Step n0-3 contributes its corrected trace
  // only; n0-2 its post-smoothed one; n0-1 all three.
  if (me.ok && s0 + n0 > 0) {
    // all loads first (one memory latency, not three); n0 is even, so steps
    // n0-2, n0-1 share a coarse step and n0-3 has the one before
    double u[3][NL], fv[3][NL], e[2][NL], c[NL], r[NL], x[NL];
    double sv = 0.0, sw = 0.0, sx = 0.0;
    const bool h3 = s0 + n0 - 3 >= 0;
#pragma unroll
    for (int l = 0; l < NL; ++l) e[0][l] = e[1][l] = u[0][l] = fv[0][l] = 0.0;
    if (h3) load_nl<NL>(up + (n0 - 3) * slab, nx, u[0]);
    load_nl<NL>(up + (n0 - 2) * slab, nx, u[1]);
    load_nl<NL>(up + (n0 - 1) * slab, nx, u[2]);
    load_nl<NL>(fp + (n0 - 2) * slab, nx, fv[1]);  // step n0-3: only v is used
    load_nl<NL>(fp + (n0 - 1) * slab, nx, fv[2]);
    if (has_c) {
      if (h3) load_nl<NL>(ep + ((n0 >> 1) - 2) * cslab, nxc, e[0]);
      load_nl<NL>(ep + ((n0 >> 1) - 1) * cslab, nxc, e[1]);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k == 0 && !h3) continue;
      if (k == 1) matvec_t<NL>(t.R1, e[1], c);
      else matvec_t<NL>(t.R2, e[k == 0 ? 0 : 1], c);
      step(u[k], fv[k], c, sv, sw, sx, r, x);
    }
    svp = sv;
    swp = sw;
    sxp = sx;
  }

  // rotating ring stages (no modulo in the loop); x and the coarse rhs go
  // out with st.global (the ping-pong pointers come from a device table, so
  // plain stores would be generic); alias-group sums with a full-warp mask
  // (every lane of the block runs every pair)
  int st_use = 0, st_iss = kRing - 1;
  double* opn = op + n0 * slab;
  double* fcn = fc + (n0 >> 1) * cslab + ((CO == 2) ? me.cidx : me.idx);
  const bool cst = (CO == 2) ? (me.cok && (tid & ((1 << DIM) - 1)) == 0) : me.ok;
  for (i64 n = n0; n < nend; n += 2) {
    double u2[2][NL], f2[2][NL], ev[NL];
    cp_async_wait<kRing - 2>();
    {
      const double* r = ring + st_use * Q * T + threadIdx.x;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          u2[e][l] = r[(e * NL + l) * T];
          f2[e][l] = r[((2 + e) * NL + l) * T];
        }
#pragma unroll
      for (int l = 0; l < NL; ++l) ev[l] = r[(4 * NL + l) * T];
    }
#if STMG_UPDOWN_PTR
    if (n + 2 * (kRing - 1) < nend) issue(st_iss);
#else
    if (n + 2 * (kRing - 1) < nend) issue(n + 2 * (kRing - 1), st_iss);
#endif
    cp_async_commit();
    st_use = (st_use == kRing - 1) ? 0 : st_use + 1;
    st_iss = (st_iss == kRing - 1) ? 0 : st_iss + 1;
    double acc[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double c[NL], r[NL], x[NL], res[NL], rt[NL];
      if (e == 0) matvec_t<NL>(t.R1, ev, c);
      else matvec_t<NL>(t.R2, ev, c);
      const double swq = swp, sxq = sxp;  // traces of step m-1
      step(u2[e], f2[e], c, svp, swp, sxp, r, x);
      if (me.ok) {
#pragma unroll
        for (int l = 0; l < NL; ++l) st_global(opn + e * slab + l * nx, x[l]);
      }
      const double d = sxq - swq;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        sumsq = fma(r[l], r[l], sumsq);
        res[l] = fma(op_.ma[l], d, om1 * r[l]);
      }
      if (e == 0) matvec<NL>(t.R1, res, rt);
      else matvec<NL>(t.R2, res, rt);
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] += (CO == 2) ? me.fac * rt[l] : rt[l];
    }
    opn += 2 * slab;
    if (CO == 2) {
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] = group_sum_full<DIM>(me.ok ? acc[l] : 0.0);
    }
    if (cst) {
#pragma unroll
      for (int l = 0; l < NL; ++l) st_global(fcn + l * nxc, acc[l]);
    }
    fcn += cslab;
  }
  return me.ok ? sumsq : 0.0;
}

// ---- Row-run staging (full coarsening, rows of whole alias-group blocks)
// The cp.async ring above moves every value through L1 (LDGSTS.ca, 8 B per
// thread): the in-flight lines need L1 capacity, and measured solves slow
// down by 25 % when the shared-memory carveout squeezes L1.  Here the block's
// loads go L2 -> shared memory without L1 allocation (16-byte cp.async.cg by
// all threads, or TMA bulk copies) as whole row segments: when the 128 / 2^DIM groups of a block lie in one
// row of the group grid (G a multiple of that), every member b of the block
// reads one contiguous run of GPB fine modes per (array, step, DG component),
// ascending or mirrored, and the coarse correction one run of GPB coarse
// modes.  Each run is copied from its 16-byte aligned-down start (GPB + 2
// doubles) into a slot of the stage; a thread reads slot[o_b + shift] with
// o_b its distance from the run's first mode.  Stages complete on an
// mbarrier; one __syncthreads per step pair frees the stage reissued next.
// 0: per-thread cp.async ring (updown_body_ops); 1: TMA bulk runs (measured
// slower: ~35-65 small copies per stage, the TMA issue rate bounds it);
// 2: the same runs in 16-byte cp.async.cg chunks by all threads (default:
// C3 114 -> 105 ms, C4 82 -> 72 ms, C5 151 -> 140 ms per solve)
#ifndef STMG_UPDOWN_TMA
#define STMG_UPDOWN_TMA 2
#endif
#ifndef STMG_TMA_STAGES
#define STMG_TMA_STAGES 3  // A/B vs 4 and 6 stages: profiles/r01_v15_tma_stages_ab.txt
#endif
constexpr int kTmaStages = STMG_TMA_STAGES;

template <int DIM, int NL, int BT = 128>
struct TmaShape {
  static constexpr int NM = 1 << DIM;       // members per alias group
  static constexpr int GPB = BT / NM;       // groups per block (one row run)
  static constexpr int SEG = GPB + 2;       // doubles per slot
  static constexpr int NU = 2 * NL * NM;    // u slots (2 steps) = f slots
  static constexpr int NC = 2 * NU + NL;    // copies per stage
  static constexpr int STAGE = NC * SEG;    // doubles per stage
  static constexpr size_t smem = size_t(kTmaStages) * STAGE * sizeof(double);
};

__device__ __forceinline__ void cp_async16cg(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// 16-byte aligned-down start of a run and the run's first element's shift
__device__ __forceinline__ const double* align16(const double* p) {
  return reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15));
}
__device__ __forceinline__ int shift16(const double* p) {
  return int((reinterpret_cast<uintptr_t>(p) >> 3) & 1);
}

template <int DIM, int NL, int BT>
__device__ __forceinline__ double updown_body_tma(const i64 tid, const i64 n0, const i64 nend,
                                                  const double* ec, const PingPong pp,
                                                  const double* f, double* fc,
                                                  const TM<NL>& t, const SP& s, const i64 n1c,
                                                  const double omega, double* ring,
                                                  const i64 s0) {
  using S = TmaShape<DIM, NL, BT>;
  constexpr int NM = S::NM, GPB = S::GPB, SEG = S::SEG, NU = S::NU;
  __shared__ alignas(8) unsigned long long bars[kTmaStages];
  __shared__ i64 segb[NM + 1];  // run start (fine mode) per member; coarse run start
  const Member me = make_member<DIM>(s, tid, n1c, true);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = ipow(n1c, DIM), cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const ModeOps<NL> op_(t, me.Mj, me.Kj, omega);
  const double fac = me.fac;
  const bool has_c = me.cok;
  const int b = int(threadIdx.x) & (NM - 1);
  if (threadIdx.x < NM) {  // group 0 of the block, member b: its run's first mode
    segb[b] = (b & 1) ? me.idx - (GPB - 1) : me.idx;
    if (b == 0) segb[NM] = me.cidx;
  }
  const unsigned bar0 = static_cast<unsigned>(__cvta_generic_to_shared(bars));
  if (threadIdx.x == 0) {
    for (int q = 0; q < kTmaStages; ++q) mbar_init(bar0 + 8u * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const i64 sb = segb[b], cb = segb[NM];
  const int ob = int(me.idx - sb);          // offset in the member's run
  const int oc = int(me.cidx - cb);         // offset in the coarse run
  pdl_wait();
  const int par = *pp.par;
  const double* ub = pp.tbl[par];
  double* op = pp.tbl[1 - par] + me.idx;
  const double* up = ub + me.idx;
  const double* fp = f + me.idx;
  const double* ep = ec + me.cidx;
  // per-slot shifts of this thread's runs (n is even: constant over pairs)
  unsigned shu = 0, shf = 0;
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      shu |= unsigned(shift16(ub + e * slab + l * nx + sb)) << (e * NL + l);
      shf |= unsigned(shift16(f + e * slab + l * nx + sb)) << (e * NL + l);
    }
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));
  const int lane = threadIdx.x & 31;
  // warp 0 issues stage st for the pair starting at n: lane i copies slots i, i+32, ...
  auto issue = [&](i64 n, int st) {
    const unsigned bar = bar0 + 8u * st;
    if (lane == 0) mbar_expect(bar, unsigned(S::NC * SEG * 8));
    __syncwarp();
    const unsigned base = ring_s + unsigned(st * S::STAGE) * 8u;
    for (int c = lane; c < S::NC; c += 32) {
      const double* src;
      if (c < 2 * NU) {
        const int arr = c / NU, r = c - arr * NU;        // r = (e * NL + l) * NM + m
        const int m = r % NM, el = r / NM, e = el / NL, l = el - e * NL;
        src = (arr ? f : ub) + (n + e) * slab + l * nx;
        src += segb[m];
      } else {
        const int l = c - 2 * NU;
        src = ec + (n >> 1) * cslab + l * nxc + cb;
      }
      bulk_g2s(base + unsigned(c * SEG) * 8u, align16(src), unsigned(SEG * 8), bar);
    }
  };
  // CG (STMG_UPDOWN_TMA == 2): the same runs, copied by all threads in
  // 16-byte cp.async.cg chunks (L2 -> shared, no L1 allocation); chunk
  // k = threadIdx.x + BT i of a stage.  Fine-run sources at n = 0 are
  // precomputed (n is even, so n * slab keeps the 16-byte alignment).
  constexpr bool CG = STMG_UPDOWN_TMA == 2;
  constexpr int HC = SEG / 2, NCH = S::NC * HC, KPT = (NCH + BT - 1) / BT;
  const double* csrc[KPT];
  unsigned cdst[KPT];
  if (CG) {
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = int(threadIdx.x) + BT * i;
      const int c = k / HC, j = k - c * HC;
      cdst[i] = unsigned(c * SEG + 2 * j) * 8u;
      csrc[i] = nullptr;
      if (c < 2 * NU) {
        const int arr = c / NU, r = c - arr * NU;
        const int m = r % NM, el = r / NM, e = el / NL, l = el - e * NL;
        csrc[i] = align16((arr ? f : ub) + e * slab + l * nx + segb[m]) + 2 * j;
      }
    }
  }
  auto issue_cg = [&](i64 n, int st) {
    const unsigned base = ring_s + unsigned(st * S::STAGE) * 8u;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = int(threadIdx.x) + BT * i;
      if (k >= NCH) break;
      const int c = k / HC;
      const double* src;
      if (c < 2 * NU) {
        src = csrc[i] + n * slab;
      } else {
        const int l = c - 2 * NU, j = k - c * HC;
        src = align16(ec + (n >> 1) * cslab + l * nxc + cb) + 2 * j;
      }
      cp_async16cg(base + cdst[i], src);
    }
  };
  unsigned phase = 0;  // bit q: parity of stage q's next completion
  if (CG) {
#pragma unroll
    for (int q = 0; q < kTmaStages - 1; ++q) {
      if (n0 + 2 * q < nend) issue_cg(n0 + 2 * q, q);
      cp_async_commit();
    }
  } else if (threadIdx.x < 32) {
#pragma unroll
    for (int q = 0; q < kTmaStages - 1; ++q)
      if (n0 + 2 * q < nend) issue(n0 + 2 * q, q);
  }

  double sumsq = 0.0;
  auto step = [&](const double (&u)[NL], const double (&fv)[NL], const double (&c)[NL],
                  double& sv, double& sw, double& sx, double (&r)[NL], double (&x)[NL]) {
    double v[NL], g[NL], w[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) v[l] = fma(fac, c[l], u[l]);
    op_.solve_w(fv, g);
    op_.sweep(v, g, sv, om1, w);
    op_.residual(fv, w, sw, r);
    op_.sweep(w, g, sw, om1, x);
    sv = trace_sum<NL>(v);
    sw = trace_sum<NL>(w);
    sx = trace_sum<NL>(x);
  };
  double svp = 0.0, swp = 0.0, sxp = 0.0;
  if (me.ok && s0 + n0 > 0) {  // warm-up, as in updown_body_ops
    double u[3][NL], fv[3][NL], e[2][NL], c[NL], r[NL], x[NL];
    double sv = 0.0, sw = 0.0, sx = 0.0;
    const bool h3 = s0 + n0 - 3 >= 0;
#pragma unroll
    for (int l = 0; l < NL; ++l) e[0][l] = e[1][l] = u[0][l] = fv[0][l] = 0.0;
    if (h3) load_nl<NL>(up + (n0 - 3) * slab, nx, u[0]);
    load_nl<NL>(up + (n0 - 2) * slab, nx, u[1]);
    load_nl<NL>(up + (n0 - 1) * slab, nx, u[2]);
    load_nl<NL>(fp + (n0 - 2) * slab, nx, fv[1]);
    load_nl<NL>(fp + (n0 - 1) * slab, nx, fv[2]);
    if (has_c) {
      if (h3) load_nl<NL>(ep + ((n0 >> 1) - 2) * cslab, nxc, e[0]);
      load_nl<NL>(ep + ((n0 >> 1) - 1) * cslab, nxc, e[1]);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k == 0 && !h3) continue;
      if (k == 1) matvec_t<NL>(t.R1, e[1], c);
      else matvec_t<NL>(t.R2, e[k == 0 ? 0 : 1], c);
      step(u[k], fv[k], c, sv, sw, sx, r, x);
    }
    svp = sv;
    swp = sw;
    sxp = sx;
  }

  int st_use = 0, st_iss = kTmaStages - 1;
  double* opn = op + n0 * slab;
  double* fcn = fc + (n0 >> 1) * cslab + me.cidx;
  const bool cst = me.cok && (tid & (NM - 1)) == 0;
  for (i64 n = n0; n < nend; n += 2) {
    if (CG) {
      cp_async_wait<kTmaStages - 2>();  // this thread's chunks of stage st_use landed
      __syncthreads();  // everyone's landed; everyone is done with stage st_iss
      if (n + 2 * (kTmaStages - 1) < nend) issue_cg(n + 2 * (kTmaStages - 1), st_iss);
      cp_async_commit();
    } else {
      __syncthreads();  // every thread is done with stage st_iss (read last pair)
      if (threadIdx.x < 32 && n + 2 * (kTmaStages - 1) < nend)
        issue(n + 2 * (kTmaStages - 1), st_iss);
      mbar_wait(bar0 + 8u * st_use, (phase >> st_use) & 1u);
      phase ^= 1u << st_use;
    }
    double u2[2][NL], f2[2][NL], ev[NL];
    {
      const double* r = ring + st_use * S::STAGE;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int k = e * NL + l;
          u2[e][l] = r[(k * NM + b) * SEG + ob + int((shu >> k) & 1u)];
          f2[e][l] = r[(NU + k * NM + b) * SEG + ob + int((shf >> k) & 1u)];
        }
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int sh = shift16(ec + (n >> 1) * cslab + l * nxc + cb);
        const double v = r[(2 * NU + l) * SEG + oc + sh];
        ev[l] = has_c ? v : 0.0;
      }
    }
    st_use = (st_use == kTmaStages - 1) ? 0 : st_use + 1;
    st_iss = (st_iss == kTmaStages - 1) ? 0 : st_iss + 1;
    double acc[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double c[NL], r[NL], x[NL], res[NL], rt[NL];
      if (e == 0) matvec_t<NL>(t.R1, ev, c);
      else matvec_t<NL>(t.R2, ev, c);
      const double swq = swp, sxq = sxp;
      step(u2[e], f2[e], c, svp, swp, sxp, r, x);
      if (me.ok) {
#pragma unroll
        for (int l = 0; l < NL; ++l) st_global(opn + e * slab + l * nx, x[l]);
      }
      const double d = sxq - swq;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        sumsq = fma(r[l], r[l], sumsq);
        res[l] = fma(op_.ma[l], d, om1 * r[l]);
      }
      if (e == 0) matvec<NL>(t.R1, res, rt);
      else matvec<NL>(t.R2, res, rt);
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] += me.fac * rt[l];
    }
    opn += 2 * slab;
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = group_sum_full<DIM>(me.ok ? acc[l] : 0.0);
    if (cst) {
#pragma unroll
      for (int l = 0; l < NL; ++l) st_global(fcn + l * nxc, acc[l]);
    }
    fcn += cslab;
  }
  return me.ok ? sumsq : 0.0;
}

// Launch bounds.  p_t <= 1: was 5 CTAs per SM (96 registers) while C2 ran
// 1024 CTAs (1.4 instead of 1.7 waves); with the 512-CTA grid of chunk target
// 148*256 all CTAs fit at 4 per SM and the 128-register budget is faster.
// p_t = 2 would spill at 96 (C3 106 -> 157 ms).
#ifndef STMG_UPDOWN_MINB3
#define STMG_UPDOWN_MINB3 3  // p_t = 2: 168 registers, 3 CTAs/SM (C3 108 -> 104 ms); 4 spills
#endif
#ifndef STMG_UPDOWN_MINB2
#define STMG_UPDOWN_MINB2 4  // p_t <= 1: 4 CTAs/SM (v16 A/B vs 5 and 3: C2 1.691 -> 1.669 ms,
                             // C4/C5 -1.5 %; profiles/r01_v16_minb_ab.txt)
#endif
// BT threads per CTA: 128, or 256 (p_t <= 1) where the level is large: twice
// the alias groups per CTA double the length of every staged run (2D: 66
// instead of 34 doubles, 3D: 34 instead of 18 -- the 2-double alignment slack
// and the per-copy issue cost halve).  The choice is made on the host from the
// GLOBAL level (pick_updown_block), so time-slab shards keep the single-shard
// partial-sum layout.
template <int DIM, int NL, int BT>
__global__ void __launch_bounds__(BT, (BT == 128 ? (NL <= 2 ? STMG_UPDOWN_MINB2 : NL == 3 ? STMG_UPDOWN_MINB3 : 1)
                                                  : STMG_UPDOWN_MINB2 / 2))
k_updown_tma(const double* __restrict__ ec, const PingPong pp, const double* __restrict__ f,
             double* __restrict__ fc, double* __restrict__ partials, const TM<NL> t, const SP s,
             const i64 n_t, const int C, const i64 n1c, const double omega, const i64 s0) {
  __shared__ double sh[32];
  extern __shared__ __align__(16) double ring[];
  const unsigned bx = blockIdx.x, by = blockIdx.y;
  const i64 tid = i64(bx) * blockDim.x + threadIdx.x;
  const i64 n0 = i64(by) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  const double sumsq =
      updown_body_tma<DIM, NL, BT>(tid, n0, nend, ec, pp, f, fc, t, s, n1c, omega, ring, s0);
  pdl_trigger();
  const double tot = block_sum(sumsq, sh);
  if (threadIdx.x == 0) partials[i64(by) * gridDim.x + bx] = tot;
}

// ---- Row-run staging for the per-level kernels (k_down / k_up) -----------
// The loader of updown_body_tma (STMG_UPDOWN_TMA = 2) as a reusable piece:
// NA fine arrays (2 steps x NL components x 2^DIM member runs each) plus,
// with HC, the NL coarse runs of the block's coarse modes, copied with
// 16-byte cp.async.cg chunks into kTmaStages stages.
template <int DIM, int NL, int NA, bool HC>
struct RowRuns {
  static constexpr int NM = 1 << DIM, GPB = 128 / NM, SEG = GPB + 2;
  static constexpr int NF = NA * 2 * NL * NM;  // fine slots
  static constexpr int NC = NF + (HC ? NL : 0);
  static constexpr int STAGE = NC * SEG;
  static constexpr int HCH = SEG / 2, NCH = NC * HCH, KPT = (NCH + 127) / 128;
  static constexpr size_t smem = size_t(kTmaStages) * STAGE * sizeof(double);
  const double* csrc[KPT];
  unsigned cdst[KPT];
  const double* ecb;  // coarse array + the block's coarse run start
  i64 slab, nxc, cslab;
  unsigned ring_s, sh;
  int ob, oc, b;
  // segb: NM + 1 shared i64 (written here, one __syncthreads inside)
  __device__ __forceinline__ void init(const double* const (&arr)[NA], const double* ec,
                                       const Member& me, const i64 nx, const i64 slab_,
                                       const i64 nxc_, const i64 cslab_, double* ring,
                                       i64* segb) {
    b = int(threadIdx.x) & (NM - 1);
    if (threadIdx.x < NM) {  // group 0 of the block, member b: its run's first mode
      segb[b] = (b & 1) ? me.idx - (GPB - 1) : me.idx;
      if (b == 0) segb[NM] = me.cidx;
    }
    __syncthreads();
    slab = slab_;
    nxc = nxc_;
    cslab = cslab_;
    const i64 sb = segb[b], cb = segb[NM];
    ob = int(me.idx - sb);
    oc = int(me.cidx - cb);
    ecb = HC ? ec + cb : nullptr;
    sh = 0;
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l)
          sh |= unsigned(shift16(arr[a] + e * slab + l * nx + sb)) << ((a * 2 + e) * NL + l);
    ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = int(threadIdx.x) + 128 * i;
      const int c = k / HCH, j = k - c * HCH;
      cdst[i] = unsigned(c * SEG + 2 * j) * 8u;
      csrc[i] = nullptr;
      if (c < NF) {
        const int a = c / (2 * NL * NM), r = c - a * (2 * NL * NM);
        const int m = r % NM, el = r / NM, e = el / NL, l = el - e * NL;
        const double* base = arr[0];
#pragma unroll
        for (int q = 1; q < NA; ++q)
          if (a == q) base = arr[q];
        csrc[i] = align16(base + e * slab + l * nx + segb[m]) + 2 * j;
      }
    }
  }
  __device__ __forceinline__ void issue(const i64 n, const int st) const {
    const unsigned base = ring_s + unsigned(st * STAGE) * 8u;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = int(threadIdx.x) + 128 * i;
      if (k >= NCH) break;
      const int c = k / HCH;
      const double* src;
      if (!HC || c < NF) {
        src = csrc[i] + n * slab;
      } else {
        const int l = c - NF, j = k - c * HCH;
        src = align16(ecb + (n >> 1) * cslab + l * nxc) + 2 * j;
      }
      cp_async16cg(base + cdst[i], src);
    }
  }
  __device__ __forceinline__ double fine(const double* ring, int st, int a, int e, int l) const {
    const int q = (a * 2 + e) * NL + l;
    return ring[st * STAGE + (q * NM + b) * SEG + ob + int((sh >> q) & 1u)];
  }
  __device__ __forceinline__ double coarse(const double* ring, int st, int l, i64 n) const {
    return ring[st * STAGE + (NF + l) * SEG + oc + shift16(ecb + (n >> 1) * cslab + l * nxc)];
  }
};

// k_down on row runs: damped Jacobi sweep + residual + full-weighting
// restriction (down_body, CO = 2) with the loads staged by RowRuns.
template <int DIM, int NL, bool ZERO>
__global__ void __launch_bounds__(128) k_down_rr(const double* __restrict__ f,
                                                 const double* __restrict__ uin,
                                                 double* __restrict__ uout,
                                                 double* __restrict__ fc, const TM<NL> t,
                                                 const SP s, const i64 n_t, const int C,
                                                 const i64 n1c, const double omega,
                                                 const bool first_global) {
  using RR = RowRuns<DIM, NL, ZERO ? 1 : 2, false>;
  constexpr int NM = RR::NM;
  extern __shared__ __align__(16) double ring[];
  __shared__ i64 segb[NM + 1];
  const i64 tid = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 n0 = i64(blockIdx.y) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  const bool has_prev = n0 > 0 || !first_global, has_prev2 = n0 - 1 > 0 || !first_global;
  const Member me = make_member<DIM>(s, tid, n1c, true);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = ipow(n1c, DIM), cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const ModeOps<NL> mo(t, me.Mj, me.Kj, omega);
  RR rr;
  const double* arrs[ZERO ? 1 : 2] = {f};
  if (!ZERO) arrs[ZERO ? 0 : 1] = uin;
  rr.init(arrs, nullptr, me, nx, slab, nxc, cslab, ring, segb);
  pdl_wait();
#pragma unroll
  for (int q = 0; q < kTmaStages - 1; ++q) {
    if (n0 + 2 * q < nend) rr.issue(n0 + 2 * q, q);
    cp_async_commit();
  }
  const double* fp = f + me.idx;
  const double* up = uin + me.idx;
  double so = 0.0, sn = 0.0;  // traces of step n-1: old iterate, smoothed
  if (me.ok && has_prev) {  // warm-up: smoothed step n0-1
    double fv[NL], g[NL], w[NL];
    load_nl<NL>(fp + (n0 - 1) * slab, nx, fv);
    mo.solve_w(fv, g);
    if (ZERO) {
      sn = trace_sum<NL>(g);
    } else {
      double u1[NL], u2[NL];
      load_nl<NL>(up + (n0 - 1) * slab, nx, u1);
#pragma unroll
      for (int l = 0; l < NL; ++l) u2[l] = 0.0;
      if (has_prev2) load_nl<NL>(up + (n0 - 2) * slab, nx, u2);
      mo.sweep(u1, g, trace_sum<NL>(u2), om1, w);
      sn = trace_sum<NL>(w);
      so = trace_sum<NL>(u1);
    }
  }
  int st_use = 0, st_iss = kTmaStages - 1;
  double* opn = uout + me.idx + n0 * slab;
  double* fcn = fc + (n0 >> 1) * cslab + me.cidx;
  const bool cst = me.cok && (tid & (NM - 1)) == 0;
  for (i64 n = n0; n < nend; n += 2) {
    cp_async_wait<kTmaStages - 2>();
    __syncthreads();
    if (n + 2 * (kTmaStages - 1) < nend) rr.issue(n + 2 * (kTmaStages - 1), st_iss);
    cp_async_commit();
    double f2[2][NL], u2[2][NL];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        f2[e][l] = rr.fine(ring, st_use, 0, e, l);
        u2[e][l] = ZERO ? 0.0 : rr.fine(ring, st_use, ZERO ? 0 : 1, e, l);
      }
    st_use = (st_use == kTmaStages - 1) ? 0 : st_use + 1;
    st_iss = (st_iss == kTmaStages - 1) ? 0 : st_iss + 1;
    double acc[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double g[NL], w[NL], res[NL], rt[NL];
      mo.solve_w(f2[e], g);
      if (ZERO) {
#pragma unroll
        for (int l = 0; l < NL; ++l) w[l] = g[l];
      } else {
        mo.sweep(u2[e], g, so, om1, w);
      }
      if (me.ok) {
#pragma unroll
        for (int l = 0; l < NL; ++l) st_global(opn + e * slab + l * nx, w[l]);
      }
      mo.residual(f2[e], w, sn, res);
      if (e == 0) matvec<NL>(t.R1, res, rt);
      else matvec<NL>(t.R2, res, rt);
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] += me.fac * rt[l];
      if (!ZERO) so = trace_sum<NL>(u2[e]);
      sn = trace_sum<NL>(w);
    }
    opn += 2 * slab;
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = group_sum_full<DIM>(me.ok ? acc[l] : 0.0);
    if (cst) {
#pragma unroll
      for (int l = 0; l < NL; ++l) st_global(fcn + l * nxc, acc[l]);
    }
    fcn += cslab;
  }
  pdl_trigger();
}

// k_up on row runs: prolongation + correction + damped Jacobi sweep
// (+ residual sum of squares) (up_body, CO = 2) with RowRuns loads.
template <int DIM, int NL, bool RESID>
__global__ void __launch_bounds__(128) k_up_rr(const double* __restrict__ ec,
                                               const double* __restrict__ uin,
                                               const double* __restrict__ f,
                                               double* __restrict__ uout,
                                               double* __restrict__ partials, const TM<NL> t,
                                               const SP s, const i64 n_t, const int C,
                                               const i64 n1c, const double omega,
                                               const bool first_global) {
  using RR = RowRuns<DIM, NL, 2, true>;
  constexpr int NM = RR::NM;
  extern __shared__ __align__(16) double ring[];
  __shared__ i64 segb[NM + 1];
  __shared__ double sh[32];
  const unsigned bx = blockIdx.x, by = blockIdx.y;
  const i64 tid = i64(bx) * blockDim.x + threadIdx.x;
  const i64 n0 = i64(by) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  const bool has_prev = n0 > 0 || !first_global, has_prev2 = n0 - 1 > 0 || !first_global;
  const Member me = make_member<DIM>(s, tid, n1c, true);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 nxc = ipow(n1c, DIM), cslab = NL * nxc;
  const double om1 = 1.0 - omega;
  const ModeOps<NL> mo(t, me.Mj, me.Kj, omega);
  const double fac = me.fac;
  const bool has_c = me.cok;
  RR rr;
  const double* arrs[2] = {uin, f};
  rr.init(arrs, ec, me, nx, slab, nxc, cslab, ring, segb);
  pdl_wait();
#pragma unroll
  for (int q = 0; q < kTmaStages - 1; ++q) {
    if (n0 + 2 * q < nend) rr.issue(n0 + 2 * q, q);
    cp_async_commit();
  }
  const double* ep = ec + me.cidx;
  const double* fp = f + me.idx;
  const double* up = uin + me.idx;
  double so = 0.0, sw = 0.0;  // traces of step n-1: corrected, smoothed
  double sumsq = 0.0;
  if (me.ok && has_prev) {
    double ev[NL], u1[NL], c1[NL], vo[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) ev[l] = 0.0;
    if (has_c) load_nl<NL>(ep + ((n0 >> 1) - 1) * cslab, nxc, ev);  // coarse step of n0-2, n0-1
    load_nl<NL>(up + (n0 - 1) * slab, nx, u1);
    matvec_t<NL>(t.R2, ev, c1);
#pragma unroll
    for (int l = 0; l < NL; ++l) vo[l] = u1[l] + fac * c1[l];
    so = trace_sum<NL>(vo);
    if (RESID) {
      double v2[NL], fv[NL], g[NL], w[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) v2[l] = 0.0;
      if (has_prev2) {
        double uu2[NL], c2[NL];
        load_nl<NL>(up + (n0 - 2) * slab, nx, uu2);
        matvec_t<NL>(t.R1, ev, c2);
#pragma unroll
        for (int l = 0; l < NL; ++l) v2[l] = uu2[l] + fac * c2[l];
      }
      load_nl<NL>(fp + (n0 - 1) * slab, nx, fv);
      mo.solve_w(fv, g);
      mo.sweep(vo, g, trace_sum<NL>(v2), om1, w);
      sw = trace_sum<NL>(w);
    }
  }
  int st_use = 0, st_iss = kTmaStages - 1;
  double* opn = uout + me.idx + n0 * slab;
  for (i64 n = n0; n < nend; n += 2) {
    cp_async_wait<kTmaStages - 2>();
    __syncthreads();
    if (n + 2 * (kTmaStages - 1) < nend) rr.issue(n + 2 * (kTmaStages - 1), st_iss);
    cp_async_commit();
    double u2[2][NL], f2[2][NL], ev[NL];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        u2[e][l] = rr.fine(ring, st_use, 0, e, l);
        f2[e][l] = rr.fine(ring, st_use, 1, e, l);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const double v = rr.coarse(ring, st_use, l, n);
      ev[l] = has_c ? v : 0.0;
    }
    st_use = (st_use == kTmaStages - 1) ? 0 : st_use + 1;
    st_iss = (st_iss == kTmaStages - 1) ? 0 : st_iss + 1;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double c[NL], v[NL], g[NL], w[NL];
      if (e == 0) matvec_t<NL>(t.R1, ev, c);
      else matvec_t<NL>(t.R2, ev, c);
#pragma unroll
      for (int l = 0; l < NL; ++l) v[l] = u2[e][l] + fac * c[l];
      mo.solve_w(f2[e], g);
      mo.sweep(v, g, so, om1, w);
      if (me.ok) {
#pragma unroll
        for (int l = 0; l < NL; ++l) st_global(opn + e * slab + l * nx, w[l]);
      }
      if (RESID) {
        double r[NL];
        mo.residual(f2[e], w, sw, r);
#pragma unroll
        for (int l = 0; l < NL; ++l) sumsq = fma(r[l], r[l], sumsq);
      }
      so = trace_sum<NL>(v);
      sw = trace_sum<NL>(w);
    }
    opn += 2 * slab;
  }
  pdl_trigger();
  if (RESID) {
    const double tot = block_sum(me.ok ? sumsq : 0.0, sh);
    if (threadIdx.x == 0) partials[i64(by) * gridDim.x + bx] = tot;
  }
}

#ifndef STMG_LEVEL_RR
#define STMG_LEVEL_RR 1
#endif
// row runs only for large levels: on small, latency-bound ones (C2 level 1,
// 1M dofs, 4-step chunks) the per-pair CTA barrier costs more than the L1
// relief gains (C2 1.77 -> 1.84 ms with row runs on every level)
#ifndef STMG_LEVEL_RR_MIN
#define STMG_LEVEL_RR_MIN (i64(1) << 22)
#endif

#ifndef STMG_UPDOWN_OPS
#define STMG_UPDOWN_OPS 1
#endif

template <int DIM, int NL, int CO>
__global__ void __launch_bounds__(128) k_updown(const double* __restrict__ ec, const PingPong pp,
                                                const double* __restrict__ f,
                                                double* __restrict__ fc,
                                                double* __restrict__ partials, const TM<NL> t,
                                                const SP s, const i64 n_t, const int C,
                                                const i64 n1c, const double omega,
                                                const i64 s0) {
  __shared__ double sh[32];
  extern __shared__ double ring[];
  const unsigned bx = blockIdx.x, by = blockIdx.y;
  const i64 tid = i64(bx) * blockDim.x + threadIdx.x;
  const i64 n0 = i64(by) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  const double sumsq =
      STMG_UPDOWN_OPS
          ? updown_body_ops<DIM, NL, CO>(tid, n0, nend, ec, pp, f, fc, t, s, n1c, omega, ring, s0)
          : updown_body<DIM, NL, CO>(tid, n0, nend, ec, pp, f, fc, t, s, n1c, omega, ring, s0);
  pdl_trigger();
  const double tot = block_sum(sumsq, sh);
  if (threadIdx.x == 0) partials[i64(by) * gridDim.x + bx] = tot;
}

// Per-mode forward substitution u_n = A_j^-1 (f_n + M_j N u_{n-1})
// (st_system.cpp:118-130 in the sine basis).
template <int DIM, int NL, bool COH>
__device__ __forceinline__ void fwdsub_body(const i64 r, const double* f, double* u,
                                            const TM<NL>& t, const SP& s, const i64 n_t) {
  if (r >= s.nx) return;
  double Mj, Kj;
  mode_eig<DIM, COH>(s, r, Mj, Kj);
  const ModeLU<NL> lu(t, Mj, Kj);
  const i64 nx = s.nx, slab = NL * nx;
  double prev[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) prev[l] = 0.0;
  for (i64 m = 0; m < n_t; ++m) {
    double fv[NL], nv[NL], x[NL];
    ld_ro<COH, NL>(f + m * slab + r, nx, fv);
    matvec<NL>(t.N, prev, nv);
#pragma unroll
    for (int l = 0; l < NL; ++l) fv[l] += Mj * nv[l];
    lu.solve(fv, x);
    store_nl<NL>(u + m * slab + r, nx, x);
#pragma unroll
    for (int l = 0; l < NL; ++l) prev[l] = x[l];
  }
}

template <int DIM, int NL, bool ZERO, int CO>
__global__ void __launch_bounds__(256) k_down(const double* __restrict__ f,
                                              const double* __restrict__ uin,
                                              double* __restrict__ uout,
                                              double* __restrict__ fc, const TM<NL> t,
                                              const SP s, const i64 n_t, const int C,
                                              const i64 n1c, const double omega,
                                              const bool first_global) {
  const i64 tid = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 n0 = i64(blockIdx.y) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  extern __shared__ double ring[];
  down_body<DIM, NL, ZERO, CO, false, bool(STMG_DOWN_ASYNC), true>(tid, n0, nend, f, uin, uout, fc, t, s, n1c, omega,
                                            n0 > 0 || !first_global, n0 - 1 > 0 || !first_global,
                                            ring);
  pdl_trigger();
}

template <int DIM, int NL, int CO, bool RESID>
__global__ void __launch_bounds__(256) k_up(const double* __restrict__ ec,
                                            const double* __restrict__ uin,
                                            const double* __restrict__ f,
                                            double* __restrict__ uout,
                                            double* __restrict__ partials, const TM<NL> t,
                                            const SP s, const i64 n_t, const int C,
                                            const i64 n1c, const double omega,
                                            const bool first_global) {
  __shared__ double sh[32];
  const unsigned bx = blockIdx.x, by = blockIdx.y;
  const i64 tid = i64(bx) * blockDim.x + threadIdx.x;
  const i64 n0 = i64(by) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  extern __shared__ double ring[];
  const double sumsq = up_body<DIM, NL, CO, RESID, false, bool(STMG_UP_ASYNC), true>(
      tid, n0, nend, ec, uin, f, uout, t, s, n1c, omega, n0 > 0 || !first_global,
      n0 - 1 > 0 || !first_global, ring);
  pdl_trigger();
  if (RESID) {
    const double tot = block_sum(sumsq, sh);
    if (threadIdx.x == 0) partials[i64(by) * gridDim.x + bx] = tot;
  }
}

// Coarse-level tail: all levels of the V-cycle from the first "small" level
// down to the coarsest and back, in ONE thread block with every vector in
// shared memory (the levels are tiny; a launch per level, or time-marching
// through L2, would dominate).  Zero initial guess on entry (mg.cpp:119),
// V(1,1), gamma = 1.  Work items are (mode lane, time chunk); the lanes of an
// alias group always share a chunk.  In: F of the first tail level (global);
// out: its corrected iterate U0 (global), as the per-level path leaves it.
template <int NL>
struct TailLevel {
  TM<NL> t;
  SP s;
  i64 n_t;
  i64 n1c;
  int mode;  // coarsening to the next level (0 on the coarsest)
  double* F;
  double* U0;
  double* U1;
};

constexpr int kTailMaxLevels = 24;

// DG/transfer blocks of every tail level as a kernel parameter (constant
// bank): indexed by the level, read with LDC instead of shared-memory loads
// in the dependent per-step chains.
template <int NL>
struct TailParams {
  TM<NL> t[kTailMaxLevels];
};

constexpr int kTailThreads = 512;  // 128 registers per thread: no spills

// cop != nullptr: coarse-operator build, one CTA per column i = blockIdx.x:
// the tail runs on the unit vector e_i (instead of the first level's F) and
// its result is column i of the n x n row-major matrix cop.
template <int DIM, int NL>
__global__ void __launch_bounds__(kTailThreads) k_tail(const TailLevel<NL>* __restrict__ lv,
                                               const int nlev, const double omega,
                                               const __grid_constant__ TailParams<NL> P,
                                               double* __restrict__ cop) {
#ifdef STMG_TAIL_STAMPS
  unsigned long long ts[32];
  int nts = 0;
  auto stamp = [&] {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (nts < 32) ts[nts++] = t;
  };
  stamp();
#define TAIL_STAMP() stamp()
#else
#define TAIL_STAMP() (void)0
#endif
  extern __shared__ double smem[];
  __shared__ TailLevel<NL> lvs[kTailMaxLevels];
  __shared__ i64 off[kTailMaxLevels + 1];
  const int T = blockDim.x;
  {  // level table -> shared memory in one cooperative copy
    static_assert(sizeof(TailLevel<NL>) % 8 == 0, "table copy in 8-byte words");
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(lv);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(lvs);
    const int words = int(nlev * sizeof(TailLevel<NL>) / 8);
    for (int i = threadIdx.x; i < words; i += T) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    off[0] = 0;
    for (int k = 0; k < nlev; ++k) off[k + 1] = off[k] + 3 * lvs[k].n_t * NL * lvs[k].s.nx;
  }
  __syncthreads();
  if (threadIdx.x < nlev) {  // point every level at its shared-memory vectors
    const int k = threadIdx.x;
    const i64 sz = lvs[k].n_t * NL * lvs[k].s.nx;
    lvs[k].F = smem + off[k];
    lvs[k].U0 = smem + off[k] + sz;
    lvs[k].U1 = smem + off[k] + 2 * sz;
  }
  {  // sine tables (mval | kval | rfac, contiguous per level) -> shared memory
    double* tab = smem + off[nlev];
    for (int k = 0; k < nlev; ++k) {
      const int n1 = int(lv[k].s.n1);
      const double* g = lv[k].s.mval;  // the three tables are contiguous
      for (int i = threadIdx.x; i < 3 * n1; i += T) tab[i] = g[i];
      if (threadIdx.x == 0) {
        lvs[k].s.mval = tab;
        lvs[k].s.kval = tab + n1;
        lvs[k].s.rfac = tab + 2 * n1;
      }
      tab += 3 * n1;
    }
  }
  const int sz0 = int(lv[0].n_t * NL * lv[0].s.nx);
  TAIL_STAMP();
  pdl_wait();  // the tables above are constants; the rhs is the previous kernel's output
  TAIL_STAMP();
  if (cop) {  // unit rhs e_i
    for (int i = threadIdx.x; i < sz0; i += T) smem[i] = (i == int(blockIdx.x)) ? 1.0 : 0.0;
  } else {  // stage the first level's rhs
    const double* g = lv[0].F;
    for (int i = threadIdx.x; i < sz0; i += T) smem[i] = g[i];
  }
  __syncthreads();
  TAIL_STAMP();
  for (int k = 0; k + 1 < nlev; ++k) {
    const TailLevel<NL>& A = lvs[k];
    const TailLevel<NL>& B = lvs[k + 1];
    const int nt = int(A.n_t);
    const int lanes = int(ipow(A.s.G, DIM) << DIM);
    int C = 2;
    while (C < nt && lanes * (nt / C) > T) C *= 2;
    const int items = lanes * ((nt + C - 1) / C);
    const int rounded = (items + T - 1) / T * T;
    for (int it = threadIdx.x; it < rounded; it += T) {
      const int lane = it % lanes, n0 = (it / lanes) * C;
      if (n0 >= nt) continue;  // whole alias groups skip together
      const int nend = min(n0 + C, nt);
      if (A.mode == 2)
        down_body<DIM, NL, true, 2, true>(lane, n0, nend, A.F, A.U1, A.U1, B.F, P.t[k], A.s,
                                          A.n1c, omega, n0 > 0, n0 - 1 > 0);
      else
        down_body<DIM, NL, true, 1, true>(lane, n0, nend, A.F, A.U1, A.U1, B.F, P.t[k], A.s,
                                          A.s.n1, omega, n0 > 0, n0 - 1 > 0);
    }
    __syncthreads();
    TAIL_STAMP();
  }
  {
    const TailLevel<NL>& A = lvs[nlev - 1];
    for (int r = threadIdx.x; r < int(A.s.nx); r += T)
      fwdsub_body<DIM, NL, true>(r, A.F, A.U0, P.t[nlev - 1], A.s, A.n_t);
  }
  __syncthreads();
  TAIL_STAMP();
  for (int k = nlev - 2; k >= 0; --k) {
    const TailLevel<NL>& A = lvs[k];
    const TailLevel<NL>& B = lvs[k + 1];
    const int nt = int(A.n_t);
    const int lanes = int(ipow(A.s.G, DIM) << DIM);
    int C = 2;
    while (C < nt && lanes * (nt / C) > T) C *= 2;
    const int items = lanes * ((nt + C - 1) / C);
    for (int it = threadIdx.x; it < items; it += T) {
      const int lane = it % lanes, n0 = (it / lanes) * C;
      const int nend = min(n0 + C, nt);
      if (A.mode == 2)
        up_body<DIM, NL, 2, false, true>(lane, n0, nend, B.U0, A.U1, A.F, A.U0, P.t[k], A.s,
                                         A.n1c, omega, n0 > 0, n0 - 1 > 0);
      else
        up_body<DIM, NL, 1, false, true>(lane, n0, nend, B.U0, A.U1, A.F, A.U0, P.t[k], A.s,
                                         A.s.n1, omega, n0 > 0, n0 - 1 > 0);
    }
    __syncthreads();
    TAIL_STAMP();
  }
  if (cop) {  // column blockIdx.x of the coarse operator
    for (int i = threadIdx.x; i < sz0; i += T) cop[i64(i) * sz0 + blockIdx.x] = smem[sz0 + i];
  } else {  // hand the first level's iterate back
    double* g = lv[0].U0;
    for (int i = threadIdx.x; i < sz0; i += T) g[i] = smem[sz0 + i];
  }
#ifdef STMG_TAIL_STAMPS
  __syncthreads();
  stamp();
  if (threadIdx.x == 0) {
    printf("TAIL");
    for (int i = 1; i < nts; ++i) printf(" %llu", ts[i] - ts[i - 1]);
    printf("\n");
  }
#endif
}

// Fused coarse levels: the V(1,1) down pass of levels a..b (zero initial
// guess, mg.cpp:106-119) and, after the tail / coarser levels, the up pass
// b..a (mg.cpp:121-131), each in ONE launch.  In the sine basis full
// coarsening only couples the 2^DIM modes of an alias group, so the modes of
// levels a..b split into independent trees: a tree is rooted at an alias
// group of level r (r = b, or a "middle" group of a level r < b, whose modes
// restrict to zero) and holds, one level finer, the groups whose coarse modes
// are the root's member modes, and so on down to level a.  Every step of the
// cycle on these levels -- smoothing, residual, restriction, prolongation --
// stays inside one tree, so a CTA runs whole trees level after level with
// __syncthreads between the levels instead of a kernel boundary per level.
// The per-mode work is down_body / up_body of the per-level kernels on the
// same global buffers (the same arithmetic and alias-group shuffle order, so
// the results are bitwise those of the per-level path).  Trees of one root
// level are packed `count` per CTA.
constexpr int kCsubMaxLevels = 8;  // levels a..b+1

template <int NL>
struct CsubLevel {
  TM<NL> t;
  SP s;
  i64 n_t;
  i64 n1c;
  double* F;
  double* U0;
  double* U1;
};

template <int NL>
struct CsubParams {
  CsubLevel<NL> lv[kCsubMaxLevels];  // index 0 = level a
  int nb;                            // index of level b (b - a)
  double omega;
};

// Global lane (alias group << DIM | member) at table level l of local lane
// `lane` of the tree rooted at group `root` of table level r.  Lane bits
// [DIM (m - l), DIM (m - l + 1)) select the member at level m; a member that
// does not exist (the mirror of a middle index) kills its subtree, whose
// lanes get an out-of-range group (make_member: ok = false, nothing stored).
template <int DIM, int NL>
__device__ __forceinline__ i64 csub_lane(const CsubParams<NL>& P, int r, unsigned root, int l,
                                         int lane) {
  int ia[DIM];
  {
    const unsigned G = unsigned(P.lv[r].s.G);
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      ia[a] = int(root % G);
      root /= G;
    }
  }
  bool dead = false;
  for (int m = r; m > l; --m) {
    const int beta = (lane >> (DIM * (m - l))) & ((1 << DIM) - 1);
    const int Gm = P.lv[m].s.G;
    const int n1m = int(P.lv[m].s.n1);
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const bool mid = ia[a] >= Gm - 1;
      const int bit = (beta >> a) & 1;
      if (bit && mid) dead = true;
      ia[a] = (bit && !mid) ? n1m - 1 - ia[a] : ia[a];
    }
  }
  const i64 Gl = P.lv[l].s.G;
  i64 gg = 0, mul = 1;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    gg += ia[a] * mul;
    mul *= Gl;
  }
  if (dead) gg = ipow(Gl, DIM);
  return (gg << DIM) | (lane & ((1 << DIM) - 1));
}

// Chunk of time steps per work item so that `lanes` lanes fill the block.
__device__ __forceinline__ int csub_chunk(int lanes, int nt, int T) {
  int C = 2;
  while (C < nt && lanes * ((nt + C - 1) / C) > T) C *= 2;
  return C;
}

struct CsubCta {
  int root;    // table level of the trees' roots
  int first;   // first tree (index into the root-group array)
  int count;   // trees in this CTA
};

template <int DIM, int NL>
__global__ void __launch_bounds__(256) k_csub_down(const CsubCta* __restrict__ ctas,
                                                   const unsigned* __restrict__ roots,
                                                   const __grid_constant__ CsubParams<NL> P) {
  const CsubCta cta = ctas[blockIdx.x];
  const int T = blockDim.x;
  pdl_wait();  // level a's rhs is the previous kernel's output
  for (int l = 0; l <= cta.root; ++l) {
    const CsubLevel<NL>& A = P.lv[l];
    const CsubLevel<NL>& B = P.lv[l + 1];
    const int per = 1 << (DIM * (cta.root - l + 1));
    const int lanes = per * cta.count;
    const int nt = int(A.n_t);
    const int C = csub_chunk(lanes, nt, T);
    const int items = lanes * ((nt + C - 1) / C);
    const int rounded = (items + T - 1) / T * T;
    for (int it = threadIdx.x; it < rounded; it += T) {
      const int lane = it % lanes, n0 = (it / lanes) * C;
      if (n0 >= nt) continue;  // whole alias groups skip together
      const i64 tid = csub_lane<DIM, NL>(P, cta.root, roots[cta.first + lane / per], l, lane % per);
      const int nend = min(n0 + C, nt);
      if (l == 0)
        down_body<DIM, NL, true, 2, false>(tid, n0, nend, A.F, A.U1, A.U1, B.F, A.t, A.s, A.n1c,
                                           P.omega, n0 > 0, n0 - 1 > 0);
      else
        down_body<DIM, NL, true, 2, true>(tid, n0, nend, A.F, A.U1, A.U1, B.F, A.t, A.s, A.n1c,
                                          P.omega, n0 > 0, n0 - 1 > 0);
    }
    __syncthreads();
  }
  pdl_trigger();
}

template <int DIM, int NL>
__global__ void __launch_bounds__(256) k_csub_up(const CsubCta* __restrict__ ctas,
                                                 const unsigned* __restrict__ roots,
                                                 const __grid_constant__ CsubParams<NL> P) {
  const CsubCta cta = ctas[blockIdx.x];
  const int T = blockDim.x;
  pdl_wait();  // the correction of level b + 1 is the previous kernel's output
  for (int l = cta.root; l >= 0; --l) {
    const CsubLevel<NL>& A = P.lv[l];
    const CsubLevel<NL>& B = P.lv[l + 1];
    const int per = 1 << (DIM * (cta.root - l + 1));
    const int lanes = per * cta.count;
    const int nt = int(A.n_t);
    const int C = csub_chunk(lanes, nt, T);
    const int items = lanes * ((nt + C - 1) / C);
    for (int it = threadIdx.x; it < items; it += T) {
      const int lane = it % lanes, n0 = (it / lanes) * C;
      const i64 tid = csub_lane<DIM, NL>(P, cta.root, roots[cta.first + lane / per], l, lane % per);
      const int nend = min(n0 + C, nt);
      up_body<DIM, NL, 2, false, true>(tid, n0, nend, B.U0, A.U1, A.F, A.U0, A.t, A.s, A.n1c,
                                       P.omega, n0 > 0, n0 - 1 > 0);
    }
    __syncthreads();
  }
  pdl_trigger();
}

// Plain damped block-Jacobi sweep per mode (ping-pong: u_out != u_in).
template <int DIM, int NL, bool ZERO>
__global__ void __launch_bounds__(128) k_smooth(const double* __restrict__ f,
                                                const double* __restrict__ uin,
                                                double* __restrict__ uout, const TM<NL> t,
                                                const SP s, const i64 n_t, const int C,
                                                const double omega, const bool first_global) {
  pdl_wait();
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.nx) return;
  double Mj, Kj;
  mode_eig<DIM>(s, r, Mj, Kj);
  const ModeLU<NL> lu(t, Mj, Kj);
  const i64 nx = s.nx, slab = NL * nx;
  const i64 n0 = i64(blockIdx.y) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  double uo[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) uo[l] = 0.0;
  if (!ZERO && (n0 > 0 || !first_global)) load_nl<NL>(uin + (n0 - 1) * slab + r, nx, uo);
  for (i64 m = n0; m < nend; ++m) {
    double fv[NL], uv[NL], nv[NL], x[NL], w[NL];
    load_nl<NL>(f + m * slab + r, nx, fv);
    if (!ZERO) {
      load_nl<NL>(uin + m * slab + r, nx, uv);
      matvec<NL>(t.N, uo, nv);
#pragma unroll
      for (int l = 0; l < NL; ++l) fv[l] += Mj * nv[l];
    }
    lu.solve(fv, x);
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      w[l] = ZERO ? omega * x[l] : (1.0 - omega) * uv[l] + omega * x[l];
      if (!ZERO) uo[l] = uv[l];
    }
    store_nl<NL>(uout + m * slab + r, nx, w);
  }
}

// Residual sum-of-squares partials of f - L u per (chunk, block).
// ZERO: u == 0 is known (zero initial guess): only f is read; every term that
// involves u is an exact zero, so the partials are bitwise those of the
// general kernel on a zero vector.
template <int DIM, int NL, bool ZERO>
__global__ void __launch_bounds__(128) k_resnorm(const double* __restrict__ u,
                                                 const double* __restrict__ f,
                                                 double* __restrict__ partials, const TM<NL> t,
                                                 const SP s, const i64 n_t, const int C,
                                                 const bool first_global) {
  pdl_wait();
  __shared__ double sh[32];
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  double sumsq = 0.0;
  if (r < s.nx) {
    double Mj, Kj;
    mode_eig<DIM>(s, r, Mj, Kj);
    const i64 nx = s.nx, slab = NL * nx;
    const i64 n0 = i64(blockIdx.y) * C;
    const i64 nend = min(n0 + i64(C), n_t);
    double up[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) up[l] = 0.0;
    if (!ZERO && (n0 > 0 || !first_global)) load_nl<NL>(u + (n0 - 1) * slab + r, nx, up);
    // UB steps per batch: all loads of a batch are issued before the first use
    // (one load pair in flight per thread left this kernel latency bound:
    // 67 us for the 66 MB of C2); the accumulation order is unchanged
    constexpr int UB = NL <= 2 ? 8 : 4;
    for (i64 m0 = n0; m0 < nend; m0 += UB) {
      double uv[UB][NL], fv[UB][NL];
#pragma unroll
      for (int j = 0; j < UB; ++j) {
        if (m0 + j < nend) {
          if (!ZERO) load_nl<NL>(u + (m0 + j) * slab + r, nx, uv[j]);
          load_nl<NL>(f + (m0 + j) * slab + r, nx, fv[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < UB; ++j) {
        if (m0 + j < nend) {
          double au[NL], np[NL];
          if (ZERO) {
#pragma unroll
            for (int l = 0; l < NL; ++l) uv[j][l] = 0.0;
          }
          apply_mode<NL>(t, Mj, Kj, uv[j], au);
          matvec<NL>(t.N, up, np);
#pragma unroll
          for (int l = 0; l < NL; ++l) {
            const double res = fv[j][l] - au[l] + Mj * np[l];
            sumsq += res * res;
            up[l] = uv[j][l];
          }
        }
      }
    }
  }
  const double tot = block_sum(sumsq, sh);
  if (threadIdx.x == 0) partials[i64(blockIdx.y) * gridDim.x + blockIdx.x] = tot;
}

template <int DIM, int NL>
__global__ void __launch_bounds__(128) k_fwdsub(const double* __restrict__ f,
                                                double* __restrict__ u, const TM<NL> t,
                                                const SP s, const i64 n_t) {
  pdl_wait();
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  fwdsub_body<DIM, NL, false>(r, f, u, t, s, n_t);
}

// Per-mode exact block solve in place.
template <int DIM, int NL>
__global__ void __launch_bounds__(256) k_modal_solve(double* __restrict__ x, const TM<NL> t,
                                                     const SP s, const i64 n_t) {
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.nx) return;
  double Mj, Kj;
  mode_eig<DIM>(s, r, Mj, Kj);
  const ModeLU<NL> lu(t, Mj, Kj);
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    double b[NL], y[NL];
    double* p = x + n * NL * s.nx + r;
    load_nl<NL>(p, s.nx, b);
    lu.solve(b, y);
    store_nl<NL>(p, s.nx, y);
  }
}

// ===================================================== physical operators
// Q1 stencils: M = (x)_a M1, K = sum_a K1 on axis a, M1 elsewhere,
// M1 = h/6 {1,4,1}, K1 = 1/h {-1,2,-1} (fem_space.cpp:40-58, + 3D).
template <int DIM>
__device__ __forceinline__ void coords(unsigned r, unsigned n1, int (&c)[3]) {
  c[0] = int(r % n1);
  c[1] = DIM > 1 ? int((r / n1) % n1) : 0;
  c[2] = DIM > 2 ? int(r / (n1 * n1)) : 0;
}

// Accumulate M v and K v at node c of one component vector v.
template <int DIM>
__device__ __forceinline__ void stencil_MK(const double* __restrict__ v, i64 n1, double h,
                                           const int (&c)[3], double& Mv, double& Kv,
                                           bool want_k) {
  const double m0 = 4.0 * h / 6.0, m1 = h / 6.0, k0 = 2.0 / h, k1 = -1.0 / h;
  Mv = 0.0;
  Kv = 0.0;
  const int dzlo = DIM > 2 ? -1 : 0, dzhi = DIM > 2 ? 1 : 0;
  const int dylo = DIM > 1 ? -1 : 0, dyhi = DIM > 1 ? 1 : 0;
  for (int dz = dzlo; dz <= dzhi; ++dz) {
    const int z = c[2] + dz;
    if (z < 0 || z >= n1) continue;
    for (int dy = dylo; dy <= dyhi; ++dy) {
      const int y = c[1] + dy;
      if (y < 0 || y >= n1) continue;
      for (int dx = -1; dx <= 1; ++dx) {
        const int x = c[0] + dx;
        if (x < 0 || x >= n1) continue;
        const double val = __ldg(v + (i64(z) * n1 + y) * n1 + x);
        const double mx = dx ? m1 : m0, my = dy ? m1 : m0, mz = dz ? m1 : m0;
        const double kx = dx ? k1 : k0, ky = dy ? k1 : k0, kz = dz ? k1 : k0;
        double wm = mx, wk = kx;
        if (DIM == 2) {
          wm = mx * my;
          wk = kx * my + mx * ky;
        } else if (DIM == 3) {
          wm = mx * my * mz;
          wk = kx * my * mz + mx * ky * mz + mx * my * kz;
        }
        Mv += wm * val;
        if (want_k) Kv += wk * val;
      }
    }
  }
}

// y_n = (M U_n) K^T + (K U_n) M^T - (M U_{n-1}) N^T; residual: r = f - y
// (st_system.cpp:18-33, 57-67).  One CTA owns a spatial tile and marches
// through a chunk of time steps: slab n (tile + 1-node halo, all DG
// components) is staged in shared memory with cp.async while slab n-1 is
// being used, so u is read from HBM once.  N_tau = a b^T is rank one
// (N[k,l] = psi_l(tau) psi_k(0)), so the jump term is a_k * sum_l b_l (M u_{n-1,l})
// and reuses the M-stencils of the previous step kept in registers.
template <int DIM>
struct ResTile {
  static constexpr int TX = DIM == 1 ? 256 : 32;
  static constexpr int TY = DIM == 1 ? 1 : (DIM == 2 ? 8 : 4);
  static constexpr int TZ = DIM == 3 ? 2 : 1;
  // cp.async ring depth: 3 in 1D/2D; 2 in 3D, where the larger halo makes a
  // third stage cost more occupancy than the extra step in flight gains
  static constexpr int STAGES = DIM == 3 ? 2 : 3;
  static constexpr int HX = TX + 2;
  static constexpr int HY = DIM >= 2 ? TY + 2 : 1;
  static constexpr int HZ = DIM == 3 ? TZ + 2 : 1;
  static constexpr int HALO = HX * HY * HZ;
  static constexpr int THREADS = TX * TY * TZ;
};


// Staging plan of one thread: the (tile + halo) x NL elements it copies each
// step, as slab-relative global offsets (-1: outside the Dirichlet domain ->
// zero fill).  Step-invariant, so computed once per CTA.
template <int DIM, int NL>
struct StagePlan {
  static constexpr int ITEMS = (NL * ResTile<DIM>::HALO + ResTile<DIM>::THREADS - 1) /
                               ResTile<DIM>::THREADS;
  int off[ITEMS];
};

template <int DIM, int NL>
__device__ __forceinline__ void make_plan(StagePlan<DIM, NL>& P, int n1, i64 nx, int x0, int y0,
                                          int z0) {
  using T = ResTile<DIM>;
#pragma unroll
  for (int i = 0; i < StagePlan<DIM, NL>::ITEMS; ++i) {
    const int e = threadIdx.x + i * T::THREADS;
    int o = -1;
    if (e < NL * T::HALO) {
      const int l = e / T::HALO;
      const int h = e - l * T::HALO;
      const int hx = h % T::HX;
      const int hy = (h / T::HX) % T::HY;
      const int hz = h / (T::HX * T::HY);
      const int x = x0 + hx - 1, y = DIM >= 2 ? y0 + hy - 1 : 0, z = DIM == 3 ? z0 + hz - 1 : 0;
      if (x >= 0 && x < n1 && y >= 0 && y < n1 && z >= 0 && z < n1)
        o = int(l * nx + (i64(z) * n1 + y) * n1 + x);
    }
    P.off[i] = o;
  }
}

// Stage slab n of u into buf (cp.async, zero fill outside the domain).
template <int DIM, int NL>
__device__ __forceinline__ void stage_slab(double* buf, const double* u, i64 n, i64 nx,
                                           const StagePlan<DIM, NL>& P) {
  using T = ResTile<DIM>;
  const double* base = u + n * NL * nx;
#pragma unroll
  for (int i = 0; i < StagePlan<DIM, NL>::ITEMS; ++i) {
    const int e = threadIdx.x + i * T::THREADS;
    if (StagePlan<DIM, NL>::ITEMS * T::THREADS == NL * T::HALO || e < NL * T::HALO)
      cp_async8(buf + e, P.off[i] >= 0 ? base + P.off[i] : base, P.off[i] >= 0);
  }
}

// M and K stencils of one staged component at tile-local (tx, ty, tz).
template <int DIM>
__device__ __forceinline__ void stencil_smem(const double* s, int tx, int ty, int tz, double h,
                                             double& Mv, double& Kv) {
  using T = ResTile<DIM>;
  const double m0 = 4.0 * h / 6.0, m1 = h / 6.0, k0 = 2.0 / h, k1 = -1.0 / h;
  auto row = [&](int yy, int zz, double& Mr, double& Kr) {
    const double* p = s + (zz * T::HY + yy) * T::HX + tx + 1;
    const double a = p[-1] + p[1], c = p[0];
    Mr = m1 * a + m0 * c;
    Kr = k1 * a + k0 * c;
  };
  auto plane = [&](int zz, double& Mp, double& Kp) {
    if (DIM == 1) {
      row(0, zz, Mp, Kp);
    } else {
      double Ma, Ka, Mb, Kb, Mc, Kc;
      row(ty, zz, Ma, Ka);
      row(ty + 1, zz, Mb, Kb);
      row(ty + 2, zz, Mc, Kc);
      const double ms = Ma + Mc;
      Mp = m1 * ms + m0 * Mb;
      Kp = m1 * (Ka + Kc) + m0 * Kb + k1 * ms + k0 * Mb;
    }
  };
  if (DIM < 3) {
    plane(0, Mv, Kv);
  } else {
    double Ma, Ka, Mb, Kb, Mc, Kc;
    plane(tz, Ma, Ka);
    plane(tz + 1, Mb, Kb);
    plane(tz + 2, Mc, Kc);
    const double ms = Ma + Mc;
    Mv = m1 * ms + m0 * Mb;
    Kv = m1 * (Ka + Kc) + m0 * Kb + k1 * ms + k0 * Mb;
  }
}

#ifndef STMG_APPLY_FREG
#define STMG_APPLY_FREG 1
#endif
template <int DIM, int NL, bool RES>
__global__ void __launch_bounds__(ResTile<DIM>::THREADS) k_apply(
    const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ y,
    const TM<NL> t, const i64 n1_, const i64 nx, const double h, const i64 n_t, const int C,
    const bool first_global, const double* __restrict__ ab) {
  using T = ResTile<DIM>;
  extern __shared__ double dsm[];
  constexpr int BS = NL * T::HALO;  // one staged slab
  const int n1 = int(n1_);
  const int tilesx = (n1 + T::TX - 1) / T::TX;
  const int tilesy = DIM >= 2 ? (n1 + T::TY - 1) / T::TY : 1;
  int tile = blockIdx.x;
  const int bx = tile % tilesx;
  tile /= tilesx;
  const int by = tile % tilesy;
  const int bz = tile / tilesy;
  const int x0 = bx * T::TX, y0 = by * T::TY, z0 = bz * T::TZ;
  const int tx = threadIdx.x % T::TX;
  const int ty = (threadIdx.x / T::TX) % T::TY;
  const int tz = threadIdx.x / (T::TX * T::TY);
  const int x = x0 + tx, yy = y0 + ty, z = z0 + tz;
  const bool inside = x < n1 && (DIM < 2 || yy < n1) && (DIM < 3 || z < n1);
  const i64 r = (i64(DIM == 3 ? z : 0) * n1 + (DIM >= 2 ? yy : 0)) * n1 + x;
  const i64 n0 = i64(blockIdx.y) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  const i64 slab = NL * nx;
  double a[NL], b[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    a[k] = ab[k];
    b[k] = ab[kMaxNL + k];
  }

  // cp.async ring: stage m holds slab m of u (tile + halo) and, for the
  // residual, this tile's f of step m; STAGES - 1 steps are in flight while
  // one is computed (the kernel is latency bound with a single slab ahead)
  constexpr int NS = T::STAGES;
  // FREG: f goes straight to registers one step ahead instead of through the
  // shared-memory ring (the ring's 8-byte LDGSTS + LDS traffic is what bounds
  // this kernel: L1 throughput 83 % on C2)
  constexpr bool FREG = RES && STMG_APPLY_FREG;
  constexpr int FS = (RES && !FREG) ? NL * T::THREADS : 0;
  constexpr int SS = BS + FS;  // doubles per stage
  auto stage = [&](int m) { return dsm + ((m + NS) % NS) * SS; };
  StagePlan<DIM, NL> plan;
  make_plan<DIM, NL>(plan, n1, nx, x0, y0, z0);
  auto issue = [&](i64 n) {  // slab n -> stage (n - n0 + 1) mod NS
    double* st = stage(int(n - n0 + 1));
    stage_slab<DIM, NL>(st, u, n, nx, plan);
    if (RES && !FREG) {
#pragma unroll
      for (int k = 0; k < NL; ++k)
        cp_async8(st + BS + k * T::THREADS + threadIdx.x,
                  inside ? f + n * slab + k * nx + r : f, inside);
    }
  };
  double mw_prev = 0.0;  // M-stencil trace of step n-1 (rank-one jump)
  const bool has_prev = n0 > 0 || !first_global;
  if (has_prev) issue(n0 - 1);
  cp_async_commit();
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    if (n0 + q < nend) issue(n0 + q);
    cp_async_commit();
  }
  cp_async_wait<NS - 1>();
  __syncthreads();
  if (has_prev && inside) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      double Mv, Kv;
      stencil_smem<DIM>(stage(0) + l * T::HALO, tx, ty, tz, h, Mv, Kv);
      mw_prev += b[l] * Mv;
    }
  }
  double fc[NL], fn[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) fc[k] = fn[k] = 0.0;
  if (FREG && inside && n0 < nend) {
#pragma unroll
    for (int k = 0; k < NL; ++k) fc[k] = __ldcs(f + n0 * slab + k * nx + r);
  }
  for (i64 n = n0; n < nend; ++n) {
    const int j = int(n - n0 + 1);
    if (FREG && inside && n + 1 < nend) {
#pragma unroll
      for (int k = 0; k < NL; ++k) fn[k] = __ldcs(f + (n + 1) * slab + k * nx + r);
    }
    cp_async_wait<NS - 2>();  // groups up to step n landed
    __syncthreads();          // slab n visible; stage of n - 1 free
    if (n + NS - 1 < nend) issue(n + NS - 1);
    cp_async_commit();
    if (inside) {
      const double* st = stage(j);
      double MU[NL], KU[NL], mw = 0.0;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        stencil_smem<DIM>(st + l * T::HALO, tx, ty, tz, h, MU[l], KU[l]);
        mw += b[l] * MU[l];
      }
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < NL; ++l) acc += MU[l] * t.K[k][l] + KU[l] * t.M[k][l];
        acc -= a[k] * mw_prev;
        const i64 o = n * slab + k * nx + r;
        const double fv = FREG ? fc[k] : (RES ? st[BS + k * T::THREADS + threadIdx.x] : 0.0);
        __stcs(y + o, RES ? fv - acc : acc);
      }
      mw_prev = mw;
    }
    if (FREG) {
#pragma unroll
      for (int k = 0; k < NL; ++k) fc[k] = fn[k];
    }
  }
}

// Register-blocked Q1 apply/residual for 2D and 3D.  A CTA of 32 x 4 threads
// owns a tile of 32 (x) x 4 (y) x R (z) nodes in 3D, or 32 (x) x 4R (y) in 2D;
// every thread computes R consecutive outputs along the blocked axis (y in
// 2D, z in 3D) with a rolling window of the 1D row (2D) or 2D plane (3D)
// stencil combinations, so one staged value feeds ~3 outputs instead of one:
// (R + 2) / R x 3 shared-memory loads per output in 2D (9 before), x 9 in 3D
// (27 before).  Staging: cp.async ring of STAGES slabs (tile + halo of u and
// the tile of f), zero fill outside the Dirichlet domain; the rank-one jump
// reuses the previous step's M-stencil traces kept in registers.
template <int DIM>
struct RbTile {
  static constexpr int TX = 32, TYT = DIM == 2 ? 8 : 4;
  static constexpr int R = 4;   // outputs per thread along the blocked axis
  static constexpr int YB = DIM == 3 ? 2 : 1;  // 3D: y rows per thread (shared plane rows)
  static constexpr int NO = R * YB;            // outputs per thread
  static constexpr int TY = DIM == 2 ? TYT * R : TYT * YB;
  static constexpr int TZ = DIM == 3 ? R : 1;
  static constexpr int HX = TX + 2, HY = TY + 2, HZ = DIM == 3 ? TZ + 2 : 1;
  static constexpr int HALO = HX * HY * HZ;
  static constexpr int OUT = TX * TY * TZ;
  static constexpr int THREADS = TX * TYT;
  static constexpr int STAGES = 2;
};

#ifndef STMG_RB_MINB
#define STMG_RB_MINB 2
#endif
template <int DIM, int NL, bool RES>
__global__ void __launch_bounds__(RbTile<DIM>::THREADS, DIM == 3 ? STMG_RB_MINB : 1) k_apply_rb(
    const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ y,
    const TM<NL> t, const i64 n1_, const i64 nx, const double h, const i64 n_t, const int C,
    const bool first_global, const double* __restrict__ ab) {
  using T = RbTile<DIM>;
  constexpr int R = T::R;
  extern __shared__ double dsm[];
  constexpr int BS = NL * T::HALO;
  constexpr int FS = RES ? NL * T::OUT : 0;
  constexpr int SS = BS + FS;
  constexpr int NS = T::STAGES;
  const int n1 = int(n1_);
  const int tilesx = (n1 + T::TX - 1) / T::TX;
  const int tilesy = (n1 + T::TY - 1) / T::TY;
  int tile = blockIdx.x;
  const int bx = tile % tilesx;
  tile /= tilesx;
  const int by = tile % tilesy;
  const int bz = tile / tilesy;
  const int x0 = bx * T::TX, y0 = by * T::TY, z0 = bz * T::TZ;
  const int tx = threadIdx.x % T::TX, ty = threadIdx.x / T::TX;
  const int x = x0 + tx;
  const i64 n0 = i64(blockIdx.y) * C;
  const i64 nend = min(n0 + i64(C), n_t);
  const i64 slab = NL * nx;
  const double m0 = 4.0 * h / 6.0, m1 = h / 6.0, k0 = 2.0 / h, k1 = -1.0 / h;
  double a[NL], b[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    a[k] = ab[k];
    b[k] = ab[kMaxNL + k];
  }
  // output j = yb * R + i of this thread: tile-local (tx, oy, oz)
  constexpr int YB = T::YB, NO = T::NO;
  auto out_y = [&](int j) { return DIM == 2 ? ty * R + j : ty * YB + j / R; };
  auto out_z = [&](int j) { return DIM == 3 ? j % R : 0; };
  auto out_inside = [&](int j) {
    return x < n1 && y0 + out_y(j) < n1 && (DIM < 3 || z0 + out_z(j) < n1);
  };
  auto out_off = [&](int j) {
    return (i64(DIM == 3 ? z0 + out_z(j) : 0) * n1 + (y0 + out_y(j))) * n1 + x;
  };
  auto stage = [&](int m) { return dsm + ((m + NS) % NS) * SS; };
  // staging plan: slab-relative offsets of this thread's (tile + halo) and f
  // elements, computed once (-1: outside the Dirichlet domain -> zero fill)
  constexpr int IH = (BS + T::THREADS - 1) / T::THREADS;
  constexpr int IF = RES ? (FS + T::THREADS - 1) / T::THREADS : 0;
  int offh[IH], offf[IF > 0 ? IF : 1];
#pragma unroll
  for (int i = 0; i < IH; ++i) {
    const int e = threadIdx.x + i * T::THREADS;
    int o = -1;
    if (e < BS) {
      const int l = e / T::HALO;
      const int hh = e - l * T::HALO;
      const int hx = hh % T::HX, hy = (hh / T::HX) % T::HY, hz = hh / (T::HX * T::HY);
      const int gx = x0 + hx - 1, gy = y0 + hy - 1, gz = DIM == 3 ? z0 + hz - 1 : 0;
      if (gx >= 0 && gx < n1 && gy >= 0 && gy < n1 && gz >= 0 && gz < n1)
        o = int(l * nx + (i64(gz) * n1 + gy) * n1 + gx);
    }
    offh[i] = o;
  }
#pragma unroll
  for (int i = 0; i < IF; ++i) {
    const int e = threadIdx.x + i * T::THREADS;
    int o = -1;
    if (e < FS) {
      const int l = e / T::OUT;
      const int q = e - l * T::OUT;
      const int gx = x0 + q % T::TX, gy = y0 + (q / T::TX) % T::TY;
      const int gz = DIM == 3 ? z0 + q / (T::TX * T::TY) : 0;
      if (gx < n1 && gy < n1 && gz < n1) o = int(l * nx + (i64(gz) * n1 + gy) * n1 + gx);
    }
    offf[i] = o;
  }
  auto issue = [&](i64 n) {  // slab n -> stage (n - n0 + 1) mod NS
    double* st = stage(int(n - n0 + 1));
    const double* base = u + n * slab;
#pragma unroll
    for (int i = 0; i < IH; ++i) {
      const int e = threadIdx.x + i * T::THREADS;
      if (IH * T::THREADS == BS || e < BS)
        cp_async8(st + e, base + (offh[i] >= 0 ? offh[i] : 0), offh[i] >= 0);
    }
    if (RES) {
      const double* fb = f + n * slab;
#pragma unroll
      for (int i = 0; i < IF; ++i) {
        const int e = threadIdx.x + i * T::THREADS;
        if (IF * T::THREADS == FS || e < FS)
          cp_async8(st + BS + e, fb + (offf[i] >= 0 ? offf[i] : 0), offf[i] >= 0);
      }
    }
  };
  // 1D row combination of staged component s at halo (hy, hz), this thread's x
  auto row = [&](const double* s, int hy, int hz, double& Mr, double& Kr) {
    const double* p = s + (hz * T::HY + hy) * T::HX + tx + 1;
    const double aa = p[-1] + p[1], c = p[0];
    Mr = m1 * aa + m0 * c;
    Kr = k1 * aa + k0 * c;
  };
  // units along the blocked axis: a row (2D, halo y = w) or the YB y-plane
  // combinations of this thread's rows (3D, halo z = w; YB + 2 rows loaded)
  auto unit = [&](const double* s, int w, double (&Mu)[YB], double (&Ku)[YB]) {
    if (DIM == 2) {
      row(s, w, 0, Mu[0], Ku[0]);
    } else {
      double Mr[YB + 2], Kr[YB + 2];
#pragma unroll
      for (int q = 0; q < YB + 2; ++q) row(s, ty * YB + q, w, Mr[q], Kr[q]);
#pragma unroll
      for (int yb = 0; yb < YB; ++yb) {
        const double ms = Mr[yb] + Mr[yb + 2];
        Mu[yb] = m1 * ms + m0 * Mr[yb + 1];
        Ku[yb] = m1 * (Kr[yb] + Kr[yb + 2]) + m0 * Kr[yb + 1] + k1 * ms + k0 * Mr[yb + 1];
      }
    }
  };
  const int w0 = DIM == 2 ? ty * R : 0;  // first halo unit of this thread's window
  double mw_prev[NO];
#pragma unroll
  for (int j = 0; j < NO; ++j) mw_prev[j] = 0.0;
  const bool has_prev = n0 > 0 || !first_global;
  if (has_prev) issue(n0 - 1);
  cp_async_commit();
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    if (n0 + q < nend) issue(n0 + q);
    cp_async_commit();
  }
  cp_async_wait<NS - 1>();
  __syncthreads();
  // Streams the outputs of this thread along the blocked axis: per output the
  // M / K stencils of every component from a rolling window of 3 units.
  auto sweep = [&](const double* st, auto&& emit) {
    double M0[NL][YB], K0[NL][YB], M1[NL][YB], K1[NL][YB];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      unit(st + l * T::HALO, w0, M0[l], K0[l]);
      unit(st + l * T::HALO, w0 + 1, M1[l], K1[l]);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      double MU[YB][NL], KU[YB][NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        double M2[YB], K2[YB];
        unit(st + l * T::HALO, w0 + i + 2, M2, K2);
#pragma unroll
        for (int yb = 0; yb < YB; ++yb) {
          const double ms = M0[l][yb] + M2[yb];
          MU[yb][l] = m1 * ms + m0 * M1[l][yb];
          KU[yb][l] = m1 * (K0[l][yb] + K2[yb]) + m0 * K1[l][yb] + k1 * ms + k0 * M1[l][yb];
          M0[l][yb] = M1[l][yb];
          K0[l][yb] = K1[l][yb];
          M1[l][yb] = M2[yb];
          K1[l][yb] = K2[yb];
        }
      }
#pragma unroll
      for (int yb = 0; yb < YB; ++yb) emit(yb * R + i, MU[yb], KU[yb]);
    }
  };
  if (has_prev) {
    sweep(stage(0), [&](int j, const double (&MU)[NL], const double (&)[NL]) {
      double mw = 0.0;
#pragma unroll
      for (int l = 0; l < NL; ++l) mw += b[l] * MU[l];
      mw_prev[j] = mw;
    });
  }
  for (i64 n = n0; n < nend; ++n) {
    const int jst = int(n - n0 + 1);
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (n + NS - 1 < nend) issue(n + NS - 1);
    cp_async_commit();
    const double* st = stage(jst);
    sweep(st, [&](int j, const double (&MU)[NL], const double (&KU)[NL]) {
      double mw = 0.0;
#pragma unroll
      for (int l = 0; l < NL; ++l) mw += b[l] * MU[l];
      if (out_inside(j)) {
        const i64 r = out_off(j);
        const int q = (out_z(j) * T::TY + out_y(j)) * T::TX + tx;
#pragma unroll
        for (int k = 0; k < NL; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < NL; ++l) acc += MU[l] * t.K[k][l] + KU[l] * t.M[k][l];
          acc -= a[k] * mw_prev[j];
          const i64 o = n * slab + k * nx + r;
          __stcs(y + o, RES ? st[BS + k * T::OUT + q] - acc : acc);
        }
      }
      mw_prev[j] = mw;
    });
  }
}

// restrict_semi / restrict_full (transfer.cpp:75-85, 138-149): one thread per
// coarse (step, node): full weighting 1/2{1 2 1} per axis of the time
// restriction c_n = U_2n R1^T + U_2n+1 R2^T.
template <int DIM, int NL, int CO>
__global__ void __launch_bounds__(256) k_restrict(const double* __restrict__ fine,
                                                  double* __restrict__ coarse, const TM<NL> t,
                                                  const i64 n1, const i64 n1c, const i64 ntc) {
  const i64 nx = ipow(n1, DIM), nxc = ipow(n1c, DIM);
  const unsigned rc = blockIdx.x * blockDim.x + threadIdx.x;
  if (rc >= nxc) return;
  int c[3];
  coords<DIM>(rc, unsigned(n1c), c);
  for (i64 nc = blockIdx.y; nc < ntc; nc += gridDim.y) {
  double v0[NL], v1[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) v0[l] = v1[l] = 0.0;
  const double* a0 = fine + (2 * nc) * NL * nx;
  const double* a1 = a0 + NL * nx;
  if (CO == 1) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      v0[l] = __ldg(a0 + l * nx + rc);
      v1[l] = __ldg(a1 + l * nx + rc);
    }
  } else {
    const int dzn = DIM > 2 ? 3 : 1, dyn = DIM > 1 ? 3 : 1;
    for (int dz = 0; dz < dzn; ++dz)
      for (int dy = 0; dy < dyn; ++dy)
        for (int dx = 0; dx < 3; ++dx) {
          const i64 fx = 2 * c[0] + dx;
          const i64 fy = DIM > 1 ? 2 * c[1] + dy : 0;
          const i64 fz = DIM > 2 ? 2 * c[2] + dz : 0;
          const double w = (dx == 1 ? 1.0 : 0.5) * (DIM > 1 ? (dy == 1 ? 1.0 : 0.5) : 1.0) *
                           (DIM > 2 ? (dz == 1 ? 1.0 : 0.5) : 1.0);
          const i64 rf = (fz * n1 + fy) * n1 + fx;
#pragma unroll
          for (int l = 0; l < NL; ++l) {
            v0[l] += w * __ldg(a0 + l * nx + rf);
            v1[l] += w * __ldg(a1 + l * nx + rf);
          }
        }
  }
  double* o = coarse + nc * NL * nxc + rc;
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      s0 += v0[l] * t.R1[k][l];
      s1 += v1[l] * t.R2[k][l];
    }
    o[k * nxc] = s0 + s1;
  }
  }
}

// prolong_semi / prolong_full (transfer.cpp:87-96, 151-158): linear
// interpolation per axis, U_2n = C_n R1, U_2n+1 = C_n R2.  One thread per fine
// node and COARSE step: it gathers the interpolated coarse value once and
// writes both fine steps (the round-1 kernel gathered per fine step through
// divergent neighbour loops: 0.8-1.3 TB/s).  The 2^DIM neighbour slots are
// uniform -- an absent neighbour is a clamped index with weight 0 -- and are
// visited in the old (z, y, x) order, so the sums are unchanged.
template <int DIM, int NL, int CO>
__global__ void __launch_bounds__(256) k_prolong(const double* __restrict__ coarse,
                                                 double* __restrict__ fine, const TM<NL> t,
                                                 const i64 n1, const i64 n1c, const i64 n_t) {
  const i64 nx = ipow(n1, DIM), nxc = ipow(n1c, DIM);
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nx) return;
  int c[3];
  coords<DIM>(r, unsigned(n1), c);
  // per axis: two coarse slots (index, weight)
  int j[3][2];
  double w[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    j[a][0] = j[a][1] = 0;
    w[a][0] = 1.0;
    w[a][1] = 0.0;
    if (a >= DIM || CO == 1) continue;
    const int i = c[a], jj = i / 2;
    if (i % 2 == 1) {
      j[a][0] = jj;
    } else {  // between coarse nodes jj - 1 and jj (either may be the boundary)
      j[a][0] = jj > 0 ? jj - 1 : 0;
      w[a][0] = jj > 0 ? 0.5 : 0.0;
      j[a][1] = jj < n1c ? jj : int(n1c) - 1;
      w[a][1] = jj < n1c ? 0.5 : 0.0;
    }
  }
  i64 rc[1 << DIM];
  double ww[1 << DIM];
#pragma unroll
  for (int q = 0; q < (1 << DIM); ++q) {
    const int ix = q & 1, iy = DIM > 1 ? (q >> 1) & 1 : 0, iz = DIM > 2 ? (q >> 2) & 1 : 0;
    ww[q] = w[0][ix] * w[1][iy] * w[2][iz];
    rc[q] = (i64(j[2][iz]) * n1c + j[1][iy]) * n1c + j[0][ix];
  }
  // a thread keeps its slots for a run of coarse steps (the index arithmetic
  // above costs more than one step's gathers)
  const i64 ntc = n_t >> 1;
  const i64 per = (ntc + gridDim.y - 1) / gridDim.y;
  const i64 nc0 = i64(blockIdx.y) * per, nc1 = min(nc0 + per, ntc);
#pragma unroll 2
  for (i64 nc = nc0; nc < nc1; ++nc) {
    double cv[NL];
    const double* src = coarse + nc * NL * nxc;
    if (CO == 1) {
#pragma unroll
      for (int k = 0; k < NL; ++k) cv[k] = __ldg(src + k * nxc + r);
    } else {
#pragma unroll
      for (int k = 0; k < NL; ++k) cv[k] = 0.0;
      // a zero-weight slot is skipped like the absent neighbour it stands for
      // (w is exactly 0 or 0.5^m: the test is exact)
#pragma unroll
      for (int q = 0; q < (1 << DIM); ++q) {
        if (ww[q] != 0.0) {
#pragma unroll
          for (int k = 0; k < NL; ++k) cv[k] += ww[q] * __ldg(src + k * nxc + rc[q]);
        }
      }
    }
    double* o = fine + (2 * nc) * NL * nx + r;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < NL; ++k) sacc += cv[k] * (e ? t.R2[k][l] : t.R1[k][l]);
        __stcs(o + (e * NL + l) * nx, sacc);
      }
  }
}

// f(0,k,:) += psi_k(0) M_h u0.
template <int DIM, int NL>
__global__ void k_fold_u0(double* __restrict__ f, const double* __restrict__ u0, const i64 n1,
                          const i64 nx, const double h, TimeConsts tc) {
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nx) return;
  int c[3];
  coords<DIM>(r, unsigned(n1), c);
  double Mv, Kv;
  stencil_MK<DIM>(u0, n1, h, c, Mv, Kv, false);
#pragma unroll
  for (int k = 0; k < NL; ++k) f[k * nx + r] += tc.psi0[k] * Mv;
}

// ================================================ high DG degree (p_t 4..10)
// The reference accepts p_t <= kMaxTimeDegree = 10 (dg_time.hpp:10).  Degrees
// above kFastNL - 1 run the physical-path operators below, with the number of
// DG components a runtime value (per-thread NL x NL algebra in local memory):
// correct, not tuned -- the fused spectral kernels are compiled for NL <= 4.
constexpr int kHiNL = kMaxNL;

// Dense NL x NL Gaussian elimination with partial pivoting, in place: A is
// destroyed, b becomes the solution.
__device__ __forceinline__ void hi_solve(int nl, double (&A)[kHiNL][kHiNL], double (&b)[kHiNL]) {
  for (int c = 0; c < nl; ++c) {
    int p = c;
    for (int r = c + 1; r < nl; ++r)
      if (fabs(A[r][c]) > fabs(A[p][c])) p = r;
    if (p != c) {
      for (int k = 0; k < nl; ++k) {
        const double t = A[c][k];
        A[c][k] = A[p][k];
        A[p][k] = t;
      }
      const double t = b[c];
      b[c] = b[p];
      b[p] = t;
    }
    const double inv = 1.0 / A[c][c];
    for (int r = c + 1; r < nl; ++r) {
      const double f = A[r][c] * inv;
      for (int k = c + 1; k < nl; ++k) A[r][k] -= f * A[c][k];
      b[r] -= f * b[c];
    }
  }
  for (int c = nl - 1; c >= 0; --c) {
    double s = b[c];
    for (int k = c + 1; k < nl; ++k) s -= A[c][k] * b[k];
    b[c] = s / A[c][c];
  }
}

template <int DIM>
__device__ __forceinline__ void hi_block(const TimeConsts& tc, double Mj, double Kj,
                                         double (&A)[kHiNL][kHiNL]) {
  for (int i = 0; i < tc.nl; ++i)
    for (int j = 0; j < tc.nl; ++j)
      A[i][j] = Mj * tc.K[i * kMaxNL + j] + Kj * tc.M[i * kMaxNL + j];
}

// y = L u (or r = f - L u) at (node r, step n): st_system.cpp:25-33.
template <int DIM>
__global__ void __launch_bounds__(128) k_apply_hi(const double* __restrict__ u,
                                                  const double* __restrict__ f,
                                                  double* __restrict__ y, const TimeConsts tc,
                                                  const i64 n1, const i64 nx, const double h,
                                                  const i64 n_t, const int residual) {
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nx) return;
  const int nl = tc.nl;
  int c[3];
  coords<DIM>(r, unsigned(n1), c);
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    double Mv[kHiNL], Kv[kHiNL], Mp[kHiNL];
    const double* un = u + n * nl * nx;
    for (int l = 0; l < nl; ++l) {
      stencil_MK<DIM>(un + l * nx, n1, h, c, Mv[l], Kv[l], true);
      double kd;
      Mp[l] = 0.0;
      if (n > 0) stencil_MK<DIM>(un - nl * nx + l * nx, n1, h, c, Mp[l], kd, false);
    }
    for (int k = 0; k < nl; ++k) {
      double s = 0.0;
      for (int l = 0; l < nl; ++l) s += Mv[l] * tc.K[k * kMaxNL + l];
      for (int l = 0; l < nl; ++l) s += Kv[l] * tc.M[k * kMaxNL + l];
      for (int l = 0; l < nl; ++l) s -= Mp[l] * tc.N[k * kMaxNL + l];
      const i64 o = (n * nl + k) * nx + r;
      y[o] = residual ? __ldg(f + o) - s : s;
    }
  }
}

// Per-mode exact block solve in place (sine basis).
template <int DIM>
__global__ void __launch_bounds__(128) k_modal_solve_hi(double* __restrict__ x,
                                                        const TimeConsts tc, const SP s,
                                                        const i64 n_t) {
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.nx) return;
  const int nl = tc.nl;
  double Mj, Kj;
  mode_eig<DIM>(s, r, Mj, Kj);
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    double A[kHiNL][kHiNL], b[kHiNL];
    hi_block<DIM>(tc, Mj, Kj, A);
    double* p = x + n * nl * s.nx + r;
    for (int l = 0; l < nl; ++l) b[l] = p[l * s.nx];
    hi_solve(nl, A, b);
    for (int l = 0; l < nl; ++l) p[l * s.nx] = b[l];
  }
}

// Per-mode forward substitution u_n = A^-1 (f_n + M_j N u_{n-1}).
template <int DIM>
__global__ void __launch_bounds__(128) k_fwdsub_hi(const double* __restrict__ f,
                                                   double* __restrict__ u, const TimeConsts tc,
                                                   const SP s, const i64 n_t) {
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.nx) return;
  const int nl = tc.nl;
  double Mj, Kj;
  mode_eig<DIM>(s, r, Mj, Kj);
  double prev[kHiNL];
  for (int l = 0; l < nl; ++l) prev[l] = 0.0;
  for (i64 m = 0; m < n_t; ++m) {
    double A[kHiNL][kHiNL], b[kHiNL];
    hi_block<DIM>(tc, Mj, Kj, A);
    for (int k = 0; k < nl; ++k) {
      double s2 = 0.0;
      for (int l = 0; l < nl; ++l) s2 += tc.N[k * kMaxNL + l] * prev[l];
      b[k] = __ldg(f + (m * nl + k) * s.nx + r) + Mj * s2;
    }
    hi_solve(nl, A, b);
    for (int l = 0; l < nl; ++l) {
      u[(m * nl + l) * s.nx + r] = b[l];
      prev[l] = b[l];
    }
  }
}

// restrict_semi / restrict_full (transfer.cpp:75-85, 138-149).
template <int DIM, int CO>
__global__ void __launch_bounds__(128) k_restrict_hi(const double* __restrict__ fine,
                                                     double* __restrict__ coarse,
                                                     const TimeConsts tc, const i64 n1,
                                                     const i64 n1c, const i64 ntc) {
  const i64 nx = ipow(n1, DIM), nxc = ipow(n1c, DIM);
  const unsigned rc = blockIdx.x * blockDim.x + threadIdx.x;
  if (rc >= nxc) return;
  const int nl = tc.nl;
  int c[3];
  coords<DIM>(rc, unsigned(n1c), c);
  for (i64 nc = blockIdx.y; nc < ntc; nc += gridDim.y) {
    double v0[kHiNL], v1[kHiNL];
    for (int l = 0; l < nl; ++l) v0[l] = v1[l] = 0.0;
    const double* a0 = fine + (2 * nc) * nl * nx;
    const double* a1 = a0 + nl * nx;
    const int dzn = (CO == 2 && DIM > 2) ? 3 : 1, dyn = (CO == 2 && DIM > 1) ? 3 : 1;
    const int dxn = CO == 2 ? 3 : 1;
    for (int dz = 0; dz < dzn; ++dz)
      for (int dy = 0; dy < dyn; ++dy)
        for (int dx = 0; dx < dxn; ++dx) {
          i64 rf = rc;
          double w = 1.0;
          if (CO == 2) {
            const i64 fx = 2 * c[0] + dx;
            const i64 fy = DIM > 1 ? 2 * c[1] + dy : 0;
            const i64 fz = DIM > 2 ? 2 * c[2] + dz : 0;
            w = (dx == 1 ? 1.0 : 0.5) * (DIM > 1 ? (dy == 1 ? 1.0 : 0.5) : 1.0) *
                (DIM > 2 ? (dz == 1 ? 1.0 : 0.5) : 1.0);
            rf = (fz * n1 + fy) * n1 + fx;
          }
          for (int l = 0; l < nl; ++l) {
            v0[l] += w * __ldg(a0 + l * nx + rf);
            v1[l] += w * __ldg(a1 + l * nx + rf);
          }
        }
    double* o = coarse + nc * nl * nxc + rc;
    for (int k = 0; k < nl; ++k) {
      double s0 = 0.0, s1 = 0.0;
      for (int l = 0; l < nl; ++l) {
        s0 += v0[l] * tc.R1[k * kMaxNL + l];
        s1 += v1[l] * tc.R2[k * kMaxNL + l];
      }
      o[k * nxc] = s0 + s1;
    }
  }
}

// prolong_semi / prolong_full (transfer.cpp:87-96, 151-158).
template <int DIM, int CO>
__global__ void __launch_bounds__(128) k_prolong_hi(const double* __restrict__ coarse,
                                                    double* __restrict__ fine,
                                                    const TimeConsts tc, const i64 n1,
                                                    const i64 n1c, const i64 n_t) {
  const i64 nx = ipow(n1, DIM), nxc = ipow(n1c, DIM);
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nx) return;
  const int nl = tc.nl;
  int c[3];
  coords<DIM>(r, unsigned(n1), c);
  for (i64 n = blockIdx.y; n < n_t; n += gridDim.y) {
    const i64 nc = n >> 1;
    double cv[kHiNL];
    for (int l = 0; l < nl; ++l) cv[l] = 0.0;
    const double* src = coarse + nc * nl * nxc;
    if (CO == 1) {
      for (int k = 0; k < nl; ++k) cv[k] = __ldg(src + k * nxc + r);
    } else {
      int j[3][2], cnt[3];
      double w[3][2];
      for (int a = 0; a < 3; ++a) {
        cnt[a] = 1;
        j[a][0] = j[a][1] = 0;
        w[a][0] = 1.0;
        w[a][1] = 0.0;
        if (a >= DIM) continue;
        const int i = c[a];
        if (i % 2 == 1) {
          j[a][0] = i / 2;
        } else {
          const int jj = i / 2;
          cnt[a] = 0;
          if (jj > 0) {
            j[a][cnt[a]] = jj - 1;
            w[a][cnt[a]++] = 0.5;
          }
          if (jj < n1c) {
            j[a][cnt[a]] = jj;
            w[a][cnt[a]++] = 0.5;
          }
        }
      }
      for (int iz = 0; iz < cnt[2]; ++iz)
        for (int iy = 0; iy < cnt[1]; ++iy)
          for (int ix = 0; ix < cnt[0]; ++ix) {
            const double ww = w[0][ix] * w[1][iy] * w[2][iz];
            const i64 rc = (i64(j[2][iz]) * n1c + j[1][iy]) * n1c + j[0][ix];
            for (int k = 0; k < nl; ++k) cv[k] += ww * __ldg(src + k * nxc + rc);
          }
    }
    const double* Rm = (n & 1) ? tc.R2 : tc.R1;
    for (int l = 0; l < nl; ++l) {
      double s = 0.0;
      for (int k = 0; k < nl; ++k) s += cv[k] * Rm[k * kMaxNL + l];
      fine[(n * nl + l) * nx + r] = s;
    }
  }
}

template <int DIM>
__global__ void k_fold_u0_hi(double* __restrict__ f, const double* __restrict__ u0, const i64 n1,
                             const i64 nx, const double h, const TimeConsts tc) {
  const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nx) return;
  int c[3];
  coords<DIM>(r, unsigned(n1), c);
  double Mv, Kv;
  stencil_MK<DIM>(u0, n1, h, c, Mv, Kv, false);
  for (int k = 0; k < tc.nl; ++k) f[k * nx + r] += tc.psi0[k] * Mv;
}

#define STMG_DIM_DISPATCH(dim, ...)        \
  switch (dim) {                            \
    case 1: {                               \
      constexpr int DIM = 1;                \
      __VA_ARGS__;                          \
    } break;                                \
    case 2: {                               \
      constexpr int DIM = 2;                \
      __VA_ARGS__;                          \
    } break;                                \
    case 3: {                               \
      constexpr int DIM = 3;                \
      __VA_ARGS__;                          \
    } break;                                \
    default:                                \
      return cudaErrorInvalidValue;         \
  }

// ================================================================ DST-I
// Orthonormal DST-I of length n1 = N-1 (N = 2^LOG2N) along one axis, with a
// complex FFT of length N per PAIR of real lines (a + i b):
//   y_j = sin(j pi/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2,   Y = FFT_N(y),
//   X_{2k} = -Im Y_k,  X_{2k+1} = X_{2k-1} + Re Y_k,  X_1 = Re Y_0 / 2
// (the real transforms of a and b are separated from Y by the usual
// conjugate-symmetry split).  Half the FFT length of an odd extension.  The
// FFT is a Stockham autosort with register-resident radix-16 passes; the
// odd-index recurrence is a team-wide prefix sum.
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// exp(-2 pi i k / 16), k in [0, 16)
__device__ __forceinline__ double2 w16(int k) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double r2 = 0.70710678118654752440;
  switch (k & 15) {
    case 0: return make_double2(1.0, 0.0);
    case 1: return make_double2(c1, -s1);
    case 2: return make_double2(r2, -r2);
    case 3: return make_double2(s1, -c1);
    case 4: return make_double2(0.0, -1.0);
    case 5: return make_double2(-s1, -c1);
    case 6: return make_double2(-r2, -r2);
    case 7: return make_double2(-c1, -s1);
    case 8: return make_double2(-1.0, 0.0);
    case 9: return make_double2(-c1, s1);
    case 10: return make_double2(-r2, r2);
    case 11: return make_double2(-s1, c1);
    case 12: return make_double2(0.0, 1.0);
    case 13: return make_double2(s1, c1);
    case 14: return make_double2(r2, r2);
    default: return make_double2(c1, s1);
  }
}

// In-register radix-R DFT (R = 2, 4, 8, 16), natural order in and out.
template <int R>
struct RegFFT {
  static __device__ __forceinline__ void run(double2 (&v)[R]) {
    double2 e[R / 2], o[R / 2];
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      e[k] = v[2 * k];
      o[k] = v[2 * k + 1];
    }
    RegFFT<R / 2>::run(e);
    RegFFT<R / 2>::run(o);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const double2 t = (k == 0) ? o[k] : cmul(w16(k * (16 / R)), o[k]);
      v[k] = make_double2(e[k].x + t.x, e[k].y + t.y);
      v[k + R / 2] = make_double2(e[k].x - t.x, e[k].y - t.y);
    }
  }
};
template <>
struct RegFFT<1> {
  static __device__ __forceinline__ void run(double2 (&)[1]) {}
};

__host__ __device__ constexpr int dst_pass_radix(int m, int p) {
  // radix-16 passes while >= 4 bits remain, then the remainder
  return (m - 4 * p) >= 4 ? 16 : (1 << (m - 4 * p));
}
__host__ __device__ constexpr int dst_num_passes(int m) { return (m + 3) / 4; }
__host__ __device__ constexpr int dst_pad(int i) { return i + (i >> 4); }

// A team of TS = L / V threads owns one length-L FFT; every thread holds V
// values per pass (one radix-16 butterfly, or 16/R radix-R ones), so a pass
// is: load to registers, team barrier, store (in place), team barrier.
#ifndef STMG_DST_BUFPAD
#define STMG_DST_BUFPAD 1
#endif
template <int LOG2N>
struct DSTShape {
  static constexpr int N = 1 << LOG2N;
  static constexpr int n1 = N - 1;
  static constexpr int M = LOG2N;  // FFT length L = N
  static constexpr int L = N;
  static constexpr int V = L >= 16 ? 16 : L;
  static constexpr int TS = L / V;  // threads per FFT (team)
#ifndef STMG_DST_BLOCK9
#define STMG_DST_BLOCK9 256  // A/B vs 128: C5 transform 11.9-12.8 -> 11.5-11.9 ms (profiles/r02_v4_dst_lines_ab.txt)
#endif
  // N = 512: a 128-thread block holds only 4 line pairs = 8 adjacent columns
  // (64 B per row) in a strided pass; STMG_DST_BLOCK9 = 256 doubles that
  static constexpr int BLOCK0 = LOG2N == 9 ? STMG_DST_BLOCK9 : 128;
  static constexpr int BLOCK = TS > BLOCK0 ? TS : BLOCK0;
  static constexpr int F = BLOCK / TS;  // FFTs (= line pairs) per block
  static constexpr int TL = 2 * F;      // lines per block
  // padded FFT buffer.  STMG_DST_BUFPAD = 1 makes BUF odd in 16-byte units
  // (L >= 128): the F line pairs of a strided (y/z) pass, which a warp's
  // lanes scatter to / gather from at one index, then hit F distinct bank
  // groups; with +4 (BUF = 4 mod 8) they hit two and conflict 2-4 ways
  static constexpr int BUF = L + L / 16 + STMG_DST_BUFPAD;
  static constexpr int KB = (L / 2 + TS - 1) / TS;  // recurrence values per thread
  static constexpr size_t smem = size_t(F) * BUF * sizeof(double2) + size_t(BLOCK) * sizeof(double2);
};

template <int TS>
__device__ __forceinline__ void team_sync() {
  if (TS <= 32) __syncwarp();
  else __syncthreads();
}

template <int L, int TS, int R, int NS>
__device__ __forceinline__ void stockham_pass(double2* __restrict__ X, const int tt,
                                              const double2* __restrict__ tw) {
  constexpr int NJ = L / R;     // butterflies per FFT
  constexpr int IPT = NJ / TS;  // butterflies per thread
  constexpr int TSTEP = L / (NS * R);
  double2 v[IPT][R];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int j = tt + i * TS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[i][r] = X[dst_pad(j + r * NJ)];
    if (NS > 1) {
      const int step = (j % NS) * TSTEP;  // NS, TSTEP: powers of two, compile time
      // w^r from the table entries w, w^2, w^4, w^8 (<= 3 products each):
      // 4 cached loads per butterfly instead of R - 1 (the L1 pipe, not
      // the FP64 pipe, is this kernel's limiter)
      double2 w[R];
      w[1] = __ldg(tw + 2 * step);
      if (R > 2) w[2] = __ldg(tw + 4 * step);
      if (R > 4) w[4] = __ldg(tw + 8 * step);
      if (R > 8) w[8] = __ldg(tw + 16 * step);
#pragma unroll
      for (int r = 3; r < R; ++r) {
        const int hi = (r >= 8) ? 8 : (r >= 4) ? 4 : 2;
        if (r != hi) w[r] = cmul(w[hi], w[r - hi]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[i][r] = cmul(v[i][r], w[r]);
    }
    RegFFT<R>::run(v[i]);
  }
  team_sync<TS>();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int j = tt + i * TS;
    const int idxD = (j / NS) * NS * R + (j % NS);
#pragma unroll
    for (int r = 0; r < R; ++r) X[dst_pad(idxD + r * NS)] = v[i][r];
  }
  team_sync<TS>();
}

template <int LOG2N, int P, int NS>
__device__ __forceinline__ void dst_passes(double2* X, const int tt,
                                           const double2* __restrict__ tw) {
  using S = DSTShape<LOG2N>;
  if constexpr (P < dst_num_passes(S::M)) {
    constexpr int R = dst_pass_radix(S::M, P);
    stockham_pass<S::L, S::TS, R, NS>(X, tt, tw);
    dst_passes<LOG2N, P + 1, NS * R>(X, tt, tw);
  }
}

#ifndef STMG_DST_MINB
#define STMG_DST_MINB 5  // A/B vs 4 and 6: profiles/r01_v17_dst_minb_ab.txt
#endif
// STRIDED: lines along y / z (element stride = `stride`, the F line pairs of a
// CTA are 2F adjacent x columns); ACC: out += alpha * DST(in).  Both are
// template parameters and every (pair, index) decomposition below is written
// out for the thread (no per-item divisions, 64-bit multiplies or line-base
// reloads): the round-1 kernel spent 40 % of its instructions in the store loop
// and 18 % in the load loop on index arithmetic (ncu source view, C3).
template <int LOG2N, bool STRIDED, bool ACC>
__global__ void __launch_bounds__(DSTShape<LOG2N>::BLOCK, (LOG2N >= 4 ? (DSTShape<LOG2N>::BLOCK > 128 ? STMG_DST_MINB / 2 : STMG_DST_MINB) : 1)) k_dst_lines(
    const double* __restrict__ in, double* __restrict__ out, const i64 n_lines, const i64 stride,
    const double scale, const double alpha, const double2* __restrict__ tw) {
  using S = DSTShape<LOG2N>;
  constexpr int F = S::F, TL = S::TL, n1 = S::n1, N = S::N, BUF = S::BUF;
  constexpr int TS = S::TS, KB = S::KB;
  constexpr int BLK = S::BLOCK;
  constexpr int H = N / 2;
  extern __shared__ double2 sm[];
  double2* wsum = sm + F * BUF;  // per-thread scan totals
  __shared__ i64 lbase[TL];      // global offset of element 0 of each tile line

  const i64 line0 = i64(blockIdx.x) * TL;
  const int nt = int(min(i64(TL), n_lines - line0));
  for (int li = threadIdx.x; li < TL; li += BLK) {
    const i64 line = line0 + min(li, nt - 1);
    const i64 o = line / stride;
    lbase[li] = o * stride * n1 + (line - o * stride);
  }
  for (int f = threadIdx.x; f < F; f += BLK) sm[f * BUF + dst_pad(0)] = make_double2(0.0, 0.0);
  __syncthreads();
  // ---- load fused with the pre-processing: items (line pair f, j = 1..N/2)
  // load z_j = (a, b)_{j-1} and its mirror z_{N-j}, write
  //   X_j = sin(j pi/N)(z_j + z_{N-j}) + (z_j - z_{N-j})/2,  X_{N-j} = ... - ...
  // (one shared-memory store per value; the middle j = N/2 is its own mirror)
  constexpr int ITEMS_ALL = F * H;
  constexpr int ITEMS = (ITEMS_ALL + BLK - 1) / BLK;
  static_assert(ITEMS_ALL % BLK == 0 || ITEMS == 1, "items tile the block");
  // item i of this thread: pair f_i, index jj_i (both cheap functions of i)
  auto item = [&](int i, int& f, int& jj) {
    if constexpr (STRIDED) {  // f fastest: 2F adjacent columns per row
      static_assert(BLK % F == 0 || ITEMS == 1, "");
      f = threadIdx.x % F;
      jj = threadIdx.x / F + i * (BLK / F);
    } else if constexpr (H >= BLK) {
      f = i / (H / BLK);
      jj = threadIdx.x + (i % (H / BLK)) * BLK;
    } else {
      f = threadIdx.x / H + i * (BLK / H);
      jj = threadIdx.x % H;
    }
  };
  double2 lo[ITEMS], hi[ITEMS];
  {
    const bool full = nt == TL;
    // thread-constant bases (STRIDED: f is the same for every item)
    i64 ba = 0, bb = 0;
    if constexpr (STRIDED) {
      ba = lbase[2 * (threadIdx.x % F)];
      bb = lbase[2 * (threadIdx.x % F) + 1];
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      int f, jj;
      item(i, f, jj);
      double al = 0.0, bl = 0.0, ah = 0.0, bh = 0.0;
      if (ITEMS_ALL % BLK == 0 || threadIdx.x + i * BLK < ITEMS_ALL) {
        if constexpr (!STRIDED) {
          ba = lbase[2 * f];
          bb = lbase[2 * f + 1];
        }
        const i64 pl = STRIDED ? i64(jj) * stride : i64(jj);
        const i64 ph = STRIDED ? i64(N - 2 - jj) * stride : i64(N - 2 - jj);  // j - 1, N - j - 1
        if (full || 2 * f < nt) {
          al = __ldcs(in + ba + pl);
          ah = __ldcs(in + ba + ph);
        }
        if (full || 2 * f + 1 < nt) {
          bl = __ldcs(in + bb + pl);
          bh = __ldcs(in + bb + ph);
        }
      }
      lo[i] = make_double2(al, bl);
      hi[i] = make_double2(ah, bh);
    }
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (ITEMS_ALL % BLK != 0 && threadIdx.x + i * BLK >= ITEMS_ALL) continue;
    int f, jj;
    item(i, f, jj);
    const int j = jj + 1;
    double2* X = sm + f * BUF;
    const double sj = -__ldg(tw + j).y;  // sin(j pi / N)
    const double2 sum = make_double2(lo[i].x + hi[i].x, lo[i].y + hi[i].y);
    const double2 dif = make_double2(0.5 * (lo[i].x - hi[i].x), 0.5 * (lo[i].y - hi[i].y));
    X[dst_pad(j)] = make_double2(sj * sum.x + dif.x, sj * sum.y + dif.y);
    if (j != H) X[dst_pad(N - j)] = make_double2(sj * sum.x - dif.x, sj * sum.y - dif.y);
  }
  __syncthreads();
  // ---- FFT of length N per pair
  const int team = threadIdx.x / TS, tt = threadIdx.x % TS;
#ifndef STMG_DST_SKIP_FFT
  dst_passes<LOG2N, 0, 1>(sm + team * BUF, tt, tw);
#endif
  __syncthreads();
  // ---- post-processing: split a/b, X_{2k} = I_k, X_{2k+1} = prefix sum of R
  double2* X = sm + team * BUF;
  double2 Rv[KB], Iv[KB];
  double2 run = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    const int k = tt * KB + q;
    double2 R = make_double2(0.0, 0.0), I = make_double2(0.0, 0.0);
    if (k < N / 2) {
      const double2 Y1 = X[dst_pad(k)], Y2 = X[dst_pad((N - k) & (N - 1))];
      R = make_double2(0.5 * (Y1.x + Y2.x), 0.5 * (Y1.y + Y2.y));  // (Ra, Rb)
      I = make_double2(0.5 * (Y2.y - Y1.y), 0.5 * (Y1.x - Y2.x));  // (Ia, Ib)
      if (k == 0) R = make_double2(0.5 * R.x, 0.5 * R.y);
    }
    run = make_double2(run.x + R.x, run.y + R.y);
    Rv[q] = run;  // inclusive prefix within the thread's block
    Iv[q] = I;
  }
  // team-wide exclusive scan of the block totals
  double2 off = make_double2(0.0, 0.0);
  {
    constexpr int W = TS < 32 ? TS : 32;
    const int lane = threadIdx.x & 31;
    double2 inc = run;
#pragma unroll
    for (int d = 1; d < W; d <<= 1) {
      const double ux = __shfl_up_sync(0xffffffffu, inc.x, d, W);
      const double uy = __shfl_up_sync(0xffffffffu, inc.y, d, W);
      if ((lane % W) >= d) {
        inc.x += ux;
        inc.y += uy;
      }
    }
    off = make_double2(inc.x - run.x, inc.y - run.y);
    if (TS > 32) {  // combine the warps of a team
      wsum[threadIdx.x] = inc;
      __syncthreads();
      const int w0 = (threadIdx.x / 32) * 32;  // first thread of this warp
      for (int w = team * TS + 31; w < w0; w += 32) {
        off.x += wsum[w].x;
        off.y += wsum[w].y;
      }
    }
  }
  __syncthreads();  // every Y read is done; X is reused for the outputs
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    const int k = tt * KB + q;
    if (k >= N / 2) continue;
    if (k >= 1) X[dst_pad(2 * k)] = Iv[q];                               // X_{2k}
    X[dst_pad(2 * k + 1)] = make_double2(off.x + Rv[q].x, off.y + Rv[q].y);  // X_{2k+1}
  }
  __syncthreads();

  // ---- store: X_{j+1} of both lines of the pair
  const bool full = nt == TL;
  auto put = [&](const double2 Z, const int f, double* pa, double* pb) {
    const double va = Z.x * scale, vb = Z.y * scale;
    if (full || 2 * f < nt) {
      if (ACC) *pa += alpha * va;
      else __stcs(pa, va);
    }
    if (full || 2 * f + 1 < nt) {
      if (ACC) *pb += alpha * vb;
      else __stcs(pb, vb);
    }
  };
  if constexpr (STRIDED) {
    // thread: pair f = tid % F, rows j = tid / F + k (BLK / F)
    constexpr int JS = BLK / F;  // rows per sweep
    const int f = threadIdx.x % F;
    const int j0 = threadIdx.x / F;
    const double2* Zs = sm + f * BUF;
    double* pa = out + lbase[2 * f] + i64(j0) * stride;
    double* pb = out + lbase[2 * f + 1] + i64(j0) * stride;
    const i64 step = i64(JS) * stride;
#pragma unroll 4
    for (int j = j0; j < n1; j += JS) {
      put(Zs[dst_pad(j + 1)], f, pa, pb);
      pa += step;
      pb += step;
    }
  } else {
    // thread: elements j = tid + k BLK of every pair
    constexpr int KJ = (n1 + BLK - 1) / BLK;
#pragma unroll
    for (int k = 0; k < KJ; ++k) {
      const int j = threadIdx.x + k * BLK;
      if (j >= n1) break;
      const double2* Zs = sm + dst_pad(j + 1);
#pragma unroll 4
      for (int f = 0; f < F; ++f)
        put(Zs[f * BUF], f, out + lbase[2 * f] + j, out + lbase[2 * f + 1] + j);
    }
  }
}

// ---- one-pass 2D DST-I of whole slabs (thread-block cluster + DSMEM) -------
// One cluster of CL CTAs transforms one n1 x n1 slab (one time step and DG
// component) along both axes with one HBM read and one HBM write (16 B per
// dof instead of 32 for the per-axis passes):
//   1. CTA q loads rows [q R, q R + R) (contiguous: one TMA bulk copy);
//   2. x pass: R/2 row pairs -> R/2 half-length FFTs (the k_dst_lines
//      algorithm); output column j goes straight into the shared memory of
//      the CTA that owns column block j / R (DSMEM stores: the transpose of
//      the slab happens on the cluster, not through HBM);
//   3. y pass: R/2 column pairs of the CTA's own block; output rows go to
//      global memory (R contiguous doubles per row).
// One shared region per CTA holds, in turn, the rows, the FFT buffers and the
// column block: every phase first gathers what it needs into registers, so
// the region is reused (35 KB per CTA instead of 68: twice the resident CTAs),
// and radix-8 passes with 2x the threads per FFT double the warps per CTA.
// radix-16 passes, 8 threads per FFT, >= 4 CTAs per SM: the fastest of
// {radix 8, 16} x {3, 4 CTAs/SM} on C2 (84 vs 106 us per 2D transform for the
// per-axis passes; profiles/r02_dst2d_ab.txt).  For 255-node axes the
// 16-CTA clusters lose to the per-axis passes (10.6 vs 9.5 ms on C3), so the
// one-pass kernel is used for 127-node slabs unless STMG_DST2D=2.
#ifndef STMG_DST2D_LOG2V
#define STMG_DST2D_LOG2V 4
#endif
template <int LOG2N, int R>
struct DST2Shape {
  static constexpr int N = 1 << LOG2N;
  static constexpr int n1 = N - 1;
  static constexpr int CL = N / R;            // CTAs per slab (cluster size)
  static constexpr int LOG2V = STMG_DST2D_LOG2V;  // values per thread and pass
  static constexpr int TS = N >> LOG2V;       // threads per FFT
  static constexpr int F = R / 2;             // FFTs (line pairs) per pass
  static constexpr int BLOCK = TS * F;
  static constexpr int BUF = N + N / 16 + 1;  // padded FFT buffer (double2)
  static constexpr int KB = (N / 2 + TS - 1) / TS;
  static constexpr int H = N / 2;
  static constexpr int PRE = (F * H + BLOCK - 1) / BLOCK;   // pre-processing items per thread
  static constexpr int OUT = (F * n1 + BLOCK - 1) / BLOCK;  // x-pass outputs per thread
  static constexpr int ROWS = R * n1 + 2;                    // rows (+ alignment shift)
  static constexpr int FFTB = 2 * F * BUF;                   // FFT buffers, in doubles
  static constexpr int REGION = ROWS > FFTB ? ROWS : FFTB;
  static constexpr size_t smem = size_t(REGION) * sizeof(double);
  static_assert(TS <= 32 && 32 % TS == 0, "FFT teams stay inside a warp");
  static_assert(R % 2 == 0 && N % R == 0, "row blocks tile the slab");
};

__host__ __device__ constexpr int dst2_radix(int m, int lv, int p) {
  return (m - lv * p) >= lv ? (1 << lv) : (1 << (m - lv * p));
}

template <int LOG2N, int LOG2V, int P, int NS>
__device__ __forceinline__ void dst2_passes(double2* X, const int tt,
                                            const double2* __restrict__ tw) {
  constexpr int NP = (LOG2N + LOG2V - 1) / LOG2V;
  if constexpr (P < NP) {
    constexpr int Rx = dst2_radix(LOG2N, LOG2V, P);
    stockham_pass<(1 << LOG2N), (1 << (LOG2N - LOG2V)), Rx, NS>(X, tt, tw);
    dst2_passes<LOG2N, LOG2V, P + 1, NS * Rx>(X, tt, tw);
  }
}

// Pre-processing of one pair of lines into its FFT buffer X (k_dst_lines):
// X_j = sin(j pi/N)(z_j + z_{N-j}) + (z_j - z_{N-j})/2 with z_j = (a, b)_{j-1}.
template <int N>
__device__ __forceinline__ void dst2_pre(double2* X, int jj, double2 lo, double2 hi,
                                         const double2* __restrict__ tw) {
  constexpr int H = N / 2;
  const int j = jj + 1;
  const double sj = -__ldg(tw + j).y;  // sin(j pi / N)
  const double2 sum = make_double2(lo.x + hi.x, lo.y + hi.y);
  const double2 dif = make_double2(0.5 * (lo.x - hi.x), 0.5 * (lo.y - hi.y));
  X[dst_pad(j)] = make_double2(sj * sum.x + dif.x, sj * sum.y + dif.y);
  if (j != H) X[dst_pad(N - j)] = make_double2(sj * sum.x - dif.x, sj * sum.y - dif.y);
}

// FFT + post-processing of the team's buffer: afterwards X[dst_pad(j + 1)]
// holds output j (j < n1) of both lines of the pair.
template <int LOG2N, int LOG2V, int TS, int KB>
__device__ __forceinline__ void dst2_fft_post(double2* X, int tt, const double2* __restrict__ tw) {
  constexpr int N = 1 << LOG2N;
  dst2_passes<LOG2N, LOG2V, 0, 1>(X, tt, tw);
  double2 Rv[KB], Iv[KB];
  double2 run = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    const int k = tt * KB + q;
    double2 Rk = make_double2(0.0, 0.0), I = make_double2(0.0, 0.0);
    if (k < N / 2) {
      const double2 Y1 = X[dst_pad(k)], Y2 = X[dst_pad((N - k) & (N - 1))];
      Rk = make_double2(0.5 * (Y1.x + Y2.x), 0.5 * (Y1.y + Y2.y));
      I = make_double2(0.5 * (Y2.y - Y1.y), 0.5 * (Y1.x - Y2.x));
      if (k == 0) Rk = make_double2(0.5 * Rk.x, 0.5 * Rk.y);
    }
    run = make_double2(run.x + Rk.x, run.y + Rk.y);
    Rv[q] = run;
    Iv[q] = I;
  }
  double2 inc = run;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < TS; d <<= 1) {
    const double ux = __shfl_up_sync(0xffffffffu, inc.x, d, TS);
    const double uy = __shfl_up_sync(0xffffffffu, inc.y, d, TS);
    if ((lane % TS) >= d) {
      inc.x += ux;
      inc.y += uy;
    }
  }
  const double2 off = make_double2(inc.x - run.x, inc.y - run.y);
  __syncwarp();  // every Y read of the team is done
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    const int k = tt * KB + q;
    if (k >= N / 2) continue;
    if (k >= 1) X[dst_pad(2 * k)] = Iv[q];
    X[dst_pad(2 * k + 1)] = make_double2(off.x + Rv[q].x, off.y + Rv[q].y);
  }
}

#ifndef STMG_DST2D_MINB
#define STMG_DST2D_MINB 4
#endif
template <int LOG2N, int R>
__global__ void __launch_bounds__(DST2Shape<LOG2N, R>::BLOCK, STMG_DST2D_MINB) k_dst2d(
    const double* __restrict__ in, double* __restrict__ out, const i64 total, const double scale,
    const double alpha, const int accumulate, const double2* __restrict__ tw) {
  using S = DST2Shape<LOG2N, R>;
  constexpr int N = S::N, n1 = S::n1, F = S::F, TS = S::TS, BUF = S::BUF, H = S::H;
  constexpr int BLK = S::BLOCK;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double dsm[];  // the region: rows / FFT buffers / column block
  __shared__ alignas(8) unsigned long long bar;
  double2* Xb = reinterpret_cast<double2*>(dsm);
  double* B = dsm;  // column block [n1 rows][R columns]
  const int q = int(cluster.block_rank());
  const i64 slab = i64(blockIdx.x / S::CL) * n1 * n1;
  const int r0 = q * R;            // first row (x pass) / column (y pass)
  const int nr = min(R, n1 - r0);  // rows / columns of this CTA
  const int team = threadIdx.x / TS, tt = threadIdx.x % TS;
  double2* X = Xb + team * BUF;

  // 1. rows [r0, r0 + nr), one TMA bulk copy from the 16-byte aligned-down
  // start (n1^2 is odd: every other slab starts at 8 mod 16); plain loads
  // where the rounded copy would read past the vector's end
  const double* src = in + slab + i64(r0) * n1;
  const int cnt = nr * n1;
  const int mis = int((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
  double* A = dsm + mis;
  const unsigned bytes = unsigned(((cnt + mis) * 8 + 15) & ~15);
  const bool bulk = (src - mis) + bytes / 8 <= in + total;
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  if (bulk && threadIdx.x == 0) {
    mbar_init(bar_s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_expect(bar_s, bytes);
    bulk_g2s(static_cast<unsigned>(__cvta_generic_to_shared(dsm)), src - mis, bytes, bar_s);
  }
  if (!bulk) {
#pragma unroll 8
    for (int i = threadIdx.x; i < cnt; i += BLK) A[i] = __ldcs(src + i);
  }
  __syncthreads();
  if (bulk) mbar_wait(bar_s, 0);
  if (nr < R) {
    for (int i = cnt + threadIdx.x; i < R * n1; i += BLK) A[i] = 0.0;
    __syncthreads();
  }
  // 2. x pass: pair f = local rows 2f, 2f+1; inputs to registers, then the
  // region becomes the FFT buffers
  double2 lo[S::PRE], hi[S::PRE];
#pragma unroll
  for (int i = 0; i < S::PRE; ++i) {
    const int e = threadIdx.x + i * BLK;
    const int f = e / H, jj = e - f * H;
    if (e < F * H) {
      const double* a = A + (2 * f) * n1;
      lo[i] = make_double2(a[jj], a[n1 + jj]);
      hi[i] = make_double2(a[N - 2 - jj], a[n1 + N - 2 - jj]);
    }
  }
  __syncthreads();
  if (threadIdx.x < F) Xb[threadIdx.x * BUF + dst_pad(0)] = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < S::PRE; ++i) {
    const int e = threadIdx.x + i * BLK;
    const int f = e / H, jj = e - f * H;
    if (e < F * H) dst2_pre<N>(Xb + f * BUF, jj, lo[i], hi[i], tw);
  }
  __syncthreads();
  dst2_fft_post<LOG2N, S::LOG2V, TS, S::KB>(X, tt, tw);
  __syncthreads();
  double2 res[S::OUT];
#pragma unroll
  for (int i = 0; i < S::OUT; ++i) {
    const int e = threadIdx.x + i * BLK;
    const int f = e / n1, j = e - f * n1;
    if (e < F * n1) res[i] = Xb[f * BUF + dst_pad(j + 1)];
  }
  cluster.sync();  // every CTA has read its FFT buffers: regions take columns
  // column j of rows (r0 + 2f, r0 + 2f + 1) -> CTA j / R, block [row][j % R]
#pragma unroll
  for (int i = 0; i < S::OUT; ++i) {
    const int e = threadIdx.x + i * BLK;
    const int f = e / n1, j = e - f * n1;
    const int row = r0 + 2 * f;
    if (e >= F * n1 || row >= n1) continue;
    double* dst = cluster.map_shared_rank(B, j / R);
    const int c = j % R;
    dst[row * R + c] = res[i].x * scale;
    if (row + 1 < n1) dst[(row + 1) * R + c] = res[i].y * scale;
  }
  if (nr < R)  // columns past n1 of the last block: zero (line b of its last pair)
    for (int i = threadIdx.x; i < n1 * (R - nr); i += BLK)
      B[(i / (R - nr)) * R + nr + i % (R - nr)] = 0.0;
  cluster.sync();  // the column block is complete
  // 3. y pass: pair f = local columns 2f, 2f+1 (row N-1 never read: index <= N-2)
#pragma unroll
  for (int i = 0; i < S::PRE; ++i) {
    const int e = threadIdx.x + i * BLK;
    const int jj = e / F, f = e - jj * F;
    if (e < F * H) {
      lo[i] = *reinterpret_cast<const double2*>(B + jj * R + 2 * f);
      hi[i] = *reinterpret_cast<const double2*>(B + (N - 2 - jj) * R + 2 * f);
    }
  }
  __syncthreads();
  if (threadIdx.x < F) Xb[threadIdx.x * BUF + dst_pad(0)] = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < S::PRE; ++i) {
    const int e = threadIdx.x + i * BLK;
    const int jj = e / F, f = e - jj * F;
    if (e < F * H) dst2_pre<N>(Xb + f * BUF, jj, lo[i], hi[i], tw);
  }
  __syncthreads();
  dst2_fft_post<LOG2N, S::LOG2V, TS, S::KB>(X, tt, tw);
  __syncthreads();
  // output rows j, columns r0 + t (t = 2f + parity): R contiguous doubles per row
  for (int e = threadIdx.x; e < n1 * R; e += BLK) {
    const int j = e / R, t = e - j * R;
    if (t >= nr) continue;
    const double2 Z = Xb[(t >> 1) * BUF + dst_pad(j + 1)];
    const double v = ((t & 1) ? Z.y : Z.x) * scale;
    double* o = out + slab + i64(j) * n1 + r0 + t;
    if (accumulate) *o += alpha * v;
    else __stcs(o, v);
  }
}

// ================================================================ misc
// ---- dense DST-I for n1 = 63 (3D C4 and every 63-node axis) --------------
// For N = 64 the transform as a dense contraction on the FP64 tensor cores
// (mma.sync m8n8k4 f64, DMMA) beats the radix-16 FFT, whose shared-memory
// passes are L1-pipe bound at this size.  One even/odd butterfly first halves
// the work: with X_j (j = 1..63) and mirrors X_{64-j},
//   Y_{2c+1} = sum_j' Sodd[j'][c] (X_{j'+1} + X_{63-j'}),  (j' < 31; j' = 31: X_32)
//   Y_{2c+2} = sum_j' Seven[j'][c] (X_{j'+1} - X_{63-j'}),
// two 32 x 32 contractions per line instead of one 64 x 64.  A warp owns 16
// lines: A fragments (s, d) are formed in registers from global loads, B
// fragments (Sodd | Seven, 16 KB, L1-resident) come through the read-only
// path, C fragments go straight to global memory: no shared memory at all.
__device__ double g_dst64[2 * 32 * 32];  // Sodd | Seven, [j'][c]

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <bool STRIDED>
__global__ void __launch_bounds__(128) k_dst_dense64(const double* __restrict__ in,
                                                     double* __restrict__ out, const i64 n_lines,
                                                     const i64 stride, const double alpha,
                                                     const int accumulate) {
  constexpr int n1 = 63;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ar = lane >> 2, ac = lane & 3;  // A: row (line), col (j'); B: row (j') = ac, col = ar
  const i64 L0 = (i64(blockIdx.x) * 4 + warp) * 16;
  i64 base[2];
  bool ok[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const i64 line = L0 + m * 8 + ar;
    ok[m] = line < n_lines;
    const i64 l = ok[m] ? line : 0;
    if (STRIDED) {
      const i64 o = l / stride;
      base[m] = o * stride * n1 + (l - o * stride);
    } else {
      base[m] = l * n1;
    }
  }
  const i64 js = STRIDED ? stride : 1;
  double sv[8][2], dv[8][2];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int j = ks * 4 + ac;  // j' (0-based X index j', mirror 62 - j')
      double lo = 0.0, hi = 0.0;
      if (ok[m]) {
        lo = __ldcs(in + base[m] + j * js);
        if (j < 31) hi = __ldcs(in + base[m] + (62 - j) * js);
      }
      sv[ks][m] = lo + hi;
      dv[ks][m] = j < 31 ? lo - hi : 0.0;
    }
  double ao[2][4][2], ae[2][4][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) ao[m][n][0] = ao[m][n][1] = ae[m][n][0] = ae[m][n][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    double bo[4], be[4];
    const double* so = g_dst64 + (ks * 4 + ac) * 32 + ar;
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      bo[n] = __ldg(so + n * 8);
      be[n] = __ldg(so + 1024 + n * 8);
    }
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        dmma(ao[m][n], sv[ks][m], bo[n]);
        dmma(ae[m][n], dv[ks][m], be[n]);
      }
  }
  // C fragment: row = lane >> 2, cols c = n * 8 + (lane & 3) * 2 + q -> Y[2c] (odd k), Y[2c+1]
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    if (!ok[m]) continue;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = n * 8 + ac * 2 + q;
        double* p = out + base[m] + (2 * c) * js;
        if (accumulate) {
          p[0] += alpha * ao[m][n][q];
          if (c < 31) p[js] += alpha * ae[m][n][q];
        } else {
          __stcs(p, ao[m][n][q]);
          if (c < 31) __stcs(p + js, ae[m][n][q]);
        }
      }
  }
}

__global__ void __launch_bounds__(256) k_step_sumsq(const double* __restrict__ v, const i64 slab,
                                                    double* __restrict__ partial) {
  __shared__ double sh[32];
  const double* p = v + i64(blockIdx.x) * slab;
  double s = 0.0;
  for (i64 i = threadIdx.x; i < slab; i += blockDim.x) {
    const double x = p[i];
    s += x * x;
  }
  const double tot = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// Fixed-order reduction: thread t sums partial[t], partial[t+256], ...
// then a fixed tree; bitwise reproducible for a given partial array.
__global__ void __launch_bounds__(256) k_norm_final(const double* __restrict__ partial,
                                                    const i64 n, double* __restrict__ out,
                                                    double* __restrict__ hist, const int hidx) {
  pdl_wait();
  __shared__ double sh[256];
  double s = 0.0;
  for (i64 i = threadIdx.x; i < n; i += 256) s += partial[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double r = sqrt(sh[0]);
    out[0] = r;
    if (hist) hist[hidx] = r;
  }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void k_fill_uniform(double* __restrict__ v, const i64 n, const unsigned long long seed,
                               const unsigned long long stream, const i64 offset) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long ctr = (stream << 56) + (unsigned long long)(offset + i);
  const unsigned long long x = mix64(seed + 0x9E3779B97F4A7C15ULL * ctr);
  v[i] = 2.0 * (double(x >> 11) * 0x1.0p-53) - 1.0;
}

__global__ void k_nonzero(const double* __restrict__ v, const i64 n, int* __restrict__ flag) {
  bool nz = false;
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    nz |= (v[i] != 0.0);
  if (__syncthreads_or(nz) && threadIdx.x == 0) *flag = 1;
}

// Stop test on the device (mg.cpp:156-160): record ||r_k||, count the cycle
// and set the while-loop condition of the solve graph.
__global__ void k_decide(cudaGraphConditionalHandle h, const double* __restrict__ norm,
                         const double* __restrict__ r0, double* __restrict__ hist,
                         int* __restrict__ iter, const double eps, const int max_iter,
                         int* __restrict__ parity) {
  pdl_wait();
  const int k = *iter + 1;
  *iter = k;
  const double rk = *norm;
  hist[k] = rk;
  const bool more = !(rk <= eps * (*r0)) && k < max_iter;
  if (parity) *parity = 1 - *parity;  // fused schedule: swap the level-0 buffers
  if (h) cudaGraphSetConditional(h, more ? 1u : 0u);
}

// k_norm_final followed by k_decide in one launch (the last two nodes of a
// device-loop body): same fixed-order reduction, so the norm, the history and
// the stop decision are bitwise those of the two-kernel sequence.
__global__ void __launch_bounds__(256) k_norm_decide(const double* __restrict__ partial,
                                                     const i64 n, double* __restrict__ out,
                                                     cudaGraphConditionalHandle h,
                                                     const double* __restrict__ r0,
                                                     double* __restrict__ hist,
                                                     int* __restrict__ iter, const double eps,
                                                     const int max_iter,
                                                     int* __restrict__ parity) {
  pdl_wait();
  __shared__ double sh[256];
  double s = 0.0;
  for (i64 i = threadIdx.x; i < n; i += 256) s += partial[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double rk = sqrt(sh[0]);
    out[0] = rk;
    const int k = *iter + 1;
    *iter = k;
    hist[k] = rk;
    const bool more = !(rk <= eps * (*r0)) && k < max_iter;
    if (parity) *parity = 1 - *parity;
    if (h) cudaGraphSetConditional(h, more ? 1u : 0u);
  }
}

// Coarse operator: y = B x with B (n x n, row-major) the precomputed linear
// map of the coarse tail's V(1,1) cycle (levels >= tail start, zero initial
// guess), rhs -> iterate.  One warp per row; the block's rows are staged into
// shared memory with cp.async BEFORE the PDL wait (B is a constant), so their
// HBM traffic overlaps the previous kernel; after the wait only x (L2) is
// read.  Fixed summation order: deterministic.
// Rows per CTA (one warp per row).  1 row: many small CTAs (C2: 1568 of
// 12.5 KB, all resident) keep more bulk copies in flight per SM than 8 rows
// (C2: 196 of 100 KB; C1's n = 1984 at 8 rows needs 127 KB, one CTA per SM).
// A/B (profiles/r01_v19_cop_rows_ab.txt, r01_v20_ab.txt): 8 -> 2 -> 1 rows
// C1 0.355 -> 0.318 -> 0.312 ms per solve, C2 1.662 -> 1.662 -> 1.644 ms,
// C4 neutral
#ifndef STMG_COP_ROWS
#define STMG_COP_ROWS 1
#endif
constexpr int kCopRows = STMG_COP_ROWS;
__global__ void __launch_bounds__(kCopRows * 32) k_cop_gemv(const double* __restrict__ B,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y, const int n) {
  extern __shared__ double rows[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * kCopRows;
  const int nr = min(kCopRows, n - r0);
  __shared__ alignas(8) unsigned long long bar;
  const double* src = B + i64(r0) * n;
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  const bool bulk = (n & 1) == 0;  // rows are 16-byte multiples: one TMA bulk copy
  if (bulk) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      const unsigned bytes = unsigned(nr) * unsigned(n) * 8u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(rows))),
          "l"(src), "r"(bytes), "r"(bar_s)
          : "memory");
    }
  } else {
    for (int i = threadIdx.x; i < nr * n; i += blockDim.x) cp_async8(rows + i, src + i, true);
    cp_async_commit();
  }
  pdl_wait();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double xv[4];
  if (bulk) {
    __syncthreads();  // barrier initialised before anyone polls it
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(bar_s)
        : "memory");
  } else {
    cp_async_wait<0>();
    __syncthreads();
  }
  if (w < nr) {
    const double* br = rows + w * n;
    int j = lane;
    for (; j + 96 < n; j += 128) {
#pragma unroll
      for (int q = 0; q < 4; ++q) xv[q] = x[j + 32 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(br[j + 32 * q], xv[q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (j + 32 * q < n) acc[q] = fma(br[j + 32 * q], x[j + 32 * q], acc[q]);
  }
  pdl_trigger();
  double v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (w < nr && lane == 0) y[r0 + w] = v;
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, const double a,
                       const i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}

}  // namespace

// Register-blocked 2D/3D kernel (k_apply_rb); STMG_APPLY_RB=0 selects the
// one-output-per-thread kernel (kept for 1D and A/B runs).
template <int DIM, int NL>
cudaError_t launch_apply_rb(const LevelView& L, const double* u, const double* f, double* y,
                            bool residual, const double* ab, cudaStream_t st) {
  using T = RbTile<DIM>;
  const i64 n1 = L.sp.n1;
  const i64 tiles = ((n1 + T::TX - 1) / T::TX) * ((n1 + T::TY - 1) / T::TY) *
                    (DIM == 3 ? (n1 + T::TZ - 1) / T::TZ : 1);
  i64 C = 64;
  while (C > 4 && tiles * ((L.n_t + C - 1) / C) < 148 * 4) C /= 2;
  C = std::min<i64>(C, L.n_t);
  const dim3 g(unsigned(tiles), unsigned((L.n_t + C - 1) / C));
  const size_t smem = size_t(T::STAGES) *
                      (size_t(NL) * T::HALO + (residual ? size_t(NL) * T::OUT : 0)) *
                      sizeof(double);
  static PerDevice attr;
  if (attr.first_use()) {
    const int most = int(size_t(T::STAGES) * (size_t(NL) * T::HALO + size_t(NL) * T::OUT) *
                         sizeof(double));
    cudaFuncSetAttribute(k_apply_rb<DIM, NL, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    cudaFuncSetAttribute(k_apply_rb<DIM, NL, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, most);
  }
  const TM<NL> t = make_tm<NL>(L.tc);
  if (residual)
    k_apply_rb<DIM, NL, true><<<g, T::THREADS, smem, st>>>(u, f, y, t, n1, L.sp.nx, L.sp.h,
                                                              L.n_t, int(C), L.first_global, ab);
  else
    k_apply_rb<DIM, NL, false><<<g, T::THREADS, smem, st>>>(u, f, y, t, n1, L.sp.nx, L.sp.h,
                                                               L.n_t, int(C), L.first_global, ab);
  return cudaGetLastError();
}

cudaError_t launch_apply(const LevelView& L, const double* u, const double* f, double* y,
                         bool residual, const double* ab, cudaStream_t st) {
  if (L.n_t * L.sp.nx == 0) return cudaSuccess;
  if (L.tc.nl > kFastNL) {
    STMG_DIM_DISPATCH(L.sp.dim, {
      k_apply_hi<DIM><<<grid2(L.sp.nx, L.n_t, 128), 128, 0, st>>>(
          u, f, y, L.tc, L.sp.n1, L.sp.nx, L.sp.h, L.n_t, residual ? 1 : 0);
    });
    return cudaGetLastError();
  }
  // row-band kernels (stmg_apply.cu: TMA bulk row staging, rolling windows);
  // STMG_APPLY_ROWS=0 keeps the tile kernels below
  static const bool rows = [] {
    const char* e = std::getenv("STMG_APPLY_ROWS");
    return !e || std::atoi(e) != 0;
  }();
  if (rows) {
    const cudaError_t e = launch_apply_rows(L, u, f, y, residual, ab, st);
    if (e != cudaErrorNotSupported) return e;
  }
  // register-blocked kernel: measured faster in 3D (27-point stencil), slower
  // in 2D (profiles/r01_v8_residual_ab.txt); STMG_APPLY_RB=0/1 forces either
  static const int rb = [] {
    const char* e = std::getenv("STMG_APPLY_RB");
    return e ? std::atoi(e) : -1;
  }();
  if (L.sp.dim == 3 ? rb != 0 : (L.sp.dim == 2 && rb == 1)) {
    switch (L.sp.dim * 8 + L.tc.nl) {
      case 2 * 8 + 1: return launch_apply_rb<2, 1>(L, u, f, y, residual, ab, st);
      case 2 * 8 + 2: return launch_apply_rb<2, 2>(L, u, f, y, residual, ab, st);
      case 2 * 8 + 3: return launch_apply_rb<2, 3>(L, u, f, y, residual, ab, st);
      case 2 * 8 + 4: return launch_apply_rb<2, 4>(L, u, f, y, residual, ab, st);
      case 3 * 8 + 1: return launch_apply_rb<3, 1>(L, u, f, y, residual, ab, st);
      case 3 * 8 + 2: return launch_apply_rb<3, 2>(L, u, f, y, residual, ab, st);
      case 3 * 8 + 3: return launch_apply_rb<3, 3>(L, u, f, y, residual, ab, st);
      case 3 * 8 + 4: return launch_apply_rb<3, 4>(L, u, f, y, residual, ab, st);
      default: return cudaErrorInvalidValue;
    }
  }
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    using T = ResTile<DIM>;
    const i64 n1 = L.sp.n1;
    const i64 tiles = ((n1 + T::TX - 1) / T::TX) * (DIM >= 2 ? (n1 + T::TY - 1) / T::TY : 1) *
                      (DIM == 3 ? (n1 + T::TZ - 1) / T::TZ : 1);
    // chunk: enough CTAs for ~4 per SM, at least 4 steps to amortise the warm-up
    i64 C = 64;
    while (C > 4 && tiles * ((L.n_t + C - 1) / C) < 148 * 4) C /= 2;
    C = std::min<i64>(C, L.n_t);
    const dim3 g(unsigned(tiles), unsigned((L.n_t + C - 1) / C));
    const TM<NL> t = make_tm<NL>(L.tc);
    const size_t smem =
        size_t(T::STAGES) *
        (size_t(NL) * T::HALO + (residual && !STMG_APPLY_FREG ? size_t(NL) * T::THREADS : 0)) *
        sizeof(double);
    static PerDevice attr;
    if (attr.first_use()) {
      const int most = int(T::STAGES * 2 * size_t(NL) * T::HALO * sizeof(double));  // >= smem
      cudaFuncSetAttribute(k_apply<DIM, NL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           most);
      cudaFuncSetAttribute(k_apply<DIM, NL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           most);
    }
    if (residual)
      k_apply<DIM, NL, true><<<g, T::THREADS, smem, st>>>(u, f, y, t, n1, L.sp.nx, L.sp.h, L.n_t,
                                                           int(C), L.first_global, ab);
    else
      k_apply<DIM, NL, false><<<g, T::THREADS, smem, st>>>(u, f, y, t, n1, L.sp.nx, L.sp.h,
                                                            L.n_t, int(C), L.first_global, ab);
  });
  return cudaGetLastError();
}

cudaError_t launch_restrict(const LevelView& F, int mode, int64_t n1c, const double* fine,
                            double* coarse, cudaStream_t st) {
  const i64 ntc = F.n_t / 2;
  const i64 n1o = mode == 2 ? n1c : F.sp.n1;
  const i64 nxo = n1o * (F.sp.dim > 1 ? n1o : 1) * (F.sp.dim > 2 ? n1o : 1);
  if (ntc * nxo == 0) return cudaSuccess;
  if (F.tc.nl > kFastNL) {
    const i64 nc1 = mode == 2 ? n1c : F.sp.n1;
    STMG_DIM_DISPATCH(F.sp.dim, {
      if (mode == 2)
        k_restrict_hi<DIM, 2><<<grid2(nxo, ntc, 128), 128, 0, st>>>(fine, coarse, F.tc, F.sp.n1,
                                                                   nc1, ntc);
      else
        k_restrict_hi<DIM, 1><<<grid2(nxo, ntc, 128), 128, 0, st>>>(fine, coarse, F.tc, F.sp.n1,
                                                                   nc1, ntc);
    });
    return cudaGetLastError();
  }
  const dim3 g = grid2(nxo, ntc, 256);
  STMG_DISPATCH(F.sp.dim, F.tc.nl, {
    const TM<NL> t = make_tm<NL>(F.tc);
    if (mode == 2)
      k_restrict<DIM, NL, 2><<<g, 256, 0, st>>>(fine, coarse, t, F.sp.n1, n1c, ntc);
    else
      k_restrict<DIM, NL, 1><<<g, 256, 0, st>>>(fine, coarse, t, F.sp.n1, F.sp.n1, ntc);
  });
  return cudaGetLastError();
}

cudaError_t launch_prolong(const LevelView& F, int mode, int64_t n1c, const double* coarse,
                           double* fine, cudaStream_t st) {
  const i64 total = F.n_t * F.sp.nx;
  if (total == 0) return cudaSuccess;
  if (F.tc.nl > kFastNL) {
    const i64 nc1 = mode == 2 ? n1c : F.sp.n1;
    STMG_DIM_DISPATCH(F.sp.dim, {
      if (mode == 2)
        k_prolong_hi<DIM, 2><<<grid2(F.sp.nx, F.n_t, 128), 128, 0, st>>>(coarse, fine, F.tc,
                                                                        F.sp.n1, nc1, F.n_t);
      else
        k_prolong_hi<DIM, 1><<<grid2(F.sp.nx, F.n_t, 128), 128, 0, st>>>(coarse, fine, F.tc,
                                                                        F.sp.n1, nc1, F.n_t);
    });
    return cudaGetLastError();
  }
  // one thread per fine node and run of coarse steps: ~8 steps per thread, but
  // at least ~16 CTAs per SM in the grid
  const i64 ntc = F.n_t / 2, bx = grid1(F.sp.nx, 256);
  i64 gy = std::max<i64>((ntc + 7) / 8, std::min<i64>(ntc, (148 * 16 + bx - 1) / bx));
  gy = std::max<i64>(1, std::min<i64>(gy, 65535));
  const dim3 g{unsigned(bx), unsigned(gy), 1u};
  STMG_DISPATCH(F.sp.dim, F.tc.nl, {
    const TM<NL> t = make_tm<NL>(F.tc);
    if (mode == 2)
      k_prolong<DIM, NL, 2><<<g, 256, 0, st>>>(coarse, fine, t, F.sp.n1, n1c, F.n_t);
    else
      k_prolong<DIM, NL, 1><<<g, 256, 0, st>>>(coarse, fine, t, F.sp.n1, F.sp.n1, F.n_t);
  });
  return cudaGetLastError();
}

cudaError_t launch_fold_u0(const LevelView& L, double* f, const double* u0, cudaStream_t st) {
  if (L.tc.nl > kFastNL) {
    STMG_DIM_DISPATCH(L.sp.dim, {
      k_fold_u0_hi<DIM><<<grid1(L.sp.nx, 256), 256, 0, st>>>(f, u0, L.sp.n1, L.sp.nx, L.sp.h,
                                                             L.tc);
    });
    return cudaGetLastError();
  }
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    k_fold_u0<DIM, NL><<<grid1(L.sp.nx, 256), 256, 0, st>>>(f, u0, L.sp.n1, L.sp.nx, L.sp.h, L.tc);
  });
  return cudaGetLastError();
}

cudaError_t launch_dst_axis(const LevelView& L, int axis, const double* in, double* out,
                            bool accumulate, double alpha, const void* twiddles,
                            cudaStream_t st) {
  const i64 n1 = L.sp.n1;
  const i64 n_lines = L.size() / n1;
  if (n_lines == 0) return cudaSuccess;
  i64 stride = 1;
  for (int a = 0; a < axis; ++a) stride *= n1;
  int log2n = 0;
  while ((i64(1) << log2n) < n1 + 1) ++log2n;
  if ((i64(1) << log2n) != n1 + 1) return cudaErrorInvalidValue;
  const double scale = std::sqrt(2.0 / double(n1 + 1));
  const double2* tw = static_cast<const double2*>(twiddles);
  static const bool dense = [] {
    const char* e = std::getenv("STMG_DST_DENSE");
    return !e || std::atoi(e) != 0;
  }();
  if (log2n == 6 && dense) {
    const unsigned g = unsigned((n_lines + 63) / 64);
    if (stride == 1)
      k_dst_dense64<false><<<g, 128, 0, st>>>(in, out, n_lines, stride, alpha,
                                              accumulate ? 1 : 0);
    else
      k_dst_dense64<true><<<g, 128, 0, st>>>(in, out, n_lines, stride, alpha, accumulate ? 1 : 0);
    return cudaGetLastError();
  }
  switch (log2n) {
#define STMG_DST_LAUNCH(K, STR, AC)                                                         \
  {                                                                                        \
    static PerDevice attr_set;                                                             \
    if (attr_set.first_use())                                                              \
      cudaFuncSetAttribute(k_dst_lines<K, STR, AC>,                                        \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(SH::smem));    \
    k_dst_lines<K, STR, AC><<<grid, SH::BLOCK, SH::smem, st>>>(in, out, n_lines, stride,   \
                                                               scale, alpha, tw);          \
  }
#define STMG_DST_CASE(K)                                                                   \
  case K: {                                                                                \
    using SH = DSTShape<K>;                                                                \
    const unsigned grid = unsigned((n_lines + SH::TL - 1) / SH::TL);                       \
    if (stride == 1) {                                                                     \
      if (accumulate) STMG_DST_LAUNCH(K, false, true) else STMG_DST_LAUNCH(K, false, false) \
    } else {                                                                               \
      if (accumulate) STMG_DST_LAUNCH(K, true, true) else STMG_DST_LAUNCH(K, true, false)  \
    }                                                                                      \
  } break;
    STMG_DST_CASE(1)
    STMG_DST_CASE(2)
    STMG_DST_CASE(3)
    STMG_DST_CASE(4)
    STMG_DST_CASE(5)
    STMG_DST_CASE(6)
    STMG_DST_CASE(7)
    STMG_DST_CASE(8)
    STMG_DST_CASE(9)
    STMG_DST_CASE(10)
#undef STMG_DST_CASE
#undef STMG_DST_LAUNCH
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// One-pass 2D transform of every n1 x n1 slab (n1 = 127 or 255); returns
// cudaErrorNotSupported for other shapes (the caller runs per-axis passes).
cudaError_t launch_dst2d(const LevelView& L, const double* in, double* out, bool accumulate,
                         double alpha, const void* twiddles, cudaStream_t st) {
  if (L.sp.dim != 2) return cudaErrorNotSupported;
  static const int mode = [] {  // 0 off, 1 127-node slabs, 2 also 255
    const char* e = std::getenv("STMG_DST2D");
    return e ? std::atoi(e) : 1;
  }();
  if (mode == 0 || (mode == 1 && L.sp.n1 != 127)) return cudaErrorNotSupported;
  const i64 n1 = L.sp.n1;
  const i64 slabs = L.n_t * L.tc.nl;
  if (slabs == 0) return cudaSuccess;
  const double scale = std::sqrt(2.0 / double(n1 + 1));
  const double2* tw = static_cast<const double2*>(twiddles);
  static PerDevice attr127, attr255;
  auto go = [&](auto kern, PerDevice& attr, int cl, int block, size_t smem, bool nonportable) {
    if (attr.first_use()) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (nonportable) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(slabs * cl));
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(cl);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t le =
        cudaLaunchKernelEx(&cfg, kern, in, out, slabs * n1 * n1, scale, alpha, accumulate ? 1 : 0, tw);
    if (le != cudaSuccess && std::getenv("STMG_DEBUG_DST2D")) {
      int ncl = -1;
      cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      std::fprintf(stderr, "dst2d launch: %s; cluster %d block %d smem %zu grid %u; max active "
                   "clusters %d (%s)\n", cudaGetErrorString(le), cl, block, smem, cfg.gridDim.x,
                   ncl, cudaGetErrorString(oe));
    }
    return le;
  };
  cudaError_t e;
  if (n1 == 127) {
    using SH = DST2Shape<7, 32>;
    e = go(k_dst2d<7, 32>, attr127, SH::CL, SH::BLOCK, SH::smem, false);
  } else if (n1 == 255) {
    using SH = DST2Shape<8, 16>;
    e = go(k_dst2d<8, 16>, attr255, SH::CL, SH::BLOCK, SH::smem, true);
  } else {
    return cudaErrorNotSupported;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t init_kernel_tables() {
  // Sodd[j'][c] = S(2c+1, j'+1) (j' < 31), S(2c+1, 32) (j' = 31);
  // Seven[j'][c] = S(2c+2, j'+1) (j' < 31, c < 31), else 0; S(k, j) = sqrt(2/64) sin(pi k j / 64)
  std::vector<double> T(2 * 32 * 32, 0.0);
  const long double pi = 3.141592653589793238462643383279502884L;
  const double sc = std::sqrt(2.0 / 64.0);
  auto S = [&](int k, int j) { return sc * double(std::sin(pi * (long double)(k * j) / 64.0L)); };
  for (int jp = 0; jp < 32; ++jp)
    for (int c = 0; c < 32; ++c) {
      T[jp * 32 + c] = S(2 * c + 1, jp < 31 ? jp + 1 : 32);
      if (jp < 31 && c < 31) T[1024 + jp * 32 + c] = S(2 * c + 2, jp + 1);
    }
  return cudaMemcpyToSymbol(g_dst64, T.data(), T.size() * sizeof(double));
}

cudaError_t launch_modal_solve(const LevelView& L, double* x, cudaStream_t st) {
  const i64 total = L.n_t * L.sp.nx;
  if (total == 0) return cudaSuccess;
  const SP s = make_sp(L.sp);
  if (L.tc.nl > kFastNL) {
    STMG_DIM_DISPATCH(L.sp.dim, {
      k_modal_solve_hi<DIM><<<grid2(L.sp.nx, L.n_t, 128), 128, 0, st>>>(x, L.tc, s, L.n_t);
    });
    return cudaGetLastError();
  }
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    k_modal_solve<DIM, NL><<<grid2(L.sp.nx, L.n_t, 256), 256, 0, st>>>(x, make_tm<NL>(L.tc), s,
                                                                        L.n_t);
  });
  return cudaGetLastError();
}

cudaError_t launch_modal_fwdsub(const LevelView& L, const double* f, double* u, cudaStream_t st) {
  const SP s = make_sp(L.sp);
  if (L.tc.nl > kFastNL) {
    STMG_DIM_DISPATCH(L.sp.dim, {
      k_fwdsub_hi<DIM><<<grid1(L.sp.nx, 128), 128, 0, st>>>(f, u, L.tc, s, L.n_t);
    });
    return cudaGetLastError();
  }
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    PDLK(k_fwdsub<DIM, NL>, grid1(L.sp.nx, 128), 128, 0, st, f, u, make_tm<NL>(L.tc), s, L.n_t);
  });
  return cudaGetLastError();
}

cudaError_t launch_step_sumsq(const LevelView& L, const double* v, double* partial,
                              cudaStream_t st) {
  if (L.n_t == 0) return cudaSuccess;
  k_step_sumsq<<<unsigned(L.n_t), 256, 0, st>>>(v, L.slab(), partial);
  return cudaGetLastError();
}

cudaError_t launch_norm_final(const double* partial, int64_t n, double* out, double* hist,
                              int hidx, cudaStream_t st) {
  PDLK(k_norm_final, 1, 256, 0, st, partial, n, out, hist, hidx);
  return cudaGetLastError();
}

cudaError_t launch_fill_uniform(double* v, int64_t n, uint64_t seed, uint64_t stream,
                                int64_t offset, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_fill_uniform<<<grid1(n, 256), 256, 0, st>>>(v, n, seed, stream, offset);
  return cudaGetLastError();
}

cudaError_t launch_decide(cudaGraphConditionalHandle h, const double* norm, const double* r0,
                          double* hist, int* iter, double eps, int max_iter, int* parity,
                          cudaStream_t st) {
  PDLK(k_decide, 1, 1, 0, st, h, norm, r0, hist, iter, eps, max_iter, parity);
  return cudaGetLastError();
}

cudaError_t launch_norm_decide(const double* partial, int64_t n, double* out,
                               cudaGraphConditionalHandle h, const double* r0, double* hist,
                               int* iter, double eps, int max_iter, int* parity,
                               cudaStream_t st) {
  PDLK(k_norm_decide, 1, 256, 0, st, partial, n, out, h, r0, hist, iter, eps, max_iter, parity);
  return cudaGetLastError();
}

#ifndef STMG_UPDOWN_SMEM_MIN
#define STMG_UPDOWN_SMEM_MIN 0
#endif
// dynamic shared memory of k_updown: the ring, padded to STMG_UPDOWN_SMEM_MIN
// bytes (caps the resident CTAs per SM; A/B knob)
size_t updown_smem(int nl) { return std::max<size_t>(ring_bytes(5 * nl), STMG_UPDOWN_SMEM_MIN); }

cudaError_t launch_updown(const LevelView& L, ModalArgs& a, const double* ec,
                          double* const* tbl, const int* par, const double* f, double* fc,
                          double* partials, cudaStream_t st, int64_t s0) {
  const SP s = make_sp(L.sp);
  const i64 lanes = ipow(s.G, L.sp.dim) << L.sp.dim;
  const bool tma = a.mode == 2 && STMG_UPDOWN_TMA;
  const int bt = (tma && a.block == 256) ? 256 : 128;
  const dim3 grid(grid1(lanes, bt), unsigned((L.n_t + a.chunk - 1) / a.chunk));
  a.n_partials = i64(grid.x) * grid.y;
  const PingPong pp{tbl, par};
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    const TM<NL> t = make_tm<NL>(L.tc);
#ifdef STMG_UPDOWN_CARVEOUT
    cudaFuncSetAttribute(k_updown<DIM, NL, 2>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         STMG_UPDOWN_CARVEOUT);
    cudaFuncSetAttribute(k_updown<DIM, NL, 1>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         STMG_UPDOWN_CARVEOUT);
#endif
    if (bt == 256) {
      if constexpr (DIM >= 2 && NL <= 2) {
        if (s.G % TmaShape<DIM, NL, 256>::GPB != 0) return cudaErrorInvalidValue;
        static PerDevice attr;
        if (attr.first_use())
          cudaFuncSetAttribute(k_updown_tma<DIM, NL, 256>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(TmaShape<DIM, NL, 256>::smem));
        PDLK(k_updown_tma<DIM, NL, 256>, grid, 256, TmaShape<DIM, NL, 256>::smem, st, ec, pp, f,
             fc, partials, t, s, L.n_t, a.chunk, a.n1c, a.omega, i64(s0));
      } else {
        return cudaErrorInvalidValue;  // pick_updown_block never asks for this
      }
    } else if (tma && s.G % TmaShape<DIM, NL>::GPB == 0)
      PDLK(k_updown_tma<DIM, NL, 128>, grid, 128, TmaShape<DIM, NL>::smem, st, ec, pp, f, fc,
           partials, t, s, L.n_t, a.chunk, a.n1c, a.omega, i64(s0));
    else if (a.mode == 2)
      PDLK(k_updown<DIM, NL, 2>, grid, 128, updown_smem(NL), st, ec, pp, f, fc, partials, t,
           s, L.n_t, a.chunk, a.n1c, a.omega, i64(s0));
    else
      PDLK(k_updown<DIM, NL, 1>, grid, 128, updown_smem(NL), st, ec, pp, f, fc, partials, t,
           s, L.n_t, a.chunk, L.sp.n1, a.omega, i64(s0));
  });
  return cudaGetLastError();
}

cudaError_t launch_cop_gemv(const double* B, const double* x, double* y, int n,
                            cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = size_t(kCopRows) * n * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static PerDevice attr;
  if (attr.first_use()) {  // maximum shared-memory carveout: all rows of B in flight in one wave
    cudaFuncSetAttribute(k_cop_gemv, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  PDLK(k_cop_gemv, grid1(n, kCopRows), kCopRows * 32, smem, st, B, x, y, n);
  return cudaGetLastError();
}

cudaError_t launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_axpy<<<grid1(n, 256), 256, 0, st>>>(y, x, a, n);
  return cudaGetLastError();
}

cudaError_t launch_nonzero(const double* v, int64_t n, int* flag, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned g = unsigned(std::min<i64>((n + 255) / 256, 148 * 8));
  k_nonzero<<<g, 256, 0, st>>>(v, n, flag);
  return cudaGetLastError();
}

template <int NL>
cudaError_t build_tail_table_t(const TailSpec* lv, int nlev, void** out, void** host_out) {
  std::vector<TailLevel<NL>> h(nlev);
  for (int k = 0; k < nlev; ++k) {
    h[k].t = make_tm<NL>(lv[k].view.tc);
    h[k].s = make_sp(lv[k].view.sp);
    h[k].n_t = lv[k].view.n_t;
    h[k].n1c = lv[k].n1c;
    h[k].mode = lv[k].mode;
    h[k].F = lv[k].F;
    h[k].U0 = lv[k].U0;
    h[k].U1 = lv[k].U1;
  }
  cudaError_t e = cudaMalloc(out, sizeof(TailLevel<NL>) * nlev);
  if (e != cudaSuccess) return e;
  void* hb = std::malloc(sizeof(TailLevel<NL>) * nlev);
  std::memcpy(hb, h.data(), sizeof(TailLevel<NL>) * nlev);
  *host_out = hb;
  return cudaMemcpy(*out, h.data(), sizeof(TailLevel<NL>) * nlev, cudaMemcpyHostToDevice);
}

cudaError_t build_tail_table(const TailSpec* levels, int nlev, void** dev_table,
                             void** host_table) {
  switch (levels[0].view.tc.nl) {
    case 1: return build_tail_table_t<1>(levels, nlev, dev_table, host_table);
    case 2: return build_tail_table_t<2>(levels, nlev, dev_table, host_table);
    case 3: return build_tail_table_t<3>(levels, nlev, dev_table, host_table);
    case 4: return build_tail_table_t<4>(levels, nlev, dev_table, host_table);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tail(int dim, int nl, const void* dev_table, const void* host_table, int nlev,
                        double omega, size_t smem_bytes, cudaStream_t st, double* cop,
                        int64_t cop_n) {
  if (nlev > kTailMaxLevels) return cudaErrorInvalidValue;
  STMG_DISPATCH(dim, nl, {
    TailParams<NL> P;
    const TailLevel<NL>* h = static_cast<const TailLevel<NL>*>(host_table);
    for (int k = 0; k < nlev; ++k) P.t[k] = h[k].t;
    cudaFuncSetAttribute(k_tail<DIM, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem_bytes));
    const unsigned grid = cop ? unsigned(cop_n) : 1u;
    PDLK(k_tail<DIM, NL>, grid, kTailThreads, smem_bytes, st,
         static_cast<const TailLevel<NL>*>(dev_table), nlev, omega, P, cop);
  });
  return cudaGetLastError();
}

template <int NL>
cudaError_t build_csub_t(const CsubSpec* lv, int nlev, int lanes_target, CsubPlan* plan) {
  if (nlev < 2 || nlev > kCsubMaxLevels) return cudaErrorInvalidValue;
  CsubParams<NL> P{};
  const int dim = lv[0].view.sp.dim;
  for (int k = 0; k < nlev; ++k) {
    P.lv[k].t = make_tm<NL>(lv[k].view.tc);
    P.lv[k].s = make_sp(lv[k].view.sp);
    P.lv[k].n_t = lv[k].view.n_t;
    P.lv[k].n1c = lv[k].n1c;
    P.lv[k].F = lv[k].F;
    P.lv[k].U0 = lv[k].U0;
    P.lv[k].U1 = lv[k].U1;
  }
  P.nb = nlev - 2;
  // trees: every group of level b, and the middle groups of levels a..b-1
  std::vector<CsubCta> ctas;
  std::vector<unsigned> roots;
  for (int r = P.nb; r >= 0; --r) {
    const i64 G = P.lv[r].s.G;
    const i64 ng = ipow(G, dim);
    const int first = int(roots.size());
    for (i64 g = 0; g < ng; ++g) {
      bool mid = false;
      i64 q = g;
      for (int a = 0; a < dim; ++a, q /= G) mid |= (q % G) == G - 1;
      if (r == P.nb || mid) roots.push_back(unsigned(g));
    }
    const int n = int(roots.size()) - first;
    const int per = 1 << (dim * (r + 1));  // level-a lanes of one tree
    const int k = std::max(1, lanes_target / per);
    for (int i = 0; i < n; i += k) ctas.push_back(CsubCta{r, first + i, std::min(k, n - i)});
  }
  free_csub(plan);
  plan->dim = dim;
  plan->nl = NL;
  plan->n_ctas = int(ctas.size());
  plan->trees = int(roots.size());
  cudaError_t e = cudaMalloc(&plan->ctas, ctas.size() * sizeof(CsubCta));
  if (e == cudaSuccess) e = cudaMalloc(&plan->roots, roots.size() * sizeof(unsigned));
  if (e == cudaSuccess)
    e = cudaMemcpy(plan->ctas, ctas.data(), ctas.size() * sizeof(CsubCta), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(plan->roots, roots.data(), roots.size() * sizeof(unsigned),
                   cudaMemcpyHostToDevice);
  plan->params = std::malloc(sizeof(P));
  std::memcpy(plan->params, &P, sizeof(P));
  return e;
}

cudaError_t build_csub(const CsubSpec* levels, int nlev, int lanes_target, CsubPlan* plan) {
  switch (levels[0].view.tc.nl) {
    case 1: return build_csub_t<1>(levels, nlev, lanes_target, plan);
    case 2: return build_csub_t<2>(levels, nlev, lanes_target, plan);
    case 3: return build_csub_t<3>(levels, nlev, lanes_target, plan);
    case 4: return build_csub_t<4>(levels, nlev, lanes_target, plan);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_csub(const CsubPlan& plan, bool up, double omega, cudaStream_t st) {
  if (!plan.params || plan.n_ctas <= 0) return cudaErrorInvalidValue;
  STMG_DISPATCH(plan.dim, plan.nl, {
    CsubParams<NL> P;
    std::memcpy(&P, plan.params, sizeof(P));
    P.omega = omega;
    const CsubCta* c = static_cast<const CsubCta*>(plan.ctas);
    const unsigned* r = static_cast<const unsigned*>(plan.roots);
    if (up)
      PDLK(k_csub_up<DIM, NL>, plan.n_ctas, plan.threads, 0, st, c, r, P);
    else
      PDLK(k_csub_down<DIM, NL>, plan.n_ctas, plan.threads, 0, st, c, r, P);
  });
  return cudaGetLastError();
}

void free_csub(CsubPlan* plan) {
  if (plan->ctas) cudaFree(plan->ctas);
  if (plan->roots) cudaFree(plan->roots);
  std::free(plan->params);
  plan->ctas = plan->roots = plan->params = nullptr;
  plan->n_ctas = plan->trees = 0;
}

int64_t partial_count(const LevelView& L, int chunk, bool grouped, int block) {
  const i64 G = (L.sp.n1 + 1) / 2;
  const i64 units = grouped ? (ipow(G, L.sp.dim) << L.sp.dim) : L.sp.nx;
  return i64(grid1(units, block)) * ((L.n_t + chunk - 1) / chunk);
}

#ifndef STMG_UPDOWN_BLOCK256_WAVES
#define STMG_UPDOWN_BLOCK256_WAVES 0  // A/B: 256 wins on C2 (-1.1 %), C4 (-2.2 %), C5 (-1 %): profiles/r02_v8_updown_block256_ab.txt
#endif
// Threads per CTA of the fused level-0 kernel (launch_updown) for the level
// `G` (the GLOBAL level: the result must not depend on the time-slab split).
int pick_updown_block(const LevelView& G, int chunk, int mode) {
  static const int forced = [] {
    const char* e = std::getenv("STMG_UPDOWN_BLOCK");
    return e ? std::atoi(e) : 0;
  }();
  if (!(mode == 2 && STMG_UPDOWN_TMA == 2 && G.sp.dim >= 2 && G.tc.nl <= 2)) return 128;
  const i64 g = (G.sp.n1 + 1) / 2;
  const int nm = 1 << G.sp.dim;
  if (g % (256 / nm) != 0) return 128;
  if (forced == 128 || forced == 256) return forced;
  static const int sms = [] {
    int d = 0, n = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
  }();
  const i64 lanes = ipow(g, G.sp.dim) << G.sp.dim;
  const i64 chunks = (G.n_t + chunk - 1) / chunk;
  // (a minimum number of waves of 256-thread CTAs can be required; measured: none needed)
  return i64(grid1(lanes, 256)) * chunks >= i64(sms) * 2 * STMG_UPDOWN_BLOCK256_WAVES ? 256 : 128;
}

#ifndef STMG_CHUNK_TARGET
#define STMG_CHUNK_TARGET (148 * 256)
#endif

// levels below STMG_CHUNK_BIG dofs (latency-bound coarse levels) may use
// their own target (A/B: 148*64 ... 148*1024 for them are all slower on C2
// than the common 148*256; profiles/r01_v17_chunk_small_ab.txt)
#ifndef STMG_CHUNK_TARGET_SMALL
#define STMG_CHUNK_TARGET_SMALL STMG_CHUNK_TARGET
#endif
#ifndef STMG_CHUNK_BIG
#define STMG_CHUNK_BIG (i64(1) << 23)
#endif
int pick_chunk(const LevelView& L, bool grouped) {
  const i64 G = (L.sp.n1 + 1) / 2;
  const i64 units = grouped ? (ipow(G, L.sp.dim) << L.sp.dim) : L.sp.nx;
  // aim for ~0.5K threads per SM worth of (lane, chunk) work items (A/B:
  // 148*256 beats 148*512 by 2 % on C2, neutral on C3-C5; profiles/
  // r01_v13_chunk_ab.txt, r01_v14_chunk_ab.txt); chunks are even and divide the
  // (power-of-two) n_t; longer chunks amortise the one-step warm-up
  const i64 target = L.size() >= STMG_CHUNK_BIG ? i64(STMG_CHUNK_TARGET) : i64(STMG_CHUNK_TARGET_SMALL);
  i64 c = 2;
  while (c < 64 && c * 2 <= L.n_t && units * (L.n_t / (c * 2)) >= target) c *= 2;
  if (c > L.n_t) c = L.n_t;
  if (c < 2) c = 2;
  return int(c);
}

cudaError_t launch_down(const LevelView& L, ModalArgs& a, bool zero_guess, const double* f,
                        const double* u_in, double* u_out, double* fc, cudaStream_t st) {
  const SP s = make_sp(L.sp);
  const i64 lanes = ipow(s.G, L.sp.dim) << L.sp.dim;
  const dim3 grid(grid1(lanes, 128), unsigned((L.n_t + a.chunk - 1) / a.chunk));
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    const TM<NL> t = make_tm<NL>(L.tc);
    if (a.mode == 2 && STMG_LEVEL_RR && L.size() >= STMG_LEVEL_RR_MIN &&
        s.G % RowRuns<DIM, NL, 1, false>::GPB == 0) {
      if (zero_guess)
        PDLK(k_down_rr<DIM, NL, true>, grid, 128, RowRuns<DIM, NL, 1, false>::smem, st, f, u_in,
             u_out, fc, t, s, L.n_t, a.chunk, a.n1c, a.omega, L.first_global);
      else
        PDLK(k_down_rr<DIM, NL, false>, grid, 128, RowRuns<DIM, NL, 2, false>::smem, st, f, u_in,
             u_out, fc, t, s, L.n_t, a.chunk, a.n1c, a.omega, L.first_global);
    } else if (a.mode == 2) {
      if (zero_guess)
        PDLK(k_down<DIM, NL, true, 2>, grid, 128, ring_bytes(2 * NL), st, f, u_in, u_out, fc, t, s, L.n_t, a.chunk,
                                                      a.n1c, a.omega, L.first_global);
      else
        PDLK(k_down<DIM, NL, false, 2>, grid, 128, ring_bytes(4 * NL), st, f, u_in, u_out, fc, t, s, L.n_t, a.chunk,
                                                       a.n1c, a.omega, L.first_global);
    } else {
      if (zero_guess)
        PDLK(k_down<DIM, NL, true, 1>, grid, 128, ring_bytes(2 * NL), st, f, u_in, u_out, fc, t, s, L.n_t, a.chunk,
                                                      L.sp.n1, a.omega, L.first_global);
      else
        PDLK(k_down<DIM, NL, false, 1>, grid, 128, ring_bytes(4 * NL), st, f, u_in, u_out, fc, t, s, L.n_t, a.chunk,
                                                       L.sp.n1, a.omega, L.first_global);
    }
  });
  return cudaGetLastError();
}

cudaError_t launch_up(const LevelView& L, ModalArgs& a, const double* ec, const double* u_in,
                      const double* f, double* u_out, double* partials, cudaStream_t st) {
  const SP s = make_sp(L.sp);
  const i64 lanes = ipow(s.G, L.sp.dim) << L.sp.dim;
  const dim3 grid(grid1(lanes, 128), unsigned((L.n_t + a.chunk - 1) / a.chunk));
  a.n_partials = i64(grid.x) * grid.y;
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    const TM<NL> t = make_tm<NL>(L.tc);
    const i64 n1c = a.mode == 2 ? a.n1c : L.sp.n1;
    if (a.mode == 2 && STMG_LEVEL_RR && L.size() >= STMG_LEVEL_RR_MIN &&
        s.G % RowRuns<DIM, NL, 2, true>::GPB == 0) {
      if (partials)
        PDLK(k_up_rr<DIM, NL, true>, grid, 128, RowRuns<DIM, NL, 2, true>::smem, st, ec, u_in, f,
             u_out, partials, t, s, L.n_t, a.chunk, n1c, a.omega, L.first_global);
      else
        PDLK(k_up_rr<DIM, NL, false>, grid, 128, RowRuns<DIM, NL, 2, true>::smem, st, ec, u_in, f,
             u_out, partials, t, s, L.n_t, a.chunk, n1c, a.omega, L.first_global);
    } else if (a.mode == 2) {
      if (partials)
        PDLK(k_up<DIM, NL, 2, true>, grid, 128, ring_bytes(5 * NL), st, ec, u_in, f, u_out, partials, t, s, L.n_t,
                                                    a.chunk, n1c, a.omega, L.first_global);
      else
        PDLK(k_up<DIM, NL, 2, false>, grid, 128, ring_bytes(5 * NL), st, ec, u_in, f, u_out, partials, t, s, L.n_t,
                                                     a.chunk, n1c, a.omega, L.first_global);
    } else {
      if (partials)
        PDLK(k_up<DIM, NL, 1, true>, grid, 128, ring_bytes(5 * NL), st, ec, u_in, f, u_out, partials, t, s, L.n_t,
                                                    a.chunk, n1c, a.omega, L.first_global);
      else
        PDLK(k_up<DIM, NL, 1, false>, grid, 128, ring_bytes(5 * NL), st, ec, u_in, f, u_out, partials, t, s, L.n_t,
                                                     a.chunk, n1c, a.omega, L.first_global);
    }
  });
  return cudaGetLastError();
}

cudaError_t launch_smooth(const LevelView& L, ModalArgs& a, bool zero_guess, const double* f,
                          const double* u_in, double* u_out, cudaStream_t st) {
  const SP s = make_sp(L.sp);
  const dim3 grid(grid1(L.sp.nx, 128), unsigned((L.n_t + a.chunk - 1) / a.chunk));
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    const TM<NL> t = make_tm<NL>(L.tc);
    if (zero_guess)
      PDLK(k_smooth<DIM, NL, true>, grid, 128, 0, st, f, u_in, u_out, t, s, L.n_t, a.chunk, a.omega,
                                                   L.first_global);
    else
      PDLK(k_smooth<DIM, NL, false>, grid, 128, 0, st, f, u_in, u_out, t, s, L.n_t, a.chunk, a.omega,
                                                    L.first_global);
  });
  return cudaGetLastError();
}

cudaError_t launch_resnorm(const LevelView& L, ModalArgs& a, const double* u, const double* f,
                           double* partials, cudaStream_t st, bool u_zero) {
  const SP s = make_sp(L.sp);
  const dim3 grid(grid1(L.sp.nx, 128), unsigned((L.n_t + a.chunk - 1) / a.chunk));
  a.n_partials = i64(grid.x) * grid.y;
  STMG_DISPATCH(L.sp.dim, L.tc.nl, {
    if (u_zero)
      PDLK(k_resnorm<DIM, NL, true>, grid, 128, 0, st, u, f, partials, make_tm<NL>(L.tc), s, L.n_t,
                                                    a.chunk, L.first_global);
    else
      PDLK(k_resnorm<DIM, NL, false>, grid, 128, 0, st, u, f, partials, make_tm<NL>(L.tc), s, L.n_t,
                                                     a.chunk, L.first_global);
  });
  return cudaGetLastError();
}

}  // namespace stmg
