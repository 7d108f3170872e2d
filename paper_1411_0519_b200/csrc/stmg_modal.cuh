// stmg_modal.cuh -- device helpers shared by the sm_100a kernel files
// (stmg_kernels.cu, stmg_spatial.cu): per-mode DG block algebra in the sine
// basis, alias-mode groups of full weighting, cp.async and PDL helpers, and
// the (dim, p_t + 1) template dispatch of the launchers.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>

#include "stmg_launch.hpp"

namespace stmg {
namespace {

using i64 = long long;

template <int NL>
struct TM {
  double K[NL][NL], M[NL][NL], N[NL][NL], R1[NL][NL], R2[NL][NL];
};

template <int NL>
TM<NL> make_tm(const TimeConsts& c) {
  TM<NL> t;
  for (int k = 0; k < NL; ++k)
    for (int l = 0; l < NL; ++l) {
      const int i = k * kMaxNL + l;
      t.K[k][l] = c.K[i];
      t.M[k][l] = c.M[i];
      t.N[k][l] = c.N[i];
      t.R1[k][l] = c.R1[i];
      t.R2[k][l] = c.R2[i];
    }
  return t;
}

struct SP {
  i64 n1, nx;
  int G;  // mode groups per axis = (n1 + 1) / 2
  double h;
  const double* __restrict__ mval;
  const double* __restrict__ kval;
  const double* __restrict__ rfac;
};

SP make_sp(const SpaceConsts& s) {
  SP p;
  p.n1 = s.n1;
  p.nx = s.nx;
  p.G = int((s.n1 + 1) / 2);
  p.h = s.h;
  p.mval = s.mval;
  p.kval = s.kval;
  p.rfac = s.rfac;
  return p;
}

__host__ __device__ constexpr i64 ipow(i64 b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// Programmatic dependent launch: the V-cycle kernels are launched with
// programmatic stream serialization, so the next kernel's CTAs are scheduled
// while this one drains; every such kernel waits for its predecessor's
// memory before touching global data.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ------------------------------------------------------------ per-mode math
// Exact per-mode block: A_j = M_j K_tau + K_j M_tau.  Its symmetric part is
// positive definite (K_tau + K_tau^T = psi(tau)psi(tau)^T + psi(0)psi(0)^T),
// so elimination without pivoting is stable.  A_j is constant along a mode's
// time line, so its factors are computed once per thread (the divisions and
// the assembly leave the time loop) and solve() runs the substitutions.
template <int NL>
struct ModeLU {
  double inv[NL];
  double L[NL][NL];  // multipliers (r > c)
  double U[NL][NL];  // eliminated rows (k > c)
  __device__ __forceinline__ ModeLU(const TM<NL>& t, double Mj, double Kj) {
    double A[NL][NL];
#pragma unroll
    for (int i = 0; i < NL; ++i)
#pragma unroll
      for (int j = 0; j < NL; ++j) A[i][j] = Mj * t.K[i][j] + Kj * t.M[i][j];
#pragma unroll
    for (int c = 0; c < NL; ++c) {
      inv[c] = 1.0 / A[c][c];
#pragma unroll
      for (int r = c + 1; r < NL; ++r) {
        const double f = A[r][c] * inv[c];
        L[r][c] = f;
#pragma unroll
        for (int k = c + 1; k < NL; ++k) A[r][k] -= f * A[c][k];
      }
    }
#pragma unroll
    for (int c = 0; c < NL; ++c)
#pragma unroll
      for (int k = c + 1; k < NL; ++k) U[c][k] = A[c][k];
  }
  __device__ __forceinline__ void solve(const double (&b)[NL], double (&x)[NL]) const {
#pragma unroll
    for (int i = 0; i < NL; ++i) x[i] = b[i];
#pragma unroll
    for (int c = 0; c < NL; ++c)
#pragma unroll
      for (int r = c + 1; r < NL; ++r) x[r] -= L[r][c] * x[c];
#pragma unroll
    for (int c = NL - 1; c >= 0; --c) {
      double s = x[c];
#pragma unroll
      for (int k = c + 1; k < NL; ++k) s -= U[c][k] * x[k];
      x[c] = s * inv[c];
    }
  }
};

// Explicit per-mode operators of one damped Jacobi step, for the time-marching
// kernels whose per-step chains are latency bound.  The DG jump is rank one,
// N_tau = a 1^T with a_k = psi_k(0) and psi_l(tau) = 1 (stmg_setup.cpp:75), so
//   sweep:    out = (1-w) cur + wAi f + h S(prev),   h = w A^-1 (M_j a)
//   residual: r   = f - A cur + ma S(prev),          ma = M_j a
// with S(v) = sum_l v_l (the end-of-step trace).  A^-1 comes from the same
// elimination as ModeLU (column by column), once per thread.  Algebraically
// identical to ModeLU::solve on f + M_j N prev; rounding differs at 1e-16.
template <int NL>
struct ModeOps {
  double wAi[NL][NL];  // omega * A_j^-1
  double A[NL][NL];    // A_j
  double h[NL];        // omega * A_j^-1 (M_j a)
  double ma[NL];       // M_j a
  __device__ __forceinline__ ModeOps(const TM<NL>& t, double Mj, double Kj, double omega) {
    const ModeLU<NL> lu(t, Mj, Kj);
#pragma unroll
    for (int i = 0; i < NL; ++i)
#pragma unroll
      for (int j = 0; j < NL; ++j) A[i][j] = Mj * t.K[i][j] + Kj * t.M[i][j];
#pragma unroll
    for (int c = 0; c < NL; ++c) {
      double e[NL], x[NL];
#pragma unroll
      for (int i = 0; i < NL; ++i) e[i] = (i == c) ? 1.0 : 0.0;
      lu.solve(e, x);
#pragma unroll
      for (int i = 0; i < NL; ++i) wAi[i][c] = omega * x[i];
    }
#pragma unroll
    for (int i = 0; i < NL; ++i) ma[i] = Mj * t.N[i][0];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NL; ++j) s += wAi[i][j] * ma[j];
      h[i] = s;
    }
  }
  // g = omega A^-1 f (shared by the sweeps of one step)
  __device__ __forceinline__ void solve_w(const double (&f)[NL], double (&g)[NL]) const {
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NL; ++j) s = fma(wAi[i][j], f[j], s);
      g[i] = s;
    }
  }
  // out = (1-w) cur + g + h * sprev
  __device__ __forceinline__ void sweep(const double (&cur)[NL], const double (&g)[NL],
                                        double sprev, double om1, double (&out)[NL]) const {
#pragma unroll
    for (int i = 0; i < NL; ++i) out[i] = fma(h[i], sprev, fma(om1, cur[i], g[i]));
  }
  // r = f - A cur + ma * sprev
  __device__ __forceinline__ void residual(const double (&f)[NL], const double (&cur)[NL],
                                           double sprev, double (&r)[NL]) const {
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NL; ++j) s = fma(A[i][j], cur[j], s);
      r[i] = fma(ma[i], sprev, f[i] - s);
    }
  }
};

template <int NL>
__device__ __forceinline__ double trace_sum(const double (&v)[NL]) {
  double s = v[0];
#pragma unroll
  for (int l = 1; l < NL; ++l) s += v[l];
  return s;
}

// y = A_j x
template <int NL>
__device__ __forceinline__ void apply_mode(const TM<NL>& t, double Mj, double Kj,
                                           const double (&x)[NL], double (&y)[NL]) {
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      a += t.K[k][l] * x[l];
      b += t.M[k][l] * x[l];
    }
    y[k] = Mj * a + Kj * b;
  }
}

template <int NL>
__device__ __forceinline__ void matvec(const double (&A)[NL][NL], const double (&x)[NL],
                                       double (&y)[NL]) {
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    double a = 0.0;
#pragma unroll
    for (int l = 0; l < NL; ++l) a += A[k][l] * x[l];
    y[k] = a;
  }
}

// y = A^T x
template <int NL>
__device__ __forceinline__ void matvec_t(const double (&A)[NL][NL], const double (&x)[NL],
                                         double (&y)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < NL; ++k) a += A[k][l] * x[k];
    y[l] = a;
  }
}

template <int DIM, bool COH = false>
__device__ __forceinline__ void mode_eig(const SP& s, i64 r, double& Mj, double& Kj) {
  double mv[DIM], kv[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const i64 q = r % s.n1;
    r /= s.n1;
    mv[a] = COH ? s.mval[q] : __ldg(s.mval + q);
    kv[a] = COH ? s.kval[q] : __ldg(s.kval + q);
  }
  Mj = 1.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) Mj *= mv[a];
  Kj = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double p = kv[a];
#pragma unroll
    for (int b = 0; b < DIM; ++b)
      if (b != a) p *= mv[b];
    Kj += p;
  }
}

template <int NL>
__device__ __forceinline__ void load_nl(const double* __restrict__ p, i64 nx, double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) v[l] = __ldg(p + l * nx);
}

template <int NL>
__device__ __forceinline__ void load_nl_cs(const double* __restrict__ p, i64 nx, double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) v[l] = __ldcs(p + l * nx);
}

template <int NL>
__device__ __forceinline__ void store_nl(double* __restrict__ p, i64 nx, const double (&v)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) p[l * nx] = v[l];
}

// Alias-mode groups: per axis the pair {i, n1-1-i} (0-based sine index) that
// full weighting maps onto coarse mode i; the middle index G-1 is alone and
// restricts to zero.  Lane bits [0, DIM) of a thread select the member of its
// group, so a group's 2^DIM members sit in adjacent lanes of one warp and the
// restriction sums with warp shuffles.
struct Member {
  i64 idx;       // fine mode (flat sine index)
  i64 cidx;      // coarse mode of the group (full coarsening)
  double Mj, Kj;
  double fac;    // full-weighting factor of this member (product over axes)
  bool ok;       // member exists (and group exists)
  bool cok;      // group has a coarse mode
};

template <int DIM, bool COH = false>
__device__ __forceinline__ Member make_member(const SP& s, i64 t, i64 n1c, bool full) {
  Member m;
  const int b = int(t & ((1 << DIM) - 1));
  const i64 gg = t >> DIM;
  const i64 ngroups = ipow(s.G, DIM);
  m.ok = gg < ngroups;
  unsigned g = m.ok ? unsigned(gg) : 0u;  // < 2^31 groups: 32-bit index math
  m.cok = m.ok;
  i64 idx = 0, mul = 1, ci = 0, cm = 1;
  double mv[DIM], kv[DIM], fac = 1.0;
  const unsigned G = unsigned(s.G);
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int ia = int(g % G);
    g /= G;
    const bool mid = ia >= s.G - 1;
    if (mid) m.cok = false;
    const int bit = (b >> a) & 1;
    if (bit && mid) m.ok = false;
    const i64 q = (bit && !mid) ? (s.n1 - 1 - ia) : i64(ia);
    idx += q * mul;
    mul *= s.n1;
    ci += ia * cm;
    cm *= n1c;
    mv[a] = COH ? s.mval[q] : __ldg(s.mval + q);
    kv[a] = COH ? s.kval[q] : __ldg(s.kval + q);
    if (full) fac *= COH ? s.rfac[q] : __ldg(s.rfac + q);
  }
  double M = 1.0, K = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) M *= mv[a];
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double p = kv[a];
#pragma unroll
    for (int c = 0; c < DIM; ++c)
      if (c != a) p *= mv[c];
    K += p;
  }
  m.idx = idx;
  m.cidx = ci;
  m.Mj = M;
  m.Kj = K;
  m.fac = fac;
  return m;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// Sum over the 2^DIM lanes of an alias group.
template <int DIM>
__device__ __forceinline__ double group_sum(double v) {
  constexpr unsigned gm = (1u << (1 << DIM)) - 1u;
  const unsigned mask = gm << ((threadIdx.x & 31) & ~((1 << DIM) - 1));
#pragma unroll
  for (int o = 1; o < (1 << DIM); o <<= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// The same with a full-warp mask: only where every lane of the warp calls it.
template <int DIM>
__device__ __forceinline__ double group_sum_full(double v) {
#pragma unroll
  for (int o = 1; o < (1 << DIM); o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Plain global store (for pointers the compiler cannot prove global).
__device__ __forceinline__ void st_global(double* p, double v) {
  asm volatile("st.global.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

// cp.async (LDGSTS) helpers: 8-byte copies, zero fill when !valid.
__device__ __forceinline__ void cp_async8(double* smem, const double* g, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async8s(unsigned s, const double* g, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g),
               "r"(valid ? 8 : 0));
}
// mbarrier + TMA bulk copy (cp.async.bulk, 16-byte aligned source, destination and size)
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity), "r"(0x989680u)  // suspend-time hint: the warp sleeps instead of spinning
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Per-thread asynchronous staging ring of the fused level kernels: stage st
// of thread t holds the loads of one step pair; element q of a stage lives at
// ring[(st * Q + q) * blockDim.x + t] (thread-fastest: conflict-free).
constexpr int kRing = 3;  // stages: two step pairs in flight while one is used
#ifndef STMG_DOWN_ASYNC
#define STMG_DOWN_ASYNC 1
#endif
#ifndef STMG_UP_ASYNC
#define STMG_UP_ASYNC 1
#endif



inline unsigned grid1(i64 n, int bs) { return unsigned((n + bs - 1) / bs); }
// cp.async ring of the fused level kernels (128 threads, q doubles per pair)
inline size_t ring_bytes(int q) { return size_t(kRing) * q * 128 * sizeof(double); }


// Launch with programmatic stream serialization (see pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#define PDLK(...)                                   \
  do {                                              \
    const cudaError_t e_ = pdl_launch(__VA_ARGS__); \
    if (e_ != cudaSuccess) return e_;               \
  } while (0)
// nodes along x (blocks of bs), time steps along y (grid-stride beyond 65535)
inline dim3 grid2(i64 nodes, i64 steps, int bs) {
  return dim3(grid1(nodes, bs), unsigned(std::max<i64>(1, std::min<i64>(steps, 65535))));
}


}  // namespace
}  // namespace stmg

// ============================================================== dispatch
#define STMG_CASE(D, Q, ...)           \
  case (D) * 8 + (Q): {                \
    constexpr int DIM = (D), NL = (Q); \
    __VA_ARGS__;                       \
  } break;

#define STMG_DISPATCH(dim, nl, ...)                                                    \
  switch ((dim) * 8 + (nl)) {                                                          \
    STMG_CASE(1, 1, __VA_ARGS__)                                                       \
    STMG_CASE(1, 2, __VA_ARGS__)                                                       \
    STMG_CASE(1, 3, __VA_ARGS__)                                                       \
    STMG_CASE(1, 4, __VA_ARGS__)                                                       \
    STMG_CASE(2, 1, __VA_ARGS__)                                                       \
    STMG_CASE(2, 2, __VA_ARGS__)                                                       \
    STMG_CASE(2, 3, __VA_ARGS__)                                                       \
    STMG_CASE(2, 4, __VA_ARGS__)                                                       \
    STMG_CASE(3, 1, __VA_ARGS__)                                                       \
    STMG_CASE(3, 2, __VA_ARGS__)                                                       \
    STMG_CASE(3, 3, __VA_ARGS__)                                                       \
    STMG_CASE(3, 4, __VA_ARGS__)                                                       \
    default:                                                                           \
      return cudaErrorInvalidValue;                                                    \
  }

