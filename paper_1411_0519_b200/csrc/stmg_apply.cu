// stmg_apply.cu -- row-band Q1 apply / residual kernels (physical space).
//
// y_n = (M U_n) K^T + (K U_n) M^T - (M U_{n-1}) N^T,  r = f - y
// (st_system.cpp:18-33, 44-67), the reference's `apply` / `residual`.
//
// The kernels in stmg_kernels.cu (k_apply, k_apply_rb) stage a 32-wide tile
// plus halo element by element (8-byte LDGSTS) and read 9 (2D) shared-memory
// values per output; ncu shows them bound by the L1/LSU pipe (C2: l1tex 77 %,
// issue slots 63 % at 40 % of DRAM peak).  Here a CTA owns FULL grid rows, so
//  * the rows y0-1 .. y0+TY of one (step, component) are ONE contiguous run
//    in the reference layout: a single TMA bulk copy (cp.async.bulk +
//    mbarrier) per component stages them, issued by one thread -- no per-
//    element copy instructions, no x halo, Dirichlet rows simply not copied
//    (the packed rows of 2^k - 1 doubles are only 8-byte aligned, so the copy
//    starts at the 16-byte aligned-down address; a multi-dimensional tensor
//    map cannot describe this layout at all: its strides must be multiples of
//    16 bytes);
//  * a thread owns one grid column and marches down the band with a rolling
//    window of the 1D row combinations (M1 u, K1 u): 3 shared-memory loads per
//    staged row and component instead of 9 per output;
//  * the CTA marches through a chunk of time steps, NS slabs in flight, the
//    rank-one jump term reusing the previous step's M-traces from registers,
//    so u and f are read once and r is written once (24 B per dof);
//  * warp specialisation: one producer warp waits on per-stage "empty"
//    mbarriers and issues the copies of the next slab (u rows and the band's f
//    rows) against the stage's "full" mbarrier; the consumer warps never meet
//    in a CTA-wide barrier.  (A first version loaded f straight into registers
//    one step ahead and reloaded each register right after its use: every
//    later use then waited for the fresh load on the shared scoreboard --
//    48 % of the stall samples -- which is why f goes through the stage.)
//  * CTAs whose band and halo lie inside the grid run a variant without any
//    range tests; time chunks are balanced and their number is rounded to a
//    whole number of waves of resident CTAs.
// Results agree with the tile kernels to rounding (the DG-block combination is
// an FMA chain here); parity with the CPU oracle: 1e-12 (tests/test_gpu_parity.py).
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "stmg_modal.cuh"

namespace stmg {
namespace {

struct PerDeviceOnce {
  std::atomic<unsigned long long> mask{0};
  bool first_use() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    return (mask.fetch_or(b) & b) == 0;
  }
};

constexpr int kRowsMaxStages = 8;

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// 1D row combinations at column x of a staged row: Mr = (M1 u)(x), Kr = (K1 u)(x).
__device__ __forceinline__ void row_mk(const double* __restrict__ p, bool has_l, bool has_r,
                                       double m0, double m1, double k0, double k1, double& Mr,
                                       double& Kr) {
  const double c = p[0];
  const double l = has_l ? p[-1] : 0.0;
  const double r = has_r ? p[1] : 0.0;
  const double a = l + r;
  Mr = m1 * a + m0 * c;
  Kr = k1 * a + k0 * c;
}

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

// ------------------------------------------------------------------ 2D
// grid = (bands of TY rows, chunks of C steps).  CW consumer warps (CW * 32 *
// XPT >= n1 columns) + one producer warp: the producer waits for a stage's
// "empty" barrier (one arrival per consumer warp) and issues the bulk copies
// of the next slab into it; consumers wait for the stage's "full" barrier and
// never meet in a CTA-wide barrier, so a warp that is done with slab n starts
// slab n + 1 while the others finish.
template <int NL, bool RES, int TYS, int YS, int XW>
__global__ void __launch_bounds__(XW * YS * 32 + 32, (XW * YS == 4 ? 3 : XW * YS == 8 ? 2 : 1))
k_apply_rows2(
    const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ y,
    const TM<NL> t, const int n1, const double h, const i64 n_t, const int NS,
    const bool first_global, const double* __restrict__ ab) {
  constexpr int CW = XW * YS, THREADS = CW * 32, TY = TYS * YS, XT = XW * 32;
  extern __shared__ __align__(16) double dsm[];  // [2 pad][NS][NL][RU + RF]
  __shared__ __align__(8) unsigned long long bars[2 * kRowsMaxStages];
  const int RU = ((TY + 2) * n1 + 2) & ~1;  // doubles per staged u component (even)
  const int RF = RES ? (TY * n1 + 2) & ~1 : 0;  // ... f component
  const int SS = NL * (RU + RF);             // doubles per stage
  const int y0 = blockIdx.x * TY;
  const int rows = min(TY, n1 - y0);
  const int ylo = max(y0 - 1, 0), yhi = min(y0 + TY, n1 - 1);
  const int len = (yhi - ylo + 1) * n1, lenf = rows * n1;
  const i64 nx = i64(n1) * n1, slab = NL * nx;
  // balanced time chunks: chunk i = steps [i n_t / nch, (i + 1) n_t / nch)
  const i64 n0 = i64(blockIdx.y) * n_t / gridDim.y, nend = i64(blockIdx.y + 1) * n_t / gridDim.y;
  const bool has_prev = n0 > 0 || !first_global;
  const i64 nbeg = has_prev ? n0 - 1 : n0;
  const int nq = int(nend - nbeg);  // slabs this CTA stages
  double* const ring = dsm + 2;
  const unsigned ring_s = smem_addr(ring), full0 = smem_addr(bars),
                 empty0 = full0 + 8u * kRowsMaxStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8u * s, 1);
      mbar_init(empty0 + 8u * s, CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (threadIdx.x >= THREADS) {  // ---- producer warp
    if (threadIdx.x == THREADS) {
      int s = 0;
      unsigned ph = 0;  // parity of the empty barrier's completed phase to wait for
      for (int q = 0; q < nq; ++q) {
        if (q >= NS) mbar_wait(empty0 + 8u * s, ph ^ 1u);
        const i64 n = nbeg + q;
        const bool with_f = RES && n >= n0;
        const unsigned bar = full0 + 8u * s;
        unsigned total = 0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const i64 off = (n * NL + l) * nx + i64(ylo) * n1;
          total += unsigned((int(off & 1) + len + 1) & ~1) * 8u;
          if (with_f) {
            const i64 offf = (n * NL + l) * nx + i64(y0) * n1;
            total += unsigned((int(offf & 1) + lenf + 1) & ~1) * 8u;
          }
        }
        mbar_expect(bar, total);
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const i64 off = (n * NL + l) * nx + i64(ylo) * n1;
          const int mis = int(off & 1);
          bulk_g2s(ring_s + unsigned(s * SS + l * RU) * 8u, u + off - mis,
                   unsigned((mis + len + 1) & ~1) * 8u, bar);
          if (with_f) {
            const i64 offf = (n * NL + l) * nx + i64(y0) * n1;
            const int misf = int(offf & 1);
            bulk_g2s(ring_s + unsigned(s * SS + NL * RU + l * RF) * 8u, f + offf - misf,
                     unsigned((misf + lenf + 1) & ~1) * 8u, bar);
          }
        }
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }

  // ---- consumer warps
  const double m0 = 4.0 * h / 6.0, m1 = h / 6.0, k0 = 2.0 / h, k1 = -1.0 / h;
  double a[NL], b[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    a[k] = ab[k];
    b[k] = ab[kMaxNL + k];
  }
  // thread -> column x of sub-band g (rows yb .. yb + TYS - 1 of the band)
  const int x = threadIdx.x % XT, g = threadIdx.x / XT;
  const int yb = y0 + g * TYS;
  const int trows = min(TYS, n1 - yb);  // <= 0: nothing to do (last band)
  const bool active = x < n1 && trows > 0;
  const bool has_l = x > 0, has_r = x < n1 - 1;
  const int odd = n1 & 1;
  double mwp[TYS];  // sum_l b_l (M u_{n-1,l}) at this thread's outputs
#pragma unroll
  for (int o = 0; o < TYS; ++o) mwp[o] = 0.0;

  // one staged slab: warm = only the jump traces of step n0 - 1
  // IN: the CTA's band and its halo rows lie inside the grid (no zero rows,
  // no partial band) -- the row loop then has no range tests at all
  auto march = [&](auto in_tag, const double* st, const i64 n, const bool warm) {
    constexpr bool IN = decltype(in_tag)::value;
    // offsets (n NL + l) nx + y n1 have the parity of (n NL + l + y) when n1 is odd
    const int pn = int(n * NL) & 1;
    const double* up[NL];  // component l, row yb - 1, column x
    const double* fp[NL];  // f of component l, row yb, column x
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      up[l] = st + l * RU + (odd & (pn + l + ylo)) + (yb - 1 - ylo) * n1 + x;
      fp[l] = st + NL * RU + l * RF + (odd & (pn + l + y0)) + g * TYS * n1 + x;
    }
    if (active) {
      double Mw0[NL], Mw1[NL], Kw0[NL], Kw1[NL];  // rows gy - 2, gy - 1
#pragma unroll
      for (int yy = 0; yy < TYS + 2; ++yy) {
        const int gy = yb - 1 + yy;
        double Mr[NL], Kr[NL];
        if (IN || (gy >= ylo && gy <= yhi)) {
#pragma unroll
          for (int l = 0; l < NL; ++l)
            row_mk(up[l] + yy * n1, has_l, has_r, m0, m1, k0, k1, Mr[l], Kr[l]);
        } else {
#pragma unroll
          for (int l = 0; l < NL; ++l) Mr[l] = Kr[l] = 0.0;
        }
        if (yy >= 2) {
          const int o = yy - 2;  // output row yb + o (centre row gy - 1)
          if (IN || o < trows) {
            double MU[NL], KU[NL], mw = 0.0;
#pragma unroll
            for (int l = 0; l < NL; ++l) {
              const double ms = Mw0[l] + Mr[l];
              MU[l] = m1 * ms + m0 * Mw1[l];
              KU[l] = m1 * (Kw0[l] + Kr[l]) + m0 * Kw1[l] + k1 * ms + k0 * Mw1[l];
              mw += b[l] * MU[l];
            }
            if (!warm) {
              const i64 o0 = n * slab + i64(yb + o) * n1 + x;
#pragma unroll
              for (int k = 0; k < NL; ++k) {
                double acc = -(a[k] * mwp[o]);
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                  acc = fma(MU[l], t.K[k][l], acc);
                  acc = fma(KU[l], t.M[k][l], acc);
                }
                __stcs(y + o0 + k * nx,
                       RES ? fp[k][o * n1] - acc : acc);
              }
            }
            mwp[o] = mw;
          }
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          Mw0[l] = Mw1[l];
          Kw0[l] = Kw1[l];
          Mw1[l] = Mr[l];
          Kw1[l] = Kr[l];
        }
      }
    }
  };

  int s = 0;
  unsigned ph = 0;
  const int lane = threadIdx.x & 31;
  auto next = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8u * s);
    if (++s == NS) {
      s = 0;
      ph ^= 1u;
    }
  };
  const bool interior = y0 >= 1 && y0 + TY <= n1 - 1;
  if (has_prev) {
    mbar_wait(full0, 0);
    march(std::false_type{}, ring, nbeg, true);
    next();
  }
  if (interior) {
    for (i64 n = n0; n < nend; ++n) {
      mbar_wait(full0 + 8u * s, ph);
      march(std::true_type{}, ring + i64(s) * SS, n, false);
      next();
    }
  } else {
    for (i64 n = n0; n < nend; ++n) {
      mbar_wait(full0 + 8u * s, ph);
      march(std::false_type{}, ring + i64(s) * SS, n, false);
      next();
    }
  }
}

// ------------------------------------------------------------------ 3D
// A CTA owns TY = TYS * YS rows (y) x TZ planes (z) x all columns (x) and
// marches through a chunk of time steps.  Per (step, component) the rows
// ylo..yhi of plane z are one contiguous run: TZ + 2 bulk copies of u and TZ
// of f.  A thread owns column x and TYS rows; per staged plane it forms the
// 2D combinations P = (M1 x M1) u, Q = (M1 x K1 + K1 x M1) u of its rows with
// a rolling window over y, and a rolling window over z turns three planes of
// (P, Q) into M_h u and K_h u (9 shared-memory loads per output for TYS = 2,
// TZ = 4, like k_apply_rb, but no per-element staging instructions, no CTA
// barriers and NS slabs in flight).
template <int NL, bool RES, int TYS, int YS, int TZ, int XW>
__global__ void __launch_bounds__(XW * YS * 32 + 32, (XW * YS <= 4 ? (TZ <= 2 ? 3 : 2) : (TYS == 1 ? 2 : 1)))
k_apply_rows3(
    const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ y,
    const TM<NL> t, const int n1, const double h, const i64 n_t, const int NS,
    const bool first_global, const double* __restrict__ ab) {
  constexpr int CW = XW * YS, THREADS = CW * 32, TY = TYS * YS, XT = XW * 32;
  extern __shared__ __align__(16) double dsm[];  // [2 pad][NS][NL][(TZ+2) RU + TZ RF]
  __shared__ __align__(8) unsigned long long bars[2 * kRowsMaxStages];
  const int RU = ((TY + 2) * n1 + 2) & ~1;
  const int RF = RES ? (TY * n1 + 2) & ~1 : 0;
  const int SU = (TZ + 2) * RU, SF = TZ * RF;  // per component
  const int SS = NL * (SU + SF);
  const int ybands = (n1 + TY - 1) / TY;
  const int y0 = (blockIdx.x % ybands) * TY, z0 = (blockIdx.x / ybands) * TZ;
  const int rows = min(TY, n1 - y0), planes = min(TZ, n1 - z0);
  const int ylo = max(y0 - 1, 0), yhi = min(y0 + TY, n1 - 1);
  const int zlo = max(z0 - 1, 0), zhi = min(z0 + TZ, n1 - 1);
  const int len = (yhi - ylo + 1) * n1, lenf = rows * n1;
  const i64 np = i64(n1) * n1, nx = np * n1, slab = NL * nx;
  const i64 n0 = i64(blockIdx.y) * n_t / gridDim.y, nend = i64(blockIdx.y + 1) * n_t / gridDim.y;
  const bool has_prev = n0 > 0 || !first_global;
  const i64 nbeg = has_prev ? n0 - 1 : n0;
  const int nq = int(nend - nbeg);
  double* const ring = dsm + 2;
  const unsigned ring_s = smem_addr(ring), full0 = smem_addr(bars),
                 empty0 = full0 + 8u * kRowsMaxStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8u * s, 1);
      mbar_init(empty0 + 8u * s, CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (threadIdx.x >= THREADS) {  // ---- producer warp: lane c issues copy c
    const int lane = threadIdx.x - THREADS;
    int s = 0;
    unsigned ph = 0;
    for (int q = 0; q < nq; ++q) {
      if (q >= NS) mbar_wait(empty0 + 8u * s, ph ^ 1u);
      const i64 n = nbeg + q;
      const bool with_f = RES && n >= n0;
      const unsigned bar = full0 + 8u * s;
      if (lane == 0) {
        unsigned total = 0;
        for (int l = 0; l < NL; ++l) {
          for (int z = zlo; z <= zhi; ++z) {
            const i64 off = (n * NL + l) * nx + i64(z) * np + i64(ylo) * n1;
            total += unsigned((int(off & 1) + len + 1) & ~1) * 8u;
          }
          if (with_f)
            for (int zo = 0; zo < planes; ++zo) {
              const i64 off = (n * NL + l) * nx + i64(z0 + zo) * np + i64(y0) * n1;
              total += unsigned((int(off & 1) + lenf + 1) & ~1) * 8u;
            }
        }
        mbar_expect(bar, total);
      }
      __syncwarp();
      // copies: c in [0, NL (TZ + 2)) = u planes, then NL TZ f planes
      for (int c = lane; c < NL * (2 * TZ + 2); c += 32) {
        if (c < NL * (TZ + 2)) {
          const int l = c / (TZ + 2), zz = c % (TZ + 2), z = z0 - 1 + zz;
          if (z >= zlo && z <= zhi) {
            const i64 off = (n * NL + l) * nx + i64(z) * np + i64(ylo) * n1;
            const int mis = int(off & 1);
            bulk_g2s(ring_s + unsigned(s * SS + l * SU + zz * RU) * 8u, u + off - mis,
                     unsigned((mis + len + 1) & ~1) * 8u, bar);
          }
        } else if (with_f) {
          const int c2 = c - NL * (TZ + 2);
          const int l = c2 / TZ, zo = c2 % TZ;
          if (zo < planes) {
            const i64 off = (n * NL + l) * nx + i64(z0 + zo) * np + i64(y0) * n1;
            const int mis = int(off & 1);
            bulk_g2s(ring_s + unsigned(s * SS + NL * SU + l * SF + zo * RF) * 8u, f + off - mis,
                     unsigned((mis + lenf + 1) & ~1) * 8u, bar);
          }
        }
      }
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  // ---- consumer warps
  const double m0 = 4.0 * h / 6.0, m1 = h / 6.0, k0 = 2.0 / h, k1 = -1.0 / h;
  double a[NL], b[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    a[k] = ab[k];
    b[k] = ab[kMaxNL + k];
  }
  const int x = threadIdx.x % XT, g = threadIdx.x / XT;
  const int yb = y0 + g * TYS;
  const int trows = min(TYS, n1 - yb);
  const bool active = x < n1 && trows > 0;
  const bool has_l = x > 0, has_r = x < n1 - 1;
  const int odd = n1 & 1;
  double mwp[TZ][TYS];
#pragma unroll
  for (int zo = 0; zo < TZ; ++zo)
#pragma unroll
    for (int o = 0; o < TYS; ++o) mwp[zo][o] = 0.0;

  auto march = [&](auto in_tag, const double* st, const i64 n, const bool warm) {
    constexpr bool IN = decltype(in_tag)::value;
    if (!active) return;
    const int pn = int(n * NL) & 1;
    double P0[TYS][NL], P1[TYS][NL], Q0[TYS][NL], Q1[TYS][NL];  // planes gz - 2, gz - 1
#pragma unroll
    for (int zz = 0; zz < TZ + 2; ++zz) {
      const int gz = z0 - 1 + zz;
      double P[TYS][NL], Q[TYS][NL];
      if (IN || (gz >= zlo && gz <= zhi)) {
        const double* up[NL];  // component l, plane gz, row yb - 1, column x
#pragma unroll
        for (int l = 0; l < NL; ++l)
          up[l] = st + l * SU + zz * RU + (odd & (pn + l + gz + ylo)) + (yb - 1 - ylo) * n1 + x;
        double Mw0[NL], Mw1[NL], Kw0[NL], Kw1[NL];
#pragma unroll
        for (int yy = 0; yy < TYS + 2; ++yy) {
          const int gy = yb - 1 + yy;
          double Mr[NL], Kr[NL];
          if (IN || (gy >= ylo && gy <= yhi)) {
#pragma unroll
            for (int l = 0; l < NL; ++l)
              row_mk(up[l] + yy * n1, has_l, has_r, m0, m1, k0, k1, Mr[l], Kr[l]);
          } else {
#pragma unroll
            for (int l = 0; l < NL; ++l) Mr[l] = Kr[l] = 0.0;
          }
          if (yy >= 2) {
#pragma unroll
            for (int l = 0; l < NL; ++l) {
              const double ms = Mw0[l] + Mr[l];
              P[yy - 2][l] = m1 * ms + m0 * Mw1[l];
              Q[yy - 2][l] = m1 * (Kw0[l] + Kr[l]) + m0 * Kw1[l] + k1 * ms + k0 * Mw1[l];
            }
          }
#pragma unroll
          for (int l = 0; l < NL; ++l) {
            Mw0[l] = Mw1[l];
            Kw0[l] = Kw1[l];
            Mw1[l] = Mr[l];
            Kw1[l] = Kr[l];
          }
        }
      } else {
#pragma unroll
        for (int o = 0; o < TYS; ++o)
#pragma unroll
          for (int l = 0; l < NL; ++l) P[o][l] = Q[o][l] = 0.0;
      }
      if (zz >= 2) {
        const int zo = zz - 2;  // output plane z0 + zo
        if (IN || zo < planes) {
#pragma unroll
          for (int o = 0; o < TYS; ++o) {
            if (IN || o < trows) {
              double MU[NL], KU[NL], mw = 0.0;
#pragma unroll
              for (int l = 0; l < NL; ++l) {
                const double ms = P0[o][l] + P[o][l];
                MU[l] = m1 * ms + m0 * P1[o][l];
                KU[l] = m1 * (Q0[o][l] + Q[o][l]) + m0 * Q1[o][l] + k1 * ms + k0 * P1[o][l];
                mw += b[l] * MU[l];
              }
              if (!warm) {
                const i64 o0 = n * slab + i64(z0 + zo) * np + i64(yb + o) * n1 + x;
#pragma unroll
                for (int k = 0; k < NL; ++k) {
                  double acc = -(a[k] * mwp[zo][o]);
#pragma unroll
                  for (int l = 0; l < NL; ++l) {
                    acc = fma(MU[l], t.K[k][l], acc);
                    acc = fma(KU[l], t.M[k][l], acc);
                  }
                  double fv = 0.0;
                  if (RES)
                    fv = st[NL * SU + k * SF + zo * RF + (odd & (pn + k + z0 + zo + y0)) +
                            (g * TYS + o) * n1 + x];
                  __stcs(y + o0 + k * nx, RES ? fv - acc : acc);
                }
              }
              mwp[zo][o] = mw;
            }
          }
        }
      }
#pragma unroll
      for (int o = 0; o < TYS; ++o)
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          P0[o][l] = P1[o][l];
          Q0[o][l] = Q1[o][l];
          P1[o][l] = P[o][l];
          Q1[o][l] = Q[o][l];
        }
    }
  };

  int s = 0;
  unsigned ph = 0;
  const int lane = threadIdx.x & 31;
  auto next = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8u * s);
    if (++s == NS) {
      s = 0;
      ph ^= 1u;
    }
  };
  const bool interior = y0 >= 1 && y0 + TY <= n1 - 1 && z0 >= 1 && z0 + TZ <= n1 - 1;
  if (has_prev) {
    mbar_wait(full0, 0);
    march(std::false_type{}, ring, nbeg, true);
    next();
  }
  if (interior) {
    for (i64 n = n0; n < nend; ++n) {
      mbar_wait(full0 + 8u * s, ph);
      march(std::true_type{}, ring + i64(s) * SS, n, false);
      next();
    }
  } else {
    for (i64 n = n0; n < nend; ++n) {
      mbar_wait(full0 + 8u * s, ph);
      march(std::false_type{}, ring + i64(s) * SS, n, false);
      next();
    }
  }
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <int NL, bool RES, int TYS, int YS, int XW>
cudaError_t launch_rows2_t(const LevelView& L, const double* u, const double* f, double* y,
                           const double* ab, cudaStream_t st) {
  constexpr int TY = TYS * YS;
  const int n1 = int(L.sp.n1);
  const int RU = ((TY + 2) * n1 + 2) & ~1;
  const int RF = RES ? (TY * n1 + 2) & ~1 : 0;
  const size_t stage = size_t(NL) * (RU + RF) * sizeof(double);
  static const int ns_env = env_int("STMG_ROWS_NS", 0);
  static const int c_env = env_int("STMG_ROWS_C", 0);
  int NS = ns_env > 0 ? ns_env : 3;
  NS = std::min(NS, kRowsMaxStages);
  while (NS > 2 && 16 + NS * stage > 200 * 1024) --NS;
  const size_t smem = 16 + NS * stage;
  if (smem > 216 * 1024) return cudaErrorNotSupported;
  const i64 bands = (n1 + TY - 1) / TY;
  static PerDeviceOnce attr;
  if (attr.first_use())
    cudaFuncSetAttribute(k_apply_rows2<NL, RES, TYS, YS, XW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024);
  // time chunks: ~32 steps amortise the one-slab warm-up; the chunk count is
  // rounded so that the grid is a whole number of waves of resident CTAs
  // (the C2 residual is a 40 us kernel of ~1 wave: a ragged last wave costs
  // up to half of it)
  static std::atomic<long long> occ_cache{-1};  // (smem << 8) | occ of the last query
  long long oc = occ_cache.load();
  if (oc < 0 || size_t(oc >> 8) != smem) {
    int o = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_apply_rows2<NL, RES, TYS, YS, XW>,
                                                  XW * YS * 32 + 32, smem);
    oc = (static_cast<long long>(smem) << 8) | (o & 255);
    occ_cache.store(oc);
  }
  const int occ = int(oc & 255);
  static const int sms = [] {
    int d = 0, n = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
  }();
  const i64 slots = i64(std::max(occ, 1)) * sms;
  i64 nch;
  if (c_env > 0) {
    nch = (L.n_t + c_env - 1) / c_env;
  } else {
    const i64 want = bands * ((L.n_t + 31) / 32);  // CTAs at 32 steps per chunk
    const i64 waves = std::max<i64>(1, (want + slots / 2) / slots);
    nch = std::max<i64>(1, waves * slots / bands);
    nch = std::min<i64>(nch, std::max<i64>(1, L.n_t / 4));  // >= 4 steps per chunk
  }
  nch = std::min<i64>(std::max<i64>(nch, 1), std::min<i64>(L.n_t, 65535));
  const dim3 g{unsigned(bands), unsigned(nch), 1u};
  const TM<NL> t = make_tm<NL>(L.tc);
  k_apply_rows2<NL, RES, TYS, YS, XW><<<g, XW * YS * 32 + 32, smem, st>>>(
      u, f, y, t, n1, L.sp.h, L.n_t, NS, L.first_global, ab);
  return cudaGetLastError();
}

// Shapes: (rows per thread TYS, sub-bands YS) per width class; STMG_ROWS_CFG
// picks one of the instantiated variants (A/B), default by (n1, NL).
template <int NL, bool RES>
cudaError_t launch_rows2(const LevelView& L, const double* u, const double* f, double* y,
                         const double* ab, cudaStream_t st) {
  const i64 n1 = L.sp.n1;
  static const int cfg_env = env_int("STMG_ROWS_CFG", -1);
  if (n1 <= 128) {
    const int cfg = cfg_env >= 0 ? cfg_env : (NL <= 2 ? 0 : 1);
    switch (cfg) {
      case 0: return launch_rows2_t<NL, RES, 8, 1, 4>(L, u, f, y, ab, st);
      case 1: return launch_rows2_t<NL, RES, 4, 1, 4>(L, u, f, y, ab, st);
      case 2: return launch_rows2_t<NL, RES, 4, 2, 4>(L, u, f, y, ab, st);
      default: return launch_rows2_t<NL, RES, 2, 4, 4>(L, u, f, y, ab, st);
    }
  } else if (n1 <= 256) {
    const int cfg = cfg_env >= 0 ? cfg_env : 0;
    switch (cfg) {
      case 0: return launch_rows2_t<NL, RES, 4, 1, 8>(L, u, f, y, ab, st);
      case 1: return launch_rows2_t<NL, RES, 2, 2, 8>(L, u, f, y, ab, st);
      case 2: return launch_rows2_t<NL, RES, 4, 2, 8>(L, u, f, y, ab, st);
      default: return launch_rows2_t<NL, RES, 2, 1, 8>(L, u, f, y, ab, st);
    }
  } else if (n1 <= 512) {
    const int cfg = cfg_env >= 0 ? cfg_env : 0;
    switch (cfg) {
      case 0: return launch_rows2_t<NL, RES, 4, 1, 16>(L, u, f, y, ab, st);
      default: return launch_rows2_t<NL, RES, 2, 1, 16>(L, u, f, y, ab, st);
    }
  }
  return cudaErrorNotSupported;
}

template <int NL, bool RES, int TYS, int YS, int TZ, int XW>
cudaError_t launch_rows3_t(const LevelView& L, const double* u, const double* f, double* y,
                           const double* ab, cudaStream_t st) {
  constexpr int TY = TYS * YS;
  const int n1 = int(L.sp.n1);
  const int RU = ((TY + 2) * n1 + 2) & ~1;
  const int RF = RES ? (TY * n1 + 2) & ~1 : 0;
  const size_t stage = size_t(NL) * (size_t(TZ + 2) * RU + size_t(TZ) * RF) * sizeof(double);
  static const int ns_env = env_int("STMG_ROWS_NS", 0);
  static const int c_env = env_int("STMG_ROWS_C", 0);
  int NS = ns_env > 0 ? ns_env : 2;
  NS = std::min(NS, kRowsMaxStages);
  while (NS > 2 && 16 + NS * stage > 200 * 1024) --NS;
  const size_t smem = 16 + NS * stage;
  if (smem > 216 * 1024) return cudaErrorNotSupported;
  const i64 bands = i64((n1 + TY - 1) / TY) * ((n1 + TZ - 1) / TZ);
  static PerDeviceOnce attr;
  if (attr.first_use())
    cudaFuncSetAttribute(k_apply_rows3<NL, RES, TYS, YS, TZ, XW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024);
  static std::atomic<long long> occ_cache{-1};  // (smem << 8) | occ of the last query
  long long oc = occ_cache.load();
  if (oc < 0 || size_t(oc >> 8) != smem) {
    int o = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_apply_rows3<NL, RES, TYS, YS, TZ, XW>,
                                                  XW * YS * 32 + 32, smem);
    oc = (static_cast<long long>(smem) << 8) | (o & 255);
    occ_cache.store(oc);
  }
  const int occ = int(oc & 255);
  static const int sms = [] {
    int d = 0, n = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
  }();
  const i64 slots = i64(std::max(occ, 1)) * sms;
  i64 nch;
  if (c_env > 0) {
    nch = (L.n_t + c_env - 1) / c_env;
  } else {
    const i64 want = bands * ((L.n_t + 31) / 32);
    const i64 waves = std::max<i64>(1, (want + slots / 2) / slots);
    nch = std::max<i64>(1, waves * slots / bands);
    nch = std::min<i64>(nch, std::max<i64>(1, L.n_t / 4));
  }
  nch = std::min<i64>(std::max<i64>(nch, 1), std::min<i64>(L.n_t, 65535));
  const dim3 g{unsigned(bands), unsigned(nch), 1u};
  const TM<NL> t = make_tm<NL>(L.tc);
  k_apply_rows3<NL, RES, TYS, YS, TZ, XW><<<g, XW * YS * 32 + 32, smem, st>>>(
      u, f, y, t, n1, L.sp.h, L.n_t, NS, L.first_global, ab);
  return cudaGetLastError();
}

template <int NL, bool RES>
cudaError_t launch_rows3(const LevelView& L, const double* u, const double* f, double* y,
                         const double* ab, cudaStream_t st) {
  const i64 n1 = L.sp.n1;
  static const int cfg_env = env_int("STMG_ROWS_CFG", -1);
  if (n1 <= 64) {
    const int cfg = cfg_env >= 0 ? cfg_env : 3;
    switch (cfg) {
      case 0: return launch_rows3_t<NL, RES, 2, 2, 4, 2>(L, u, f, y, ab, st);
      case 1: return launch_rows3_t<NL, RES, 2, 4, 4, 2>(L, u, f, y, ab, st);
      case 2: return launch_rows3_t<NL, RES, 1, 4, 4, 2>(L, u, f, y, ab, st);
      default: return launch_rows3_t<NL, RES, 2, 2, 2, 2>(L, u, f, y, ab, st);
    }
  } else if (n1 <= 128) {
    const int cfg = cfg_env >= 0 ? cfg_env : 0;
    switch (cfg) {
      case 0: return launch_rows3_t<NL, RES, 2, 2, 4, 4>(L, u, f, y, ab, st);
      default: return launch_rows3_t<NL, RES, 2, 1, 4, 4>(L, u, f, y, ab, st);
    }
  }
  return cudaErrorNotSupported;
}

}  // namespace

// Row-band apply/residual; cudaErrorNotSupported when the level has no such
// kernel (1D, small or very wide grids, unaligned vectors, p_t > 3).
cudaError_t launch_apply_rows(const LevelView& L, const double* u, const double* f, double* y,
                              bool residual, const double* ab, cudaStream_t st) {
  if (L.tc.nl > kFastNL || L.sp.dim < 2) return cudaErrorNotSupported;
  if (L.sp.n1 < (L.sp.dim == 2 ? 96 : 48)) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(u) & 15) != 0) return cudaErrorNotSupported;
  // the 16-byte rounded copy of the vector's last run would read one double
  // past the end when the vector has an odd number of entries (n_t = 1 with an
  // odd number of DG components): leave those to the tile kernels
  if ((L.size() & 1) != 0) return cudaErrorNotSupported;
  if (residual && (reinterpret_cast<uintptr_t>(f) & 15) != 0) return cudaErrorNotSupported;
#define STMG_ROWS_CASE(D, Q, R)                                           \
  case (D) * 16 + (Q) * 2 + (R):                                          \
    return (D) == 2 ? launch_rows2<Q, (R) != 0>(L, u, f, y, ab, st)       \
                    : launch_rows3<Q, (R) != 0>(L, u, f, y, ab, st);
  switch (L.sp.dim * 16 + L.tc.nl * 2 + (residual ? 1 : 0)) {
    STMG_ROWS_CASE(2, 1, 0) STMG_ROWS_CASE(2, 1, 1) STMG_ROWS_CASE(2, 2, 0) STMG_ROWS_CASE(2, 2, 1)
    STMG_ROWS_CASE(2, 3, 0) STMG_ROWS_CASE(2, 3, 1) STMG_ROWS_CASE(2, 4, 0) STMG_ROWS_CASE(2, 4, 1)
    STMG_ROWS_CASE(3, 1, 0) STMG_ROWS_CASE(3, 1, 1) STMG_ROWS_CASE(3, 2, 0) STMG_ROWS_CASE(3, 2, 1)
    STMG_ROWS_CASE(3, 3, 0) STMG_ROWS_CASE(3, 3, 1) STMG_ROWS_CASE(3, 4, 0) STMG_ROWS_CASE(3, 4, 1)
    default: return cudaErrorNotSupported;
  }
#undef STMG_ROWS_CASE
}

}  // namespace stmg
