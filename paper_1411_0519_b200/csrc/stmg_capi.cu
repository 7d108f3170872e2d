// stmg_capi.cu -- context, device memory, cycle driver and the C ABI
// (include/stmg_b200.h).  Host code; kernels live in stmg_kernels.cu.
//
// Solve path (STMG_PATH_SPECTRAL, default): f and u are transformed once to
// orthonormal sine coefficients (dim passes of the batched DST-I kernel), the
// V-cycles run as fused per-mode kernels (k_down / k_up, stmg_kernels.cu)
// captured in a CUDA graph, and u is transformed back at the end.  The
// iteration is the reference's V-cycle (mg.cpp:96-166) in an orthogonal basis:
// identical in exact arithmetic, same stop rule on ||r||_2 (the basis is
// orthonormal, so the norm is the same).
//
// Physical path (STMG_PATH_PHYSICAL): the reference call structure on nodal
// values, one kernel family per reference entry point; used for the operator
// API and as a second GPU implementation in the parity tests.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/stmg_b200.h"
#include "stmg_launch.hpp"
#include "stmg_lfa.hpp"
#include "stmg_setup.hpp"

namespace {

using i64 = int64_t;
thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error in ") + what + " (stmg_capi.cu:" + std::to_string(line) +
                    "): " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x, __LINE__)

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return STMG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return STMG_EINVAL;
  } catch (const std::domain_error& e) {  // lfa: theta_x = 0 (lfa.cpp:207-211)
    g_err = e.what();
    return STMG_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return STMG_ERUNTIME;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// Calls of this library's own C ABI from inside another entry point.
#define CK_ABI(call)                                                   \
  do {                                                                 \
    const int st_ = (call);                                            \
    if (st_ == STMG_EINVAL) throw std::invalid_argument(g_err);        \
    if (st_ != STMG_OK) throw std::runtime_error(g_err);               \
  } while (0)

// Device buffer with `halo` leading slabs (multi-GPU halo exchange lands there).
struct DevBuf {
  double* raw = nullptr;
  double* base = nullptr;
  i64 count = 0;
  // kTailPad zeroed doubles after the vector: the TMA-staged k_updown copies
  // whole 16-byte aligned row runs, which may end up to 2 elements past the
  // last mode
  static constexpr i64 kTailPad = 16;
  void alloc(i64 n, i64 halo_elems) {
    release();
    CK(cudaMalloc(&raw, size_t(n + halo_elems + kTailPad) * sizeof(double)));
    CK(cudaMemset(raw, 0, size_t(n + halo_elems + kTailPad) * sizeof(double)));
    base = raw + halo_elems;
    count = n;
  }
  void release() {
    if (raw) cudaFree(raw);
    raw = base = nullptr;
    count = 0;
  }
};

struct Level {
  stmg::LevelSpec spec;
  stmg::LevelView view;
  double* d_tables = nullptr;  // mval | kval | rfac
  void* d_twiddle = nullptr;
  // spectral V-cycle buffers (allocated on first solve)
  DevBuf F, U[2];
  // physical-path temporaries (allocated on first use)
  DevBuf R, RC, EC, CORR;
};

struct ProfSlot {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;  // eager launches
  size_t used = 0;
  cudaEvent_t ga = nullptr, gb = nullptr;  // pair recorded inside the cycle graph
  bool in_graph = false;
  double total_ms = 0.0;
  i64 launches = 0;
  double bytes = 0.0;
};

}  // namespace

namespace {
struct ShardSet;
}

struct stmg_ctx {
  int device = 0;
  std::unique_ptr<ShardSet> shards;  // time-slab sharding (virtual or NCCL)
  cudaStream_t stream = nullptr;
  std::vector<Level> levels;
  int p_t = 0, dim = 1;
  // p_t > 3: the physical-path operators with a runtime DG size (the fused
  // spectral kernels are compiled for p_t <= 3); every cycle runs there
  bool hi_degree = false;
  // scratch
  DevBuf partials;       // norm partial sums of the spectral cycle (graph-resident)
  DevBuf partials_phys;  // per-step partials of stmg_norm
  double* d_norm = nullptr;
  double* d_hist = nullptr;
  int hist_cap = 0;
  double* h_norm = nullptr;  // pinned
  DevBuf user_f, user_u;     // for stmg_solve_host (and set 0 of the batch)
  // stmg_solve_host_batch: staging sets 1..2 (set 0 = user_f/user_u), copy
  // streams and their events
  static constexpr int kSets = 3;
  DevBuf batch_f[kSets - 1], batch_u[kSets - 1];
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[kSets] = {}, ev_free[kSets] = {};
  cudaEvent_t ev_done = nullptr;
  // graphs of one spectral V-cycle keyed by (cfg, starting buffer parity)
  struct GraphKey {
    int nu1, nu2, gamma, cur0;
    double omega;
    int bs, nu1x, nu2x, gx;
    double omx;
    bool operator<(const GraphKey& o) const {
      if (nu1 != o.nu1) return nu1 < o.nu1;
      if (nu2 != o.nu2) return nu2 < o.nu2;
      if (gamma != o.gamma) return gamma < o.gamma;
      if (cur0 != o.cur0) return cur0 < o.cur0;
      if (omega != o.omega) return omega < o.omega;
      if (bs != o.bs) return bs < o.bs;
      if (nu1x != o.nu1x) return nu1x < o.nu1x;
      if (nu2x != o.nu2x) return nu2x < o.nu2x;
      if (gx != o.gx) return gx < o.gx;
      return omx < o.omx;
    }
  };
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int cur0_after = 0;
    i64 kernels = 0;
  };
  std::map<GraphKey, GraphEntry> graphs;
  std::vector<int> cur;  // current U buffer per level
  // profiling
  bool profile = false;
  ProfSlot prof[6];
  i64 launches = 0;
  bool capturing = false;
  i64 captured_kernels = 0;
  cudaEvent_t ev_solve[2] = {nullptr, nullptr};
  cudaEvent_t ev_host = nullptr;  // host waits for a mapped word, not for the whole stream
  // single-CTA coarse tail (levels >= tail_start), built on first solve
  void* tail_table = nullptr;
  void* tail_host = nullptr;
  int tail_start = -1;
  size_t tail_smem = 0;
  int* d_flag = nullptr;
  int* h_flag = nullptr;  // pinned
  // mailbox: pinned host words the solve path's tiny kernels write directly
  // (k_tiny) instead of cudaMemcpyAsync, so the solve never queues behind a
  // bulk transfer on the copy engines (stmg_solve_host_batch)
  double* h_hist = nullptr;  // pinned, hist_cap entries
  int* h_iter = nullptr;     // pinned
  // device-side solve loop (conditional while node): cached per configuration
  std::map<std::string, cudaGraphExec_t> loops;
  std::map<std::string, i64> loop_kernels;  // kernels per body iteration
  // fused schedule: device ping-pong table {U0[0], U0[1]} and its selector
  double** d_pp = nullptr;
  int* d_par = nullptr;
  std::map<std::string, cudaGraphExec_t> fused_bodies;  // per-cycle graphs (profiling)
  // buffer indices (c->cur, then every shard's cur) a captured loop / body
  // leaves behind; restored when the cached graph is replayed instead of
  // re-captured, so host code after it (the fused suffix) reads the buffers
  // the graph actually wrote
  std::map<std::string, std::vector<std::vector<int>>> cur_after;
  int* d_iter = nullptr;
  double* d_r0 = nullptr;
  bool use_device_loop = true;
  bool use_fused = true;  // fused level-0 schedule for V(1,1) solves
  // a device-loop body may leave its final norm reduction to device_loop,
  // which then launches it fused with the stop test (k_norm_decide)
  i64 pending_norm = -1;  // number of partials, or -1
  // inexact block solver: sine tables per spatial grid level and one
  // workspace (X, B per sub-level) shared by all levels, sized for level 0
  std::map<int, double*> space_tab;
  DevBuf svc_pool;
  // coarse operator: the tail's V(1,1) map F -> U as a dense matrix per omega_t
  std::map<double, double*> cop;
  bool use_cop = true;
  // fused coarse levels csub_a..csub_b (alias-group trees, stmg_kernels.cu)
  stmg::CsubPlan csub;
  int csub_a = -1, csub_b = -1;
  bool csub_decided = false;
  // off by default: slower than the per-level kernels on C2-C5
  // (profiles/r02_csub_ab.txt); STMG_CSUB=1 enables
  bool use_csub = false;
};

namespace {

// ---------------------------------------------------------------- helpers
// Entry points that take a context run on its device and restore the caller's.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const stmg_ctx* c) {
    if (c) enter(c->device);
  }
  explicit DevGuard(int device) { enter(device); }
  void enter(int device) {
    int d = 0;
    if (cudaGetDevice(&d) == cudaSuccess && d != device) {
      prev = d;
      cudaSetDevice(device);
    }
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DevGuard(const DevGuard&) = delete;
  DevGuard& operator=(const DevGuard&) = delete;
};

template <class F>
int cguard(const stmg_ctx* c, F&& fn) {
  return guard([&] {
    DevGuard dg(c);
    fn();
  });
}

Level& lev(stmg_ctx* c, int level) {
  require(c != nullptr, "null context");
  require(level >= 0 && level < int(c->levels.size()), "level index out of range");
  return c->levels[level];
}

void count(stmg_ctx* c, i64 k = 1) {
  if (c->capturing) c->captured_kernels += k;
  else c->launches += k;
}

void prof_begin(stmg_ctx* c, int id) {
  if (!c->profile) return;
  ProfSlot& s = c->prof[id];
  if (c->capturing) {
    CK(cudaEventRecordWithFlags(s.ga, c->stream, cudaEventRecordExternal));
    return;
  }
  if (s.used == s.pool.size()) {
    std::pair<cudaEvent_t, cudaEvent_t> e;
    CK(cudaEventCreate(&e.first));
    CK(cudaEventCreate(&e.second));
    s.pool.push_back(e);
  }
  CK(cudaEventRecord(s.pool[s.used].first, c->stream));
}

void prof_end(stmg_ctx* c, int id, double bytes) {
  if (!c->profile) return;
  ProfSlot& s = c->prof[id];
  s.bytes = bytes;
  if (c->capturing) {
    CK(cudaEventRecordWithFlags(s.gb, c->stream, cudaEventRecordExternal));
    s.in_graph = true;
    return;
  }
  CK(cudaEventRecord(s.pool[s.used].second, c->stream));
  ++s.used;
}

// Collect eager event pairs (after a synchronisation).
void prof_collect(stmg_ctx* c) {
  if (!c->profile) return;
  for (auto& s : c->prof) {
    for (size_t i = 0; i < s.used; ++i) {
      float ms = 0.f;
      CK(cudaEventSynchronize(s.pool[i].second));
      CK(cudaEventElapsedTime(&ms, s.pool[i].first, s.pool[i].second));
      s.total_ms += ms;
      s.launches += 1;
    }
    s.used = 0;
  }
}

// Collect the pairs recorded by one replay of a cycle graph.
void prof_collect_graph(stmg_ctx* c) {
  if (!c->profile) return;
  for (auto& s : c->prof) {
    if (!s.in_graph) continue;
    float ms = 0.f;
    CK(cudaEventSynchronize(s.gb));
    CK(cudaEventElapsedTime(&ms, s.ga, s.gb));
    s.total_ms += ms;
    s.launches += 1;
  }
}

// Sine tables of one grid: mval | kval | rfac (n1 each), then `extra` zeros.
std::vector<double> sine_tables(i64 n1, double h, size_t extra) {
  const double N = double(n1 + 1);
  const i64 G = (n1 + 1) / 2;
  std::vector<double> tab(3 * n1 + extra, 0.0);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (i64 q = 0; q < n1; ++q) {
    const long double th = pi * (long double)(q + 1) / (long double)N;
    const double c = double(std::cos(th));
    const double s2 = double(std::sin(th / 2));
    tab[q] = h / 3.0 * (2.0 + c);             // M1 eigenvalue (h/3)(2 + cos)
    tab[n1 + q] = 4.0 / h * s2 * s2;          // K1 eigenvalue (2/h)(1 - cos)
    const double c2 = double(std::cos(th / 2));
    const double f = 2.0 * c2 * c2 / std::sqrt(2.0);  // (1 + cos)/sqrt(2)
    tab[2 * n1 + q] = q < G - 1 ? f : (q == G - 1 ? 0.0 : -f);
  }
  return tab;
}

void build_level_tables(Level& L) {
  const i64 n1 = L.spec.n1();
  const double h = L.spec.h, N = double(n1 + 1);
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<double> tab = sine_tables(n1, h, 2 * stmg::kMaxNL);
  {  // N_tau = a b^T with a_k = psi_k(0), b_l = psi_l(tau) (Legendre: psi_0 = 1)
    const stmg::DGBlock dg0 = stmg::dg_block(L.spec.p_t, L.spec.tau);
    const int nl = L.spec.p_t + 1;
    for (int k = 0; k < nl; ++k) {
      tab[3 * n1 + k] = dg0.N[k * nl + 0];
      tab[3 * n1 + stmg::kMaxNL + k] = dg0.N[0 * nl + k];
    }
  }
  CK(cudaMalloc(&L.d_tables, tab.size() * sizeof(double)));
  CK(cudaMemcpy(L.d_tables, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
  // twiddles exp(-2 pi i k / L), L = 2N, full circle (k < L; indices in the
  // Stockham passes stay below L)
  std::vector<double> tw(4 * (n1 + 1));
  for (i64 k = 0; k < 2 * (n1 + 1); ++k) {
    const long double a = -pi * (long double)k / (long double)N;
    tw[2 * k] = double(std::cos(a));
    tw[2 * k + 1] = double(std::sin(a));
  }
  CK(cudaMalloc(&L.d_twiddle, tw.size() * sizeof(double)));
  CK(cudaMemcpy(L.d_twiddle, tw.data(), tw.size() * sizeof(double), cudaMemcpyHostToDevice));

  stmg::LevelView& v = L.view;
  v.n_t = L.spec.n_t;
  v.first_global = true;
  v.sp.dim = L.spec.dim;
  v.sp.n1 = n1;
  v.sp.nx = L.spec.nx();
  v.sp.h = h;
  v.sp.mval = L.d_tables;
  v.sp.kval = L.d_tables + n1;
  v.sp.rfac = L.d_tables + 2 * n1;
  const int nl = L.spec.p_t + 1;
  v.tc.nl = nl;
  const stmg::DGBlock dg = stmg::dg_block(L.spec.p_t, L.spec.tau);
  std::vector<double> R1, R2;
  stmg::time_transfer(L.spec.p_t, L.spec.tau, R1, R2);
  for (int k = 0; k < nl; ++k) {
    for (int l = 0; l < nl; ++l) {
      const int i = k * stmg::kMaxNL + l;
      v.tc.K[i] = dg.K[k * nl + l];
      v.tc.M[i] = dg.M[k * nl + l];
      v.tc.N[i] = dg.N[k * nl + l];
      v.tc.R1[i] = R1[k * nl + l];
      v.tc.R2[i] = R2[k * nl + l];
    }
    v.tc.psi0[k] = (k % 2 == 0) ? 1.0 : -1.0;
  }
}

// ------------------------------------------------------- tiny moves (k_tiny)
// Scalar bookkeeping of the solve path (flags, norms, iteration counts, the
// history, the ping-pong table) as one 1-CTA kernel: a copy of `bytes` from
// src, or a 4/8-byte immediate when src is null.  Host-side ends are pinned
// (mapped) words, written over PCIe by the kernel, so nothing on the solve
// path goes through the copy engines.
struct TinyOp {
  void* dst;
  const void* src;
  unsigned long long imm;
  int bytes;
};
struct TinyOps {
  TinyOp op[8];
  int n;
};

__global__ void k_tiny(TinyOps t) {
  for (int k = 0; k < t.n; ++k) {
    const TinyOp o = t.op[k];
    if (o.src) {
      for (int i = threadIdx.x; i < o.bytes / 4; i += blockDim.x)
        static_cast<unsigned*>(o.dst)[i] = static_cast<const unsigned*>(o.src)[i];
    } else if (threadIdx.x == 0) {
      if (o.bytes == 4) *static_cast<unsigned*>(o.dst) = unsigned(o.imm);
      else *static_cast<unsigned long long*>(o.dst) = o.imm;
    }
    __syncthreads();
  }
}

void* mapped(void* h) {
  void* d = nullptr;
  CK(cudaHostGetDevicePointer(&d, h, 0));
  return d;
}

void tiny(stmg_ctx* c, std::initializer_list<TinyOp> ops) {
  TinyOps t{};
  require(ops.size() <= sizeof(t.op) / sizeof(t.op[0]), "internal: too many tiny ops");
  for (const TinyOp& o : ops) {
    require(o.bytes > 0 && o.bytes % 4 == 0 && (o.src || o.bytes <= 8),
            "internal: tiny op size must be a positive multiple of 4 bytes");
    t.op[t.n++] = o;
  }
  k_tiny<<<1, 128, 0, c->stream>>>(t);
  CK(cudaGetLastError());
  count(c);
}

TinyOp to_host(void* h, const void* d, int bytes) { return TinyOp{mapped(h), d, 0ull, bytes}; }
TinyOp set4(void* d, unsigned v) { return TinyOp{d, nullptr, v, 4}; }
TinyOp set8(void* d, unsigned long long v) { return TinyOp{d, nullptr, v, 8}; }
TinyOp copy(void* d, const void* s, int bytes) { return TinyOp{d, s, 0ull, bytes}; }

void ensure(DevBuf& b, i64 n, i64 halo = 0) {
  if (b.count != n) b.alloc(n, halo);
}

// ----------------------------------------------------- physical operators
// out = DST(in) over all axes.  accumulate: out += alpha DST(in); then `in`
// is overwritten (it holds the partial transforms of the first dim-1 axes).
void dst_all(stmg_ctx* c, Level& L, const double* in, double* out, bool accumulate = false,
             double alpha = 1.0) {
  const int dim = L.spec.dim;
  prof_begin(c, 2);
  if (dim == 2) {
    const cudaError_t e =
        stmg::launch_dst2d(L.view, in, out, accumulate, alpha, L.d_twiddle, c->stream);
    if (e != cudaErrorNotSupported) {
      CK(e);
      count(c);
      prof_end(c, 2, 16.0 * double(L.view.size()));  // algorithmic: read + write once
      return;
    }
  }
  double* mid = accumulate ? const_cast<double*>(in) : out;
  for (int a = 0; a < dim; ++a) {
    const bool last = a + 1 == dim;
    CK(stmg::launch_dst_axis(L.view, a, a == 0 ? in : mid, last ? out : mid, last && accumulate,
                             alpha, L.d_twiddle, c->stream));
    count(c);
  }
  prof_end(c, 2, 16.0 * double(L.view.size()));  // algorithmic: read + write once
}

// Exact block solve on every step: x = A^-1 b (x may equal b).  When
// accumulate, u += alpha * A^-1 b instead (x is scratch).
void block_solve(stmg_ctx* c, Level& L, const double* b, double* x, double* acc_into = nullptr,
                 double alpha = 1.0) {
  const int dim = L.spec.dim;
  // forward transform: one-pass cluster kernel where the shape has one (2D,
  // 127-node slabs), else one pass per axis
  cudaError_t e2 = dim == 2 ? stmg::launch_dst2d(L.view, b, x, false, 1.0, L.d_twiddle, c->stream)
                            : cudaErrorNotSupported;
  if (e2 != cudaErrorNotSupported) {
    CK(e2);
    count(c);
  } else {
    CK(stmg::launch_dst_axis(L.view, 0, b, x, false, 1.0, L.d_twiddle, c->stream));
    count(c);
    for (int a = 1; a < dim; ++a) {
      CK(stmg::launch_dst_axis(L.view, a, x, x, false, 1.0, L.d_twiddle, c->stream));
      count(c);
    }
  }
  CK(stmg::launch_modal_solve(L.view, x, c->stream));
  count(c);
  double* out = acc_into ? acc_into : x;
  e2 = dim == 2 ? stmg::launch_dst2d(L.view, x, out, acc_into != nullptr, alpha, L.d_twiddle,
                                     c->stream)
                : cudaErrorNotSupported;
  if (e2 != cudaErrorNotSupported) {
    CK(e2);
    count(c);
    return;
  }
  for (int a = 0; a < dim; ++a) {
    const bool last = a + 1 == dim;
    if (last && acc_into) {
      CK(stmg::launch_dst_axis(L.view, a, x, acc_into, true, alpha, L.d_twiddle, c->stream));
    } else {
      CK(stmg::launch_dst_axis(L.view, a, x, x, false, 1.0, L.d_twiddle, c->stream));
    }
    count(c);
  }
}

void residual(stmg_ctx* c, Level& L, const double* u, const double* f, double* r) {
  prof_begin(c, 3);
  CK(stmg::launch_apply(L.view, u, f, r, true, L.d_tables + 3 * L.spec.n1(), c->stream));
  prof_end(c, 3, 24.0 * double(L.view.size()));
  count(c);
}

void smooth_spectral(stmg_ctx* c, int level, double* u, const double* f, double omega, int nu);

struct Spatial;
void svc_smooth_phys(stmg_ctx* c, int level, double* u, const double* f, double omega, int nu,
                     const Spatial& sp);

void smooth_phys(stmg_ctx* c, int level, double* u, const double* f, double omega, int nu,
                 const Spatial* inexact = nullptr) {
  if (inexact) {
    svc_smooth_phys(c, level, u, f, omega, nu, *inexact);
    return;
  }
  Level& L = c->levels[level];
  if (nu >= 2 && L.spec.p_t + 1 <= stmg::kFastNL) {
    // several sweeps: transform u and f once, sweep in the sine basis (one
    // 24 B/dof pass per sweep, k_smooth), transform back -- 3 transforms
    // instead of 2 per sweep.  Same iteration in an orthonormal basis.
    smooth_spectral(c, level, u, f, omega, nu);
    return;
  }
  ensure(L.R, L.view.size());
  for (int s = 0; s < nu; ++s) {
    prof_begin(c, 5);
    residual(c, L, u, f, L.R.base);
    block_solve(c, L, L.R.base, L.R.base, u, omega);
    prof_end(c, 5, 24.0 * double(L.view.size()));  // the reference's unit: read u, f; write u
  }
}

i64 coarse_n1(const Level& L, int mode) { return mode == 2 ? (L.spec.n1() - 1) / 2 : L.spec.n1(); }

int resolve_mode(const Level& L, int mode) {
  if (mode == 0) mode = L.spec.coarsen;
  require(mode == 1 || mode == 2, "level has no coarser level");
  require(L.spec.n_t % 2 == 0, "restrict_semi requires an even step count");
  if (mode == 2) require(L.spec.space_level > 0, "cannot coarsen the level-0 space grid");
  return mode;
}

void fwdsub_phys(stmg_ctx* c, Level& L, const double* f, double* u) {
  ensure(L.R, L.view.size());
  dst_all(c, L, f, L.R.base);
  CK(stmg::launch_modal_fwdsub(L.view, L.R.base, u, c->stream));
  count(c);
  dst_all(c, L, u, u);
}

const Spatial* phys_spatial(const stmg_cycle_config& cfg);

void phys_cycle(stmg_ctx* c, int level, double* u, const double* f, const stmg_cycle_config& cfg) {
  Level& L = c->levels[level];
  if (level + 1 == int(c->levels.size())) {
    fwdsub_phys(c, L, f, u);
    return;
  }
  const Spatial* ix = phys_spatial(cfg);
  smooth_phys(c, level, u, f, cfg.omega_t, cfg.nu1, ix);
  ensure(L.R, L.view.size());
  residual(c, L, u, f, L.R.base);
  Level& C = c->levels[level + 1];
  ensure(C.RC, C.view.size());
  ensure(C.EC, C.view.size());
  ensure(L.CORR, L.view.size());
  const int mode = L.spec.coarsen;
  CK(stmg::launch_restrict(L.view, mode, C.spec.n1(), L.R.base, C.RC.base, c->stream));
  count(c);
  CK(cudaMemsetAsync(C.EC.base, 0, size_t(C.view.size()) * sizeof(double), c->stream));
  for (int g = 0; g < cfg.gamma; ++g) phys_cycle(c, level + 1, C.EC.base, C.RC.base, cfg);
  CK(stmg::launch_prolong(L.view, mode, C.spec.n1(), C.EC.base, L.CORR.base, c->stream));
  count(c);
  CK(stmg::launch_axpy(u, L.CORR.base, 1.0, L.view.size(), c->stream));
  count(c);
  smooth_phys(c, level, u, f, cfg.omega_t, cfg.nu2, ix);
}

double norm_phys(stmg_ctx* c, Level& L, const double* v) {
  // own buffer: the spectral partials are baked into cached graphs
  ensure(c->partials_phys, std::max<i64>(L.view.n_t, 1));
  CK(stmg::launch_step_sumsq(L.view, v, c->partials_phys.base, c->stream));
  CK(stmg::launch_norm_final(c->partials_phys.base, L.view.n_t, c->d_norm, nullptr, 0, c->stream));
  count(c, 2);
  CK(cudaMemcpyAsync(c->h_norm, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return *c->h_norm;
}

// --------------------------------------------------------- spectral cycle
void ensure_spectral(stmg_ctx* c, int from_level) {
  for (int l = from_level; l < int(c->levels.size()); ++l) {
    Level& L = c->levels[l];
    const i64 n = L.view.size(), halo = 2 * L.view.slab();
    ensure(L.F, n, halo);
    ensure(L.U[0], n, halo);
    ensure(L.U[1], n, halo);
  }
  if (int(c->cur.size()) != int(c->levels.size())) c->cur.assign(c->levels.size(), 0);
  // partial sums: largest (blocks x chunks) grid of the residual-norm kernels
  i64 need = 16;
  for (int l = from_level; l < int(c->levels.size()); ++l) {
    const Level& L = c->levels[l];
    const i64 G = (L.spec.n1() + 1) / 2;
    i64 lanes = 1;
    for (int a = 0; a < L.spec.dim; ++a) lanes *= 2 * G;
    const i64 bx = (std::max(lanes, L.spec.nx()) + 127) / 128;
    const int ch = std::min(stmg::pick_chunk(L.view, true), stmg::pick_chunk(L.view, false));
    need = std::max<i64>(need, bx * ((L.view.n_t + ch - 1) / ch));
  }
  if (c->partials.count < need) {  // grow only; cached graphs bake the pointer in
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
    c->graphs.clear();
    for (auto& kv : c->loops) cudaGraphExecDestroy(kv.second);
    c->loops.clear();
    c->partials.alloc(need, 0);
  }
}

// The suffix of levels whose vectors (f, u, u') fit in one SM's shared
// memory runs inside the single-CTA tail kernel.
constexpr i64 kTailSmemBytes = 180 * 1024;

// First level of the small suffix that runs in the tail kernel (0: none),
// from the level vector sizes (doubles).
int tail_start_from(const std::vector<i64>& sizes, i64* bytes_out) {
  const int nl = int(sizes.size());
  int start = nl;
  i64 bytes = 0;
  while (start - 1 >= 1) {
    const i64 b = 24 * sizes[start - 1];
    if (bytes + b > kTailSmemBytes || nl - (start - 1) > 24) break;
    bytes += b;
    --start;
  }
  if (bytes_out) *bytes_out = bytes;
  return start >= nl ? 0 : start;
}

int tail_start_of(const stmg_ctx* c, i64* bytes_out) {
  std::vector<i64> sizes;
  for (const Level& L : c->levels) sizes.push_back(L.view.size());
  return tail_start_from(sizes, bytes_out);
}

// Gather level of a ladder for S shards: first level with fewer than 2 steps
// per shard, or the first tail level if that comes earlier.
int gather_level_of(const std::vector<stmg::LevelSpec>& specs, int S) {
  const int nl = int(specs.size());
  int lg = nl - 1;
  for (int l = 0; l < nl; ++l)
    if (specs[l].n_t < 2 * S) {
      lg = l;
      break;
    }
  std::vector<i64> sizes;
  for (const auto& L : specs) sizes.push_back(L.size());
  const int ts = tail_start_from(sizes, nullptr);
  if (ts > 0) lg = std::min(lg, ts);
  return lg;
}

// Build the tail's device table (the buffers of levels >= start must exist).
void ensure_tail(stmg_ctx* c) {
  if (c->tail_table || c->tail_start == 0) return;
  const int nl = int(c->levels.size());
  i64 bytes = 0;
  const int start = tail_start_of(c, &bytes);
  if (start == 0) {
    c->tail_start = 0;  // not even the coarsest fits: per-level path
    return;
  }
  std::vector<stmg::TailSpec> spec(nl - start);
  for (int l = start; l < nl; ++l) {
    Level& L = c->levels[l];
    require(L.F.base != nullptr, "internal: tail buffers not allocated");
    stmg::TailSpec& t = spec[l - start];
    t.view = L.view;
    t.mode = L.spec.coarsen;
    t.n1c = (l + 1 < nl) ? c->levels[l + 1].spec.n1() : L.spec.n1();
    t.F = L.F.base;
    t.U0 = L.U[0].base;
    t.U1 = L.U[1].base;
  }
  CK(stmg::build_tail_table(spec.data(), int(spec.size()), &c->tail_table, &c->tail_host));
  c->tail_start = start;
  i64 tab = 0;  // the sine tables are staged too
  for (int l = start; l < nl; ++l) tab += 3 * c->levels[l].spec.n1() * i64(sizeof(double));
  c->tail_smem = size_t(bytes + tab);
}

// ---- fused coarse levels ---------------------------------------------------
// Levels a..b of a V(1,1) cycle (zero initial guess) run as two launches
// (k_csub_down / k_csub_up) when they are small enough to be latency bound:
// a = the first coarse level (>= 1) with at most kCsubMaxDofs unknowns,
// b = the last level before the tail (or before the first level that is not
// fully coarsened), at most kCsubMaxDepth levels.  Env: STMG_CSUB=0 disables,
// STMG_CSUB_DEPTH / STMG_CSUB_LANES / STMG_CSUB_THREADS tune.
constexpr i64 kCsubMaxDofs = i64(4) << 20;

void ensure_csub(stmg_ctx* c) {
  if (c->csub_decided) return;
  c->csub_decided = true;
  if (!c->use_csub) return;
  const int nl = int(c->levels.size());
  int a = -1;
  i64 maxdofs = kCsubMaxDofs;
  if (const char* e = std::getenv("STMG_CSUB_MAXDOFS")) maxdofs = std::atoll(e);
  for (int l = 1; l < nl; ++l)
    if (c->levels[l].view.size() <= maxdofs) {
      a = l;
      break;
    }
  if (a < 0) return;
  int depth = 3;
  if (const char* e = std::getenv("STMG_CSUB_DEPTH")) depth = std::atoi(e);
  int b = a - 1;
  const int stop = (c->tail_table && c->tail_start > 0) ? c->tail_start : nl - 1;
  while (b + 1 < stop && b + 1 - a < depth && c->levels[b + 1].spec.coarsen == 2 &&
         c->levels[b + 1].F.base && c->levels[b + 2].F.base)
    ++b;
  if (b < a || b + 1 >= nl) return;
  std::vector<stmg::CsubSpec> spec(b + 2 - a);
  for (int l = a; l <= b + 1; ++l) {
    Level& L = c->levels[l];
    stmg::CsubSpec& q = spec[l - a];
    q.view = L.view;
    q.n1c = (l + 1 < nl) ? c->levels[l + 1].spec.n1() : L.spec.n1();
    q.F = L.F.base;
    q.U0 = L.U[0].base;
    q.U1 = L.U[1].base;
  }
  int lanes = 64;
  if (const char* e = std::getenv("STMG_CSUB_LANES")) lanes = std::atoi(e);
  CK(stmg::build_csub(spec.data(), int(spec.size()), lanes, &c->csub));
  if (const char* e = std::getenv("STMG_CSUB_THREADS")) c->csub.threads = std::atoi(e);
  c->csub_a = a;
  c->csub_b = b;
}

// ---- coarse operator ------------------------------------------------------
// The tail (levels >= tail_start, V(1,1), zero initial guess) is a fixed
// linear map F -> U of the tail's first level.  When that level has at most
// kCopMax unknowns it is precomputed once per omega_t (column i = the tail
// kernel applied to e_i) and applied as one multi-CTA GEMV, which replaces the
// tail's ~20 dependent single-CTA phases.  Exact in exact arithmetic;
// rounding-level differences only (tests: STMG_COARSE_OP=0 vs 1).
constexpr i64 kCopMax = 3200;

i64 cop_size(const stmg_ctx* c) {
  if (c->tail_start <= 0) return 0;
  return c->levels[c->tail_start].view.size();
}

bool v11_exact(const stmg_cycle_config& cfg) {
  return cfg.path == STMG_PATH_SPECTRAL && cfg.block_solver == STMG_BLOCK_EXACT && cfg.nu1 == 1 &&
         cfg.nu2 == 1 && cfg.gamma == 1;
}

void launch_tail_kernel(stmg_ctx* c, double omega) {
  CK(stmg::launch_tail(c->dim, c->p_t + 1, c->tail_table, c->tail_host,
                       int(c->levels.size()) - c->tail_start, omega, c->tail_smem, c->stream));
  count(c);
}

// Build the operator for omega (outside any graph capture).
void ensure_cop(stmg_ctx* c, double omega) {
  if (!c->use_cop || !c->tail_table || c->cop.count(omega)) return;
  const i64 n = cop_size(c);
  if (n <= 0 || n > kCopMax) return;
  double* B = nullptr;
  CK(cudaMalloc(&B, size_t(n * n) * sizeof(double)));
  // one launch: CTA i runs the tail kernel on e_i and writes column i
  CK(stmg::launch_tail(c->dim, c->p_t + 1, c->tail_table, c->tail_host,
                       int(c->levels.size()) - c->tail_start, omega, c->tail_smem, c->stream, B,
                       n));
  count(c);
  CK(cudaStreamSynchronize(c->stream));
  c->cop[omega] = B;
}

// The tail of a V(1,1) cycle: the coarse operator if built, else the kernel.
void run_tail(stmg_ctx* c, double omega) {
  auto it = c->cop.find(omega);
  if (it != c->cop.end()) {
    Level& T = c->levels[c->tail_start];
    CK(stmg::launch_cop_gemv(it->second, T.F.base, T.U[0].base, int(cop_size(c)), c->stream));
    count(c);
  } else {
    launch_tail_kernel(c, omega);
  }
  for (int l = c->tail_start; l < int(c->levels.size()); ++l) c->cur[l] = 0;
}

stmg::ModalArgs modal_args(const Level& L, const Level* C, double omega, bool grouped) {
  stmg::ModalArgs a;
  a.omega = omega;
  a.chunk = stmg::pick_chunk(L.view, grouped);
  a.mode = L.spec.coarsen ? L.spec.coarsen : 1;
  a.n1c = C ? C->spec.n1() : L.spec.n1();
  a.block = stmg::pick_updown_block(L.view, stmg::pick_chunk(L.view, true), a.mode);
  return a;
}

// nu damped block-Jacobi sweeps of the physical vectors u, f through the sine
// basis (the level's spectral buffers are scratch here; a solve re-fills them).
void smooth_spectral(stmg_ctx* c, int level, double* u, const double* f, double omega, int nu) {
  Level& L = c->levels[level];
  const i64 n = L.view.size(), halo = 2 * L.view.slab();
  ensure(L.F, n, halo);
  ensure(L.U[0], n, halo);
  ensure(L.U[1], n, halo);
  dst_all(c, L, f, L.F.base);
  dst_all(c, L, u, L.U[0].base);
  int cur = 0;
  for (int s = 0; s < nu; ++s) {
    stmg::ModalArgs a = modal_args(L, nullptr, omega, false);
    CK(stmg::launch_smooth(L.view, a, false, L.F.base, L.U[cur].base, L.U[1 - cur].base,
                           c->stream));
    count(c);
    cur = 1 - cur;
  }
  dst_all(c, L, L.U[cur].base, u);
}

// Enqueue one gamma-cycle from `level` on the spectral buffers.  zero_guess:
// the level's iterate is 0 (coarse levels).  want_resid: compute the residual
// norm partials of the finest result (returns their count via *np).
void inexact_cycle(stmg_ctx* c, int level, bool zero_guess, const stmg_cycle_config& cfg,
                   bool want_resid, i64* np);

void spectral_cycle(stmg_ctx* c, int level, bool zero_guess, const stmg_cycle_config& cfg,
                    bool want_resid, i64* np) {
  if (cfg.block_solver == STMG_BLOCK_VCYCLE) {
    inexact_cycle(c, level, zero_guess, cfg, want_resid, np);
    return;
  }
  if (zero_guess && !want_resid && level == c->csub_a && v11_exact(cfg)) {
    // levels a..b fused: down pass, the levels below b, up pass
    CK(stmg::launch_csub(c->csub, false, cfg.omega_t, c->stream));
    count(c);
    const int nb = c->csub_b + 1;
    if (c->tail_table && nb == c->tail_start) run_tail(c, cfg.omega_t);
    else spectral_cycle(c, nb, true, cfg, false, nullptr);
    CK(stmg::launch_csub(c->csub, true, cfg.omega_t, c->stream));
    count(c);
    for (int l = c->csub_a; l <= c->csub_b; ++l) c->cur[l] = 0;
    return;
  }
  Level& L = c->levels[level];
  int& cur = c->cur[level];
  if (zero_guess) cur = 0;
  const bool last = level + 1 == int(c->levels.size());
  if (last) {
    CK(stmg::launch_modal_fwdsub(L.view, L.F.base, L.U[cur].base, c->stream));
    count(c);
    if (want_resid) {
      stmg::ModalArgs a = modal_args(L, nullptr, cfg.omega_t, false);
      CK(stmg::launch_resnorm(L.view, a, L.U[cur].base, L.F.base, c->partials.base, c->stream));
      count(c);
      *np = a.n_partials;
    }
    return;
  }
  Level& C = c->levels[level + 1];
  const int nu1 = std::max(cfg.nu1, 0), nu2 = std::max(cfg.nu2, 0);
  // pre-smoothing: nu1-1 plain sweeps, the last fused with residual+restriction
  for (int s = 0; s + 1 < nu1; ++s) {
    stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, false);
    CK(stmg::launch_smooth(L.view, a, zero_guess, L.F.base, L.U[cur].base, L.U[1 - cur].base,
                           c->stream));
    count(c);
    cur ^= 1;
    zero_guess = false;
  }
  {
    stmg::ModalArgs a = modal_args(L, &C, nu1 > 0 ? cfg.omega_t : 0.0, true);
    if (level == 0) prof_begin(c, 0);
    CK(stmg::launch_down(L.view, a, zero_guess, L.F.base, L.U[cur].base, L.U[1 - cur].base,
                         C.F.base, c->stream));
    if (level == 0)
      prof_end(c, 0, 8.0 * double((zero_guess ? 2 : 3) * L.view.size() + C.view.size()));
    count(c);
    cur ^= 1;
  }
  const bool fused = nu1 == 1 && nu2 == 1 && cfg.gamma == 1;
  if (fused && c->tail_table && level + 1 == c->tail_start) {
    run_tail(c, cfg.omega_t);
  } else {
    for (int g = 0; g < std::max(cfg.gamma, 1); ++g)
      spectral_cycle(c, level + 1, g == 0, cfg, false, nullptr);
  }
  // prolong + correct + first post-sweep (+ residual norm on the finest level)
  const bool fuse_resid = want_resid && nu2 <= 1;
  {
    stmg::ModalArgs a = modal_args(L, &C, nu2 > 0 ? cfg.omega_t : 0.0, true);
    if (level == 0) prof_begin(c, 1);
    CK(stmg::launch_up(L.view, a, C.U[c->cur[level + 1]].base, L.U[cur].base, L.F.base,
                       L.U[1 - cur].base, fuse_resid ? c->partials.base : nullptr, c->stream));
    if (level == 0) prof_end(c, 1, 8.0 * double(3 * L.view.size() + C.view.size()));
    count(c);
    if (fuse_resid) *np = a.n_partials;
    cur ^= 1;
  }
  for (int s = 1; s < nu2; ++s) {
    stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, false);
    CK(stmg::launch_smooth(L.view, a, false, L.F.base, L.U[cur].base, L.U[1 - cur].base,
                           c->stream));
    count(c);
    cur ^= 1;
  }
  if (want_resid && !fuse_resid) {
    stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, false);
    CK(stmg::launch_resnorm(L.view, a, L.U[cur].base, L.F.base, c->partials.base, c->stream));
    count(c);
    *np = a.n_partials;
  }
}

// ------------------------------------------- inexact block solver (f2)
// SpatialVCycleSolver (smoother.cpp:8-78) on every time step of a level, in
// the sine basis (kernels: stmg_spatial.cu).  Sub-level sigma = 0..s of a
// level with space level s is the grid of level s - sigma; the workspace
// holds X_sigma, B_sigma for every sub-level.
struct Spatial {
  double omega_x = 2.0 / 3.0;
  int nu1_x = 2, nu2_x = 2, gamma_x = 1;
};

Spatial spatial_of(const stmg_cycle_config& c) { return {c.omega_x, c.nu1_x, c.nu2_x, c.gamma_x}; }
Spatial spatial_of(const stmg_smoother_config& c) {
  return {c.omega_x, c.nu1_x, c.nu2_x, c.gamma_x};
}

const double* space_tables(stmg_ctx* c, int g) {
  auto it = c->space_tab.find(g);
  if (it != c->space_tab.end()) return it->second;
  const i64 n1 = (i64(1) << (g + 1)) - 1;
  const std::vector<double> tab = sine_tables(n1, std::ldexp(1.0, -(g + 1)), 0);
  double* d = nullptr;
  CK(cudaMalloc(&d, tab.size() * sizeof(double)));
  CK(cudaMemcpy(d, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
  c->space_tab[g] = d;
  return d;
}

// Kronecker diagonals of M_h and K_h on grid level g (uniform grid: one value
// each, smoother.cpp:16-20): M(0,0) = md^dim, K(0,0) = dim kd md^(dim-1).
void space_diag(int dim, int g, double& md, double& kd) {
  const double h = std::ldexp(1.0, -(g + 1));
  const double m1 = 4.0 * h / 6.0, k1 = 2.0 / h;
  md = std::pow(m1, dim);
  kd = dim * k1 * std::pow(m1, dim - 1);
}

stmg::SvcArgs svc_args(stmg_ctx* c, int dim, int g, const Spatial& sp, int nu) {
  stmg::SvcArgs a;
  const i64 n1 = (i64(1) << (g + 1)) - 1;
  const double* tab = space_tables(c, g);
  a.sp.dim = dim;
  a.sp.n1 = n1;
  a.sp.nx = 1;
  for (int d = 0; d < dim; ++d) a.sp.nx *= n1;
  a.sp.h = std::ldexp(1.0, -(g + 1));
  a.sp.mval = tab;
  a.sp.kval = tab + n1;
  a.sp.rfac = tab + 2 * n1;
  a.n1c = g > 0 ? (i64(1) << g) - 1 : 1;
  space_diag(dim, g, a.md, a.kd);
  space_diag(dim, 0, a.mc, a.kc);  // the 1-node grid: its block is diagonal
  a.omega_x = sp.omega_x;
  a.nu = nu;
  return a;
}

// Workspace doubles of level L's sub-levels (X and B each).
i64 svc_sub_size(const Level& L, int sigma) {
  const int g = L.spec.space_level - sigma;
  i64 nx = 1;
  for (int d = 0; d < L.spec.dim; ++d) nx *= (i64(1) << (g + 1)) - 1;
  return L.spec.n_t * (L.spec.p_t + 1) * nx;
}

struct SvcBufs {
  std::vector<double*> X, B;
};

SvcBufs svc_bufs(stmg_ctx* c, const Level& L) {
  if (!c->svc_pool.base) {  // once, for the largest level (never grows: graphs bake pointers)
    i64 need = 0;
    for (const Level& K : c->levels) {
      i64 t = 0;
      for (int sg = 0; sg <= K.spec.space_level; ++sg) t += 2 * svc_sub_size(K, sg);
      need = std::max(need, t);
    }
    c->svc_pool.alloc(need, 0);
  }
  SvcBufs b;
  double* p = c->svc_pool.base;
  for (int sg = 0; sg <= L.spec.space_level; ++sg) {
    const i64 n = svc_sub_size(L, sg);
    b.X.push_back(p);
    b.B.push_back(p + n);
    p += 2 * n;
  }
  require(p - c->svc_pool.base <= c->svc_pool.count, "internal: spatial workspace too small");
  return b;
}

// Workspace and sine tables of every grid, outside any graph capture.
void ensure_svc(stmg_ctx* c, const stmg_cycle_config& cfg) {
  if (cfg.block_solver != STMG_BLOCK_VCYCLE) return;
  svc_bufs(c, c->levels[0]);
  for (int g = 0; g <= c->levels[0].spec.space_level; ++g) space_tables(c, g);
}

// One spatial cycle per time step of level L.  f != null: B_0 = f - L u (u =
// u_in, sine basis); else B_0 is set by the caller.  zero0: X_0 starts at 0
// (else the caller set it).  u_final != null: u_final += omega_t x, else the
// result is left in X_0.
void svc_run(stmg_ctx* c, Level& L, const Spatial& sp, const double* f, const double* u_in,
             double* u_final, bool zero0, double omega_t) {
  const SvcBufs w = svc_bufs(c, L);
  const int s = L.spec.space_level, dim = L.spec.dim;
  if (s == 0) {
    const stmg::SvcArgs a = svc_args(c, dim, 0, sp, 0);
    CK(stmg::launch_svc_direct(L.view, a, f != nullptr, f, u_in, w.B[0], w.X[0], u_final, omega_t,
                               c->stream));
    count(c);
    return;
  }
  std::function<void(int, bool)> rec = [&](int sg, bool zero) {
    const int g = s - sg;
    const bool to_c = g - 1 == 0;
    const stmg::SvcArgs down = svc_args(c, dim, g, sp, sp.nu1_x);
    CK(stmg::launch_svc_down(L.view, down, sg == 0 && f, zero, to_c, f, u_in, w.B[sg], w.X[sg],
                             to_c ? w.X[sg + 1] : w.B[sg + 1], c->stream));
    count(c);
    if (!to_c)
      for (int k = 0; k < sp.gamma_x; ++k) rec(sg + 1, k == 0);
    const stmg::SvcArgs up = svc_args(c, dim, g, sp, sp.nu2_x);
    CK(stmg::launch_svc_up(L.view, up, w.X[sg + 1], w.B[sg], w.X[sg], sg == 0 ? u_final : nullptr,
                           omega_t, c->stream));
    count(c);
  };
  rec(0, zero0);
}

// block_jacobi_step with spatial-V-cycle blocks on the spectral iterate.
void svc_smooth_spectral(stmg_ctx* c, Level& L, const Spatial& sp, const double* f, double* u,
                         double omega_t, int nu) {
  for (int k = 0; k < nu; ++k) svc_run(c, L, sp, f, u, u, true, omega_t);
}

// mg_cycle (mg.cpp:96-132) on the sine coefficients with inexact block
// solves: smoothing by svc_smooth_spectral; residual + restriction and
// prolongation + correction by the fused level kernels with omega = 0
// (their smoothing sweep is then the identity).
void inexact_cycle(stmg_ctx* c, int level, bool zero_guess, const stmg_cycle_config& cfg,
                   bool want_resid, i64* np) {
  Level& L = c->levels[level];
  int& cur = c->cur[level];
  const Spatial sp = spatial_of(cfg);
  if (zero_guess) {
    cur = 0;
    CK(cudaMemsetAsync(L.U[0].base, 0, size_t(L.view.size()) * sizeof(double), c->stream));
  }
  if (level + 1 == int(c->levels.size())) {
    CK(stmg::launch_modal_fwdsub(L.view, L.F.base, L.U[cur].base, c->stream));
    count(c);
    if (want_resid) {
      stmg::ModalArgs a = modal_args(L, nullptr, cfg.omega_t, false);
      CK(stmg::launch_resnorm(L.view, a, L.U[cur].base, L.F.base, c->partials.base, c->stream));
      count(c);
      *np = a.n_partials;
    }
    return;
  }
  Level& C = c->levels[level + 1];
  svc_smooth_spectral(c, L, sp, L.F.base, L.U[cur].base, cfg.omega_t, std::max(cfg.nu1, 0));
  {
    stmg::ModalArgs a = modal_args(L, &C, 0.0, true);
    CK(stmg::launch_down(L.view, a, false, L.F.base, L.U[cur].base, L.U[1 - cur].base, C.F.base,
                         c->stream));
    count(c);
    cur ^= 1;
  }
  for (int g = 0; g < std::max(cfg.gamma, 1); ++g)
    inexact_cycle(c, level + 1, g == 0, cfg, false, nullptr);
  {
    stmg::ModalArgs a = modal_args(L, &C, 0.0, true);
    CK(stmg::launch_up(L.view, a, C.U[c->cur[level + 1]].base, L.U[cur].base, L.F.base,
                       L.U[1 - cur].base, nullptr, c->stream));
    count(c);
    cur ^= 1;
  }
  svc_smooth_spectral(c, L, sp, L.F.base, L.U[cur].base, cfg.omega_t, std::max(cfg.nu2, 0));
  if (want_resid) {
    stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, false);
    CK(stmg::launch_resnorm(L.view, a, L.U[cur].base, L.F.base, c->partials.base, c->stream));
    count(c);
    *np = a.n_partials;
  }
}

void check_spatial(double omega_x, int nu1_x, int nu2_x, int gamma_x) {
  require(nu1_x >= 0 && nu2_x >= 0, "spatial smoothing step counts must be >= 0");
  require(gamma_x >= 1, "gamma_x must be >= 1");
  require(std::isfinite(omega_x), "omega_x must be finite");
}

// Physical path: residual -> DST -> spatial cycles -> inverse DST, u += w x.
void svc_smooth_phys(stmg_ctx* c, int level, double* u, const double* f, double omega, int nu,
                     const Spatial& sp) {
  Level& L = c->levels[level];
  ensure(L.R, L.view.size());
  for (int k = 0; k < nu; ++k) {
    residual(c, L, u, f, L.R.base);
    const SvcBufs w = svc_bufs(c, L);
    dst_all(c, L, L.R.base, w.B[0]);
    svc_run(c, L, sp, nullptr, nullptr, nullptr, true, omega);
    dst_all(c, L, w.X[0], u, true, omega);
  }
}

const Spatial* phys_spatial(const stmg_cycle_config& cfg) {
  static thread_local Spatial sp;
  if (cfg.block_solver != STMG_BLOCK_VCYCLE) return nullptr;
  sp = spatial_of(cfg);
  return &sp;
}

void check_cfg(const stmg_cycle_config* cfg) {
  require(cfg != nullptr, "null cycle config");
  require(cfg->nu1 >= 0 && cfg->nu2 >= 0, "smoothing step counts must be >= 0");
  require(cfg->gamma >= 1, "gamma must be >= 1");
  require(cfg->path == STMG_PATH_SPECTRAL || cfg->path == STMG_PATH_PHYSICAL, "unknown cycle path");
  require(cfg->block_solver == STMG_BLOCK_EXACT || cfg->block_solver == STMG_BLOCK_VCYCLE,
          "block_solver must be 'exact' or 'vcycle'");
  if (cfg->block_solver == STMG_BLOCK_VCYCLE)
    check_spatial(cfg->omega_x, cfg->nu1_x, cfg->nu2_x, cfg->gamma_x);
}

// The cycle configuration a context actually runs: p_t > 3 takes the
// physical path (same iteration, reference call structure).
stmg_cycle_config effective_cfg(const stmg_ctx* c, const stmg_cycle_config& cfg) {
  stmg_cycle_config e = cfg;
  if (c->hi_degree) {
    require(cfg.block_solver == STMG_BLOCK_EXACT,
            "spatial V-cycle block solves support p_t <= 3 on the B200 path");
    e.path = STMG_PATH_PHYSICAL;
  }
  return e;
}

void ensure_hist(stmg_ctx* c, int n) {
  if (c->hist_cap >= n) return;
  n = std::max(n, 1024);
  // every cached loop and fused body bakes d_hist in (k_decide / k_norm_decide)
  for (auto& kv : c->loops) cudaGraphExecDestroy(kv.second);
  c->loops.clear();
  for (auto& kv : c->fused_bodies) cudaGraphExecDestroy(kv.second);
  c->fused_bodies.clear();
  c->cur_after.clear();
  if (c->d_hist) cudaFree(c->d_hist);
  if (c->h_hist) cudaFreeHost(c->h_hist);
  c->h_hist = nullptr;
  CK(cudaMalloc(&c->d_hist, size_t(n) * sizeof(double)));
  CK(cudaMallocHost(&c->h_hist, size_t(n) * sizeof(double)));
  c->hist_cap = n;
}

// Residual norm of the spectral iterate at level 0 (synchronising).
// Enqueue only: the norm lands in d_norm and (mapped) h_norm; ev_host marks it.
void spectral_resnorm_async(stmg_ctx* c, int level, bool u_zero) {
  Level& L = c->levels[level];
  stmg::ModalArgs a = modal_args(L, nullptr, 0.5, false);
  CK(stmg::launch_resnorm(L.view, a, L.U[c->cur[level]].base, L.F.base, c->partials.base,
                          c->stream, u_zero));
  CK(stmg::launch_norm_final(c->partials.base, a.n_partials, c->d_norm, nullptr, 0, c->stream));
  count(c, 2);
  tiny(c, {to_host(c->h_norm, c->d_norm, 8)});
  CK(cudaEventRecord(c->ev_host, c->stream));
}

double spectral_resnorm(stmg_ctx* c, int level, bool u_zero = false) {
  spectral_resnorm_async(c, level, u_zero);
  CK(cudaEventSynchronize(c->ev_host));
  return *c->h_norm;
}

// One full V-cycle from level 0 + residual norm into d_norm/h_norm, as a
// captured graph (replayed every iteration).
stmg_ctx::GraphEntry& cycle_graph(stmg_ctx* c, const stmg_cycle_config& cfg) {
  const bool ix = cfg.block_solver == STMG_BLOCK_VCYCLE;
  stmg_ctx::GraphKey key{cfg.nu1,          cfg.nu2,           cfg.gamma,         c->cur[0],
                         cfg.omega_t,      cfg.block_solver,  ix ? cfg.nu1_x : 0, ix ? cfg.nu2_x : 0,
                         ix ? cfg.gamma_x : 0, ix ? cfg.omega_x : 0.0};
  auto it = c->graphs.find(key);
  if (it != c->graphs.end()) return it->second;
  const int cur0 = c->cur[0];
  cudaGraph_t graph;
  c->capturing = true;
  c->captured_kernels = 0;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    i64 np = 0;
    spectral_cycle(c, 0, false, cfg, true, &np);
    CK(stmg::launch_norm_final(c->partials.base, np, c->d_norm, nullptr, 0, c->stream));
    count(c);
    CK(cudaMemcpyAsync(c->h_norm, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  } catch (...) {
    cudaStreamEndCapture(c->stream, &graph);
    c->capturing = false;
    throw;
  }
  CK(cudaStreamEndCapture(c->stream, &graph));
  c->capturing = false;
  stmg_ctx::GraphEntry e;
  CK(cudaGraphInstantiate(&e.exec, graph, 0));
  CK(cudaGraphDestroy(graph));
  e.cur0_after = c->cur[0];
  e.kernels = c->captured_kernels;
  c->cur[0] = cur0;
  return c->graphs[key] = e;
}

std::vector<std::vector<int>> cur_snapshot(const stmg_ctx* c);
void cur_restore(stmg_ctx* c, const std::vector<std::vector<int>>& s);

// Buffer flips of the finest level per V-cycle (each sweep ping-pongs).
int nu_flips(const stmg_cycle_config& cfg) { return std::max(cfg.nu1, 1) + std::max(cfg.nu2, 1); }

// The whole iteration as one graph: a conditional WHILE node whose body is a
// V-cycle + residual norm + the device-side stop test (k_decide), so the host
// does not synchronise per cycle.  Requires the cycle to leave the finest
// iterate in the buffer it started from (true for V(1,1), any nu1 + nu2 even).
template <class Body>
cudaGraphExec_t device_loop(stmg_ctx* c, const std::string& key, double eps, int max_iter,
                            Body&& body, int* parity = nullptr) {
  auto it = c->loops.find(key);
  if (it != c->loops.end()) {
    cur_restore(c, c->cur_after.at(key));
    return it->second;
  }
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t bodyg = np.conditional.phGraph_out[0];
  c->capturing = true;
  c->captured_kernels = 0;
  CK(cudaStreamBeginCaptureToGraph(c->stream, bodyg, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  try {
    c->pending_norm = -1;
    body();
    if (c->pending_norm >= 0)
      CK(stmg::launch_norm_decide(c->partials.base, c->pending_norm, c->d_norm, h, c->d_r0,
                                  c->d_hist, c->d_iter, eps, max_iter, parity, c->stream));
    else
      CK(stmg::launch_decide(h, c->d_norm, c->d_r0, c->d_hist, c->d_iter, eps, max_iter, parity,
                             c->stream));
    c->pending_norm = -1;
    count(c);
  } catch (...) {
    c->pending_norm = -1;
    cudaGraph_t dummy;
    cudaStreamEndCapture(c->stream, &dummy);
    c->capturing = false;
    cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t captured;
  CK(cudaStreamEndCapture(c->stream, &captured));
  c->capturing = false;
  cudaGraphExec_t exec;
  CK(cudaGraphInstantiate(&exec, g, 0));
  CK(cudaGraphDestroy(g));
  c->loops[key] = exec;
  c->loop_kernels[key] = c->captured_kernels;
  c->cur_after[key] = cur_snapshot(c);
  return exec;
}

std::string loop_key(const char* kind, const stmg_cycle_config& cfg, int cur0, double eps,
                     int max_iter) {
  char b[256];
  std::snprintf(b, sizeof(b), "%s/%d/%d/%d/%.17g/%d/%.17g/%d", kind, cfg.nu1, cfg.nu2, cfg.gamma,
                cfg.omega_t, cur0, eps, max_iter);
  std::string k(b);
  if (cfg.block_solver == STMG_BLOCK_VCYCLE) {
    std::snprintf(b, sizeof(b), "/vc/%d/%d/%d/%.17g", cfg.nu1_x, cfg.nu2_x, cfg.gamma_x,
                  cfg.omega_x);
    k += b;
  }
  return k;
}

// Run the remaining cycles on the device; fills r and history from the device.
void run_device_loop(stmg_ctx* c, cudaGraphExec_t exec, int max_iter, double* history,
                     int history_cap, int* nh, stmg_solve_report& r, double eps) {
  tiny(c, {set4(c->d_iter, 0u)});
  CK(cudaGraphLaunch(exec, c->stream));
  tiny(c, {to_host(c->h_iter, c->d_iter, 4),
           to_host(c->h_hist, c->d_hist, (max_iter + 1) * int(sizeof(double)))});
  CK(cudaStreamSynchronize(c->stream));
  const int it = *c->h_iter;
  const std::vector<double> h(c->h_hist, c->h_hist + it + 1);
  for (int k = 1; k <= it; ++k) {
    if (history && *nh < history_cap) history[*nh] = h[k];
    ++*nh;
  }
  r.iterations = it;
  r.r_final = it > 0 ? h[it] : r.r0;
  r.converged = (it > 0 && h[it] <= eps * r.r0) ? 1 : 0;
  (void)max_iter;
}

// ---- fused V(1,1) schedule: one pass over level 0 per cycle ----------------
// prefix: down(0) of cycle 1; then per cycle k: coarse levels of cycle k,
// k_updown (post-smooth k + stop-test residual + pre-smooth/restrict k+1),
// norm, stop test (+ swap of the level-0 buffers); suffix: up(0) of the last
// cycle recomputed from its inputs (still intact) to produce the result.
bool fused_eligible(const stmg_ctx* c, const stmg_cycle_config& cfg) {
  return c->use_fused && cfg.path == STMG_PATH_SPECTRAL && cfg.block_solver == STMG_BLOCK_EXACT &&
         cfg.nu1 == 1 && cfg.nu2 == 1 &&
         cfg.gamma == 1 && c->levels.size() >= 2 && c->levels[0].spec.coarsen != 0;
}

// Coarse part (levels >= 1) of one V(1,1) cycle, zero initial guess.
void coarse_cycle(stmg_ctx* c, const stmg_cycle_config& cfg) {
  if (c->tail_table && c->tail_start == 1) {
    run_tail(c, cfg.omega_t);
  } else {
    spectral_cycle(c, 1, true, cfg, false, nullptr);
  }
}

// One fused cycle body (captured): coarse(k), k_updown, norm.
void fused_body(stmg_ctx* c, const stmg_cycle_config& cfg, i64* np, bool defer_norm = false) {
  Level& L = c->levels[0];
  Level& C = c->levels[1];
  prof_begin(c, 4);
  coarse_cycle(c, cfg);
  prof_end(c, 4, 0.0);
  stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, true);
  prof_begin(c, 0);
  CK(stmg::launch_updown(L.view, a, C.U[c->cur[1]].base, c->d_pp, c->d_par, L.F.base, C.F.base,
                         c->partials.base, c->stream));
  prof_end(c, 0, 8.0 * double(3 * L.view.size() + 2 * C.view.size()));
  count(c);
  *np = a.n_partials;
  if (defer_norm) {
    c->pending_norm = *np;
    return;
  }
  CK(stmg::launch_norm_final(c->partials.base, *np, c->d_norm, nullptr, 0, c->stream));
  count(c);
}

// Runs the cycles of a solve whose finest iterate is in U0[0] (r0 known and
// > 0); leaves the result in U0[c->cur[0]].  Fills r and history.
// prefix of the fused schedule: pre-smooth + restriction of cycle 1 into U0[1], F1
void fused_prefix(stmg_ctx* c, const stmg_cycle_config& cfg, bool u_zero) {
  Level& L = c->levels[0];
  Level& C = c->levels[1];
  stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, true);
  CK(stmg::launch_down(L.view, a, u_zero, L.F.base, L.U[0].base, L.U[1].base, C.F.base,
                       c->stream));
  count(c);
}

void run_fused(stmg_ctx* c, const stmg_cycle_config& cfg, double eps, int max_iter,
               double* history, int history_cap, int* nh, stmg_solve_report& r,
               bool u_zero, bool prefix_done = false, bool r0_deferred = false) {
  // r0_deferred (zero guess, device loop): the host has not read r0; it comes
  // back as history[0] with the loop's results, so the whole solve is enqueued
  // without a host round trip.  r0 == 0 then means f == 0: the one cycle the
  // loop ran worked on zeros and the report is the reference's (0 iterations).
  Level& L = c->levels[0];
  Level& C = c->levels[1];
  ensure_hist(c, max_iter + 1);
  if (!prefix_done) fused_prefix(c, cfg, u_zero);
  tiny(c, {set8(c->d_pp, reinterpret_cast<unsigned long long>(L.U[0].base)),
           set8(c->d_pp + 1, reinterpret_cast<unsigned long long>(L.U[1].base)),
           set4(c->d_par, 1u), copy(c->d_r0, c->d_norm, 8), copy(c->d_hist, c->d_norm, 8),
           set4(c->d_iter, 0u)});
  int iters = 0;
  if (c->use_device_loop && !c->profile) {
    cudaGraphExec_t ex = device_loop(
        c, loop_key("fused", cfg, 0, eps, max_iter), eps, max_iter,
        [&] {
          i64 np = 0;
          fused_body(c, cfg, &np, true);
        },
        c->d_par);
    CK(cudaGraphLaunch(ex, c->stream));
    tiny(c, {to_host(c->h_iter, c->d_iter, 4),
             to_host(c->h_hist, c->d_hist, (max_iter + 1) * int(sizeof(double)))});
    CK(cudaStreamSynchronize(c->stream));
    iters = *c->h_iter;
    c->launches += iters * c->loop_kernels[loop_key("fused", cfg, 0, eps, max_iter)];
  } else {  // host-driven cycles (profiling: event records around k_updown)
    const std::string key = loop_key("fusedbody", cfg, 0, eps, max_iter);
    auto it = c->fused_bodies.find(key);
    if (it == c->fused_bodies.end()) {
      cudaGraph_t g;
      c->capturing = true;
      c->captured_kernels = 0;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        i64 np = 0;
        fused_body(c, cfg, &np);
        CK(stmg::launch_decide(0, c->d_norm, c->d_r0, c->d_hist, c->d_iter, eps, max_iter,
                               c->d_par, c->stream));
        count(c);
        CK(cudaMemcpyAsync(c->h_norm, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
      } catch (...) {
        cudaStreamEndCapture(c->stream, &g);
        c->capturing = false;
        throw;
      }
      CK(cudaStreamEndCapture(c->stream, &g));
      c->capturing = false;
      cudaGraphExec_t ex;
      CK(cudaGraphInstantiate(&ex, g, 0));
      CK(cudaGraphDestroy(g));
      it = c->fused_bodies.emplace(key, ex).first;
      c->cur_after[key] = cur_snapshot(c);
    } else {
      cur_restore(c, c->cur_after.at(key));
    }
    for (int k = 0; k < max_iter; ++k) {
      CK(cudaGraphLaunch(it->second, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      prof_collect_graph(c);
      ++iters;
      if (*c->h_norm <= eps * r.r0) break;
    }
  }
  // history and report (the device loop fetched it with the iteration count)
  if (!(c->use_device_loop && !c->profile)) {
    tiny(c, {to_host(c->h_hist, c->d_hist, (iters + 1) * int(sizeof(double)))});
    CK(cudaStreamSynchronize(c->stream));
  }
  const std::vector<double> h(c->h_hist, c->h_hist + iters + 1);
  if (r0_deferred) {
    r.r0 = r.r_final = h[0];
    if (history && *nh < history_cap) history[*nh] = h[0];
    ++*nh;
    if (h[0] == 0.0) iters = 0;
  }
  for (int k = 1; k <= iters; ++k) {
    if (history && *nh < history_cap) history[*nh] = h[k];
    ++*nh;
  }
  r.iterations = iters;
  r.r_final = iters > 0 ? h[iters] : r.r0;
  r.converged = ((iters > 0 && h[iters] <= eps * r.r0) || (r0_deferred && r.r0 == 0.0)) ? 1 : 0;
  // suffix: the last cycle's post-smooth from its (intact) inputs; after an
  // even number of cycles the last input A is U0[1], after an odd number U0[0]
  const int a_last = (iters % 2 == 1) ? 1 : 0;
  {
    stmg::ModalArgs a = modal_args(L, &C, cfg.omega_t, true);
    CK(stmg::launch_up(L.view, a, C.U[c->cur[1]].base, L.U[a_last].base, L.F.base,
                       L.U[1 - a_last].base, nullptr, c->stream));
    count(c);
  }
  c->cur[0] = 1 - a_last;
}

// known_zero: the caller guarantees u == 0 on the device (it zeroed the buffer
// itself): no k_nonzero pass and no flag round trip.
void solve_impl(stmg_ctx* c, const double* f, double* u, const stmg_cycle_config& cfg, double eps,
                int max_iter, double* history, int history_cap, stmg_solve_report* rep,
                bool known_zero = false) {
  require(eps > 0.0, "eps_mg must be positive");
  require(f != nullptr && u != nullptr, "null vector");
  require(max_iter >= 0, "max_iter must be >= 0");
  Level& L0 = c->levels[0];
  stmg_solve_report r{};
  int nh = 0;
  auto push = [&](double v) {
    if (history && nh < history_cap) history[nh] = v;
    ++nh;
  };
  CK(cudaStreamSynchronize(c->stream));
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaEventRecord(c->ev_solve[0], c->stream));
  if (cfg.path == STMG_PATH_PHYSICAL) {
    ensure(L0.R, L0.view.size());
    residual(c, L0, u, f, L0.R.base);
    const double r0 = norm_phys(c, L0, L0.R.base);
    r.r0 = r.r_final = r0;
    push(r0);
    if (r0 == 0.0) r.converged = 1;
    for (int k = 0; k < max_iter && !r.converged; ++k) {
      phys_cycle(c, 0, u, f, cfg);
      residual(c, L0, u, f, L0.R.base);
      const double rk = norm_phys(c, L0, L0.R.base);
      push(rk);
      r.r_final = rk;
      ++r.iterations;
      if (rk <= eps * r0) r.converged = 1;
    }
  } else {
    ensure_spectral(c, 0);
    ensure_tail(c);
    ensure_csub(c);
    if (v11_exact(cfg)) ensure_cop(c, cfg.omega_t);
    ensure_svc(c, cfg);
    c->cur[0] = 0;
    // a zero initial guess (the usual case) needs no transform
    bool u_zero = true;
    if (known_zero) {
      dst_all(c, L0, f, L0.F.base);
    } else {
      tiny(c, {set4(c->d_flag, 0u)});
      CK(stmg::launch_nonzero(u, L0.view.size(), c->d_flag, c->stream));
      count(c);
      tiny(c, {to_host(c->h_flag, c->d_flag, 4)});
      CK(cudaEventRecord(c->ev_host, c->stream));
      dst_all(c, L0, f, L0.F.base);
      // the host reads the flag while the transform of f runs: no stream-wide
      // synchronisation (and no idle GPU) before the next kernels are enqueued
      CK(cudaEventSynchronize(c->ev_host));
      u_zero = !*c->h_flag;
    }
    if (!u_zero) dst_all(c, L0, u, L0.U[0].base);
    // zero guess: r0 = ||f|| from F alone (bitwise the general kernel's value)
    spectral_resnorm_async(c, 0, u_zero);
    // the fused schedule's prefix does not depend on r0: enqueue it before the
    // host waits for r0 (if r0 turns out to be 0 its output is simply unused)
    const bool may_fuse = fused_eligible(c, cfg) && max_iter > 0;
    if (may_fuse) fused_prefix(c, cfg, u_zero);
    // zero guess + device loop: r0 is not needed on the host before the loop
    const bool defer = may_fuse && u_zero && c->use_device_loop && !c->profile;
    double r0 = 0.0;
    if (!defer) {
      CK(cudaEventSynchronize(c->ev_host));
      r0 = *c->h_norm;
      r.r0 = r.r_final = r0;
      push(r0);
      if (r0 == 0.0) r.converged = 1;
    }
    const bool fused = may_fuse && !r.converged;
    // the fused schedule's zero-guess prefix never reads U[0]; every other
    // path (and the immediate return when f == 0) needs the zero iterate there
    if (u_zero && !fused)
      CK(cudaMemsetAsync(L0.U[0].base, 0, size_t(L0.view.size()) * sizeof(double), c->stream));
    if (fused) run_fused(c, cfg, eps, max_iter, history, history_cap, &nh, r, u_zero, true, defer);
    // the device-side loop needs the finest iterate back in its buffer after
    // a cycle; the per-cycle graph (kept for profiling) reports where it ends
    bool loop_ok = false;
    i64 probe_kernels = 0;
    if (!fused) {
      const stmg_ctx::GraphEntry& probe = cycle_graph(c, cfg);
      loop_ok = c->use_device_loop && !c->profile && probe.cur0_after == c->cur[0];
      probe_kernels = probe.kernels;
    }
    if (loop_ok && !r.converged && max_iter > 0) {
      ensure_hist(c, max_iter + 1);
      tiny(c, {copy(c->d_r0, c->d_norm, 8), copy(c->d_hist, c->d_norm, 8)});
      const int cur0 = c->cur[0];
      cudaGraphExec_t ex = device_loop(c, loop_key("single", cfg, cur0, eps, max_iter), eps,
                                       max_iter, [&] {
                                         i64 np = 0;
                                         spectral_cycle(c, 0, false, cfg, true, &np);
                                         c->pending_norm = np;  // fused with the stop test
                                       });
      c->cur[0] = cur0;
      run_device_loop(c, ex, max_iter, history, history_cap, &nh, r, eps);
      c->launches += r.iterations * probe_kernels;
    }
    for (int k = 0; k < max_iter && !r.converged && !loop_ok && !fused; ++k) {
      stmg_ctx::GraphEntry& g = cycle_graph(c, cfg);
      CK(cudaGraphLaunch(g.exec, c->stream));
      c->launches += g.kernels;
      CK(cudaStreamSynchronize(c->stream));
      prof_collect_graph(c);
      c->cur[0] = g.cur0_after;
      const double rk = *c->h_norm;
      push(rk);
      r.r_final = rk;
      ++r.iterations;
      if (rk <= eps * r0) r.converged = 1;
    }
    dst_all(c, L0, L0.U[c->cur[0]].base, u);
  }
  CK(cudaEventRecord(c->ev_solve[1], c->stream));
  CK(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev_solve[0], c->ev_solve[1]));
    r.device_time_seconds = 1e-3 * double(ms);
  }
  r.wall_time_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rep) *rep = r;
}

// ======================================================= time-slab sharding
// Level l < lg of the hierarchy is split into S contiguous time slabs (one per
// shard); the rest (l >= lg, small) is gathered onto shard 0 ("root").  Each
// fused kernel on a sharded level needs the end-of-slab halo of its left
// neighbour (2 u slabs, 1 f slab, 1 coarse e slab), which lands in the halo
// slabs in front of every buffer.  Norm partials are concatenated in global
// chunk order, so iterates AND norms are bitwise identical for any S.
// Transports: virtual shards on one device (D2D copies on the ctx stream) or
// one rank per GPU over NCCL (send/recv, all-gather; dlopen'ed, graph-capturable).
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGetErrorString) ErrStr = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw std::runtime_error(std::string("cannot load NCCL: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.ErrStr = reinterpret_cast<decltype(api.ErrStr)>(sym("ncclGetErrorString"));
  api.h = h;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL error in ") + what + ": " + nccl().ErrStr(r));
}

struct ShardLevel {
  stmg::LevelView view;  // local n_t, first_global
  DevBuf F, U[2];
};

struct Shard {
  int g = 0;  // global shard index
  std::vector<ShardLevel> lv;  // sharded levels 0..lg-1
  std::vector<int> cur;
  DevBuf Fg;  // local part of F_lg (written by down(lg-1))
  DevBuf Eg;  // local part of the coarse correction at lg (+2 halo slabs)
  DevBuf tbl;  // {U0[0], U0[1]} base pointers (fused schedule's ping-pong table)
};

struct ShardSet {
  int S = 1;
  int lg = 0;  // first gathered level
  bool nccl = false;
  ncclComm_t comm = nullptr;
  std::vector<Shard> local;  // virtual: all S shards; nccl: this rank's
  DevBuf partials;           // S * P partial sums (global chunk order)
  DevBuf par01;              // device ints {0, 1}: fixed ping-pong parities
  i64 P = 0;                 // partials per shard (level-0 residual)
  i64 m = 0;                 // coarse steps per shard at lg
  bool built = false;
};

bool is_root(const ShardSet& ss, const Shard& sh) { return sh.g == 0; }

std::vector<std::vector<int>> cur_snapshot(const stmg_ctx* c) {
  std::vector<std::vector<int>> s{c->cur};
  if (c->shards)
    for (const Shard& sh : c->shards->local) s.push_back(sh.cur);
  return s;
}

void cur_restore(stmg_ctx* c, const std::vector<std::vector<int>>& s) {
  c->cur = s.at(0);
  if (c->shards)
    for (size_t i = 0; i < c->shards->local.size() && i + 1 < s.size(); ++i)
      c->shards->local[i].cur = s[i + 1];
}

int gather_level(stmg_ctx* c, int S) {
  std::vector<stmg::LevelSpec> specs;
  for (const Level& L : c->levels) specs.push_back(L.spec);
  return gather_level_of(specs, S);
}

// Chunk of a sharded level: the single-shard choice, so partial sums line up.
int shard_chunk(const Level& G, const stmg::LevelView& local, bool grouped) {
  int ch = stmg::pick_chunk(G.view, grouped);
  while (ch > 2 && (local.n_t % ch) != 0) ch /= 2;
  return int(std::min<i64>(ch, local.n_t));
}

void build_shards(stmg_ctx* c) {
  ShardSet& ss = *c->shards;
  if (ss.built) return;
  ss.lg = gather_level(c, ss.S);
  require(ss.lg >= 1, "too few time steps for this many shards (need >= 2 per shard)");
  const int lg = ss.lg;
  ss.m = c->levels[lg].spec.n_t / ss.S;
  require(ss.m >= 1 && ss.m * ss.S == c->levels[lg].spec.n_t, "time steps do not split evenly");
  for (Shard& sh : ss.local) {
    sh.lv.resize(lg);
    sh.cur.assign(lg, 0);
    for (int l = 0; l < lg; ++l) {
      ShardLevel& s = sh.lv[l];
      s.view = c->levels[l].view;
      s.view.n_t = c->levels[l].spec.n_t / ss.S;
      s.view.first_global = sh.g == 0;
      // level 0: 3 halo slabs (the fused k_updown's warm-up reads steps -3..-1)
      const i64 n = s.view.size(), halo = (l == 0 ? 3 : 2) * s.view.slab();
      s.F.alloc(n, halo);
      s.U[0].alloc(n, halo);
      s.U[1].alloc(n, halo);
    }
    const i64 cslab = c->levels[lg].view.slab();
    sh.Fg.alloc(ss.m * cslab, 2 * cslab);
    sh.Eg.alloc(ss.m * cslab, 2 * cslab);
    sh.tbl.alloc(2, 0);
    double* t2[2] = {sh.lv[0].U[0].base, sh.lv[0].U[1].base};
    CK(cudaMemcpy(sh.tbl.base, t2, sizeof(t2), cudaMemcpyHostToDevice));
  }
  {
    ss.par01.alloc(1, 0);
    const int p01[2] = {0, 1};
    CK(cudaMemcpy(ss.par01.base, p01, sizeof(p01), cudaMemcpyHostToDevice));
  }
  // root holds the gathered levels (full size)
  bool have_root = false;
  for (Shard& sh : ss.local) have_root |= sh.g == 0;
  if (have_root) {
    ensure_spectral(c, lg);
    ensure_tail(c);
  }
  if (int(c->cur.size()) != int(c->levels.size())) c->cur.assign(c->levels.size(), 0);
  // level-0 residual partials per shard (k_up grouped, k_resnorm per mode)
  {
    const stmg::LevelView& v = ss.local[0].lv[0].view;
    ss.P = std::max(stmg::partial_count(v, shard_chunk(c->levels[0], v, true), true),
                    stmg::partial_count(v, shard_chunk(c->levels[0], v, false), false));
  }
  ss.partials.alloc(ss.S * ss.P + 16, 0);
  ss.built = true;
}

// Copy the last `ns` slabs of every shard's buffer into its right
// neighbour's halo.  get(sh) -> the buffer base of that shard.
template <class Get>
void halo(stmg_ctx* c, i64 n_loc, i64 slab, int ns, Get get) {
  ShardSet& ss = *c->shards;
  const size_t bytes = size_t(ns) * size_t(slab) * sizeof(double);
  if (!ss.nccl) {
    for (size_t i = 1; i < ss.local.size(); ++i) {
      double* dst = get(ss.local[i]) - ns * slab;
      const double* src = get(ss.local[i - 1]) + (n_loc - ns) * slab;
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    }
    return;
  }
  Shard& sh = ss.local[0];
  NcclApi& N = nccl();
  nccl_check(N.GroupStart(), "group start");
  if (sh.g + 1 < ss.S)
    nccl_check(N.Send(get(sh) + (n_loc - ns) * slab, size_t(ns) * slab, ncclDouble, sh.g + 1,
                      ss.comm, c->stream), "halo send");
  if (sh.g > 0)
    nccl_check(N.Recv(get(sh) - ns * slab, size_t(ns) * slab, ncclDouble, sh.g - 1, ss.comm,
                      c->stream), "halo recv");
  nccl_check(N.GroupEnd(), "group end");
}

// Fg of every shard -> root's full F at lg.
void gather_rhs(stmg_ctx* c) {
  ShardSet& ss = *c->shards;
  const i64 cslab = c->levels[ss.lg].view.slab();
  const size_t bytes = size_t(ss.m * cslab) * sizeof(double);
  if (!ss.nccl) {
    double* F = c->levels[ss.lg].F.base;
    for (Shard& sh : ss.local)
      CK(cudaMemcpyAsync(F + sh.g * ss.m * cslab, sh.Fg.base, bytes, cudaMemcpyDeviceToDevice,
                         c->stream));
    return;
  }
  Shard& sh = ss.local[0];
  NcclApi& N = nccl();
  nccl_check(N.GroupStart(), "group start");
  if (sh.g == 0) {
    double* F = c->levels[ss.lg].F.base;
    CK(cudaMemcpyAsync(F, sh.Fg.base, bytes, cudaMemcpyDeviceToDevice, c->stream));
    for (int g = 1; g < ss.S; ++g)
      nccl_check(N.Recv(F + g * ss.m * cslab, size_t(ss.m * cslab), ncclDouble, g, ss.comm,
                        c->stream), "gather recv");
  } else {
    nccl_check(N.Send(sh.Fg.base, size_t(ss.m * cslab), ncclDouble, 0, ss.comm, c->stream),
               "gather send");
  }
  nccl_check(N.GroupEnd(), "group end");
}

// root's coarse correction at lg -> every shard's Eg (+ the two steps before:
// k_up reads one, the fused k_updown's warm-up two).
void scatter_corr(stmg_ctx* c) {
  ShardSet& ss = *c->shards;
  const i64 cslab = c->levels[ss.lg].view.slab();
  auto nh = [&](int g) { return std::min<i64>(2, i64(g) * ss.m); };
  auto src_of = [&](int g) {
    const double* E = c->levels[ss.lg].U[c->cur[ss.lg]].base;
    return E + (g * ss.m - nh(g)) * cslab;
  };
  auto count_of = [&](int g) { return size_t((ss.m + nh(g)) * cslab); };
  auto dst_of = [&](Shard& sh) { return sh.Eg.base - nh(sh.g) * cslab; };
  if (!ss.nccl) {
    for (Shard& sh : ss.local)
      CK(cudaMemcpyAsync(dst_of(sh), src_of(sh.g), count_of(sh.g) * sizeof(double),
                         cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  Shard& sh = ss.local[0];
  NcclApi& N = nccl();
  nccl_check(N.GroupStart(), "group start");
  if (sh.g == 0) {
    CK(cudaMemcpyAsync(dst_of(sh), src_of(0), count_of(0) * sizeof(double),
                       cudaMemcpyDeviceToDevice, c->stream));
    for (int g = 1; g < ss.S; ++g)
      nccl_check(N.Send(src_of(g), count_of(g), ncclDouble, g, ss.comm, c->stream),
                 "scatter send");
  } else {
    nccl_check(N.Recv(dst_of(sh), count_of(sh.g), ncclDouble, 0, ss.comm, c->stream),
               "scatter recv");
  }
  nccl_check(N.GroupEnd(), "group end");
}

void allgather_partials(stmg_ctx* c, i64 np) {
  ShardSet& ss = *c->shards;
  if (!ss.nccl) return;  // virtual shards write their segments in place
  NcclApi& N = nccl();
  const Shard& sh = ss.local[0];
  nccl_check(N.AllGather(ss.partials.base + sh.g * np, ss.partials.base, size_t(np), ncclDouble,
                         ss.comm, c->stream), "partials all-gather");
}

// Partial sums of one shard's level-0 residual kernel (same on every shard).
i64 shard_np(stmg_ctx* c, bool grouped) {
  const stmg::LevelView& v = c->shards->local[0].lv[0].view;
  return stmg::partial_count(v, shard_chunk(c->levels[0], v, grouped), grouped);
}

// Partial sums of one shard's launch_updown (its CTAs may be 256 threads wide).
i64 shard_np_updown(stmg_ctx* c) {
  const stmg::LevelView& v = c->shards->local[0].lv[0].view;
  const Level& G = c->levels[0];
  const int mode = G.spec.coarsen ? G.spec.coarsen : 1;
  const int block = stmg::pick_updown_block(G.view, stmg::pick_chunk(G.view, true), mode);
  return stmg::partial_count(v, shard_chunk(G, v, true), true, block);
}

stmg::ModalArgs shard_args(stmg_ctx* c, int l, const ShardLevel& s, double omega, bool grouped) {
  stmg::ModalArgs a;
  a.omega = omega;
  a.chunk = shard_chunk(c->levels[l], s.view, grouped);
  a.mode = c->levels[l].spec.coarsen ? c->levels[l].spec.coarsen : 1;
  a.n1c = c->levels[l + 1].spec.n1();
  // from the GLOBAL level: every shard uses the single-shard block size
  a.block = stmg::pick_updown_block(c->levels[l].view,
                                    stmg::pick_chunk(c->levels[l].view, true), a.mode);
  return a;
}

// One V-cycle (gamma = 1) over the sharded levels + the root's tail, plus the
// residual norm into d_norm (and h_norm).  from = 1: only the coarse part
// (levels >= 1, zero guess) of the fused schedule -- no norm.
void sharded_cycle(stmg_ctx* c, const stmg_cycle_config& cfg, bool copy_norm = true,
                   int from = 0) {
  ShardSet& ss = *c->shards;
  const int lg = ss.lg;
  const int nu1 = cfg.nu1, nu2 = cfg.nu2;
  for (int l = from; l < lg; ++l) {
    const stmg::LevelView& v = ss.local[0].lv[l].view;
    const i64 n_loc = v.n_t, slab = v.slab();
    bool zero = l > 0;
    if (zero)
      for (Shard& sh : ss.local) sh.cur[l] = 0;
    if (l > 0) halo(c, n_loc, slab, 1, [&](Shard& sh) { return sh.lv[l].F.base; });
    for (int s = 0; s + 1 < nu1; ++s) {
      if (!zero) halo(c, n_loc, slab, 1, [&](Shard& sh) { return sh.lv[l].U[sh.cur[l]].base; });
      for (Shard& sh : ss.local) {
        ShardLevel& L = sh.lv[l];
        stmg::ModalArgs a = shard_args(c, l, L, cfg.omega_t, false);
        CK(stmg::launch_smooth(L.view, a, zero, L.F.base, L.U[sh.cur[l]].base,
                               L.U[1 - sh.cur[l]].base, c->stream));
        count(c);
        sh.cur[l] ^= 1;
      }
      zero = false;
    }
    if (!zero) halo(c, n_loc, slab, 2, [&](Shard& sh) { return sh.lv[l].U[sh.cur[l]].base; });
    for (Shard& sh : ss.local) {
      ShardLevel& L = sh.lv[l];
      stmg::ModalArgs a = shard_args(c, l, L, cfg.omega_t, true);
      double* fc = (l + 1 < lg) ? sh.lv[l + 1].F.base : sh.Fg.base;
      const bool p = l == 0 && sh.g == 0;
      if (p) prof_begin(c, 0);
      CK(stmg::launch_down(L.view, a, zero, L.F.base, L.U[sh.cur[l]].base, L.U[1 - sh.cur[l]].base,
                           fc, c->stream));
      if (p) prof_end(c, 0, 8.0 * double((zero ? 2 : 3) * L.view.size() + L.view.size() / 8));
      count(c);
      sh.cur[l] ^= 1;
    }
  }
  gather_rhs(c);
  bool have_root = false;
  for (Shard& sh : ss.local) have_root |= sh.g == 0;
  if (have_root) {
    if (c->tail_table && lg == c->tail_start && nu1 == 1 && nu2 == 1) {  // tail = V(1,1)
      run_tail(c, cfg.omega_t);
    } else {
      spectral_cycle(c, lg, true, cfg, false, nullptr);
    }
  }
  scatter_corr(c);
  for (int l = lg - 1; l >= from; --l) {
    const stmg::LevelView& v = ss.local[0].lv[l].view;
    const i64 n_loc = v.n_t, slab = v.slab();
    if (l + 1 < lg) {
      const stmg::LevelView& vc = ss.local[0].lv[l + 1].view;
      halo(c, vc.n_t, vc.slab(), 1,
           [&](Shard& sh) { return sh.lv[l + 1].U[sh.cur[l + 1]].base; });
    }
    halo(c, n_loc, slab, 2, [&](Shard& sh) { return sh.lv[l].U[sh.cur[l]].base; });
    const bool resid = l == 0 && nu2 == 1;
    const i64 npu = shard_np(c, true);
    for (Shard& sh : ss.local) {
      ShardLevel& L = sh.lv[l];
      stmg::ModalArgs a = shard_args(c, l, L, cfg.omega_t, true);
      const double* ec = (l + 1 < lg) ? sh.lv[l + 1].U[sh.cur[l + 1]].base : sh.Eg.base;
      const bool p = l == 0 && sh.g == 0;
      if (p) prof_begin(c, 1);
      CK(stmg::launch_up(L.view, a, ec, L.U[sh.cur[l]].base, L.F.base, L.U[1 - sh.cur[l]].base,
                         resid ? ss.partials.base + sh.g * npu : nullptr, c->stream));
      if (p) prof_end(c, 1, 8.0 * double(3 * L.view.size() + L.view.size() / 8));
      count(c);
      if (resid) require(a.n_partials == npu, "partial count mismatch");
      sh.cur[l] ^= 1;
    }
    for (int s = 1; s < nu2; ++s) {
      halo(c, n_loc, slab, 1, [&](Shard& sh) { return sh.lv[l].U[sh.cur[l]].base; });
      for (Shard& sh : ss.local) {
        ShardLevel& L = sh.lv[l];
        stmg::ModalArgs a = shard_args(c, l, L, cfg.omega_t, false);
        CK(stmg::launch_smooth(L.view, a, false, L.F.base, L.U[sh.cur[l]].base,
                               L.U[1 - sh.cur[l]].base, c->stream));
        count(c);
        sh.cur[l] ^= 1;
      }
    }
    if (l == 0 && !resid) {
      halo(c, n_loc, slab, 1, [&](Shard& sh) { return sh.lv[0].U[sh.cur[0]].base; });
      const i64 npr = shard_np(c, false);
      for (Shard& sh : ss.local) {
        ShardLevel& L = sh.lv[0];
        stmg::ModalArgs a = shard_args(c, 0, L, cfg.omega_t, false);
        CK(stmg::launch_resnorm(L.view, a, L.U[sh.cur[0]].base, L.F.base,
                                ss.partials.base + sh.g * npr, c->stream));
        count(c);
        require(a.n_partials == npr, "partial count mismatch");
      }
    }
  }
  if (from > 0) return;
  const i64 np = shard_np(c, nu2 == 1);
  allgather_partials(c, np);
  CK(stmg::launch_norm_final(ss.partials.base, ss.S * np, c->d_norm, nullptr, 0, c->stream));
  count(c);
  if (copy_norm)
    CK(cudaMemcpyAsync(c->h_norm, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

// ---- fused V(1,1) schedule on time slabs (see run_fused) -------------------
// Same passes as the single-device schedule; per cycle the level-0 exchange is
// 3 slabs of the pre-smoothed iterate A (k_updown's warm-up rebuilds steps
// -3..-1) and 2 coarse-correction slabs; the rhs halo (2 slabs) is sent once
// per solve.  Buffer parity alternates per cycle, so the host drives the
// cycles with two captured graphs (A = U0[1], A = U0[0]).
bool sharded_fused_ok(stmg_ctx* c, const stmg_cycle_config& cfg) {
  const ShardSet& ss = *c->shards;
  return fused_eligible(c, cfg) && ss.local[0].lv[0].view.n_t >= 4;
}

const double* shard_ec(stmg_ctx* c, Shard& sh) {
  return c->shards->lg > 1 ? sh.lv[1].U[sh.cur[1]].base : sh.Eg.base;
}

double* shard_fc(stmg_ctx* c, Shard& sh) {
  return c->shards->lg > 1 ? sh.lv[1].F.base : sh.Fg.base;
}

// One cycle body: coarse part, halos, k_updown per shard, norm, stop test.
void sharded_fused_body(stmg_ctx* c, const stmg_cycle_config& cfg, int pa, double eps,
                        int max_iter) {
  ShardSet& ss = *c->shards;
  sharded_cycle(c, cfg, false, 1);
  if (ss.lg > 1) {
    const stmg::LevelView& v1 = ss.local[0].lv[1].view;
    halo(c, v1.n_t, v1.slab(), 2, [&](Shard& sh) { return sh.lv[1].U[sh.cur[1]].base; });
  }
  const stmg::LevelView& v0 = ss.local[0].lv[0].view;
  halo(c, v0.n_t, v0.slab(), 3, [&](Shard& sh) { return sh.lv[0].U[pa].base; });
  const i64 np = shard_np_updown(c);
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    stmg::ModalArgs a = shard_args(c, 0, L, cfg.omega_t, true);
    const bool p = sh.g == 0;
    if (p) prof_begin(c, 0);
    CK(stmg::launch_updown(L.view, a, shard_ec(c, sh),
                           reinterpret_cast<double* const*>(sh.tbl.base),
                           reinterpret_cast<const int*>(ss.par01.base) + pa, L.F.base,
                           shard_fc(c, sh), ss.partials.base + sh.g * np, c->stream,
                           int64_t(sh.g) * v0.n_t));
    if (p) {
      const Level& C = c->levels[1];
      prof_end(c, 0, 8.0 * double(3 * L.view.size() + 2 * C.view.size() / ss.S));
    }
    count(c);
    require(np == a.n_partials, "partial count mismatch");
  }
  allgather_partials(c, np);
  CK(stmg::launch_norm_final(ss.partials.base, ss.S * np, c->d_norm, nullptr, 0, c->stream));
  count(c);
  CK(stmg::launch_decide(0, c->d_norm, c->d_r0, c->d_hist, c->d_iter, eps, max_iter, nullptr,
                         c->stream));
  count(c);
  CK(cudaMemcpyAsync(c->h_norm, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

void run_sharded_fused(stmg_ctx* c, const stmg_cycle_config& cfg, double eps, int max_iter,
                       double* history, int history_cap, int* nh, stmg_solve_report& r,
                       bool u_zero) {
  ShardSet& ss = *c->shards;
  const stmg::LevelView& v0 = ss.local[0].lv[0].view;
  ensure_hist(c, max_iter + 1);
  halo(c, v0.n_t, v0.slab(), 2, [&](Shard& sh) { return sh.lv[0].F.base; });
  // prefix: pre-smooth + restriction of cycle 1 into U0[1]
  if (!u_zero) halo(c, v0.n_t, v0.slab(), 2, [&](Shard& sh) { return sh.lv[0].U[0].base; });
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    stmg::ModalArgs a = shard_args(c, 0, L, cfg.omega_t, true);
    CK(stmg::launch_down(L.view, a, u_zero, L.F.base, L.U[0].base, L.U[1].base, shard_fc(c, sh),
                         c->stream));
    count(c);
  }
  CK(cudaMemcpyAsync(c->d_r0, c->d_norm, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(c->d_hist, c->d_norm, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemsetAsync(c->d_iter, 0, sizeof(int), c->stream));
  int iters = 0;
  for (int k = 0; k < max_iter; ++k) {
    const int pa = (k % 2 == 0) ? 1 : 0;  // A of cycle k
    const std::string key = loop_key(pa ? "shfused1" : "shfused0", cfg, 0, eps, max_iter);
    auto it = c->fused_bodies.find(key);
    if (it == c->fused_bodies.end()) {
      cudaGraph_t g;
      c->capturing = true;
      c->captured_kernels = 0;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        sharded_fused_body(c, cfg, pa, eps, max_iter);
      } catch (...) {
        cudaStreamEndCapture(c->stream, &g);
        c->capturing = false;
        throw;
      }
      CK(cudaStreamEndCapture(c->stream, &g));
      c->capturing = false;
      cudaGraphExec_t ex;
      CK(cudaGraphInstantiate(&ex, g, 0));
      CK(cudaGraphDestroy(g));
      c->loop_kernels[key] = c->captured_kernels;
      it = c->fused_bodies.emplace(key, ex).first;
      c->cur_after[key] = cur_snapshot(c);
    } else {
      cur_restore(c, c->cur_after.at(key));
    }
    CK(cudaGraphLaunch(it->second, c->stream));
    c->launches += c->loop_kernels[key];
    CK(cudaStreamSynchronize(c->stream));
    prof_collect_graph(c);
    ++iters;
    if (*c->h_norm <= eps * r.r0) break;
  }
  std::vector<double> h(size_t(iters) + 1);
  CK(cudaMemcpy(h.data(), c->d_hist, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int k = 1; k <= iters; ++k) {
    if (history && *nh < history_cap) history[*nh] = h[k];
    ++*nh;
  }
  r.iterations = iters;
  r.r_final = iters > 0 ? h[iters] : r.r0;
  r.converged = (iters > 0 && h[iters] <= eps * r.r0) ? 1 : 0;
  // suffix: the last cycle's post-smooth from its intact inputs (A and the
  // correction, whose halos the last body already exchanged)
  const int a_last = (iters % 2 == 1) ? 1 : 0;
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    stmg::ModalArgs a = shard_args(c, 0, L, cfg.omega_t, true);
    CK(stmg::launch_up(L.view, a, shard_ec(c, sh), L.U[a_last].base, L.F.base,
                       L.U[1 - a_last].base, nullptr, c->stream));
    count(c);
    sh.cur[0] = 1 - a_last;
  }
}

// Full sine transform of one shard's finest slabs (the kernels dst_all uses,
// so sharded iterates stay bitwise those of one shard).
void shard_dst(stmg_ctx* c, const stmg::LevelView& v, const double* in, double* out) {
  const void* tw = c->levels[0].d_twiddle;
  if (c->dim == 2) {
    const cudaError_t e = stmg::launch_dst2d(v, in, out, false, 1.0, tw, c->stream);
    if (e != cudaErrorNotSupported) {
      CK(e);
      count(c);
      return;
    }
  }
  for (int a = 0; a < c->dim; ++a) {
    CK(stmg::launch_dst_axis(v, a, a == 0 ? in : out, out, false, 1.0, tw, c->stream));
    count(c);
  }
}

// Sharded solve: f, u are this process's time slabs (virtual shards: the whole
// vectors, split here).
void solve_sharded(stmg_ctx* c, const double* f, double* u, const stmg_cycle_config& cfg,
                   double eps, int max_iter, double* history, int history_cap,
                   stmg_solve_report* rep) {
  require(eps > 0.0, "eps_mg must be positive");
  require(f != nullptr && u != nullptr, "null vector");
  require(max_iter >= 0, "max_iter must be >= 0");
  require(cfg.path == STMG_PATH_SPECTRAL, "sharded solves run on the spectral path");
  require(cfg.block_solver == STMG_BLOCK_EXACT,
          "sharded solves use exact block solves (block_solver = 'exact')");
  require(cfg.gamma == 1 && cfg.nu1 >= 1 && cfg.nu2 >= 1,
          "sharded solves support V(nu1, nu2) cycles with nu1, nu2 >= 1");
  build_shards(c);
  if (v11_exact(cfg)) ensure_cop(c, cfg.omega_t);
  ShardSet& ss = *c->shards;
  stmg_solve_report r{};
  int nh = 0;
  auto push = [&](double v) {
    if (history && nh < history_cap) history[nh] = v;
    ++nh;
  };
  CK(cudaStreamSynchronize(c->stream));
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaEventRecord(c->ev_solve[0], c->stream));
  const i64 nloc0 = ss.local[0].lv[0].view.size();
  auto part = [&](const Shard& sh) { return ss.nccl ? 0 : sh.g * nloc0; };
  // zero initial guess detection (OR over shards)
  CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  for (Shard& sh : ss.local) {
    CK(stmg::launch_nonzero(u + part(sh), nloc0, c->d_flag, c->stream));
    count(c);
  }
  if (ss.nccl)
    nccl_check(nccl().AllReduce(c->d_flag, c->d_flag, 1, ncclInt32, ncclMax, ss.comm, c->stream),
               "flag all-reduce");
  CK(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    shard_dst(c, L.view, f + part(sh), L.F.base);
    sh.cur[0] = 0;
  }
  CK(cudaStreamSynchronize(c->stream));
  const bool u_nonzero = *c->h_flag != 0;
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    if (u_nonzero) {
      shard_dst(c, L.view, u + part(sh), L.U[0].base);
    } else {
      CK(cudaMemsetAsync(L.U[0].base, 0, size_t(nloc0) * sizeof(double), c->stream));
    }
  }
  const stmg::LevelView& v0 = ss.local[0].lv[0].view;
  halo(c, v0.n_t, v0.slab(), 1, [&](Shard& sh) { return sh.lv[0].F.base; });
  halo(c, v0.n_t, v0.slab(), 1, [&](Shard& sh) { return sh.lv[0].U[0].base; });
  const i64 npr = shard_np(c, false);
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    stmg::ModalArgs a = shard_args(c, 0, L, cfg.omega_t, false);
    CK(stmg::launch_resnorm(L.view, a, L.U[0].base, L.F.base, ss.partials.base + sh.g * npr,
                            c->stream));
    count(c);
    require(a.n_partials == npr, "partial count mismatch");
  }
  allgather_partials(c, npr);
  CK(stmg::launch_norm_final(ss.partials.base, ss.S * npr, c->d_norm, nullptr, 0, c->stream));
  count(c);
  CK(cudaMemcpyAsync(c->h_norm, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const double r0 = *c->h_norm;
  r.r0 = r.r_final = r0;
  push(r0);
  if (r0 == 0.0) r.converged = 1;
  const bool fused = sharded_fused_ok(c, cfg) && !r.converged && max_iter > 0;
  if (fused) run_sharded_fused(c, cfg, eps, max_iter, history, history_cap, &nh, r, !u_nonzero);
  // virtual shards: all cycles in one graph (device-side stop test); the
  // finest parity is preserved when nu1 + nu2 is even
  const bool loop_ok = !fused && !ss.nccl && c->use_device_loop && !c->profile &&
                       (nu_flips(cfg) % 2 == 0);
  if (loop_ok && !r.converged && max_iter > 0) {
    ensure_hist(c, max_iter + 1);
    CK(cudaMemcpyAsync(c->d_r0, c->d_norm, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_hist, c->d_norm, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    std::vector<int> cur0(ss.local.size());
    for (size_t i = 0; i < ss.local.size(); ++i) cur0[i] = ss.local[i].cur[0];
    cudaGraphExec_t ex = device_loop(c, loop_key("sharded", cfg, cur0[0], eps, max_iter), eps,
                                     max_iter, [&] { sharded_cycle(c, cfg, false); });
    for (size_t i = 0; i < ss.local.size(); ++i) ss.local[i].cur[0] = cur0[i];
    run_device_loop(c, ex, max_iter, history, history_cap, &nh, r, eps);
  }
  for (int k = 0; k < max_iter && !r.converged && !loop_ok && !fused; ++k) {
    // the cycle's buffer parity pattern is the same every iteration (coarse
    // levels restart at buffer 0) except the finest level's, so at most two
    // graphs; key on shard 0's finest parity
    stmg_ctx::GraphKey key{cfg.nu1, cfg.nu2, -1 - ss.local[0].cur[0], 0, cfg.omega_t};
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      std::vector<int> cur0(ss.local.size());
      for (size_t i = 0; i < ss.local.size(); ++i) cur0[i] = ss.local[i].cur[0];
      cudaGraph_t graph;
      c->capturing = true;
      c->captured_kernels = 0;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        sharded_cycle(c, cfg);
      } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        c->capturing = false;
        throw;
      }
      CK(cudaStreamEndCapture(c->stream, &graph));
      c->capturing = false;
      stmg_ctx::GraphEntry e;
      CK(cudaGraphInstantiate(&e.exec, graph, 0));
      CK(cudaGraphDestroy(graph));
      e.cur0_after = ss.local[0].cur[0];
      e.kernels = c->captured_kernels;
      for (size_t i = 0; i < ss.local.size(); ++i) ss.local[i].cur[0] = cur0[i];
      it = c->graphs.emplace(key, e).first;
    }
    CK(cudaGraphLaunch(it->second.exec, c->stream));
    c->launches += it->second.kernels;
    CK(cudaStreamSynchronize(c->stream));
    prof_collect_graph(c);
    for (Shard& sh : ss.local) sh.cur[0] = it->second.cur0_after;
    const double rk = *c->h_norm;
    push(rk);
    r.r_final = rk;
    ++r.iterations;
    if (rk <= eps * r0) r.converged = 1;
  }
  for (Shard& sh : ss.local) {
    ShardLevel& L = sh.lv[0];
    shard_dst(c, L.view, L.U[sh.cur[0]].base, u + part(sh));
  }
  CK(cudaEventRecord(c->ev_solve[1], c->stream));
  CK(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev_solve[0], c->ev_solve[1]));
    r.device_time_seconds = 1e-3 * double(ms);
  }
  r.wall_time_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rep) *rep = r;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* stmg_last_error(void) { return g_err.c_str(); }

double stmg_critical_mu(int p_t) {
  double v = NAN;
  guard([&] { v = stmg::critical_mu(p_t); });
  return v;
}

int stmg_dg_block(int p_t, double tau, double* K, double* M, double* N) {
  return guard([&] {
    require(K && M && N, "null output");
    const stmg::DGBlock b = stmg::dg_block(p_t, tau);
    std::memcpy(K, b.K.data(), b.K.size() * sizeof(double));
    std::memcpy(M, b.M.data(), b.M.size() * sizeof(double));
    std::memcpy(N, b.N.data(), b.N.size() * sizeof(double));
  });
}

int stmg_time_transfer(int p_t, double tau, double* R1, double* R2) {
  return guard([&] {
    require(R1 && R2, "null output");
    std::vector<double> a, b;
    stmg::time_transfer(p_t, tau, a, b);
    std::memcpy(R1, a.data(), a.size() * sizeof(double));
    std::memcpy(R2, b.data(), b.size() * sizeof(double));
  });
}

int stmg_create(const stmg_hierarchy_params* p, stmg_ctx** out) {
  return guard([&] {
    require(p != nullptr && out != nullptr, "null argument");
    require(p->shards >= 0 && p->shards <= 4096, "shard count out of range");
    *out = nullptr;
    auto specs = stmg::build_ladder(p->p_t, p->dim, p->space_level, p->time_level, p->t_final,
                                    p->mu_star, p->policy, p->two_grid);
    // (build_ladder already rejected p_t outside 0..kMaxTimeDegree = 10)
    require(p->p_t + 1 <= stmg::kMaxNL, "p_t out of range");
    require(p->p_t + 1 <= stmg::kFastNL || p->shards <= 1,
            "time-slab sharding runs the spectral kernels: p_t <= 3");
    int ndev = 0;
    const cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      throw std::runtime_error("no CUDA device available (the B200 library has no CPU fallback)");
    require(p->device >= 0 && p->device < ndev, "device ordinal out of range");
    auto c = std::make_unique<stmg_ctx>();
    c->device = p->device;
    DevGuard dg(c->device);  // the caller's current device is restored on return
    CK(stmg::init_kernel_tables());
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->p_t = p->p_t;
    c->dim = p->dim;
    c->hi_degree = p->p_t + 1 > stmg::kFastNL;
    c->levels.resize(specs.size());
    for (size_t i = 0; i < specs.size(); ++i) {
      c->levels[i].spec = specs[i];
      build_level_tables(c->levels[i]);
    }
    if (p->shards > 1) {
      c->shards = std::make_unique<ShardSet>();
      c->shards->S = p->shards;
      c->shards->local.resize(p->shards);
      for (int g = 0; g < p->shards; ++g) c->shards->local[g].g = g;
    }
    CK(cudaMalloc(&c->d_norm, sizeof(double)));
    CK(cudaMallocHost(&c->h_norm, sizeof(double)));
    CK(cudaMalloc(&c->d_flag, sizeof(int)));
    CK(cudaMalloc(&c->d_iter, sizeof(int)));
    CK(cudaMalloc(&c->d_pp, 2 * sizeof(double*)));
    CK(cudaMalloc(&c->d_par, sizeof(int)));
    CK(cudaMalloc(&c->d_r0, sizeof(double)));
    if (const char* e = std::getenv("STMG_DEVICE_LOOP")) c->use_device_loop = std::atoi(e) != 0;
    if (const char* e = std::getenv("STMG_FUSED")) c->use_fused = std::atoi(e) != 0;
    if (const char* e = std::getenv("STMG_COARSE_OP")) c->use_cop = std::atoi(e) != 0;
    if (const char* e = std::getenv("STMG_CSUB")) c->use_csub = std::atoi(e) != 0;
    CK(cudaMallocHost(&c->h_flag, sizeof(int)));
    CK(cudaMallocHost(&c->h_iter, sizeof(int)));
    CK(cudaEventCreate(&c->ev_solve[0]));
    CK(cudaEventCreate(&c->ev_solve[1]));
    CK(cudaEventCreateWithFlags(&c->ev_host, cudaEventDisableTiming));
    for (auto& s : c->prof) {
      CK(cudaEventCreate(&s.ga));
      CK(cudaEventCreate(&s.gb));
    }
    c->cur.assign(c->levels.size(), 0);
    *out = c.release();
  });
}

int stmg_destroy(stmg_ctx* c) {
  return guard([&] {
    if (!c) return;
    DevGuard dg(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
    if (c->shards) {
      for (Shard& sh : c->shards->local) {
        for (ShardLevel& L : sh.lv)
          for (DevBuf* b : {&L.F, &L.U[0], &L.U[1]}) b->release();
        sh.Fg.release();
        sh.Eg.release();
        sh.tbl.release();
      }
      c->shards->partials.release();
      c->shards->par01.release();
      if (c->shards->comm) nccl().CommDestroy(c->shards->comm);
      c->shards.reset();
    }
    for (auto& L : c->levels) {
      cudaFree(L.d_tables);
      cudaFree(L.d_twiddle);
      for (DevBuf* b : {&L.F, &L.U[0], &L.U[1], &L.R, &L.RC, &L.EC, &L.CORR}) b->release();
    }
    c->partials.release();
    c->partials_phys.release();
    c->svc_pool.release();
    for (auto& kv : c->space_tab) cudaFree(kv.second);
    for (auto& kv : c->cop) cudaFree(kv.second);
    stmg::free_csub(&c->csub);
    c->user_f.release();
    c->user_u.release();
    for (int s = 0; s < stmg_ctx::kSets; ++s) {
      if (s > 0) {
        c->batch_f[s - 1].release();
        c->batch_u[s - 1].release();
      }
      if (c->ev_in[s]) cudaEventDestroy(c->ev_in[s]);
      if (c->ev_free[s]) cudaEventDestroy(c->ev_free[s]);
    }
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    for (auto& s : c->prof) {
      for (auto& e : s.pool) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
      if (s.ga) cudaEventDestroy(s.ga);
      if (s.gb) cudaEventDestroy(s.gb);
    }
    cudaEventDestroy(c->ev_solve[0]);
    cudaEventDestroy(c->ev_solve[1]);
    if (c->ev_host) cudaEventDestroy(c->ev_host);
    cudaFree(c->d_norm);
    cudaFree(c->d_hist);
    cudaFree(c->d_flag);
    cudaFree(c->d_iter);
    cudaFree(c->d_pp);
    cudaFree(c->d_par);
    for (auto& kv : c->fused_bodies) cudaGraphExecDestroy(kv.second);
    cudaFree(c->d_r0);
    for (auto& kv : c->loops) cudaGraphExecDestroy(kv.second);
    cudaFreeHost(c->h_flag);
    cudaFreeHost(c->h_iter);
    if (c->h_hist) cudaFreeHost(c->h_hist);
    if (c->tail_table) cudaFree(c->tail_table);
    std::free(c->tail_host);
    cudaFreeHost(c->h_norm);
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

int stmg_num_levels(const stmg_ctx* c, int* out) {
  return cguard(c, [&] {
    require(c && out, "null argument");
    *out = int(c->levels.size());
  });
}

int stmg_get_level_info(const stmg_ctx* cc, int level, stmg_level_info* o) {
  return cguard(cc, [&] {
    stmg_ctx* c = const_cast<stmg_ctx*>(cc);
    require(o != nullptr, "null output");
    const Level& L = lev(c, level);
    o->n_t = L.spec.n_t;
    o->n_x = L.spec.nx();
    o->n_loc = L.spec.p_t + 1;
    o->n1 = L.spec.n1();
    o->dim = L.spec.dim;
    o->space_level = L.spec.space_level;
    o->coarsen_to_next = L.spec.coarsen;
    o->tau = L.spec.tau;
    o->h = L.spec.h;
    o->mu = L.spec.mu;
  });
}

int stmg_level_size(const stmg_ctx* cc, int level, int64_t* out) {
  return cguard(cc, [&] {
    require(out != nullptr, "null output");
    *out = lev(const_cast<stmg_ctx*>(cc), level).spec.size();
  });
}

int stmg_device_alloc(stmg_ctx* c, size_t bytes, void** dptr) {
  return cguard(c, [&] {
    require(c && dptr, "null argument");
    CK(cudaMalloc(dptr, bytes ? bytes : 8));
  });
}

int stmg_device_free(stmg_ctx* c, void* dptr) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaFree(dptr));
  });
}

int stmg_upload(stmg_ctx* c, void* dst, const void* src, size_t bytes) {
  return cguard(c, [&] {
    require(c && (bytes == 0 || (dst && src)), "null argument");
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  });
}

int stmg_download(stmg_ctx* c, void* dst, const void* src, size_t bytes) {
  return cguard(c, [&] {
    require(c && (bytes == 0 || (dst && src)), "null argument");
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int stmg_memset_zero(stmg_ctx* c, void* dst, size_t bytes) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    CK(cudaMemsetAsync(dst, 0, bytes, c->stream));
  });
}

int stmg_host_alloc(stmg_ctx* c, size_t bytes, void** hptr) {
  return cguard(c, [&] {
    require(c && hptr, "null argument");
    CK(cudaHostAlloc(hptr, bytes ? bytes : 8, cudaHostAllocDefault));
  });
}

int stmg_host_free(stmg_ctx* c, void* hptr) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaFreeHost(hptr));
  });
}

int stmg_synchronize(stmg_ctx* c) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    CK(cudaStreamSynchronize(c->stream));
    prof_collect(c);
  });
}

int stmg_fill_uniform(stmg_ctx* c, double* dst, int64_t n, uint64_t seed, uint64_t stream,
                      int64_t offset) {
  return cguard(c, [&] {
    require(c && (n == 0 || dst), "null argument");
    CK(stmg::launch_fill_uniform(dst, n, seed, stream, offset, c->stream));
    count(c);
  });
}

int stmg_fill_random_host(double* dst, int64_t n, uint64_t seed) {
  return guard([&] {
    require(n >= 0 && (n == 0 || dst), "null argument");
    std::mt19937_64 gen(seed);  // mg.cpp:168-173
    for (int64_t i = 0; i < n; ++i) dst[i] = double(gen() >> 11) * 0x1.0p-53;
  });
}

int stmg_fold_u0(stmg_ctx* c, double* f, const double* u0) {
  return cguard(c, [&] {
    require(f && u0, "null vector");
    Level& L = lev(c, 0);
    CK(stmg::launch_fold_u0(L.view, f, u0, c->stream));
    count(c);
  });
}

int stmg_apply(stmg_ctx* c, int level, const double* u, double* y) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(u && y, "null vector");
    CK(stmg::launch_apply(L.view, u, nullptr, y, false, L.d_tables + 3 * L.spec.n1(), c->stream));
    count(c);
  });
}

int stmg_residual(stmg_ctx* c, int level, const double* u, const double* f, double* r) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(u && f && r, "null vector");
    residual(c, L, u, f, r);
  });
}

int stmg_norm(stmg_ctx* c, int level, const double* v, double* out) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(v && out, "null argument");
    *out = norm_phys(c, L, v);
  });
}

int stmg_block_solve(stmg_ctx* c, int level, const double* b, double* x) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(b && x, "null vector");
    block_solve(c, L, b, x);
  });
}

int stmg_smooth(stmg_ctx* c, int level, double* u, const double* f, double omega_t, int nu) {
  return cguard(c, [&] {
    lev(c, level);
    require(u && f, "null vector");
    require(nu >= 0, "nu must be >= 0");
    smooth_phys(c, level, u, f, omega_t, nu);
  });
}

int stmg_cycle_config_init(stmg_cycle_config* cfg) {
  return guard([&] {
    require(cfg != nullptr, "null cycle config");
    *cfg = stmg_cycle_config{2, 2, 1, 0.5, STMG_PATH_SPECTRAL, STMG_BLOCK_EXACT, 2.0 / 3.0, 2, 2, 1};
  });
}

int stmg_smoother_config_init(stmg_smoother_config* cfg) {
  return guard([&] {
    require(cfg != nullptr, "null smoother config");
    *cfg = stmg_smoother_config{0.5, 1, STMG_BLOCK_EXACT, 2.0 / 3.0, 2, 2, 1};
  });
}

int stmg_block_jacobi_step(stmg_ctx* c, int level, double* u, const double* f,
                           const stmg_smoother_config* cfg) {
  return cguard(c, [&] {
    lev(c, level);
    require(cfg != nullptr, "null smoother config");
    require(u && f, "null vector");
    require(cfg->nu >= 0, "nu must be >= 0");
    require(cfg->block_solver == STMG_BLOCK_EXACT || cfg->block_solver == STMG_BLOCK_VCYCLE,
            "block_solver must be 'exact' or 'vcycle'");
    if (cfg->block_solver == STMG_BLOCK_VCYCLE) {
      check_spatial(cfg->omega_x, cfg->nu1_x, cfg->nu2_x, cfg->gamma_x);
      require(!c->hi_degree, "spatial V-cycle block solves support p_t <= 3 on the B200 path");
      const Spatial sp = spatial_of(*cfg);
      smooth_phys(c, level, u, f, cfg->omega_t, cfg->nu, &sp);
    } else {
      smooth_phys(c, level, u, f, cfg->omega_t, cfg->nu);
    }
  });
}

int stmg_spatial_vcycle(stmg_ctx* c, int level, const double* b, const double* x0, double* x,
                        const stmg_smoother_config* cfg) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(cfg != nullptr, "null smoother config");
    require(b && x, "null vector");
    check_spatial(cfg->omega_x, cfg->nu1_x, cfg->nu2_x, cfg->gamma_x);
    require(!c->hi_degree, "spatial V-cycle block solves support p_t <= 3 on the B200 path");
    const Spatial sp = spatial_of(*cfg);
    const SvcBufs w = svc_bufs(c, L);
    dst_all(c, L, b, w.B[0]);
    if (x0) dst_all(c, L, x0, w.X[0]);
    svc_run(c, L, sp, nullptr, nullptr, nullptr, x0 == nullptr, 1.0);
    dst_all(c, L, w.X[0], x);
  });
}

int stmg_restrict(stmg_ctx* c, int level, int mode, const double* fine, double* coarse) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(fine && coarse, "null vector");
    mode = resolve_mode(L, mode);
    CK(stmg::launch_restrict(L.view, mode, coarse_n1(L, mode), fine, coarse, c->stream));
    count(c);
  });
}

int stmg_prolong(stmg_ctx* c, int level, int mode, const double* coarse, double* fine) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(fine && coarse, "null vector");
    mode = resolve_mode(L, mode);
    CK(stmg::launch_prolong(L.view, mode, coarse_n1(L, mode), coarse, fine, c->stream));
    count(c);
  });
}

int stmg_forward_substitution(stmg_ctx* c, int level, const double* f, double* u) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    require(f && u, "null vector");
    fwdsub_phys(c, L, f, u);
  });
}

int stmg_mg_cycle(stmg_ctx* c, int level, double* u, const double* f,
                  const stmg_cycle_config* cfg) {
  return cguard(c, [&] {
    Level& L = lev(c, level);
    check_cfg(cfg);
    require(u && f, "null vector");
    const stmg_cycle_config ecfg = effective_cfg(c, *cfg);
    cfg = &ecfg;
    if (cfg->path == STMG_PATH_PHYSICAL) {
      phys_cycle(c, level, u, f, *cfg);
      return;
    }
    ensure_spectral(c, 0);
    ensure_tail(c);
    ensure_csub(c);
    if (v11_exact(*cfg)) ensure_cop(c, cfg->omega_t);
    c->cur[level] = 0;
    dst_all(c, L, f, L.F.base);
    dst_all(c, L, u, L.U[0].base);
    spectral_cycle(c, level, false, *cfg, false, nullptr);
    dst_all(c, L, L.U[c->cur[level]].base, u);
  });
}

int stmg_solve(stmg_ctx* c, const double* f, double* u, const stmg_cycle_config* cfg, double eps,
               int max_iter, double* history, int history_cap, stmg_solve_report* report) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    check_cfg(cfg);
    const stmg_cycle_config ec = effective_cfg(c, *cfg);
    if (c->shards) solve_sharded(c, f, u, ec, eps, max_iter, history, history_cap, report);
    else solve_impl(c, f, u, ec, eps, max_iter, history, history_cap, report);
  });
}

int stmg_solve_host(stmg_ctx* c, const double* f_host, double* u_host,
                    const stmg_cycle_config* cfg, double eps, int max_iter, double* history,
                    int history_cap, stmg_solve_report* report) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    check_cfg(cfg);
    require(f_host && u_host, "null vector");
    const stmg_cycle_config ecfg = effective_cfg(c, *cfg);
    cfg = &ecfg;
    Level& L0 = c->levels[0];
    const i64 n = (c->shards && c->shards->nccl) ? L0.view.size() / c->shards->S : L0.view.size();
    ensure(c->user_f, n);
    ensure(c->user_u, n);
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaMemcpyAsync(c->user_f.base, f_host, size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMemcpyAsync(c->user_u.base, u_host, size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    stmg_solve_report r{};
    if (c->shards)
      solve_sharded(c, c->user_f.base, c->user_u.base, *cfg, eps, max_iter, history, history_cap,
                    &r);
    else
      solve_impl(c, c->user_f.base, c->user_u.base, *cfg, eps, max_iter, history, history_cap, &r);
    CK(cudaMemcpyAsync(u_host, c->user_u.base, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    r.wall_time_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (report) *report = r;
  });
}

// Streams a batch of independent solves through one context: the H2D of
// problems i+1, i+2 (copy stream s_in) and the D2H of problem i-1 (s_out) run
// on the two copy engines while problem i solves on the context stream.  Three
// device staging sets {f, u} rotate, so an upload never waits for the download
// of the problem just before it (with two sets it would, and the upload -- the
// longest of the three phases -- would serialise behind it).  The solve path
// itself uses no copy engine (k_tiny), so it never queues behind a bulk copy.
// Each solve is exactly stmg_solve_host's (same kernels, same result bits).
// STMG_BATCH_TRACE=1 prints per-problem phase times (ms from the batch start,
// CUDA events) to stderr.
int stmg_solve_host_batch(stmg_ctx* c, int count, const double* const* f_host,
                          const double* const* u0_host, double* const* u_host,
                          const stmg_cycle_config* cfg, double eps, int max_iter,
                          stmg_solve_report* reports) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    check_cfg(cfg);
    const stmg_cycle_config ecfg = effective_cfg(c, *cfg);
    cfg = &ecfg;
    require(count >= 0, "count must be >= 0");
    if (count == 0) return;
    require(f_host != nullptr && u_host != nullptr, "null vector array");
    for (int i = 0; i < count; ++i) require(f_host[i] && u_host[i], "null vector");
    require(eps > 0.0, "eps_mg must be positive");
    require(max_iter >= 0, "max_iter must be >= 0");
    constexpr int NS = stmg_ctx::kSets;
    Level& L0 = c->levels[0];
    const i64 n = (c->shards && c->shards->nccl) ? L0.view.size() / c->shards->S : L0.view.size();
    const size_t bytes = size_t(n) * sizeof(double);
    {  // uploads run NS-1 problems ahead of the downloads: the buffers read by
       // problem j's upload must not overlap u_host[i] of the NS-1 problems
       // before it, whose results may still be in flight
      auto overlap = [&](const void* a, const void* b) {
        const char* x = static_cast<const char*>(a);
        const char* y = static_cast<const char*>(b);
        return x < y + bytes && y < x + bytes;
      };
      for (int j = 1; j < count; ++j)
        for (int i = std::max(0, j - (NS - 1)); i < j; ++i) {
          const void* src_u = u0_host ? static_cast<const void*>(u0_host[j]) : u_host[j];
          require(!overlap(f_host[j], u_host[i]) && !(src_u && overlap(src_u, u_host[i])),
                  "stmg_solve_host_batch: an input of problem j overlaps the output of one of "
                  "the 2 problems before it (results are downloaded while later inputs upload)");
        }
    }
    DevBuf* F[NS] = {&c->user_f};
    DevBuf* U[NS] = {&c->user_u};
    for (int s = 1; s < NS; ++s) {
      F[s] = &c->batch_f[s - 1];
      U[s] = &c->batch_u[s - 1];
    }
    for (int s = 0; s < NS; ++s) {
      ensure(*F[s], n);
      ensure(*U[s], n);
    }
    if (!c->s_in) {
      CK(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
      for (int s = 0; s < NS; ++s) {
        CK(cudaEventCreateWithFlags(&c->ev_in[s], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_free[s], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    }
    const char* te = std::getenv("STMG_BATCH_TRACE");
    const bool trace = te && std::atoi(te) != 0;
    std::vector<cudaEvent_t> tev;  // per problem: h2d start/end, solve start/end, d2h end
    auto mark = [&](cudaStream_t st) {
      if (!trace) return;
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      CK(cudaEventRecord(e, st));
      tev.push_back(e);
    };
    std::vector<int> tslot(size_t(count) * 5, -1);
    auto tmark = [&](int i, int k, cudaStream_t st) {
      if (!trace) return;
      tslot[size_t(i) * 5 + k] = int(tev.size());
      mark(st);
    };
    // a set may be refilled once the D2H of its previous problem has drained
    // (its f was consumed by that solve's forward transform before that)
    CK(cudaStreamSynchronize(c->s_out));
    auto upload = [&](int i) {
      const int s = i % NS;
      const double* u0 = u0_host ? u0_host[i] : u_host[i];
      if (i >= NS) CK(cudaStreamWaitEvent(c->s_in, c->ev_free[s], 0));
      tmark(i, 0, c->s_in);
      CK(cudaMemcpyAsync(F[s]->base, f_host[i], bytes, cudaMemcpyHostToDevice, c->s_in));
      if (u0) CK(cudaMemcpyAsync(U[s]->base, u0, bytes, cudaMemcpyHostToDevice, c->s_in));
      else CK(cudaMemsetAsync(U[s]->base, 0, bytes, c->s_in));  // zero initial guess
      CK(cudaEventRecord(c->ev_in[s], c->s_in));
      tmark(i, 1, c->s_in);
    };
    // uploads run NS-1 (= 2) problems ahead: problem j's set was last used by
    // problem j-NS, whose D2H (and its ev_free record) is already enqueued
    for (int j = 0; j < std::min(count, NS - 1); ++j) upload(j);
    for (int i = 0; i < count; ++i) {
      const int s = i % NS;
      if (i + NS - 1 < count) upload(i + NS - 1);
      CK(cudaStreamWaitEvent(c->stream, c->ev_in[s], 0));
      tmark(i, 2, c->stream);
      const auto t0 = std::chrono::steady_clock::now();
      stmg_solve_report r{};
      if (c->shards)
        solve_sharded(c, F[s]->base, U[s]->base, *cfg, eps, max_iter, nullptr, 0, &r);
      else
        solve_impl(c, F[s]->base, U[s]->base, *cfg, eps, max_iter, nullptr, 0, &r,
                   /*known_zero=*/(u0_host ? u0_host[i] : u_host[i]) == nullptr);
      CK(cudaEventRecord(c->ev_done, c->stream));
      tmark(i, 3, c->stream);
      CK(cudaStreamWaitEvent(c->s_out, c->ev_done, 0));
      CK(cudaMemcpyAsync(u_host[i], U[s]->base, bytes, cudaMemcpyDeviceToHost, c->s_out));
      CK(cudaEventRecord(c->ev_free[s], c->s_out));
      tmark(i, 4, c->s_out);
      r.wall_time_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (reports) reports[i] = r;
    }
    CK(cudaStreamSynchronize(c->s_out));
    CK(cudaStreamSynchronize(c->s_in));
    if (trace) {
      for (int i = 0; i < count; ++i) {
        std::fprintf(stderr, "batch %d:", i);
        static const char* nm[5] = {"h2d0", "h2d1", "solve0", "solve1", "d2h1"};
        for (int k = 0; k < 5; ++k) {
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, tev[0], tev[size_t(tslot[size_t(i) * 5 + k])]));
          std::fprintf(stderr, " %s=%.3f", nm[k], ms);
        }
        std::fprintf(stderr, "\n");
      }
      for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
  });
}

int stmg_nccl_unique_id(void* out, size_t len) {
  return guard([&] {
    require(out != nullptr && len >= sizeof(ncclUniqueId), "buffer too small for an NCCL id");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "get unique id");
    std::memcpy(out, &id, sizeof(id));
  });
}

int stmg_create_distributed(const stmg_hierarchy_params* p, int rank, int world,
                            const void* nccl_id, size_t id_len, stmg_ctx** out) {
  return guard([&] {
    require(p && out && nccl_id, "null argument");
    require(world >= 1 && rank >= 0 && rank < world, "rank/world out of range");
    require(id_len >= sizeof(ncclUniqueId), "NCCL id too short");
    stmg_hierarchy_params q = *p;
    q.shards = 0;
    stmg_ctx* c = nullptr;
    const int rc = stmg_create(&q, &c);
    if (rc != STMG_OK) {
      if (rc == STMG_EINVAL) throw std::invalid_argument(g_err);
      throw std::runtime_error(g_err);
    }
    std::unique_ptr<stmg_ctx, int (*)(stmg_ctx*)> hold(c, stmg_destroy);
    if (world > 1) {
      require(!c->hi_degree, "time-slab sharding runs the spectral kernels: p_t <= 3");
      c->shards = std::make_unique<ShardSet>();
      c->shards->S = world;
      c->shards->nccl = true;
      c->shards->local.resize(1);
      c->shards->local[0].g = rank;
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      DevGuard dg(c->device);
      nccl_check(nccl().CommInitRank(&c->shards->comm, world, id, rank), "comm init");
      build_shards(c);
    }
    *out = hold.release();
  });
}

int stmg_shard_plan(const stmg_hierarchy_params* p, int shards, int* gather_level,
                    int64_t* steps_per_shard) {
  return guard([&] {
    require(p && gather_level && steps_per_shard, "null argument");
    require(shards >= 1, "shard count must be >= 1");
    const auto specs = stmg::build_ladder(p->p_t, p->dim, p->space_level, p->time_level,
                                          p->t_final, p->mu_star, p->policy, p->two_grid);
    const int lg = gather_level_of(specs, shards);
    require(shards == 1 || lg >= 1, "too few time steps for this many shards (need >= 2 per shard)");
    *gather_level = lg;
    *steps_per_shard = specs[0].n_t / shards;
  });
}

int stmg_local_steps(const stmg_ctx* c, int64_t* first_step, int64_t* n_steps) {
  return cguard(c, [&] {
    require(c && first_step && n_steps, "null argument");
    const i64 nt = c->levels[0].spec.n_t;
    if (c->shards && c->shards->nccl) {
      const i64 loc = nt / c->shards->S;
      *first_step = c->shards->local[0].g * loc;
      *n_steps = loc;
    } else {
      *first_step = 0;
      *n_steps = nt;
    }
  });
}

int stmg_profile_enable(stmg_ctx* c, int on) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    if (bool(on) != c->profile) {  // re-capture with / without event nodes
      CK(cudaStreamSynchronize(c->stream));
      for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
      c->graphs.clear();
      for (auto& kv : c->fused_bodies) cudaGraphExecDestroy(kv.second);
      c->fused_bodies.clear();
    }
    c->profile = on != 0;
  });
}

int stmg_profile_read(stmg_ctx* c, int id, double* total_ms, int64_t* launches,
                      double* bytes_per_launch) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    require(id >= 0 && id < 6, "kernel id out of range");
    CK(cudaStreamSynchronize(c->stream));
    prof_collect(c);
    if (total_ms) *total_ms = c->prof[id].total_ms;
    if (launches) *launches = c->prof[id].launches;
    if (bytes_per_launch) *bytes_per_launch = c->prof[id].bytes;
  });
}

int stmg_profile_reset(stmg_ctx* c) {
  return cguard(c, [&] {
    require(c != nullptr, "null context");
    CK(cudaStreamSynchronize(c->stream));
    prof_collect(c);
    for (auto& s : c->prof) {
      s.total_ms = 0.0;
      s.launches = 0;
      s.in_graph = false;
    }
  });
}

int stmg_launch_count(const stmg_ctx* c, int64_t* out) {
  return cguard(c, [&] {
    require(c && out, "null argument");
    *out = c->launches;
  });
}

// ---------------------------------------------------------------- LFA (host)
namespace {
void check_lfa(int p_t, double mu) {
  require(p_t >= 0 && p_t <= stmg::kMaxTimeDegree, "p_t out of range");
  require(mu > 0.0, "mu must be positive");
}
void check_mode(int mode) {
  require(mode == STMG_COARSEN_SEMI || mode == STMG_COARSEN_FULL,
          "LFA needs semi or full coarsening");
}
}  // namespace

int stmg_lfa_beta(double theta_x, double* out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    *out = stmg::lfa::beta(theta_x);
  });
}

int stmg_lfa_alpha(int p_t, double mu, double theta_x, double* out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    require(p_t >= 0 && p_t <= stmg::kMaxTimeDegree, "p_t out of range");
    *out = stmg::lfa::alpha(p_t, mu, theta_x);
  });
}

int stmg_lfa_smoother_rho(int p_t, double mu, double omega_t, double theta_x, double theta_t,
                          double* rho, double* rho_closed_form) {
  return guard([&] {
    check_lfa(p_t, mu);
    const stmg::lfa::Symbols s(p_t, mu);
    if (rho) *rho = s.smoother_rho(omega_t, theta_x, theta_t);
    if (rho_closed_form) *rho_closed_form = s.smoother_rho_closed_form(omega_t, theta_x, theta_t);
  });
}

int stmg_lfa_smoother_symbol(int p_t, double mu, double omega_t, double theta_x, double theta_t,
                             double* re, double* im) {
  return guard([&] {
    check_lfa(p_t, mu);
    require(re && im, "null argument");
    const stmg::lfa::Symbols s(p_t, mu);
    s.smoother_symbol(omega_t, theta_x, theta_t, re, im);
  });
}

int stmg_lfa_twogrid_symbol(int p_t, double mu, const stmg_cycle_config* cfg, int mode,
                            double theta_x, double theta_t, double* re, double* im) {
  return guard([&] {
    check_lfa(p_t, mu);
    check_mode(mode);
    require(cfg && re && im, "null argument");
    require(cfg->nu1 >= 0 && cfg->nu2 >= 0, "nu must be >= 0");
    const stmg::lfa::Symbols s(p_t, mu);
    s.twogrid_symbol(cfg->omega_t, cfg->nu1, cfg->nu2, mode, theta_x, theta_t, re, im);
  });
}

int stmg_lfa_spectral_radius(int n, const double* re, const double* im, double* out) {
  return guard([&] {
    require(n >= 1 && re && out, "bad argument");
    *out = stmg::lfa::spectral_radius(n, re, im);
  });
}

int stmg_lfa_smoothing_factor(int p_t, double mu, double omega_t, int mode, int n_theta_x,
                              int n_theta_t, double* out) {
  return guard([&] {
    check_lfa(p_t, mu);
    check_mode(mode);
    require(out != nullptr, "null argument");
    *out = stmg::lfa::smoothing_factor(p_t, mu, omega_t, mode, n_theta_x, n_theta_t);
  });
}

int stmg_lfa_twogrid_factor(int p_t, double mu, const stmg_cycle_config* cfg, int mode,
                            int n_theta_x, int n_theta_t, double* out) {
  return guard([&] {
    check_lfa(p_t, mu);
    check_mode(mode);
    require(cfg && out, "null argument");
    require(cfg->nu1 >= 0 && cfg->nu2 >= 0, "nu must be >= 0");
    *out = stmg::lfa::twogrid_factor(p_t, mu, cfg->omega_t, cfg->nu1, cfg->nu2, mode, n_theta_x,
                                     n_theta_t);
  });
}

int stmg_lfa_twogrid_factor_inexact(int p_t, double mu, const stmg_cycle_config* cfg,
                                    double omega_x, int nu1_x, int nu2_x, int mode, int n_theta_x,
                                    int n_theta_t, double* out) {
  return guard([&] {
    check_lfa(p_t, mu);
    check_mode(mode);
    require(cfg && out, "null argument");
    require(cfg->nu1 >= 0 && cfg->nu2 >= 0 && nu1_x >= 0 && nu2_x >= 0, "nu must be >= 0");
    *out = stmg::lfa::twogrid_factor_inexact(p_t, mu, cfg->omega_t, cfg->nu1, cfg->nu2, omega_x,
                                             nu1_x, nu2_x, mode, n_theta_x, n_theta_t);
  });
}

// ------------------------------------------- two-grid factor measurement (GPU)
int stmg_measure_convergence_factor(const stmg_rho_problem* pr, const stmg_cycle_config* cfg,
                                    uint64_t seed, int n_theta_x, int n_theta_t,
                                    stmg_rho_measurement* out) {
  stmg_ctx* c = nullptr;
  double* u = nullptr;
  double* f = nullptr;
  double* r = nullptr;
  const int st = guard([&] {
    require(pr && cfg && out, "null argument");
    check_cfg(cfg);
    check_mode(pr->mode);
    require(pr->mu > 0.0, "mu must be positive");
    require(pr->time_level >= 1 && pr->time_level <= 30, "time_level out of range");
    require(pr->space_level >= 0 && pr->space_level <= 20, "space_level out of range");
    // tau = mu h^2 with h = 1 / (n1 + 1) (bench.cpp:81-83)
    const double h = 1.0 / double(int64_t(1) << (pr->space_level + 1));
    const int64_t n_t = int64_t(1) << pr->time_level;
    stmg_hierarchy_params hp{};
    hp.p_t = pr->p_t;
    hp.dim = pr->dim;
    hp.space_level = pr->space_level;
    hp.time_level = pr->time_level;
    hp.t_final = pr->mu * h * h * double(n_t);
    hp.mu_star = 0.0;
    hp.policy = STMG_POLICY_MU_DRIVEN;
    hp.two_grid = pr->mode;
    hp.device = pr->device;
    hp.shards = 1;
    if (stmg_create(&hp, &c) != STMG_OK) throw std::runtime_error(g_err);
    int64_t n = 0;
    CK_ABI(stmg_level_size(c, 0, &n));
    CK_ABI(stmg_device_alloc(c, size_t(n) * 8, reinterpret_cast<void**>(&u)));
    CK_ABI(stmg_device_alloc(c, size_t(n) * 8, reinterpret_cast<void**>(&f)));
    CK_ABI(stmg_device_alloc(c, size_t(n) * 8, reinterpret_cast<void**>(&r)));
    CK_ABI(stmg_memset_zero(c, f, size_t(n) * 8));
    stmg_rho_measurement m{};
    m.seed_used = seed;
    double r0 = 0.0;
    for (bool first = true;; first = false) {  // a zero initial residual reseeds (bench.cpp:107-121)
      if (!first) ++m.seed_used;
      CK_ABI(stmg_fill_uniform(c, u, n, m.seed_used, 1, 0));
      CK_ABI(stmg_residual(c, 0, u, f, r));
      CK_ABI(stmg_norm(c, 0, r, &r0));
      if (r0 > 0.0) break;
      require(m.seed_used - seed < 16, "initial guess keeps solving the system");
    }
    const double floor = 1e-13 * r0;
    double prev = r0, rho = 0.0;
    for (int k = 0; k < 250; ++k) {
      CK_ABI(stmg_mg_cycle(c, 0, u, f, cfg));
      double rk = 0.0;
      CK_ABI(stmg_residual(c, 0, u, f, r));
      CK_ABI(stmg_norm(c, 0, r, &rk));
      ++m.n_iterations_used;
      if (prev > floor) rho = std::max(rho, rk / prev);
      prev = rk;
      if (rk <= floor) break;
    }
    m.measured_rho = rho;
    // exact blocks: lfa::twogrid_factor (bench.cpp:142-143); inexact blocks
    // (an extension of the reference harness): the inexact-block symbol
    m.predicted_rho =
        cfg->block_solver == STMG_BLOCK_VCYCLE
            ? stmg::lfa::twogrid_factor_inexact(pr->p_t, pr->mu, cfg->omega_t, cfg->nu1, cfg->nu2,
                                                cfg->omega_x, cfg->nu1_x, cfg->nu2_x, pr->mode,
                                                n_theta_x, n_theta_t)
            : stmg::lfa::twogrid_factor(pr->p_t, pr->mu, cfg->omega_t, cfg->nu1, cfg->nu2,
                                        pr->mode, n_theta_x, n_theta_t);
    *out = m;
  });
  if (c) {
    if (u) stmg_device_free(c, u);
    if (f) stmg_device_free(c, f);
    if (r) stmg_device_free(c, r);
    stmg_destroy(c);
  }
  return st;
}

}  // extern "C"
