/*
 * stmg_b200.h -- C ABI of the B200-native space-time multigrid library.
 *
 * Drop-in boundary for the reference's hot path (arXiv 1411.0519 space-time
 * multigrid, /root/reference/proj).  The reference has no FFI: its boundary is
 * the C++ header API of the static library `stmg`.  Each entry point below
 * names the reference function it replaces (file:line, relative to
 * /root/reference/proj).  A C++ shim with the reference's own signatures is in
 * include/stmg_b200.hpp.
 *
 * Conventions
 *  - Every function returns an int status: STMG_OK (0), STMG_EINVAL (1, the
 *    reference's std::invalid_argument), STMG_ERUNTIME (2, std::runtime_error,
 *    CUDA or NCCL failures).  stmg_last_error() returns the message of the last
 *    failure on the calling thread.
 *  - Vectors are DEVICE pointers (double, FP64) in the reference BlockVector
 *    layout (block_vector.hpp:12-29): flat index (n*n_loc + l)*n_x + r with
 *    r = (iz*n1 + iy)*n1 + ix.  Only stmg_solve_host takes host pointers.
 *  - All compute calls are stream-ordered on the context's stream; only
 *    stmg_norm, stmg_solve*, stmg_download and stmg_synchronize synchronise.
 *  - The context is not thread-safe (one driver thread, like the reference).
 *  - There is no CPU fallback: without a CUDA device stmg_create fails.
 */
#ifndef STMG_B200_H
#define STMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STMG_OK 0
#define STMG_EINVAL 1
#define STMG_ERUNTIME 2

/* Coarsening policy (mg.hpp:47, CoarseningPolicy). */
#define STMG_POLICY_MU_DRIVEN 0
#define STMG_POLICY_ALWAYS_SEMI 1
#define STMG_POLICY_PREFER_FULL 2

/* Coarsening mode of a level (mg.hpp:12, Coarsening). */
#define STMG_COARSEN_NONE 0
#define STMG_COARSEN_SEMI 1
#define STMG_COARSEN_FULL 2

/* Cycle execution path. */
#define STMG_PATH_SPECTRAL 0 /* fused V-cycle on sine coefficients (default) */
#define STMG_PATH_PHYSICAL 1 /* reference call structure on nodal values */

typedef struct stmg_ctx stmg_ctx;

/* HierarchyParams (mg.hpp:49-58) + build_two_grid's mode (mg.hpp:81). */
typedef struct {
  int p_t;          /* DG degree in time, 0..10 (4..10: physical-path kernels) */
  int dim;          /* 1, 2 or 3 */
  int space_level;  /* finest space level L: n1 = 2^(L+1)-1 nodes per axis */
  int time_level;   /* finest n_t = 2^time_level */
  double t_final;   /* T; tau = T / n_t on the finest level */
  double mu_star;   /* full-coarsening threshold; <= 0 -> lfa::critical_mu(p_t) */
  int policy;       /* STMG_POLICY_* */
  int two_grid;     /* 0: full ladder; STMG_COARSEN_SEMI/FULL: build_two_grid */
  int device;       /* CUDA device ordinal */
  int shards;       /* >1: time-slab sharding emulated on this device (same
                       halo/gather/scatter logic as the multi-GPU path) */
} stmg_hierarchy_params;

/* Block solver behind the smoother (smoother.hpp:13, BlockSolverKind). */
#define STMG_BLOCK_EXACT 0  /* exact inverse of every time-step block */
#define STMG_BLOCK_VCYCLE 1 /* one spatial V-cycle per block (spatial_vcycle) */

/* CycleConfig + SmootherConfig (mg.hpp:66-71, smoother.hpp:15-24).  The
 * spatial fields are read only when block_solver == STMG_BLOCK_VCYCLE;
 * stmg_cycle_config_init fills the reference defaults. */
typedef struct {
  int nu1;          /* pre-smoothing sweeps */
  int nu2;          /* post-smoothing sweeps */
  int gamma;        /* 1 = V-cycle */
  double omega_t;   /* block-Jacobi damping */
  int path;         /* STMG_PATH_* */
  int block_solver; /* STMG_BLOCK_* (0 = exact when zero-initialised) */
  double omega_x;   /* spatial damped-Jacobi weight (2/3) */
  int nu1_x;        /* spatial pre-smoothing sweeps (2) */
  int nu2_x;        /* spatial post-smoothing sweeps (2) */
  int gamma_x;      /* spatial cycle index (1 = V) */
} stmg_cycle_config;

/* SmootherConfig (smoother.hpp:15-24) for the single-operator entry points. */
typedef struct {
  double omega_t;   /* damping of the block Jacobi iteration (0.5) */
  int nu;           /* smoothing steps per call (1) */
  int block_solver; /* STMG_BLOCK_* */
  double omega_x;   /* (2/3) */
  int nu1_x, nu2_x; /* (2, 2) */
  int gamma_x;      /* (1) */
} stmg_smoother_config;

/* SolveReport (mg.hpp:83-89). */
typedef struct {
  int iterations;
  int converged;
  double wall_time_seconds;   /* host wall clock of the whole call */
  double device_time_seconds; /* CUDA events around the solve on the ctx stream
                                 (basis transforms included, host I/O excluded) */
  double r0;
  double r_final;
  uint64_t seed;
} stmg_solve_report;

/* STLevel summary (mg.hpp:19-36). */
typedef struct {
  int64_t n_t, n_x, n_loc, n1;
  int dim, space_level, coarsen_to_next;
  double tau, h, mu;
} stmg_level_info;

const char* stmg_last_error(void);

/* lfa::critical_mu (lfa.cpp:317-328); returns NaN on invalid p_t. */
double stmg_critical_mu(int p_t);
/* assemble_dg_block (dg_time.cpp:125-166): row-major (p_t+1)^2 blocks. */
int stmg_dg_block(int p_t, double tau, double* K, double* M, double* N);
/* build_time_transfer (transfer.cpp:50-73): row-major R1, R2. */
int stmg_time_transfer(int p_t, double tau, double* R1, double* R2);

/* build_hierarchy / build_two_grid (mg.cpp:10-94) + device setup. */
int stmg_create(const stmg_hierarchy_params* params, stmg_ctx** out);
int stmg_destroy(stmg_ctx* ctx);
int stmg_num_levels(const stmg_ctx* ctx, int* out);
int stmg_get_level_info(const stmg_ctx* ctx, int level, stmg_level_info* out);
/* Number of doubles of a level vector (BlockVector::size). */
int stmg_level_size(const stmg_ctx* ctx, int level, int64_t* out);

/* Device memory plumbing (plain pointers and sizes). */
int stmg_device_alloc(stmg_ctx* ctx, size_t bytes, void** dptr);
int stmg_device_free(stmg_ctx* ctx, void* dptr);
int stmg_upload(stmg_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
int stmg_download(stmg_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);
int stmg_memset_zero(stmg_ctx* ctx, void* dst_dev, size_t bytes);
/* Page-locked host buffers for the end-to-end path (cudaHostAlloc). */
int stmg_host_alloc(stmg_ctx* ctx, size_t bytes, void** hptr);
int stmg_host_free(stmg_ctx* ctx, void* hptr);
int stmg_synchronize(stmg_ctx* ctx);
/* Seeded counter-based uniform[-1,1) fill; identical to the
 * host generator for the same (seed, stream, global offset). */
int stmg_fill_uniform(stmg_ctx* ctx, double* dst_dev, int64_t n, uint64_t seed,
                      uint64_t stream, int64_t offset);
/* f(0,k,:) += psi_k(0) * M_h u0 on the finest level (u0: n_x nodal values). */
int stmg_fold_u0(stmg_ctx* ctx, double* f_dev, const double* u0_dev);
/* fill_random (mg.cpp:168-173), reference-exact, on the HOST (no GPU needed):
 * std::mt19937_64 gen(seed); dst[i] = (gen() >> 11) * 2^-53, i = 0..n-1. */
int stmg_fill_random_host(double* dst_host, int64_t n, uint64_t seed);

/* Reference defaults: CycleConfig (mg.hpp:66-71: nu1 = nu2 = 2, gamma = 1)
 * with SmootherConfig (smoother.hpp:15-24: omega_t = 1/2, exact blocks,
 * omega_x = 2/3, nu1_x = nu2_x = 2, gamma_x = 1), spectral path. */
int stmg_cycle_config_init(stmg_cycle_config* cfg);
int stmg_smoother_config_init(stmg_smoother_config* cfg);

/* ---- operators: reference entry points (device pointers) ---------------- */
/* apply (st_system.cpp:44-49): y = L u. */
int stmg_apply(stmg_ctx* ctx, int level, const double* u, double* y);
/* residual (st_system.cpp:57-67): r = f - L u. */
int stmg_residual(stmg_ctx* ctx, int level, const double* u, const double* f,
                  double* r);
/* BlockVector::norm (st_system.cpp:8-16); synchronising. */
int stmg_norm(stmg_ctx* ctx, int level, const double* v, double* out);
/* BlockSolver::solve on every time step (st_system.cpp:110-116). */
int stmg_block_solve(stmg_ctx* ctx, int level, const double* b, double* x);
/* block_jacobi_step, exact blocks (smoother.cpp:96-106): nu sweeps of
 * u <- u + omega_t A^-1 (f - L u). */
int stmg_smooth(stmg_ctx* ctx, int level, double* u, const double* f,
                double omega_t, int nu);
/* block_jacobi_step with a full SmootherConfig (smoother.cpp:96-106): nu
 * sweeps of u <- u + omega_t D~^-1 (f - L u), D~^-1 = the exact block inverse
 * or one spatial V-cycle per time step (block_solver). */
int stmg_block_jacobi_step(stmg_ctx* ctx, int level, double* u, const double* f,
                           const stmg_smoother_config* cfg);
/* SpatialVCycleSolver::cycle (smoother.cpp:71-78) on every time step of the
 * level: x_n = cycle(b_n, x0_n); x0 NULL = zero initial guess (the smoother's
 * D~ approximation).  Uses omega_x, nu1_x, nu2_x, gamma_x of cfg. */
int stmg_spatial_vcycle(stmg_ctx* ctx, int level, const double* b, const double* x0,
                        double* x, const stmg_smoother_config* cfg);
/* restrict_semi / restrict_full (transfer.cpp:75-85, 138-149).  mode 0 uses
 * the level's coarsen_to_next. */
int stmg_restrict(stmg_ctx* ctx, int level, int mode, const double* fine,
                  double* coarse);
/* prolong_semi / prolong_full (transfer.cpp:87-96, 151-158). */
int stmg_prolong(stmg_ctx* ctx, int level, int mode, const double* coarse,
                 double* fine);
/* forward_substitution_solve (st_system.cpp:118-130). */
int stmg_forward_substitution(stmg_ctx* ctx, int level, const double* f,
                              double* u);
/* mg_cycle (mg.cpp:96-132): one gamma-cycle from `level` on u in place. */
int stmg_mg_cycle(stmg_ctx* ctx, int level, double* u, const double* f,
                  const stmg_cycle_config* cfg);
/* solve (mg.cpp:134-166): cycles until ||r_k|| <= eps ||r_0|| or max_iter.
 * history (optional, capacity history_cap) receives ||r_0||, ||r_1||, ... */
int stmg_solve(stmg_ctx* ctx, const double* f, double* u,
               const stmg_cycle_config* cfg, double eps, int max_iter,
               double* history, int history_cap, stmg_solve_report* report);
/* Same with HOST f and u (pinned or pageable): H2D, solve, D2H. */
int stmg_solve_host(stmg_ctx* ctx, const double* f_host, double* u_host,
                    const stmg_cycle_config* cfg, double eps, int max_iter,
                    double* history, int history_cap, stmg_solve_report* report);
/* Extension (no reference counterpart; solve, mg.cpp:134-166, takes one f per
 * call): a batch of independent solves (many right-hand sides / initial
 * guesses) streamed through one context.  Problem i solves from u0_host[i]
 * (u0_host NULL: u_host[i] in place) into u_host[i] while the H2D of problem
 * i+1 and i+2 and the D2H of problem i-1 run on the copy engines (three
 * device staging sets).  Each result is bitwise stmg_solve_host's.  Because
 * uploads run two problems ahead, the inputs of problem j (f_host[j] and
 * u0_host[j], or u_host[j] in place) must not overlap u_host[j-1] or
 * u_host[j-2]; an overlapping batch fails with STMG_EINVAL.  A NULL entry
 * u0_host[i] (u0_host itself non-NULL) is a zero initial guess: nothing is
 * uploaded for it (the device buffer is cleared), so only f crosses PCIe.  reports (optional) gets
 * count entries; wall_time_seconds there is per solve, without the overlapped
 * copies.  Host buffers should be pinned (stmg_host_alloc) for the copies to
 * overlap. */
int stmg_solve_host_batch(stmg_ctx* ctx, int count, const double* const* f_host,
                          const double* const* u0_host, double* const* u_host,
                          const stmg_cycle_config* cfg, double eps,
                          int max_iter, stmg_solve_report* reports);

/* ---- multi-GPU: time slabs over ranks (one process per GPU, NCCL) ------- */
/* 128-byte NCCL unique id, created on rank 0 and broadcast by the caller. */
int stmg_nccl_unique_id(void* out, size_t len);
/* Context owning time steps [rank*n_t/world, (rank+1)*n_t/world) of the finest
 * level; stmg_solve / stmg_solve_host then take this rank's slabs of f and u.
 * Coarse levels with fewer than 2 steps per rank run on rank 0. */
int stmg_create_distributed(const stmg_hierarchy_params* params, int rank,
                            int world, const void* nccl_id, size_t id_len,
                            stmg_ctx** out);
/* Sharding plan (host only, no GPU needed): first level gathered onto rank 0
 * and finest-level steps per shard. */
int stmg_shard_plan(const stmg_hierarchy_params* params, int shards,
                    int* gather_level, int64_t* steps_per_shard);
/* Finest-level time steps owned by this context. */
int stmg_local_steps(const stmg_ctx* ctx, int64_t* first_step,
                     int64_t* n_steps);

/* ---- live per-kernel timing (CUDA events inside the cycle) --------------- */
/* Kernel ids: 0 = fused pre-smooth+residual+restrict on the finest level
 *                 (fused V(1,1) schedule: the k_updown pass),
 *             1 = fused prolong+correct+post-smooth+residual-norm (finest),
 *             2 = basis transform pass, 3 = physical residual,
 *             4 = coarse part of a fused V(1,1) cycle (levels >= 1, all
 *                 kernels between two finest-level passes; bytes = 0),
 *             5 = one damped block-Jacobi sweep of the physical smoother
 *                 (stmg_smooth, exact blocks: residual + transforms + modal
 *                 solve + update; bytes = 24 per dof, the reference's unit). */
int stmg_profile_enable(stmg_ctx* ctx, int on);
int stmg_profile_read(stmg_ctx* ctx, int kernel_id, double* total_ms,
                      int64_t* launches, double* bytes_per_launch);
int stmg_profile_reset(stmg_ctx* ctx);
/* Kernel launches issued by the library since creation (all kinds). */
int stmg_launch_count(const stmg_ctx* ctx, int64_t* out);

/* ---- local Fourier analysis (lfa.hpp:15-150; host only, no GPU) ----------
 * Nondimensionalised like the reference: h = 1, tau = mu; mode is
 * STMG_COARSEN_SEMI or STMG_COARSEN_FULL; cfg supplies nu1, nu2, omega_t. */
/* beta(theta_x) = 6 (1 - cos)/(2 + cos) (lfa.hpp:15-17). */
int stmg_lfa_beta(double theta_x, double* out);
/* alpha = R(-mu beta(theta_x)) (lfa.hpp:19-20). */
int stmg_lfa_alpha(int p_t, double mu, double theta_x, double* out);
/* Spectral radius of the damped block-Jacobi symbol, by eigenvalues and by
 * the closed form (SymbolBuilder::smoother_symbol / smoother_rho_closed_form,
 * lfa.hpp:75-85). */
int stmg_lfa_smoother_rho(int p_t, double mu, double omega_t, double theta_x,
                          double theta_t, double* rho, double* rho_closed_form);
/* (p_t+1)^2 smoother symbol, row-major real / imaginary parts (lfa.hpp:75-77). */
int stmg_lfa_smoother_symbol(int p_t, double mu, double omega_t, double theta_x,
                             double theta_t, double* re, double* im);
/* (4(p_t+1))^2 two-grid symbol on the four harmonics (lfa.hpp:93-99);
 * STMG_EINVAL for theta_x = 0 (the reference's std::domain_error). */
int stmg_lfa_twogrid_symbol(int p_t, double mu, const stmg_cycle_config* cfg, int mode,
                            double theta_x, double theta_t, double* re, double* im);
/* Spectral radius of an n x n complex matrix (lfa.hpp:50); im may be NULL. */
int stmg_lfa_spectral_radius(int n, const double* re, const double* im, double* out);
/* smoothing_factor (lfa.hpp:125-132): sup over the closed high-frequency
 * region, grid n_theta_x x n_theta_t (each at least 64). */
int stmg_lfa_smoothing_factor(int p_t, double mu, double omega_t, int mode,
                              int n_theta_x, int n_theta_t, double* out);
/* twogrid_factor (lfa.hpp:137-141): max over the sampled low quarter. */
int stmg_lfa_twogrid_factor(int p_t, double mu, const stmg_cycle_config* cfg, int mode,
                            int n_theta_x, int n_theta_t, double* out);
/* twogrid_factor_inexact (lfa.hpp:142-145): block solves replaced by one
 * spatial two-grid iteration (damped Jacobi omega_x, nu1_x / nu2_x sweeps). */
int stmg_lfa_twogrid_factor_inexact(int p_t, double mu, const stmg_cycle_config* cfg,
                                    double omega_x, int nu1_x, int nu2_x, int mode,
                                    int n_theta_x, int n_theta_t, double* out);

/* ---- two-grid factor measurement on the GPU (bench.hpp:12-39) ------------ */
typedef struct {
  int p_t;
  int dim;
  int space_level;
  int time_level;
  double mu;      /* tau = mu h^2 */
  int mode;       /* STMG_COARSEN_SEMI / STMG_COARSEN_FULL */
  int device;
} stmg_rho_problem;

typedef struct {
  double measured_rho;   /* largest ||r_k+1|| / ||r_k|| above the 1e-13 guard */
  double predicted_rho;  /* stmg_lfa_twogrid_factor of the same problem */
  int n_iterations_used;
  uint64_t seed_used;
} stmg_rho_measurement;

/* measure_convergence_factor (bench.cpp:77-145): f = 0, seeded random initial
 * guess (this library's uniform generator, stream 1), two-grid cycles with
 * exact block solves until ||r|| <= 1e-13 ||r_0|| or 250 cycles. */
int stmg_measure_convergence_factor(const stmg_rho_problem* problem,
                                    const stmg_cycle_config* cfg, uint64_t seed,
                                    int n_theta_x, int n_theta_t,
                                    stmg_rho_measurement* out);

#ifdef __cplusplus
}
#endif
#endif /* STMG_B200_H */
