/*
 * stmg_oracle.h -- C ABI of the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * The oracle is a plain C++/OpenMP restatement of the reference space-time
 * multigrid (arXiv 1411.0519, /root/reference/proj) used as the parity checker
 * for the B200 library and as the CPU baseline timed by bench.py.  Only
 * tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference) may load it.  The product library never links it.
 *
 * Parity pinning: the reference cannot be built here (Eigen3/doctest absent,
 * proj/CMakeLists.txt:11), so the oracle is pinned against every known-answer
 * test the reference's own unit tests hold for this path (tests/golden/kats.json)
 * and against scipy.sparse.linalg.splu for the exact block solve (the
 * reference's Eigen SparseLU boundary, st_system.cpp:103-116).
 *
 * Vector layout = reference BlockVector (block_vector.hpp:12-29):
 *   flat index (n * n_loc + l) * n_x + r,  r = (iz * n1 + iy) * n1 + ix.
 */
#ifndef STMG_ORACLE_H
#define STMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_hier or_hier;

typedef struct {
  int p_t;          /* DG degree in time, 0..10 */
  int dim;          /* 1, 2 or 3 (3 = extension; the reference throws) */
  int space_level;  /* finest space level L: n1 = 2^(L+1) - 1 */
  int time_level;   /* finest n_t = 2^time_level */
  double t_final;   /* T; tau = T / n_t */
  double mu_star;   /* <= 0: use critical_mu(p_t) */
  int policy;       /* 0 mu_driven, 1 always_semi, 2 prefer_full */
  int two_grid;     /* 0 full ladder; 1 semi two-grid; 2 full two-grid */
} or_params;

/* CycleConfig + its SmootherConfig (mg.hpp:66-71, smoother.hpp:15-24).
 * block_solver: 0 exact, 1 spatial_vcycle (omega_x, nu1_x, nu2_x, gamma_x). */
typedef struct {
  int nu1, nu2, gamma;
  double omega_t;
  int block_solver;
  double omega_x;
  int nu1_x, nu2_x, gamma_x;
} or_cycle;

/* SmootherConfig (smoother.hpp:15-24). */
typedef struct {
  double omega_t;
  int nu;
  int block_solver;
  double omega_x;
  int nu1_x, nu2_x, gamma_x;
} or_smoother;

typedef struct {
  int64_t n_t, n_x, n_loc, n1;
  int dim, space_level, coarsen_to_next; /* 0 none, 1 semi, 2 full */
  double tau, h, mu;
} or_level_info;

/* errors: 0 ok, 1 invalid_argument, 2 runtime_error */
const char* or_last_error(void);

/* dg_time.cpp:125-166, transfer.cpp:50-73, lfa.cpp:317-328 */
int or_assemble_dg(int p_t, double tau, double* K, double* M, double* N);
int or_time_transfer(int p_t, double tau, double* R1, double* R2);
double or_pade(int p_t, double z);
double or_critical_mu(int p_t);

/* mg.cpp:10-75 / 77-94 */
int or_hier_create(const or_params* p, or_hier** out);
void or_hier_destroy(or_hier* h);
int or_hier_levels(const or_hier* h);
int or_level_info_get(const or_hier* h, int level, or_level_info* out);

/* st_system.cpp */
int or_apply(const or_hier* h, int level, const double* u, double* y);
int or_residual(const or_hier* h, int level, const double* u, const double* f,
                double* r);
double or_norm(const or_hier* h, int level, const double* v);
/* norm(residual(u, f)) without a residual vector (bitwise the same value). */
double or_residual_norm(const or_hier* h, int level, const double* u,
                        const double* f);
int or_block_solve(const or_hier* h, int level, const double* b, double* x);
int or_forward_substitution(const or_hier* h, int level, const double* f,
                            double* u);
/* smoother.cpp:96-106 */
int or_smooth(const or_hier* h, int level, double* u, const double* f,
              double omega_t, int nu);
/* block_jacobi_step with a full SmootherConfig (smoother.cpp:96-106). */
int or_smooth_ex(const or_hier* h, int level, double* u, const double* f,
                 const or_smoother* cfg);
/* SpatialVCycleSolver::cycle (smoother.cpp:71-78) on every time step of the
 * level: x_n = cycle(b_n, x0_n) (x0 may be NULL = zero guess). */
int or_spatial_vcycle(const or_hier* h, int level, const double* b,
                      const double* x0, double* x, const or_smoother* cfg);
/* transfer.cpp: mode 1 semi, 2 full, 0 = level's coarsen_to_next */
int or_restrict(const or_hier* h, int level, int mode, const double* fine,
                double* coarse);
int or_prolong(const or_hier* h, int level, int mode, const double* coarse,
               double* fine);
/* mg.cpp:96-166 */
int or_mg_cycle(const or_hier* h, int level, double* u, const double* f,
                const or_cycle* cfg);
int or_solve(const or_hier* h, const double* f, double* u, const or_cycle* cfg,
             double eps, int max_iter, double* history, int history_cap,
             int* iterations, int* converged, double* wall_seconds);

/* Synthetic inputs: splitmix64 counter generator. */
void or_fill_uniform(double* v, int64_t n, uint64_t seed, uint64_t stream,
                     int64_t offset);
/* f(0,k,:) += psi_k(0) * M_h u0 (u0: n_x interior nodal values). */
int or_fold_u0(const or_hier* h, double* f, const double* u0);

#ifdef __cplusplus
}
#endif
#endif
