/*
 * pcal_oracle.h — CPU restatement of the reference PCAL path (TEST INFRASTRUCTURE).
 *
 * This is the parity CHECKER for the B200 implementation, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  Every function restates one reference routine of
 * /root/reference/proj/core (cited file:line) with the same floating-point
 * operation order; compiled with -ffp-contract=off it reproduces the reference
 * bit for bit on the dense models (pinned by tests/golden/, generated from the
 * reference itself via oracle/_ref).  The stencil and Kohn–Sham-like models of
 * configs 3–5 have no reference implementation: they follow DESIGN.md §3
 * and are pinned by finite differences and by a dense
 * operator cross-check on tiny grids ("parity unpinned" by any reference test).
 */
#ifndef PCAL_ORACLE_H
#define PCAL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: xoshiro256++ seeded by splitmix64, Box–Muller normals (rng.hpp:13-55,
 *      kernels.cpp:65-78) ---------------------------------------------------- */
typedef struct {
  uint64_t s[4];
  double spare;
  int has_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
/* random_normal / random_uniform (kernels.cpp:49-63): column-major fill.
 * threads > 1 splits the Box–Muller work over checkpointed generator states;
 * the output is bitwise identical to the sequential fill. */
void orc_random_normal(int64_t count, uint64_t seed, double* out, int threads);
void orc_random_uniform(int64_t count, uint64_t seed, double* out);

/* ---- dense kernels (kernels.cpp) ---------------------------------------- */
void orc_sym_part(const double* m, int64_t n, double* out);              /* :28-36 */
void orc_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t ncols,
                double* c, int threads);                                 /* :105-122 */
void orc_matmul_at_b(const double* a, int64_t n, int64_t m, const double* b,
                     int64_t ncols, double* c, int threads);             /* :124-137 */
void orc_gram(const double* x, int64_t n, int64_t p, double* g, int threads); /* :139-153 */
double orc_dot(const double* a, const double* b, int64_t n);             /* :20-24 */
double orc_frobenius_norm(const double* a, int64_t count);               /* :311-313 */
/* orthonormalize (kernels.cpp:250-265): CholeskyQR2 with MGS2 fallback.
 * Returns 0, or ORC_E_RANK when the fallback hits the pivot floor. */
int orc_orthonormalize(const double* x, int64_t n, int64_t p, double* q);
int orc_orthonormalize_t(const double* x, int64_t n, int64_t p, double* q, int threads);
/* mgs2 (kernels.cpp:212-246) alone: ORC_E_RANK when a column norm² ≤ floor. */
int orc_mgs2(const double* x, int64_t n, int64_t p, double floor_, double* q);
/* blocked restatements (orc_blas.c), bitwise equal to the reference loops */
void orc_blas_matmul(const double* a, int64_t m, int64_t kdim, const double* b, int64_t ncols,
                     double* c, int threads);
void orc_blas_at_b(const double* a, int64_t n, int64_t m, const double* b, int64_t ncols,
                   double* c, int threads);
void orc_blas_gram(const double* x, int64_t n, int64_t p, double* g, int threads);
/* spectral_norm_estimate (kernels.cpp:267-293). */
double orc_spectral_norm_estimate(const double* a, int64_t n, uint64_t seed, int threads);

/* ---- objective models (problems.hpp:28-111 + DESIGN.md §3) -------------- */
enum { ORC_MODEL_DENSE = 1, ORC_MODEL_STENCIL = 2, ORC_MODEL_KOHN_SHAM = 3 };

typedef struct {
  int kind;
  int64_t n, p;
  double s;              /* curvature_scale() */
  const double* a;       /* dense: n×n column-major symmetric */
  const double* g0;      /* dense: optional n×p linear term (NULL = 0) */
  int64_t nx, ny, nz;    /* grid models: n = nx·ny·nz, row i = x + nx(y + ny z) */
  const double* v;       /* stencil: V (n); Kohn–Sham: V_ion (n) */
  void* work;            /* Kohn–Sham: spectral tables (orc_model_prepare) */
} orc_model;

int orc_model_prepare(orc_model* m);  /* allocates KS tables; no-op otherwise */
void orc_model_release(orc_model* m);
/* ObjectiveModel::evaluate: returns 0, or ORC_E_EVAL for a non-finite f or G
 * (check_finite, problems.cpp:27-30). */
int orc_evaluate(const orc_model* m, const double* x, double* f, double* g, int threads);
/* Operator pieces for the grid models (exposed for tests). */
void orc_laplacian_apply(const double* x, int64_t nx, int64_t ny, int64_t nz,
                         int64_t p, double* lx);
int orc_pseudo_inverse_laplacian(const orc_model* m, const double* rho, double* out);
/* Fourier basis of the periodic N-point second difference. */
void orc_fourier_basis(int64_t N, double* q /* N×N, q[i + N*m] */, double* lam /* N */);
/* Finite-difference gradient check (problems.cpp:296-325). */
double orc_fd_gradient_check(const orc_model* m, const double* x, double h, uint64_t seed);

/* ---- solver (solver.hpp:13-42, solver.cpp) ------------------------------ */
enum { ORC_ETA_CONSTANT = 0, ORC_ETA_DIFFERENTIAL = 1, ORC_ETA_BB1 = 2, ORC_ETA_BB2 = 3,
       ORC_ETA_ABB = 4 };
enum { ORC_MULT_PLAM = 0, ORC_MULT_PCAL = 1 };
enum { ORC_CONVERGED = 0, ORC_MAXITER = 1, ORC_DIVERGED = 2 };
enum { ORC_OK = 0, ORC_E_PARAM = -1, ORC_E_DIM = -2, ORC_E_RANK = -3, ORC_E_EVAL = -4,
       ORC_E_DIVERGE = -5, ORC_E_ALLOC = -6 };

/* Algorithm (diagnostics.hpp:10), reference enum order */
enum { ORC_ALG_PLAM = 0, ORC_ALG_PCAL = 1, ORC_ALG_ALM = 2, ORC_ALG_MOPTQR = 3, ORC_ALG_PLAMDA = 4,
       ORC_ALG_PCALDA = 5 };

typedef struct {
  double beta;            /* < 0: per-algorithm default (solver.cpp:120-134) */
  int eta_kind;           /* ORC_ETA_* (StepsizeRule::Kind order) */
  double gamma, eta_min, eta_max, eta0;
  int multiplier_rule;    /* ORC_MULT_* */
  double tol_rel_kkt;
  int64_t max_iter;
  int threads;
  int final_orth;
  int algorithm;          /* ORC_ALG_* (ALM is not restated: ORC_E_PARAM) */
} orc_config;

void orc_config_default(orc_config* c); /* SolverConfig defaults, solver.hpp:13-42 */

#define ORC_TRACE_COLS 7 /* iter, fval, kkt_abs, kkt_rel, feas, eta, elapsed */

typedef struct {
  double* trace;          /* (max_iter+1) × ORC_TRACE_COLS, caller-owned */
  int64_t trace_len;
  double final_pre[4];    /* fval, kkt_abs, kkt_rel, feas */
  double final_post[4];
  int has_post;
  double* stop_x;         /* n×p or NULL */
  double* final_x;        /* n×p or NULL */
  int has_x;
  int64_t iterations;
  int64_t degenerate_steps;
  double wall_time;
  int status;
  double beta_used, eta0_used;
  /* optional snapshots of the iterate X_k (k = snap_iters[i]) */
  const int64_t* snap_iters;
  int nsnap;
  double* snaps;          /* nsnap × n × p */
  double* snap_eta;       /* eta used to produce X_k (k ≥ 1), per snapshot */
} orc_report;

/* solve() — iterate_main (solver.cpp:320-474, 626-633) for PLAM, PCAL,
 * MOptQR, PLAM-DA and PCAL-DA.  Returns 0 or a negative ORC_E_* for errors the
 * reference throws out of solve(). */
int orc_solve(const orc_model* m, const orc_config* c, const double* x0, orc_report* r);
int orc_solve_pcal(const orc_model* m, const orc_config* c, const double* x0, orc_report* r);

/* Building blocks (solver.hpp:74-113) */
double orc_stepsize_select(const orc_config* c, int64_t iter, double eta_prev, double eta0,
                           const double* x, const double* xp, const double* gl,
                           const double* glp, int64_t count);
int orc_pcal_step(const double* x, const double* gl, int64_t n, int64_t p, double eta,
                  double* out, int64_t* degenerate, int threads);
/* PCAL multiplier + aug-Lagrangian gradient at x (solver.cpp:67-88 + 385-409):
 * returns grad_l (n×p) and f/kkt_abs/feas. */
int orc_pcal_grad_l(const orc_model* m, const double* x, double beta, int mult_rule,
                    double* grad_l, double* f, double* kkt_abs, double* feas, int threads);

double orc_flops_estimate_pcal(int64_t n, int64_t p); /* diagnostics.cpp:100-114 */

#ifdef __cplusplus
}
#endif
#endif
