/*
 * pcal_b200.h — C ABI of the B200-native PCAL iteration (libpcal_b200.so).
 *
 * This is the drop-in boundary for the reference's solver entry point
 *   orthopt::RunReport orthopt::solve(const ObjectiveModel&, const SolverConfig&,
 *                                      const DenseMatrix& x0, CategoryTimers*)
 *   (/root/reference/proj/core/include/orthopt/solver.hpp:120-121)
 * restated with plain pointers and sizes.  Matrices are FP64, column-major
 * (element (i,j) at data[i + j*rows]) exactly like orthopt::DenseMatrix
 * (matrix.hpp:38-45), so host buffers round-trip without transposes.
 *
 * The reference's virtual gradient callback ObjectiveModel::evaluate
 * (problems.hpp:39) cannot be a host callback here (X lives in HBM), so the
 * model is a descriptor of a device-evaluated objective (pcal_model_desc):
 * dense quadratic (QuadraticModel, problems.hpp:53-69), 7-point periodic
 * stencil + diagonal potential, or the Kohn–Sham-like density model.  An
 * unsupported model is an error; there is no CPU fallback.
 *
 * Errors the reference throws out of solve() (parameter_error, dimension_error,
 * solver.cpp:106-118,628-630) are returned as negative codes with a message in
 * pcal_last_error().  In-run failures (divergence_error / evaluation_error /
 * rank_error, solver.cpp:460-471) are NOT errors: the report carries
 * status = PCAL_STATUS_DIVERGED and a partial trace, as in the reference.
 */
#ifndef PCAL_B200_H
#define PCAL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define PCAL_OK 0
#define PCAL_E_PARAMETER (-1)   /* orthopt::parameter_error   (errors.hpp:24-28) */
#define PCAL_E_DIMENSION (-2)   /* orthopt::dimension_error   (errors.hpp:9-13)  */
#define PCAL_E_RANK (-3)        /* orthopt::rank_error        (errors.hpp:15-19) */
#define PCAL_E_UNSUPPORTED (-4) /* model/algorithm not provided by this library   */
#define PCAL_E_CUDA (-5)        /* CUDA runtime failure / no device               */
#define PCAL_E_STATE (-6)       /* API misuse (e.g. reading an unfinished run)     */
#define PCAL_E_DIVERGENCE (-7)  /* building blocks only: orthopt::divergence_error (errors.hpp:33-45) */
#define PCAL_E_EVALUATION (-8)  /* building blocks only: orthopt::evaluation_error (errors.hpp:27-31) */

/* run status — orthopt::RunStatus (report.hpp:37) */
#define PCAL_STATUS_CONVERGED 0
#define PCAL_STATUS_MAX_ITER 1
#define PCAL_STATUS_DIVERGED 2

/* model kinds */
#define PCAL_MODEL_DENSE 1      /* f = ½tr(XᵀAX) + tr(G0ᵀX), A n×n symmetric (problems.cpp:130-141) */
#define PCAL_MODEL_STENCIL 2    /* f = ½tr(XᵀLX) + ½tr(XᵀVX), L = −Δ_h 7-point periodic */
#define PCAL_MODEL_KOHN_SHAM 3  /* E = ¼tr(XᵀLX)+½tr(XᵀV_ionX)+¼ρᵀL†ρ+½ρᵀε_xc(ρ) */
#define PCAL_MODEL_DEVICE_CALLBACK 4  /* any f: the caller's own device gradient (below) */
#define PCAL_MODEL_BILINEAR 5   /* f = ½tr(XᵀAXB), A n×n, B p×p symmetric (problems.cpp:143-156, P4) */
#define PCAL_MODEL_DENSITY 6    /* f = ½tr(XᵀLX) + density term of ρ = rowsq(X), h = L⁻¹ρ
                                   (DensityModel, problems.cpp:158-206, P1 / P6) */

/* DensityModel's two density terms (problems.cpp:179-203) */
#define PCAL_DENSITY_P1 0       /* + ¼·coeff·ρᵀh,            G += coeff·h∘X          */
#define PCAL_DENSITY_P6 1       /* + ½ρᵀh − ¾·coeff·Σρ^{4/3}, G += (2h − 2coeff·ρ^{1/3})∘X */

/* ObjectiveModel::evaluate (problems.hpp:39) for a caller-defined model, on the
 * device: enqueue on `stream` (a cudaStream_t) the work that writes G = ∇f(X)
 * into g (n×p, leading dimension ld, column-major) and f(X) into the device
 * scalar *f, reading X (same layout).  Rows n..ld-1 of x are zero and those of
 * g must stay zero.  The call only ENQUEUES: it may be made while the stream is
 * being captured into a CUDA graph, so it must not synchronise, allocate or
 * copy to/from the host.  Return 0 on success.  Non-finite G or f is detected
 * by the library (evaluation_error ⇒ status Diverged, solver.cpp:460-466). */
typedef int (*pcal_gradient_fn)(const double* x, int64_t ld, int64_t n, int64_t p, double* g,
                                double* f, void* stream, void* ctx);

/* pointer location for model data / x0 */
#define PCAL_HOST 0
#define PCAL_DEVICE 1
/* x0 only (session create / solve): x0 points to a uint64_t seed and the
 * library builds initial_point({Qr}, seed) itself — orthonormalize(random_normal
 * (n, p, Rng(seed))), solver.cpp:136-142 — on the device.  A sharded session
 * draws only its own rows of the Gaussian (checkpointed reference stream) and
 * orthonormalises them with the chunk-ordered Gram of the final CholeskyQR2,
 * so no rank ever holds the global n×p start point and X0 is bitwise the same
 * for every rank count. */
#define PCAL_X0_SEED 2

/* StepsizeRule::Kind (solver.hpp:13-20), same order */
#define PCAL_ETA_CONSTANT 0
#define PCAL_ETA_DIFFERENTIAL 1
#define PCAL_ETA_BB1 2
#define PCAL_ETA_BB2 3
#define PCAL_ETA_ABB 4

/* MultiplierRule (solver.hpp:22) */
#define PCAL_MULT_PLAM_FORMULA 0
#define PCAL_MULT_PCAL_FORMULA 1

/* Algorithm (diagnostics.hpp:10), reference enum order. */
#define PCAL_ALG_PLAM 0
#define PCAL_ALG_PCAL 1
#define PCAL_ALG_ALM 2         /* alm_outer (solver.cpp:478-624); single GPU and row-sharded */
#define PCAL_ALG_MOPTQR 3
#define PCAL_ALG_PLAMDA 4
#define PCAL_ALG_PCALDA 5

typedef struct pcal_model_desc {
  int32_t kind;          /* PCAL_MODEL_* */
  int32_t location;      /* PCAL_HOST / PCAL_DEVICE for a, g0, v */
  int64_t n, p;          /* ObjectiveModel::n(), p() */
  double s;              /* ObjectiveModel::curvature_scale() (sets eta0 = s + 2β) */
  const double* a;       /* dense: n×n column-major, symmetric */
  const double* g0;      /* dense: n×p linear term or NULL (zero) */
  int64_t nx, ny, nz;    /* grid models: n = nx·ny·nz, row i = x + nx·(y + ny·z) */
  const double* v;       /* stencil: V (n); Kohn–Sham: V_ion (n) */
  pcal_gradient_fn grad; /* PCAL_MODEL_DEVICE_CALLBACK: the gradient callback */
  void* grad_ctx;        /* its context pointer */
  const double* b;       /* bilinear: B p×p column-major, symmetric (location as a) */
  const double* linv;    /* density: L⁻¹ rows (the a slab's rows, all n_glob columns; ld = rows),
                            from pcal_density_inverse — the reference's LinearSolver */
  double coeff;          /* density: α (P1) or γ (P6) */
  int32_t density_variant; /* PCAL_DENSITY_P1 / PCAL_DENSITY_P6 */
} pcal_model_desc;

typedef struct pcal_config {  /* orthopt::SolverConfig (solver.hpp:30-42) */
  int32_t algorithm;          /* PCAL_ALG_* (PCAL default; PLAM, ALM, MOptQR, PLAM-DA, PCAL-DA) */
  double beta;                /* < 0: PCAL default 1.0 (solver.cpp:120-125) */
  int32_t eta_kind;           /* PCAL_ETA_* */
  double gamma;               /* Constant rule only */
  double eta_min, eta_max;    /* safeguard interval */
  double eta0;                /* <= 0: s + 2β */
  int32_t multiplier_rule;    /* PCAL_MULT_* */
  double tol_rel_kkt;
  int64_t max_iter;
  int32_t final_orth;
  int32_t device;             /* CUDA device ordinal ("threads" is never ambient, SPEC §) */
  int32_t alm_inner_max;      /* AlmOptions (solver.hpp:24-28): gradient steps per multiplier update */
  int32_t alm_outer_max;      /*   multiplier updates */
  double alm_inner_tol_scale; /*   inner target max(scale·tol, scale^k)·kkt0 */
} pcal_config;

#define PCAL_TRACE_COLS 7     /* iter, fval, kkt_abs, kkt_rel, feas, eta, elapsed (report.hpp:13-21) */

typedef struct pcal_report {  /* orthopt::RunReport (report.hpp:51-64) */
  double* trace;              /* caller buffer: trace_capacity × PCAL_TRACE_COLS (row-major) */
  int64_t trace_capacity;     /* >= max_iter + 1 */
  int64_t trace_len;
  double final_pre[4];        /* fval, kkt_abs, kkt_rel, feas */
  double final_post[4];
  int32_t has_post;
  double* stop_x;             /* caller buffer n×p, or NULL */
  double* final_x;            /* caller buffer n×p, or NULL */
  int32_t has_x;              /* 0 when the run diverged (reference leaves them empty) */
  int64_t iterations;
  int64_t degenerate_steps;
  double wall_time;           /* seconds */
  int32_t status;             /* PCAL_STATUS_* */
  double beta;                /* resolved penalty */
  double eta0;                /* resolved first stepsize */
  int64_t outer_iterations;   /* ALM multiplier updates (report.hpp:59) */
  int64_t inner_cap_hits;     /* ALM inner loops stopped by a cap (report.hpp:60) */
} pcal_report;

typedef struct pcal_category_timers { /* orthopt::CategoryTimers (report.hpp:66-72), seconds */
  double blas3, func, orth;
} pcal_category_timers;

/* Defaults of SolverConfig (PCAL, β auto, ABB, PcalFormula, tol 1e-8, 3000 iters). */
void pcal_config_default(pcal_config* c);

/* orthopt::solve — the drop-in entry point (host buffers; copies in/out inside). */
int pcal_solve(const pcal_model_desc* model, const pcal_config* config, const double* x0,
               int32_t x0_location, pcal_report* report, pcal_category_timers* timers);

/* Thread-local message for the last failing call. */
const char* pcal_last_error(void);

/* ---- device-resident session (the same solver, split into its phases) -----
 * create uploads/adopts the model and x0 and evaluates the start point (trace
 * row 0); run enqueues iterations on the session stream without a host sync;
 * finish performs the final orthonormalization and fills the report. */
typedef struct pcal_session pcal_session;

int pcal_session_create(const pcal_model_desc* model, const pcal_config* config,
                        const double* x0, int32_t x0_location, pcal_session** out);
/* Enqueue up to `iters` more iterations (stops early once converged/diverged). */
int pcal_session_run(pcal_session* s, int64_t iters);
int pcal_session_sync(pcal_session* s);
/* cudaStream_t of the session, as void*, for event timing by the caller. */
void* pcal_session_stream(pcal_session* s);
int pcal_session_finish(pcal_session* s, pcal_report* report);
void pcal_session_destroy(pcal_session* s);
/* Teacher forcing: replace the state by (X_{k-1}, X_k) at iteration k with the
 * previous stepsize eta_prev (k = 0: x_prev ignored).  Host buffers. */
int pcal_session_set_state(pcal_session* s, const double* x_prev, const double* x, int64_t k,
                           double eta_prev);
/* Copy the current iterate X_k (host buffer n×p) and the last stepsize. */
int pcal_session_get_x(pcal_session* s, double* x_out, double* eta_out, int64_t* k_out);
/* Device pointer of the current iterate (column-major, leading dimension *ld). */
int pcal_session_device_x(pcal_session* s, const double** x, int64_t* ld);
/* Number of kernels this library launched since session creation. */
int64_t pcal_session_kernel_launches(pcal_session* s);
/* Run `iters` iterations WITHOUT graphs, timing each phase with CUDA events on
 * the session stream; ms_out[4] = mean ms per iteration of {streaming step
 * (stepsize + pcal_step), gradient, Gram + p×p, X·[W|C] + reductions}. */
int pcal_session_profile(pcal_session* s, int64_t iters, double* ms_out);
/* Same, per kernel: an event after every launch; writes "name mean_ms\n" lines
 * (mean ms per iteration, kernels of one name summed) into buf (cap bytes). */
int pcal_session_profile_kernels(pcal_session* s, int64_t iters, char* buf, int64_t cap);
/* Per-iteration launch count of the captured iteration graph. */
int64_t pcal_session_kernels_per_iteration(pcal_session* s);
/* Form of the X·[W|C] product of PCAL / PLAM: 1 = single block P = G − X·M1
 * with M1 = W − βC and Σ kkt² from Σ P² by the identity (one GPU, p > 96),
 * 0 = the two-block product.  *fallbacks (may be NULL) = evaluations so far in
 * which the identity cancelled too much and the gated two-block product ran. */
int pcal_session_xm_mode(pcal_session* s, int64_t* fallbacks);

/* ---- row-sharded multi-GPU solve (one process per GPU, NCCL) -------------
 * Rows are split into fixed global row chunks (pcal_row_chunks: whole z-plane
 * groups for the grid models, row blocks for dense) and rank r of R owns the
 * chunks [⌊r·NC/R⌋, ⌊(r+1)·NC/R⌋).  Every n×p object is row-local, p×p
 * objects are replicated, and per iteration the ranks exchange per-chunk
 * partials of the Gram, column sums, stepsize inner products and column norms
 * (all-gathered and summed in global chunk order, so results are bitwise
 * identical for every rank count — the reference's thread-count invariance,
 * harness.cpp:131-137) plus the halo planes / X allgather.  A
 * sharded session takes the GLOBAL sizes in `model` (n, p, nx, ny, nz) but
 * LOCAL data: dense `a` = rows [row0, row0+nrows) of A for all n columns
 * (ld = nrows), `g0`, `v` and x0 = the owned rows.  pcal_partition tells each
 * rank its rows. */
typedef struct pcal_comm pcal_comm;
int pcal_partition(const pcal_model_desc* model, int32_t nranks, int32_t rank, int64_t* row0,
                   int64_t* nrows);
/* Number of visible CUDA devices (0 without a GPU; never fails). */
int pcal_device_count(int32_t* count);
/* The fixed row chunking of the sharded path: rows per chunk and chunk count
 * (the largest usable rank count). */
int pcal_row_chunks(const pcal_model_desc* model, int64_t* chunk_rows, int64_t* nchunks);
/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it). */
int pcal_nccl_unique_id(void* out);
int pcal_comm_create_nccl(int32_t nranks, int32_t rank, const void* unique_id, int32_t device,
                          pcal_comm** out);
void pcal_comm_destroy(pcal_comm* comm);
int pcal_session_create_sharded(const pcal_model_desc* local_model, const pcal_config* config,
                                const double* x0_local, int32_t x0_location, pcal_comm* comm,
                                pcal_session** out);
/* report rows (stop_x / final_x) are the local rows (nrows × p). */
int pcal_solve_sharded(const pcal_model_desc* local_model, const pcal_config* config,
                       const double* x0_local, int32_t x0_location, pcal_comm* comm,
                       pcal_report* report, pcal_category_timers* timers /* nullable */);
/* The sharded algorithm with `nranks` emulated ranks on ONE GPU (host threads,
 * loopback collectives): validates the multi-GPU path where one GPU exists.
 * Global host data in, global report out. */
int pcal_solve_emulated(const pcal_model_desc* model, const pcal_config* config, const double* x0,
                        int32_t nranks, pcal_report* report,
                        pcal_category_timers* timers /* nullable: rank 0's categories */);

/* ---- building blocks (host buffers; for parity tests and tools) ---------- */
/* C = Aᵀ·B for n×pa and n×pb (kernels.cpp:124-137 matmul_at_b). */
int pcal_matmul_at_b(const double* a, const double* b, int64_t n, int64_t pa, int64_t pb,
                     double* c, int32_t device);
/* C = A·B, m×k times k×nc (kernels.cpp:105-122 matmul). */
int pcal_matmul(const double* a, const double* b, int64_t m, int64_t k, int64_t nc, double* c,
                int32_t device);
/* XᵀX, exactly symmetric (kernels.cpp:139-153 gram). */
int pcal_gram(const double* x, int64_t n, int64_t p, double* g, int32_t device);
/* CholeskyQR2 with MGS2 fallback (kernels.cpp:250-265 orthonormalize);
 * PCAL_E_RANK when rank-deficient. */
int pcal_orthonormalize(const double* x, int64_t n, int64_t p, double* q, int32_t device);
/* ObjectiveModel::evaluate on the device (f and G = ∇f at x). */
int pcal_evaluate(const pcal_model_desc* model, const double* x, double* f, double* g,
                  int32_t device);
/* fd_gradient_check (problems.hpp:148-149, problems.cpp:296-325) with the device
 * evaluation: the worst |fd − g| / (1 + |g|) over up to 50 distinct seeded
 * coordinates (reference default seed 0x5EEDC0DE), central differences with
 * step h·(1 + |x_ij|).  h must be positive. */
int pcal_fd_gradient_check(const pcal_model_desc* model, const double* x, double h, uint64_t seed,
                           int32_t device, double* worst);
/* pcal_step (solver.cpp:264-307): per-column normalized proximal step. */
int pcal_pcal_step(const double* x, const double* grad_l, int64_t n, int64_t p, double eta,
                   double* out, int64_t* degenerate_columns, int32_t device);
/* Power iteration on A² (kernels.cpp:267-293 spectral_norm_estimate), device matvecs,
 * start vector from the reference Rng(seed). */
int pcal_spectral_norm_estimate(const double* a, int64_t n, uint64_t seed, double* s,
                                int32_t device);
/* flops_estimate(Pcal, n, p) (diagnostics.cpp:100-114). */
double pcal_flops_estimate(int64_t n, int64_t p);

/* ---- problem setup on the host (reference generators, problems.cpp) ------ */
/* random_normal(rows, cols, Rng(seed)) (kernels.cpp:49-55), bitwise equal;
 * `threads` host threads (checkpointed generator states). */
int pcal_random_normal(int64_t rows, int64_t cols, uint64_t seed, double* out, int32_t threads);
int pcal_random_uniform(int64_t count, uint64_t seed, double* out);
/* spectral_norm_estimate(A, seed) (kernels.cpp:267-293) on the host, bitwise equal to
 * the reference's (problem setup of small instances; the device version is
 * pcal_spectral_norm_estimate). */
int pcal_spectral_norm_estimate_host(const double* a, int64_t n, uint64_t seed, int32_t threads,
                                     double* out);
/* sym_part(random_normal(n, n, Rng(seed))) — the dense operator of configs 1–2
 * (problems.cpp:45-48). */
int pcal_gen_dense_operator(int64_t n, uint64_t seed, double* a, int32_t threads);

/* L⁻¹ of a symmetric n×n L (column-major, host), for PCAL_MODEL_DENSITY: the
 * reference's LinearSolver factorisation (linsolve.cpp:30-68 — Cholesky when it
 * succeeds, else LU with partial pivoting) applied to the unit vectors with its
 * own substitution loops (linsolve.cpp:70-102).  PCAL_E_PARAMETER (the
 * reference's generation_error) when L is numerically singular. */
int pcal_density_inverse(const double* l, int64_t n, double* linv, int32_t threads);
/* Diagnostic: the branch of orthonormalize (kernels.cpp:250-261) the calling
 * thread's last device orthonormalisation took — 0 CholeskyQR2; 1 / 2 MGS2
 * after the first / second Cholesky pass hit the pivot floor 1e-14·‖XᵀX‖_F;
 * -1 MGS2 failed too (rank_error). */
int32_t pcal_last_orthonormalize_path(void);
/* initial_point({Qr}, n, p) on the device: orthonormalize(random_normal(n,p,Rng(seed)))
 * (solver.cpp:136-142). */
int pcal_initial_point_qr(int64_t n, int64_t p, uint64_t seed, double* x0, int32_t device);
/* initial_point(InitialPointSpec{mode, sigma_lower, seed}, n, p) (solver.cpp:136-170,
 * solver.hpp:47-59): Q = orthonormalize(random_normal(n,p,Rng(seed))) on the
 * device, then for the Assumption-A2 starts the column scaling of the
 * reference — type I: last column ·√(1−σ²) (σ ∈ (0,1), σ² ≤ ½); type II:
 * column j ·√(1 + b·(2u_j − 1)), b = 0.9/√p, u_j the next uniforms of the same
 * stream, |·−1| floored at 0.1·b.  Invalid arguments: PCAL_E_PARAMETER. */
#define PCAL_INIT_QR 0
#define PCAL_INIT_A2_TYPE_I 1
#define PCAL_INIT_A2_TYPE_II 2
int pcal_initial_point(int64_t n, int64_t p, int32_t mode, double sigma_lower, uint64_t seed,
                       double* x0, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* PCAL_B200_H */
