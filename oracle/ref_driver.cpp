// ref_driver.cpp — C entry points into the UNMODIFIED reference library
// (/root/reference/proj/core, compiled from its own sources by oracle/Makefile
// into oracle/_ref/).  TEST INFRASTRUCTURE: used to generate the golden
// fixtures, to pin the C restatement (pcal_oracle.c), and as bench.py's
// `--impl reference` CPU arm.  Nothing of the product links this.
//
// The grid models of configs 3–5 do not exist in the reference; they are
// plugged into the reference solve() as ObjectiveModel subclasses whose
// evaluate() calls the restatement in pcal_oracle.c.
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "orthopt/diagnostics.hpp"
#include "orthopt/kernels.hpp"
#include "orthopt/linsolve.hpp"
#include "orthopt/problems.hpp"
#include "orthopt/rng.hpp"
#include "orthopt/solver.hpp"
#include "pcal_oracle.h"

using namespace orthopt;

namespace {

thread_local std::string g_err;

// Grid model adapter: reference ObjectiveModel backed by the oracle restatement.
class GridModel : public ObjectiveModel {
 public:
  GridModel(const orc_model& m, std::vector<double> v)
      : ObjectiveModel(m.n, m.p, m.kind == ORC_MODEL_STENCIL ? ProblemKind::P3 : ProblemKind::P6,
                       m.s),
        m_(m),
        v_(std::move(v)) {
    m_.v = v_.data();
    m_.work = nullptr;
    orc_model_prepare(&m_);
  }
  ~GridModel() override { orc_model_release(&m_); }
  Evaluation evaluate(const DenseMatrix& x, int threads) const override {
    if (x.rows() != n_ || x.cols() != p_) throw dimension_error("evaluate: iterate shape mismatch");
    Evaluation ev;
    ev.gradient = DenseMatrix(n_, p_);
    const int rc = orc_evaluate(&m_, x.data(), &ev.value, ev.gradient.data(), threads);
    if (rc) throw evaluation_error("GridModel: non-finite objective or gradient");
    return ev;
  }
  void save(std::ostream&) const override { throw io_error("GridModel: not serializable"); }

 private:
  orc_model m_;
  std::vector<double> v_;
};

DenseMatrix from_ptr(const double* p, std::int64_t r, std::int64_t c) {
  DenseMatrix m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

SquareSymmetric sym_from_ptr(const double* p, std::int64_t n) {
  SquareSymmetric s(n);
  for (std::int64_t j = 0; j < n; ++j)
    for (std::int64_t i = 0; i <= j; ++i) s.set_mirrored(i, j, p[i + j * n]);
  return s;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const parameter_error& e) {
    g_err = e.what();
    return ORC_E_PARAM;
  } catch (const dimension_error& e) {
    g_err = e.what();
    return ORC_E_DIM;
  } catch (const rank_error& e) {
    g_err = e.what();
    return ORC_E_RANK;
  } catch (const evaluation_error& e) {
    g_err = e.what();
    return ORC_E_EVAL;
  } catch (const divergence_error& e) {
    g_err = e.what();
    return ORC_E_DIVERGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -99;
  }
}

// AlmOptions for the next solves and the ALM counters of the last one
// (orc_config / orc_report carry neither; set through ref_set_alm).
AlmOptions g_alm{};
std::int64_t g_alm_counts[2] = {0, 0};

SolverConfig to_config(const orc_config* c) {
  SolverConfig cfg;
  cfg.alm = g_alm;
  cfg.algorithm = static_cast<Algorithm>(c->algorithm);
  cfg.beta = c->beta;
  cfg.eta_rule.kind = static_cast<StepsizeRule::Kind>(c->eta_kind);
  cfg.eta_rule.gamma = c->gamma;
  cfg.eta_rule.eta_min = c->eta_min;
  cfg.eta_rule.eta_max = c->eta_max;
  cfg.eta_rule.eta0 = c->eta0;
  cfg.multiplier_rule =
      c->multiplier_rule == ORC_MULT_PCAL ? MultiplierRule::PcalFormula : MultiplierRule::PlamFormula;
  cfg.tol_rel_kkt = c->tol_rel_kkt;
  cfg.max_iter = c->max_iter;
  cfg.threads = c->threads;
  cfg.final_orth = c->final_orth != 0;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- problem construction (problems.cpp) --------------------------------
// Dense trace minimization of configs 1–2: A = sym_part(random_normal(n,n,Rng(seed)))
// (problems.cpp:45-48 via gen_problem1(α=0, RandomSym)); s from
// spectral_norm_estimate(A, seed ^ 0x73706563) (problems.cpp:215) unless s_in >= 0.
void* ref_make_dense_trace_min(std::int64_t n, std::int64_t p, std::uint64_t seed, double s_in,
                               int threads, double* a_out, double* s_out) {
  void* out = nullptr;
  guarded([&] {
    Rng rng(seed);
    SquareSymmetric a = sym_part(random_normal(n, n, rng));
    const double s = s_in >= 0.0 ? s_in : spectral_norm_estimate(a, seed ^ 0x73706563u, threads);
    if (a_out) std::memcpy(a_out, a.matrix().data(), sizeof(double) * static_cast<size_t>(n * n));
    if (s_out) *s_out = s;
    out = make_quadratic(std::move(a), DenseMatrix(n, p), ProblemKind::P3, s, threads).release();
    return 0;
  });
  return out;
}

void* ref_make_quadratic(const double* a, const double* g0, std::int64_t n, std::int64_t p,
                         double s) {
  void* out = nullptr;
  guarded([&] {
    DenseMatrix g = g0 ? from_ptr(g0, n, p) : DenseMatrix(n, p);
    out = make_quadratic(sym_from_ptr(a, n), std::move(g), g0 ? ProblemKind::P2 : ProblemKind::P3,
                         s)
              .release();
    return 0;
  });
  return out;
}

void* ref_make_grid_model(int kind, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                          std::int64_t p, const double* v, double s) {
  void* out = nullptr;
  guarded([&] {
    orc_model m{};
    m.kind = kind;
    m.nx = nx;
    m.ny = ny;
    m.nz = nz;
    m.n = nx * ny * nz;
    m.p = p;
    m.s = s;
    out = new GridModel(m, std::vector<double>(v, v + m.n));
    return 0;
  });
  return out;
}

void ref_free_model(void* m) { delete static_cast<ObjectiveModel*>(m); }

int ref_evaluate(void* model, const double* x, double* f, double* g) {
  return guarded([&] {
    auto* m = static_cast<ObjectiveModel*>(model);
    Evaluation ev = m->evaluate(from_ptr(x, m->n(), m->p()), 1);
    *f = ev.value;
    std::memcpy(g, ev.gradient.data(), sizeof(double) * ev.gradient.size());
    return 0;
  });
}

double ref_fd_gradient_check(void* model, const double* x, double h, std::uint64_t seed) {
  double r = -1.0;
  guarded([&] {
    auto* m = static_cast<ObjectiveModel*>(model);
    r = fd_gradient_check(*m, from_ptr(x, m->n(), m->p()), h, seed);
    return 0;
  });
  return r;
}

// --- kernels / setup -------------------------------------------------------
int ref_random_normal(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double* out) {
  return guarded([&] {
    Rng rng(seed);
    DenseMatrix m = random_normal(rows, cols, rng);
    std::memcpy(out, m.data(), sizeof(double) * m.size());
    return 0;
  });
}

int ref_initial_point(int mode, double sigma, std::uint64_t seed, std::int64_t n, std::int64_t p,
                      double* out) {
  return guarded([&] {
    DenseMatrix x = initial_point({static_cast<InitMode>(mode), sigma, seed}, n, p);
    std::memcpy(out, x.data(), sizeof(double) * x.size());
    return 0;
  });
}

double ref_spectral_norm_estimate(const double* a, std::int64_t n, std::uint64_t seed, int threads) {
  double r = -1.0;
  guarded([&] {
    r = spectral_norm_estimate(sym_from_ptr(a, n), seed, threads);
    return 0;
  });
  return r;
}

int ref_orthonormalize(const double* x, std::int64_t n, std::int64_t p, double* q) {
  return guarded([&] {
    DenseMatrix r = orthonormalize(from_ptr(x, n, p));
    std::memcpy(q, r.data(), sizeof(double) * r.size());
    return 0;
  });
}

int ref_gram(const double* x, std::int64_t n, std::int64_t p, double* g) {
  return guarded([&] {
    SquareSymmetric s = gram(from_ptr(x, n, p), 1);
    std::memcpy(g, s.matrix().data(), sizeof(double) * static_cast<size_t>(p * p));
    return 0;
  });
}

int ref_matmul_at_b(const double* a, const double* b, std::int64_t n, std::int64_t pa,
                    std::int64_t pb, double* c) {
  return guarded([&] {
    DenseMatrix r = matmul_at_b(from_ptr(a, n, pa), from_ptr(b, n, pb), 1);
    std::memcpy(c, r.data(), sizeof(double) * r.size());
    return 0;
  });
}

int ref_matmul(const double* a, const double* b, std::int64_t m, std::int64_t k, std::int64_t nc,
               double* c, int threads) {
  return guarded([&] {
    DenseMatrix r = matmul(from_ptr(a, m, k), from_ptr(b, k, nc), threads);
    std::memcpy(c, r.data(), sizeof(double) * r.size());
    return 0;
  });
}

int ref_pcal_step(const double* x, const double* gl, std::int64_t n, std::int64_t p, double eta,
                  double* out, std::int64_t* degenerate) {
  return guarded([&] {
    PcalStepResult r = pcal_step(from_ptr(x, n, p), from_ptr(gl, n, p), eta, 1);
    std::memcpy(out, r.x.data(), sizeof(double) * r.x.size());
    *degenerate = r.degenerate_columns;
    return 0;
  });
}

double ref_stepsize_select(const orc_config* c, std::int64_t iter, double eta_prev, double eta0,
                           const double* x, const double* xp, const double* gl,
                           const double* glp, std::int64_t n, std::int64_t p) {
  double r = -1.0;
  guarded([&] {
    SolverState st;
    st.x = from_ptr(x, n, p);
    st.grad_l = from_ptr(gl, n, p);
    if (xp) st.prev_x = from_ptr(xp, n, p);
    if (glp) st.prev_grad_l = from_ptr(glp, n, p);
    st.iter = iter;
    st.eta = eta_prev;
    st.eta0 = eta0;
    r = stepsize_select(to_config(c).eta_rule, st);
    return 0;
  });
  return r;
}

double ref_kkt_violation(void* model, const double* x) {
  double r = -1.0;
  guarded([&] {
    auto* m = static_cast<ObjectiveModel*>(model);
    r = kkt_violation(*m, from_ptr(x, m->n(), m->p()), 1);
    return 0;
  });
  return r;
}

double ref_feasibility_violation(const double* x, std::int64_t n, std::int64_t p) {
  return feasibility_violation(from_ptr(x, n, p), 1);
}

double ref_flops_estimate_pcal(std::int64_t n, std::int64_t p) {
  return flops_estimate(Algorithm::Pcal, n, p);
}

// --- solve() ---------------------------------------------------------------
// Fills the same orc_report layout as the restatement.  Returns a negative
// ORC_E_* code when solve() throws (parameter/dimension errors).
int ref_solve(void* model, const orc_config* c, const double* x0, orc_report* r,
              double* timers /* blas3, func, orth or NULL */) {
  return guarded([&] {
    auto* m = static_cast<ObjectiveModel*>(model);
    CategoryTimers t;
    RunReport rep = solve(*m, to_config(c), from_ptr(x0, m->n(), m->p()), timers ? &t : nullptr);
    g_alm_counts[0] = rep.outer_iterations;
    g_alm_counts[1] = rep.inner_cap_hits;
    r->trace_len = static_cast<std::int64_t>(rep.trace.size());
    for (size_t i = 0; i < rep.trace.size(); ++i) {
      double* row = r->trace + i * ORC_TRACE_COLS;
      const MetricSample& s = rep.trace[i];
      row[0] = static_cast<double>(s.iter);
      row[1] = s.fval;
      row[2] = s.kkt_abs;
      row[3] = s.kkt_rel;
      row[4] = s.feas;
      row[5] = s.eta;
      row[6] = s.elapsed;
    }
    r->final_pre[0] = rep.final_pre_orth.fval;
    r->final_pre[1] = rep.final_pre_orth.kkt_abs;
    r->final_pre[2] = rep.final_pre_orth.kkt_rel;
    r->final_pre[3] = rep.final_pre_orth.feas;
    r->has_post = rep.final_post_orth.has_value();
    if (r->has_post) {
      r->final_post[0] = rep.final_post_orth->fval;
      r->final_post[1] = rep.final_post_orth->kkt_abs;
      r->final_post[2] = rep.final_post_orth->kkt_rel;
      r->final_post[3] = rep.final_post_orth->feas;
    }
    r->has_x = !rep.stop_iterate.empty();
    if (r->has_x && r->stop_x)
      std::memcpy(r->stop_x, rep.stop_iterate.data(), sizeof(double) * rep.stop_iterate.size());
    if (r->has_x && r->final_x)
      std::memcpy(r->final_x, rep.final_x.data(), sizeof(double) * rep.final_x.size());
    r->iterations = rep.iterations;
    r->degenerate_steps = rep.degenerate_steps;
    r->wall_time = rep.wall_time;
    r->status = rep.status == RunStatus::Converged ? ORC_CONVERGED
                : rep.status == RunStatus::MaxIter ? ORC_MAXITER
                                                    : ORC_DIVERGED;
    r->beta_used = rep.config.beta;
    r->eta0_used = rep.trace.empty() ? 0.0 : rep.trace.front().eta;
    if (timers) {
      timers[0] = t.blas3;
      timers[1] = t.func;
      timers[2] = t.orth;
    }
    return 0;
  });
}

}  // extern "C"

// --- report I/O and the problem container of the reference (report_io.cpp,
//     problems.cpp:327-416): golden text for the product's formatter tests ----
#include <fstream>
#include <sstream>

#include "orthopt/harness.hpp"
#include "orthopt/report_io.hpp"

extern "C" {

// run_single(P1 α=0 / RandomSym, seed) with PCAL defaults and max_iter; writes
// the reference's JSON (no timing) and trace CSV (time column zeroed) into bufs.
int ref_run_single_text(std::int64_t n, std::int64_t p, std::uint64_t seed, std::int64_t max_iter,
                        char* json_buf, std::int64_t json_cap, char* csv_buf,
                        std::int64_t csv_cap) {
  return guarded([&] {
    ProblemSpec spec;
    spec.kind = ProblemKind::P1;
    spec.alpha = 0.0;
    spec.n = n;
    spec.p = p;
    spec.seed = seed;
    SolverConfig cfg;
    cfg.max_iter = max_iter;
    RunReport rep = run_single(spec, cfg, {InitMode::Qr, 0.5, 0});
    for (auto& s : rep.trace) s.elapsed = 0.0;
    const std::string js = to_json(rep, false);
    std::ostringstream cs;
    write_trace_csv(rep, cs);
    if ((std::int64_t)js.size() + 1 > json_cap || (std::int64_t)cs.str().size() + 1 > csv_cap)
      throw io_error("buffer too small");
    std::memcpy(json_buf, js.c_str(), js.size() + 1);
    std::memcpy(csv_buf, cs.str().c_str(), cs.str().size() + 1);
    return 0;
  });
}

// to_json of a hand-built RunReport whose trace row k carries vals[k] in every
// metric (iter = k): the reference's number formatting over any magnitudes.
int ref_report_json_values(const double* vals, std::int64_t count, char* json_buf,
                           std::int64_t json_cap) {
  return guarded([&] {
    RunReport rep;
    rep.config.problem = "p3";
    rep.config.n = 8;
    rep.config.p = 2;
    rep.config.solver = "pcal";
    rep.config.curvature_scale = count > 0 ? vals[0] : 0.0;
    for (std::int64_t k = 0; k < count; ++k)
      rep.trace.push_back({k, vals[k], vals[k], vals[k], vals[k], vals[k], 0.0});
    if (count > 0) {
      rep.final_pre_orth = {vals[count - 1], vals[0], vals[0], vals[count - 1]};
      rep.final_post_orth = FinalMetrics{vals[0], vals[count - 1], vals[0], vals[0]};
    }
    rep.iterations = count;
    const std::string js = to_json(rep, false);
    if ((std::int64_t)js.size() + 1 > json_cap) throw io_error("buffer too small");
    std::memcpy(json_buf, js.c_str(), js.size() + 1);
    return 0;
  });
}

// run_single(ProblemSpec, SolverConfig{max_iter}, InitialPointSpec) as the
// reference's JSON report (elapsed times zeroed); kind 1..6 = P1..P6 names.
int ref_run_single_json(int kind, std::int64_t n, std::int64_t p, double alpha, double kappa,
                        double theta, double zeta, double xi, int block_tridiag,
                        std::uint64_t seed, int init_mode, double sigma, std::int64_t max_iter,
                        char* json_buf, std::int64_t json_cap) {
  return guarded([&] {
    ProblemSpec spec;
    spec.kind = kind == 1 ? ProblemKind::P1 : kind == 2 ? ProblemKind::P2
                : kind == 3 ? ProblemKind::P3 : kind == 4 ? ProblemKind::P4 : ProblemKind::P6;
    spec.n = n;
    spec.p = p;
    spec.alpha = alpha;
    spec.kappa = kappa;
    spec.theta = theta;
    spec.zeta = zeta;
    spec.xi = xi;
    spec.mode = block_tridiag ? OperatorMode::BlockTridiag : OperatorMode::RandomSym;
    spec.seed = seed;
    SolverConfig cfg;
    cfg.max_iter = max_iter;
    RunReport rep = run_single(spec, cfg, {static_cast<InitMode>(init_mode), sigma, 0});
    for (auto& s : rep.trace) s.elapsed = 0.0;
    const std::string js = to_json(rep, false);
    if ((std::int64_t)js.size() + 1 > json_cap) throw io_error("buffer too small");
    std::memcpy(json_buf, js.c_str(), js.size() + 1);
    return 0;
  });
}

// make_problem(ProblemSpec) (harness.cpp:31-46) as a model handle for
// ref_solve (freed by ref_free_model): the reference's own instance of every
// problem kind, for runs from caller-chosen start points.
void* ref_make_problem(int kind, std::int64_t n, std::int64_t p, double alpha, double kappa,
                       double theta, double zeta, double xi, int block_tridiag,
                       std::uint64_t seed) {
  void* out = nullptr;
  const int rc = guarded([&] {
    ProblemSpec spec;
    spec.kind = kind == 1 ? ProblemKind::P1 : kind == 2 ? ProblemKind::P2
                : kind == 3 ? ProblemKind::P3 : kind == 4 ? ProblemKind::P4 : ProblemKind::P6;
    spec.n = n;
    spec.p = p;
    spec.alpha = alpha;
    spec.kappa = kappa;
    spec.theta = theta;
    spec.zeta = zeta;
    spec.xi = xi;
    spec.mode = block_tridiag ? OperatorMode::BlockTridiag : OperatorMode::RandomSym;
    spec.seed = seed;
    out = make_problem(spec).release();
    return 0;
  });
  return rc == 0 ? out : nullptr;
}

int ref_save_quadratic(const double* a, const double* g0, std::int64_t n, std::int64_t p, double s,
                       const char* path) {
  return guarded([&] {
    DenseMatrix g = g0 ? from_ptr(g0, n, p) : DenseMatrix(n, p);
    auto m = make_quadratic(sym_from_ptr(a, n), std::move(g), g0 ? ProblemKind::P2 : ProblemKind::P3, s);
    std::ofstream out(path, std::ios::binary);
    save_problem(*m, out);
    return 0;
  });
}

// LinearSolver (linsolve.cpp) of a symmetric a, solved against the identity's
// columns: pins pcal_density_inverse.  1 when the constructor throws
// generation_error (numerically singular).
int ref_linear_inverse(const double* a, std::int64_t n, double* out) {
  return guarded([&] {
    std::unique_ptr<LinearSolver> ls;
    try {
      ls = std::make_unique<LinearSolver>(sym_from_ptr(a, n));
    } catch (const generation_error&) {
      return 1;
    }
    std::vector<double> e((size_t)n, 0.0);
    for (std::int64_t c = 0; c < n; ++c) {
      e[(size_t)c] = 1.0;
      const std::vector<double> y = ls->solve(e);
      e[(size_t)c] = 0.0;
      std::memcpy(out + c * n, y.data(), sizeof(double) * (size_t)n);
    }
    return 0;
  });
}

// gen_problem{1,4,6}(…, seed) evaluated at x (problems.cpp:130-206): pins the
// device Bilinear / Density models.  kind 1 = P1 (alpha), 4 = P4, 6 = P6.
int ref_evaluate_problem(int kind, std::int64_t n, std::int64_t p, double alpha, int block_tridiag,
                         std::uint64_t seed, const double* x, double* f, double* g,
                         double* fd) {
  return guarded([&] {
    const OperatorMode mode = block_tridiag ? OperatorMode::BlockTridiag : OperatorMode::RandomSym;
    std::unique_ptr<ObjectiveModel> m =
        kind == 1 ? gen_problem1(n, p, alpha, mode, seed, 1)
        : kind == 4 ? gen_problem4(n, p, seed, 1)
                    : gen_problem6(n, p, mode, seed, 1);
    const Evaluation ev = m->evaluate(from_ptr(x, n, p), 1);
    *f = ev.value;
    std::memcpy(g, ev.gradient.data(), sizeof(double) * (size_t)(n * p));
    if (fd) *fd = fd_gradient_check(*m, from_ptr(x, n, p));  // defaults h = 1e-5, seed 0x5eedc0de
    return 0;
  });
}

// AlmOptions of the following ref_solve calls (solver.hpp:24-28).
void ref_set_alm(int inner_max, int outer_max, double inner_tol_scale) {
  g_alm.inner_max = inner_max;
  g_alm.outer_max = outer_max;
  g_alm.inner_tol_scale = inner_tol_scale;
}
// RunReport::outer_iterations / inner_cap_hits of the last ref_solve.
void ref_last_alm_counts(std::int64_t* out) {
  out[0] = g_alm_counts[0];
  out[1] = g_alm_counts[1];
}

// run_matrix (harness.cpp:75-104) over a fixed spec (tests/golden/ref_matrix.csv):
// P2 40×4, P4 30×3, P1 (α = 1) 30×3, P6 block 30×3 and a P1 block cell with
// n = 32 whose generation fails; PCAL, PLAM, ALM; seeds 1, 2; max_iter 500.
int ref_run_matrix_csv(char* buf, std::int64_t cap) {
  return guarded([&] {
    MatrixSpec m;
    ProblemSpec p2;
    p2.kind = ProblemKind::P2;
    p2.n = 40;
    p2.p = 4;
    ProblemSpec p4 = p2;
    p4.kind = ProblemKind::P4;
    p4.n = 30;
    p4.p = 3;
    ProblemSpec p1 = p4;
    p1.kind = ProblemKind::P1;
    ProblemSpec p6 = p4;
    p6.kind = ProblemKind::P6;
    p6.mode = OperatorMode::BlockTridiag;
    ProblemSpec bad = p1;
    bad.n = 32;
    bad.mode = OperatorMode::BlockTridiag;
    m.problems = {p2, p4, p1, p6, bad};
    m.solvers = {Algorithm::Pcal, Algorithm::Plam, Algorithm::Alm};
    m.seeds = {1, 2};
    m.base.max_iter = 500;
    std::ostringstream out;
    run_matrix(m, out);
    const std::string t = out.str();
    if ((std::int64_t)t.size() + 1 > cap) throw io_error("buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
  });
}

// diagnostics.cpp on gen_problem{1,4,6}(…, seed) at x: out = {kkt_violation,
// feasibility_violation, merit_h(beta), bound.applicable, delta, lhs, rhs, holds, slack}.
int ref_diagnostics(int kind, std::int64_t n, std::int64_t p, double alpha, int block_tridiag,
                    std::uint64_t seed, const double* x, double beta, double* out) {
  return guarded([&] {
    const OperatorMode mode = block_tridiag ? OperatorMode::BlockTridiag : OperatorMode::RandomSym;
    std::unique_ptr<ObjectiveModel> m =
        kind == 1 ? gen_problem1(n, p, alpha, mode, seed, 1)
        : kind == 4 ? gen_problem4(n, p, seed, 1)
                    : gen_problem6(n, p, mode, seed, 1);
    const DenseMatrix xm = from_ptr(x, n, p);
    out[0] = kkt_violation(*m, xm);
    out[1] = feasibility_violation(xm);
    out[2] = merit_h(*m, xm, beta);
    const FeasibilityBoundResult b = feasibility_bound_check(*m, xm, beta);
    out[3] = b.applicable ? 1.0 : 0.0;
    out[4] = b.delta;
    out[5] = b.lhs;
    out[6] = b.rhs;
    out[7] = b.holds ? 1.0 : 0.0;
    out[8] = b.slack;
    return 0;
  });
}

// save_problem of gen_problem{1,4,6}(…, seed) (problems.cpp:341-365): the
// Bilinear / Density container forms.
int ref_save_generated(int kind, std::int64_t n, std::int64_t p, double alpha, int block_tridiag,
                       std::uint64_t seed, const char* path) {
  return guarded([&] {
    const OperatorMode mode = block_tridiag ? OperatorMode::BlockTridiag : OperatorMode::RandomSym;
    std::unique_ptr<ObjectiveModel> m =
        kind == 1 ? gen_problem1(n, p, alpha, mode, seed, 1)
        : kind == 4 ? gen_problem4(n, p, seed, 1)
                    : gen_problem6(n, p, mode, seed, 1);
    std::ofstream out(path, std::ios::binary);
    save_problem(*m, out);
    return 0;
  });
}

}  // extern "C"
