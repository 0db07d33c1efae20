// orthopt_b200/solver.hpp — header-only C++ mirror of the reference solver API
// (/root/reference/proj/core/include/orthopt/solver.hpp, report.hpp, errors.hpp,
// problems.hpp), implemented over the C ABI of libpcal_b200.so
// (include/pcal_b200.h).  A caller of orthopt::solve() switches by changing the
// namespace and constructing a device-evaluated model descriptor instead of a
// virtual ObjectiveModel subclass:
//
//   orthopt_b200::QuadraticModel model(a, p, s);           // problems.hpp:53-69
//   orthopt_b200::SolverConfig cfg;                        // solver.hpp:30-42
//   orthopt_b200::RunReport rep = orthopt_b200::solve(model, cfg, x0);
//
// Errors mirror errors.hpp: parameter_error / dimension_error are thrown before
// iterating; divergence inside the run is reported via RunStatus::Diverged.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <cmath>
#include <vector>

#include "../pcal_b200.h"

namespace orthopt_b200 {

// ---- errors (errors.hpp:9-50) -------------------------------------------------
struct dimension_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct parameter_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct rank_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {  // CUDA failure / no B200: no CPU fallback
  using std::runtime_error::runtime_error;
};
struct generation_error : std::runtime_error {  // errors.hpp:27-31
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == PCAL_OK) return;
  const std::string msg = pcal_last_error();
  switch (rc) {
    case PCAL_E_PARAMETER: throw parameter_error(msg);
    case PCAL_E_DIMENSION: throw dimension_error(msg);
    case PCAL_E_RANK: throw rank_error(msg);
    default: throw device_error(msg);
  }
}

// ---- DenseMatrix (matrix.hpp:16-67): column-major FP64 -----------------------
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(std::int64_t rows, std::int64_t cols) : rows_(rows), cols_(cols) {
    if (rows < 1 || cols < 1) throw dimension_error("DenseMatrix: dimensions must be positive");
    data_.assign(static_cast<size_t>(rows * cols), 0.0);
  }
  std::int64_t rows() const { return rows_; }
  std::int64_t cols() const { return cols_; }
  bool empty() const { return data_.empty(); }
  double& operator()(std::int64_t i, std::int64_t j) { return data_[i + j * rows_]; }
  double operator()(std::int64_t i, std::int64_t j) const { return data_[i + j * rows_]; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  std::size_t size() const { return data_.size(); }

 private:
  std::int64_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

// ---- configuration (solver.hpp:13-42) -----------------------------------------
struct StepsizeRule {
  enum class Kind { Constant, Differential, Bb1, Bb2, Abb };
  Kind kind = Kind::Abb;
  double gamma = 1.0;
  double eta_min = 1e-10;
  double eta_max = 1e10;
  double eta0 = 0.0;
};
enum class MultiplierRule { PlamFormula, PcalFormula };
// Algorithm (diagnostics.hpp:10), reference order
enum class Algorithm { Plam = PCAL_ALG_PLAM, Pcal = PCAL_ALG_PCAL, Alm = PCAL_ALG_ALM,
                       MoptQr = PCAL_ALG_MOPTQR, PlamDa = PCAL_ALG_PLAMDA, PcalDa = PCAL_ALG_PCALDA };
struct AlmOptions {  // solver.hpp:24-28
  int inner_max = 500;
  int outer_max = 50;
  double inner_tol_scale = 0.1;
};

struct SolverConfig {
  Algorithm algorithm = Algorithm::Pcal;
  double beta = -1.0;
  StepsizeRule eta_rule{};
  MultiplierRule multiplier_rule = MultiplierRule::PcalFormula;
  double tol_rel_kkt = 1e-8;
  std::int64_t max_iter = 3000;
  int threads = 1;  // accepted for source compatibility (SolverConfig::threads); echoed,
                    // not used: parallelism is the device's
  int device = 0;   // the explicit GPU ordinal (never ambient)
  AlmOptions alm{};
  bool final_orth = true;
};

// ---- results (report.hpp:13-72) --------------------------------------------------
struct MetricSample {
  std::int64_t iter = 0;
  double fval = 0, kkt_abs = 0, kkt_rel = 0, feas = 0, eta = 0, elapsed = 0;
};
enum class RunStatus { Converged, MaxIter, Diverged };
struct FinalMetrics {
  double fval = 0, kkt_abs = 0, kkt_rel = 0, feas = 0;
};
struct CategoryTimers {
  double blas3 = 0, func = 0, orth = 0;
};
// ConfigEcho (report.hpp:35-49): what solve() ran with, filled like the
// reference's iterate_main (solver.cpp:333-342); run_single-level fields
// (seed, init, alpha…) stay at their defaults unless the caller's harness sets them.
struct ConfigEcho {
  std::string problem;
  std::int64_t n = 0;
  std::int64_t p = 0;
  std::string solver;
  double beta = 0.0;
  std::string eta_rule;
  double tol_rel_kkt = 0.0;
  std::int64_t max_iter = 0;
  int threads = 1;
  std::string init;
  std::uint64_t seed = 0;
  double alpha = 0.0, kappa = 0.0, theta = 0.0, zeta = 0.0, xi = 0.0;
  double curvature_scale = 0.0;
};
struct RunReport {
  ConfigEcho config;
  std::vector<MetricSample> trace;
  FinalMetrics final_pre_orth;
  std::optional<FinalMetrics> final_post_orth;
  DenseMatrix stop_iterate;
  DenseMatrix final_x;
  std::int64_t iterations = 0;
  std::int64_t outer_iterations = 0;  // ALM multiplier updates
  std::int64_t inner_cap_hits = 0;    // ALM inner loops stopped by a cap
  std::int64_t degenerate_steps = 0;
  double wall_time = 0.0;
  RunStatus status = RunStatus::MaxIter;
  double beta = 0.0;
};

// ---- models: device-evaluated descriptors of ObjectiveModel (problems.hpp:28-111)
enum class ProblemKind { P1 = 1, P2 = 2, P3 = 3, P4 = 4, P6 = 6 };
inline const char* problem_kind_name(ProblemKind k) {  // problems.cpp:114-123
  switch (k) {
    case ProblemKind::P1: return "p1";
    case ProblemKind::P2: return "p2";
    case ProblemKind::P3: return "p3";
    case ProblemKind::P4: return "p4";
    case ProblemKind::P6: return "p6";
  }
  return "?";
}

class ObjectiveModel {
 public:
  virtual ~ObjectiveModel() = default;
  std::int64_t n() const { return desc_.n; }
  std::int64_t p() const { return desc_.p; }
  double curvature_scale() const { return desc_.s; }
  ProblemKind kind() const { return kind_; }
  // ConfigEcho::problem: the reference's kind name; the models it does not
  // have (grid, Kohn–Sham, caller-defined) echo their own names
  virtual const char* problem_name() const { return problem_kind_name(kind_); }
  const pcal_model_desc& desc() const { return desc_; }

 protected:
  pcal_model_desc desc_{};
  ProblemKind kind_ = ProblemKind::P2;  // make_quadratic's default (problems.hpp:141-142)
};

// f(X) = ½tr(XᵀAX) + tr(GᵀX); A and G are host matrices owned by the caller.
class QuadraticModel : public ObjectiveModel {
 public:
  QuadraticModel(const DenseMatrix& a, std::int64_t p, double s, const DenseMatrix* g = nullptr,
                 ProblemKind kind = ProblemKind::P2) {
    if (a.rows() != a.cols()) throw dimension_error("QuadraticModel: A must be square");
    kind_ = kind;
    if (g && (g->rows() != a.rows() || g->cols() != p))
      throw dimension_error("QuadraticModel: G row count must equal n");
    desc_.kind = PCAL_MODEL_DENSE;
    desc_.location = PCAL_HOST;
    desc_.n = a.rows();
    desc_.p = p;
    desc_.s = s;
    desc_.a = a.data();
    desc_.g0 = g ? g->data() : nullptr;
  }
};

// f(X) = ½tr(XᵀLX) + ½tr(XᵀVX), L = −Δ_h 7-point periodic.
class StencilModel : public ObjectiveModel {
 public:
  StencilModel(std::int64_t nx, std::int64_t ny, std::int64_t nz, const std::vector<double>& v,
               std::int64_t p, double s, int32_t kind = PCAL_MODEL_STENCIL) {
    if (static_cast<std::int64_t>(v.size()) != nx * ny * nz)
      throw dimension_error("StencilModel: |V| must equal nx*ny*nz");
    desc_.kind = kind;
    desc_.location = PCAL_HOST;
    desc_.n = nx * ny * nz;
    desc_.p = p;
    desc_.s = s;
    desc_.nx = nx;
    desc_.ny = ny;
    desc_.nz = nz;
    desc_.v = v.data();
  }
  const char* problem_name() const override {
    return desc_.kind == PCAL_MODEL_KOHN_SHAM ? "kohn_sham" : "stencil";
  }
};

// f(X) = ½tr(XᵀAXB) (BilinearModel, problems.cpp:143-156; problem P4); A n×n and
// B p×p symmetric host matrices owned by the caller.
class BilinearModel : public ObjectiveModel {
 public:
  BilinearModel(const DenseMatrix& a, const DenseMatrix& b, double s) {
    if (a.rows() != a.cols() || b.rows() != b.cols())
      throw dimension_error("BilinearModel: A and B must be square");
    kind_ = ProblemKind::P4;
    desc_.kind = PCAL_MODEL_BILINEAR;
    desc_.location = PCAL_HOST;
    desc_.n = a.rows();
    desc_.p = b.rows();
    desc_.s = s;
    desc_.a = a.data();
    desc_.b = b.data();
  }
};

// DensityModel (problems.cpp:158-206): ½tr(XᵀLX) plus the density term of
// ρ = rowsq(X) and h = L⁻¹ρ — P1: ¼·coeff·ρᵀh; P6: ½ρᵀh − ¾·coeff·Σρ^{4/3}.
// Like the reference's constructor (which builds its LinearSolver), this forms
// L⁻¹ and throws generation_error when L is numerically singular.
class DensityModel : public ObjectiveModel {
 public:
  DensityModel(const DenseMatrix& l, std::int64_t p, double coeff, ProblemKind kind, double s)
      : linv_(l.rows(), l.cols()) {
    if (l.rows() != l.cols()) throw dimension_error("DensityModel: L must be square");
    if (p < 1 || 2 * p > l.rows())
      throw parameter_error("DensityModel: dimensions must satisfy 2p <= n");
    if (kind != ProblemKind::P1 && kind != ProblemKind::P6)
      throw parameter_error("DensityModel: kind must be P1 or P6");
    if (pcal_density_inverse(l.data(), l.rows(), linv_.data(), 8) != PCAL_OK)
      throw generation_error("LinearSolver: matrix is numerically singular");
    kind_ = kind;
    desc_.kind = PCAL_MODEL_DENSITY;
    desc_.location = PCAL_HOST;
    desc_.n = l.rows();
    desc_.p = p;
    desc_.s = s;
    desc_.a = l.data();
    desc_.linv = linv_.data();
    desc_.coeff = coeff;
    desc_.density_variant = kind == ProblemKind::P6 ? PCAL_DENSITY_P6 : PCAL_DENSITY_P1;
  }
  DensityModel(const DensityModel&) = delete;
  DensityModel& operator=(const DensityModel&) = delete;

 private:
  DenseMatrix linv_;
};

// A caller-defined objective on the device: the counterpart of subclassing
// orthopt::ObjectiveModel and overriding evaluate() (problems.hpp:24-51).
// enqueue_gradient() receives device pointers and the solver's CUDA stream
// (as void*) and must only ENQUEUE the work writing G = ∇f(X) and f(X) (see
// pcal_gradient_fn in pcal_b200.h).  The object must outlive the solve.
class DeviceModel : public ObjectiveModel {
 public:
  DeviceModel(std::int64_t n, std::int64_t p, double s) {
    desc_.kind = PCAL_MODEL_DEVICE_CALLBACK;
    desc_.location = PCAL_DEVICE;
    desc_.n = n;
    desc_.p = p;
    desc_.s = s;
    desc_.grad = &DeviceModel::trampoline;
    desc_.grad_ctx = this;
  }
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;
  virtual int enqueue_gradient(const double* x, std::int64_t ld, double* g, double* f,
                               void* stream) const = 0;
  const char* problem_name() const override { return "device"; }

 private:
  static int trampoline(const double* x, int64_t ld, int64_t n, int64_t p, double* g, double* f,
                        void* stream, void* ctx) {
    (void)n;
    (void)p;
    return static_cast<const DeviceModel*>(ctx)->enqueue_gradient(x, ld, g, f, stream);
  }
};

// E(X) = ¼tr(XᵀLX) + ½tr(XᵀV_ion X) + ¼ρᵀL†ρ + ½ρᵀε_xc(ρ).
class KohnShamModel : public StencilModel {
 public:
  KohnShamModel(std::int64_t nx, std::int64_t ny, std::int64_t nz, const std::vector<double>& v_ion,
                std::int64_t p, double s)
      : StencilModel(nx, ny, nz, v_ion, p, s, PCAL_MODEL_KOHN_SHAM) {}
};

// ---- solve (solver.hpp:120-121) ------------------------------------------------
inline RunReport solve(const ObjectiveModel& model, const SolverConfig& config,
                       const DenseMatrix& x0, CategoryTimers* timers = nullptr) {
  if (x0.rows() != model.n() || x0.cols() != model.p())
    throw dimension_error("solve: start point shape mismatch");
  pcal_config c;
  pcal_config_default(&c);
  c.algorithm = static_cast<int32_t>(config.algorithm);
  c.alm_inner_max = config.alm.inner_max;
  c.alm_outer_max = config.alm.outer_max;
  c.alm_inner_tol_scale = config.alm.inner_tol_scale;
  c.beta = config.beta;
  c.eta_kind = static_cast<int32_t>(config.eta_rule.kind);
  c.gamma = config.eta_rule.gamma;
  c.eta_min = config.eta_rule.eta_min;
  c.eta_max = config.eta_rule.eta_max;
  c.eta0 = config.eta_rule.eta0;
  c.multiplier_rule = config.multiplier_rule == MultiplierRule::PcalFormula
                          ? PCAL_MULT_PCAL_FORMULA
                          : PCAL_MULT_PLAM_FORMULA;
  c.tol_rel_kkt = config.tol_rel_kkt;
  c.max_iter = config.max_iter;
  c.final_orth = config.final_orth ? 1 : 0;
  c.device = config.device;
  if (config.max_iter < 1) throw parameter_error("SolverConfig: max_iter must be at least 1");
  RunReport rep;
  std::vector<double> trace(static_cast<size_t>(config.max_iter + 1) * PCAL_TRACE_COLS);
  rep.stop_iterate = DenseMatrix(model.n(), model.p());
  rep.final_x = DenseMatrix(model.n(), model.p());
  pcal_report r{};
  r.trace = trace.data();
  r.trace_capacity = config.max_iter + 1;
  r.stop_x = rep.stop_iterate.data();
  r.final_x = rep.final_x.data();
  pcal_category_timers t{};
  check(pcal_solve(&model.desc(), &c, x0.data(), PCAL_HOST, &r, timers ? &t : nullptr));
  if (timers) {
    timers->blas3 += t.blas3;
    timers->func += t.func;
    timers->orth += t.orth;
  }
  rep.trace.resize(static_cast<size_t>(r.trace_len));
  for (std::int64_t k = 0; k < r.trace_len; ++k) {
    const double* row = trace.data() + k * PCAL_TRACE_COLS;
    rep.trace[k] = {static_cast<std::int64_t>(row[0]), row[1], row[2], row[3], row[4], row[5],
                    row[6]};
  }
  rep.final_pre_orth = {r.final_pre[0], r.final_pre[1], r.final_pre[2], r.final_pre[3]};
  if (r.has_post)
    rep.final_post_orth = FinalMetrics{r.final_post[0], r.final_post[1], r.final_post[2],
                                       r.final_post[3]};
  if (!r.has_x) {
    rep.stop_iterate = DenseMatrix();
    rep.final_x = DenseMatrix();
  }
  rep.iterations = r.iterations;
  rep.outer_iterations = r.outer_iterations;
  rep.inner_cap_hits = r.inner_cap_hits;
  rep.degenerate_steps = r.degenerate_steps;
  rep.wall_time = r.wall_time;
  rep.status = r.status == PCAL_STATUS_CONVERGED ? RunStatus::Converged
               : r.status == PCAL_STATUS_MAX_ITER ? RunStatus::MaxIter
                                                  : RunStatus::Diverged;
  rep.beta = r.beta;
  // ConfigEcho as iterate_main fills it (solver.cpp:333-342)
  static const char* const alg_names[] = {"plam", "pcal", "alm", "moptqr", "plam-da",
                                          "pcal-da"};  // algorithm_name, diagnostics.cpp:9-19
  rep.config.solver = alg_names[static_cast<int>(config.algorithm)];
  rep.config.beta = r.beta;
  switch (config.eta_rule.kind) {  // eta_rule_name (solver.cpp:41-50)
    case StepsizeRule::Kind::Constant:
      rep.config.eta_rule = "const:" + std::to_string(config.eta_rule.gamma);
      break;
    case StepsizeRule::Kind::Differential: rep.config.eta_rule = "diff"; break;
    case StepsizeRule::Kind::Bb1: rep.config.eta_rule = "bb1"; break;
    case StepsizeRule::Kind::Bb2: rep.config.eta_rule = "bb2"; break;
    case StepsizeRule::Kind::Abb: rep.config.eta_rule = "abb"; break;
  }
  rep.config.tol_rel_kkt = config.tol_rel_kkt;
  rep.config.max_iter = config.max_iter;
  rep.config.threads = config.threads;
  rep.config.n = model.n();
  rep.config.p = model.p();
  rep.config.problem = model.problem_name();
  rep.config.curvature_scale = model.curvature_scale();
  return rep;
}

// initial_point({Qr}, n, p) with Rng(seed) (solver.cpp:136-142)
inline DenseMatrix initial_point_qr(std::int64_t n, std::int64_t p, std::uint64_t seed,
                                    int device = 0) {
  DenseMatrix x(n, p);
  check(pcal_initial_point_qr(n, p, seed, x.data(), device));
  return x;
}

// InitMode / InitialPointSpec / initial_point (solver.hpp:47-59, solver.cpp:136-170)
enum class InitMode { Qr = PCAL_INIT_QR, A2TypeI = PCAL_INIT_A2_TYPE_I, A2TypeII = PCAL_INIT_A2_TYPE_II };
struct InitialPointSpec {
  InitMode mode = InitMode::Qr;
  double sigma_lower = 0.5;  // a2-i only; requires sigma² <= 1/2
  std::uint64_t seed = 0;
};
inline DenseMatrix initial_point(const InitialPointSpec& spec, std::int64_t n, std::int64_t p,
                                 int device = 0) {
  DenseMatrix x(n, p);
  check(pcal_initial_point(n, p, static_cast<int32_t>(spec.mode), spec.sigma_lower, spec.seed,
                           x.data(), device));
  return x;
}

// flops_estimate(Pcal, n, p) (diagnostics.cpp:100-114)
inline double flops_estimate(std::int64_t n, std::int64_t p) { return pcal_flops_estimate(n, p); }

// ---- evaluation and diagnostics (problems.hpp:39,148-149; diagnostics.hpp) ----------
struct Evaluation {  // problems.hpp:18-22
  double value = 0.0;
  DenseMatrix gradient;
};
inline Evaluation evaluate(const ObjectiveModel& model, const DenseMatrix& x, int device = 0) {
  Evaluation ev;
  ev.gradient = DenseMatrix(x.rows(), x.cols());
  check(pcal_evaluate(&model.desc(), x.data(), &ev.value, ev.gradient.data(), device));
  return ev;
}

// fd_gradient_check with the device evaluation (problems.cpp:296-325)
inline double fd_gradient_check(const ObjectiveModel& model, const DenseMatrix& x,
                                double h = 1e-5, std::uint64_t seed = 0x5eedc0de,
                                int device = 0) {
  double w = 0.0;
  check(pcal_fd_gradient_check(&model.desc(), x.data(), h, seed, device, &w));
  return w;
}

namespace detail {
inline DenseMatrix sym_at_b(const DenseMatrix& a, const DenseMatrix& b, int device) {
  DenseMatrix m(a.cols(), b.cols());
  check(pcal_matmul_at_b(a.data(), b.data(), a.rows(), a.cols(), b.cols(), m.data(), device));
  DenseMatrix w(m.rows(), m.cols());
  for (std::int64_t j = 0; j < m.cols(); ++j)
    for (std::int64_t i = 0; i < m.rows(); ++i) w(i, j) = 0.5 * (m(i, j) + m(j, i));
  return w;
}
inline DenseMatrix gram_minus_identity(const DenseMatrix& x, int device) {
  DenseMatrix c(x.cols(), x.cols());
  check(pcal_gram(x.data(), x.rows(), x.cols(), c.data(), device));
  for (std::int64_t j = 0; j < c.cols(); ++j) c(j, j) -= 1.0;
  return c;
}
inline double fro(const DenseMatrix& m) {
  double s = 0.0;
  for (std::size_t k = 0; k < m.size(); ++k) s += m.data()[k] * m.data()[k];
  return std::sqrt(s);
}
}  // namespace detail

// ‖G − X·Ψ(GᵀX)‖_F (diagnostics.cpp:21-30): the n×p products on the device
inline double kkt_violation(const DenseMatrix& grad_f, const DenseMatrix& x, int device = 0) {
  if (grad_f.rows() != x.rows() || grad_f.cols() != x.cols())
    throw dimension_error("kkt_violation: shape mismatch");
  const DenseMatrix w = detail::sym_at_b(grad_f, x, device);
  DenseMatrix xw(x.rows(), x.cols());
  check(pcal_matmul(x.data(), w.data(), x.rows(), x.cols(), x.cols(), xw.data(), device));
  for (std::size_t k = 0; k < xw.size(); ++k) xw.data()[k] = grad_f.data()[k] - xw.data()[k];
  return detail::fro(xw);
}
inline double kkt_violation(const ObjectiveModel& model, const DenseMatrix& x, int device = 0) {
  return kkt_violation(evaluate(model, x, device).gradient, x, device);
}
// ‖XᵀX − I‖_F (diagnostics.cpp:32-36)
inline double feasibility_violation(const DenseMatrix& x, int device = 0) {
  return detail::fro(detail::gram_minus_identity(x, device));
}
// f(X) − ½⟨Ψ(GᵀX), XᵀX − I⟩ + β/4‖XᵀX − I‖² (diagnostics.cpp:38-47)
inline double merit_h(const ObjectiveModel& model, const DenseMatrix& x, double beta,
                      int device = 0) {
  const Evaluation ev = evaluate(model, x, device);
  const DenseMatrix w = detail::sym_at_b(ev.gradient, x, device);
  const DenseMatrix c = detail::gram_minus_identity(x, device);
  double cross = 0.0, feas2 = 0.0;
  for (std::size_t k = 0; k < c.size(); ++k) {
    cross += w.data()[k] * c.data()[k];
    feas2 += c.data()[k] * c.data()[k];
  }
  return ev.value - 0.5 * cross + 0.25 * beta * feas2;
}

}  // namespace orthopt_b200
