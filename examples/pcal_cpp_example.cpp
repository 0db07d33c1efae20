// pcal_cpp_example.cpp — the reference's Rayleigh–Ritz acceptance check
// (acceptance_main.cpp:50-73 shape: n=200, p=10, PCAL defaults) written against
// the C++ mirror (include/orthopt_b200/solver.hpp).  Exit code 0 on success.
//   usage: pcal_cpp_example [n p]
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "orthopt_b200/solver.hpp"

int main(int argc, char** argv) {
  using namespace orthopt_b200;
  const std::int64_t n = argc > 2 ? std::atoll(argv[1]) : 200;
  const std::int64_t p = argc > 2 ? std::atoll(argv[2]) : 10;
  try {
    DenseMatrix a(n, n);
    check(pcal_gen_dense_operator(n, 101, a.data(), 4));  // sym_part(random_normal(n,n,Rng(101)))
    double s = 0.0;
    check(pcal_spectral_norm_estimate(a.data(), n, 0x73706563, &s, 0));
    QuadraticModel model(a, p, s);
    SolverConfig cfg;
    const DenseMatrix x0 = initial_point_qr(n, p, 102);
    CategoryTimers timers;
    const RunReport rep = solve(model, cfg, x0, &timers);
    std::printf("status=%d iterations=%lld f_post=%.12f feas_post=%.3e blas3=%.4fs func=%.4fs orth=%.4fs\n",
                static_cast<int>(rep.status), static_cast<long long>(rep.iterations),
                rep.final_post_orth ? rep.final_post_orth->fval : NAN,
                rep.final_post_orth ? rep.final_post_orth->feas : NAN, timers.blas3, timers.func,
                timers.orth);
    if (rep.status != RunStatus::Converged || !rep.final_post_orth ||
        rep.final_post_orth->feas > 1e-12)
      return 1;
    // ConfigEcho as the reference's solve() fills it (solver.cpp:333-342)
    const ConfigEcho& ce = rep.config;
    std::printf("echo: problem=%s solver=%s beta=%g eta_rule=%s n=%lld p=%lld threads=%d s=%.6f\n",
                ce.problem.c_str(), ce.solver.c_str(), ce.beta, ce.eta_rule.c_str(),
                static_cast<long long>(ce.n), static_cast<long long>(ce.p), ce.threads,
                ce.curvature_scale);
    if (ce.problem != "p2" || ce.solver != "pcal" || ce.beta != 1.0 || ce.eta_rule != "abb" ||
        ce.n != n || ce.p != p || ce.max_iter != cfg.max_iter || ce.curvature_scale != s ||
        ce.threads != cfg.threads)
      return 6;
    // the P6 density model on the same operator (problems.cpp:276-285)
    {
      DensityModel p6(a, p, 2.0 * std::cbrt(3.0 / 3.14159265358979323846), ProblemKind::P6, s);
      const RunReport r6 = solve(p6, SolverConfig{}, x0);
      std::printf("p6: status=%d iterations=%lld f_post=%.12f feas_post=%.3e\n",
                  static_cast<int>(r6.status), static_cast<long long>(r6.iterations),
                  r6.final_post_orth ? r6.final_post_orth->fval : NAN,
                  r6.final_post_orth ? r6.final_post_orth->feas : NAN);
      if (!r6.final_post_orth || r6.final_post_orth->feas > 1e-12) return 4;
      // the reference's diagnostics on the final iterate (diagnostics.cpp:21-47)
      const double kkt = kkt_violation(p6, r6.final_x), feas = feasibility_violation(r6.final_x);
      const double fd = fd_gradient_check(p6, r6.final_x);
      std::printf("p6 diagnostics: kkt=%.3e (report %.3e) feas=%.3e fd=%.3e merit=%.12f\n", kkt,
                  r6.final_post_orth->kkt_abs, feas, fd, merit_h(p6, r6.final_x, 1.0));
      if (std::abs(kkt - r6.final_post_orth->kkt_abs) > 1e-6 * std::max(kkt, 1e-300) + 1e-12 ||
          feas > 1e-12 || fd > 1e-6)
        return 5;
    }
    // parameter errors are thrown before iterating (solver.cpp:106-118)
    cfg.tol_rel_kkt = 0.0;
    try {
      solve(model, cfg, x0);
      return 2;
    } catch (const parameter_error&) {
    }
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
