// test_shim.cpp — the C++ mirror API (paper_2203_10148_b200/host/pit_gpu.hpp)
// on c1: PiTSBiCG to 1e-10 must converge at k=5 with one restart (the
// reference's history, tests/golden/c1_reference.npz) and raise the
// reference's exception types on bad input.
#include <cmath>
#include <cstdio>

#include "../../paper_2203_10148_b200/host/pit_gpu.hpp"

int main() {
  pit_gpu::Problem1D p;
  p.M = 100;
  p.N = 16;
  p.T = 1.0;
  p.fine_steps = 100;
  p.coarse_steps = 1;
  const double h = 1.0 / (p.M + 1);
  const double mu_h2 = 1.0 / (h * h);
  p.band_lo = -mu_h2;
  p.band_diag = 2.0 * mu_h2;
  p.band_up = -mu_h2;
  p.y0.resize(p.M);
  for (int i = 0; i < p.M; ++i) p.y0[i] = std::sin(M_PI * (i + 1) * h);
  pit_gpu::BlockOperatorContext ctx(p);
  pit_gpu::SolverConfig cfg;
  cfg.tolerance = 1e-10;
  const auto r = pit_gpu::pitsbicg_solve(ctx, cfg);
  const auto& last = r.history.records.back();
  std::printf("k=%d restarts=%d residual=%.6e fine=%ld\n", last.k, r.history.restarts,
              last.residual_norm, last.fine_applications);
  bool ok = last.k == 5 && r.history.restarts == 1 && last.residual_norm <= 1e-10 &&
            r.history.status == pit_gpu::SolveStatus::Converged;
  try {
    pit_gpu::apply_F(ctx, pit_gpu::BlockVector(10));
    ok = false;
  } catch (const std::invalid_argument&) {
  }
  try {
    pit_gpu::SolverConfig bad;
    bad.tolerance = 1e-13;
    pit_gpu::pitsbicg_solve(ctx, bad);
    ok = false;
  } catch (const pit_gpu::ConfigError&) {
  }
  // the reference's desk rotation preset (K6, BiCGStab inner solves) with a
  // reference solution: converges, every row carries error_vs_reference
  const auto pr = pit_gpu::make_preset(pit_gpu::CaseName::AdvectionDiffusionReaction,
                                       pit_gpu::Scale::Desk);
  pit_gpu::BlockOperatorContext c2(pit_gpu::build_problem(pr, 8));
  const pit_gpu::BlockVector ref = pit_gpu::sequential_fine_solve(c2);
  pit_gpu::SolveOptions opts;
  opts.reference = &ref;
  const auto r2 = pit_gpu::pitsbicg_solve(c2, pit_gpu::SolverConfig{}, opts);
  const auto& l2 = r2.history.records.back();
  std::printf("desk rotation N=8: k=%d residual=%.3e error=%.3e\n", l2.k, l2.residual_norm,
              l2.error_vs_reference ? *l2.error_vs_reference : -1.0);
  ok = ok && r2.history.status == pit_gpu::SolveStatus::Converged && l2.residual_norm <= 1e-8 &&
       l2.error_vs_reference && *l2.error_vs_reference < 1e-7;
  // a general SourceFn (pde.hpp:13) and a variable-coefficient tridiagonal
  // operator through the mirror: the sequential fine solution is the fixed
  // point of F lambda = b, and PiTSBiCG reaches it
  auto fixed_point = [](const pit_gpu::BlockOperatorContext& c, const char* what, double tol) {
    const pit_gpu::BlockVector seq = pit_gpu::sequential_fine_solve(c);
    const pit_gpu::BlockVector Fl = pit_gpu::apply_F(c, seq);
    const pit_gpu::BlockVector b = pit_gpu::assemble_rhs(c);
    double gap = 0.0, scale = 0.0;
    for (size_t i = 0; i < seq.size(); ++i) {
      gap = std::fmax(gap, std::fabs(Fl[i] - b[i]));
      scale = std::fmax(scale, std::fabs(seq[i]));
    }
    pit_gpu::SolveOptions o;
    o.reference = &seq;
    pit_gpu::SolverConfig sc;
    sc.tolerance = tol;
    const auto rr = pit_gpu::pitsbicg_solve(c, sc, o);
    const auto& lr = rr.history.records.back();
    std::printf("%s: |F seq - b|=%.3e (scale %.3e) k=%d residual=%.3e error=%.3e\n", what, gap,
                scale, lr.k, lr.residual_norm, lr.error_vs_reference ? *lr.error_vs_reference : -1.0);
    return scale > 0.0 && gap <= 1e-13 * std::fmax(1.0, scale) &&
           rr.history.status == pit_gpu::SolveStatus::Converged && lr.error_vs_reference &&
           *lr.error_vs_reference <= 100.0 * tol * std::fmax(1.0, scale);
  };
  pit_gpu::Problem1D ps = p;
  ps.N = 8;
  ps.T = 0.5;
  ps.source_fn = [](double t, double x) { return std::exp(-t) * x * (1.0 - x) + std::sin(3.0 * t * x); };
  ok = ok && fixed_point(pit_gpu::BlockOperatorContext(ps), "source_fn", 1e-10);
  pit_gpu::Problem1D pv = p;
  pv.N = 8;
  pv.T = 0.05;
  pv.fine_steps = 20;
  pv.stencil.resize(3 * static_cast<size_t>(pv.M));
  for (int i = 0; i < pv.M; ++i) {
    const double xl = (i + 0.5) * h, xr = (i + 1.5) * h;
    const double kl = 1.0 + 0.5 * std::sin(2.0 * M_PI * xl), kr = 1.0 + 0.5 * std::sin(2.0 * M_PI * xr);
    pv.stencil[i] = i > 0 ? -kl * mu_h2 : 0.0;
    pv.stencil[pv.M + i] = (kl + kr) * mu_h2;
    pv.stencil[2 * static_cast<size_t>(pv.M) + i] = i + 1 < pv.M ? -kr * mu_h2 : 0.0;
  }
  ok = ok && fixed_point(pit_gpu::BlockOperatorContext(pv), "stencil", 1e-9);
  std::printf("%s\n", ok ? "SHIM OK" : "SHIM FAIL");
  return ok ? 0 : 1;
}
