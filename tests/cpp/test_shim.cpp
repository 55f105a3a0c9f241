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
  std::printf("%s\n", ok ? "SHIM OK" : "SHIM FAIL");
  return ok ? 0 : 1;
}
