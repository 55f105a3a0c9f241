// test_adapter.cpp — the reference's own API driving the B200 path through
// integration/pit_gpu_backend.hpp, checked against the reference's CPU path
// on c1 (1D heat, M=100, N=16, 100/1 BE steps, tol 1e-10).  Built by
// oracle/Makefile (needs the reference headers; runs on the GPU box).
#include <cmath>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "pit/block_system.hpp"
#include "pit/pde.hpp"
#include "pit/presets.hpp"
#include "pit/propagator.hpp"
#include "pit/runner.hpp"
#include "pit/solvers.hpp"
#include "pit_gpu_backend.hpp"

using namespace pit;

static double rel(const BlockVector& a, const BlockVector& b) {
  double worst = 0.0;
  for (int n = 0; n < a.block_count(); ++n) {
    double d = 0, s = 0;
    for (size_t i = 0; i < a[n].size(); ++i) {
      d += (a[n][i] - b[n][i]) * (a[n][i] - b[n][i]);
      s += b[n][i] * b[n][i];
    }
    worst = std::fmax(worst, std::sqrt(d) / (s > 0 ? std::sqrt(s) : 1.0));
  }
  return worst;
}

// max_n ||a_n - b_n|| / max_n ||b_n|| (blocks decay by orders of magnitude
// over the desk horizon, so per-block relative errors of tiny blocks say
// nothing about the solve)
static double relmax(const BlockVector& a, const BlockVector& b) {
  double d = 0.0, s = 0.0;
  for (int n = 0; n < a.block_count(); ++n) {
    double dn = 0, sn = 0;
    for (size_t i = 0; i < a[n].size(); ++i) {
      dn += (a[n][i] - b[n][i]) * (a[n][i] - b[n][i]);
      sn += b[n][i] * b[n][i];
    }
    d = std::fmax(d, std::sqrt(dn));
    s = std::fmax(s, std::sqrt(sn));
  }
  return d / (s > 0 ? s : 1.0);
}

int main() {
  const int M = 100, N = 16;
  const GridPtr g = SpatialGrid::make(1, 0.0, 1.0, M + 2);
  PDECoefficients c;
  c.diffusion = 1.0;
  const SpatialOperator op = assemble_spatial_operator(c, g);
  const TimeSlabPartition part(1.0, N);
  std::vector<double> y0(M);
  for (int i = 0; i < M; ++i) y0[i] = std::sin(M_PI * g->interior_coord(i));
  BlockOperatorContext ctx(Propagator(op, part, 100, PropagatorRole::Fine),
                           Propagator(op, part, 1, PropagatorRole::Coarse),
                           ScalarField(g, y0));
  gpu::Backend gpu(ctx);
  SlabExecutor exec(2);
  BlockVector L = ctx.zero_vector();
  for (int n = 0; n < N; ++n)
    for (int i = 0; i < M; ++i) L[n][i] = std::cos(0.37 * n + 0.011 * i);
  RunStats st_cpu, st_gpu;
  const double eF = rel(gpu.apply_F(L, exec, &st_gpu), apply_F(ctx, L, exec, &st_cpu));
  const double eG = rel(gpu.apply_G_inverse(L), apply_G_inverse(ctx, L));
  SolverConfig cfg;
  cfg.tolerance = 1e-10;
  const SolveResult rc = pitsbicg_solve(ctx, cfg, exec);
  const SolveResult rg = gpu.pitsbicg_solve(cfg, exec);
  const double eS = rel(rg.solution, rc.solution);
  const int kc = rc.history.records.back().k, kg = rg.history.records.back().k;
  std::printf("apply_F rel %.3e, apply_G_inverse rel %.3e, pitsbicg k cpu %d gpu %d, restarts %d/%d, "
              "lambda rel %.3e, fine apps %ld/%ld\n",
              eF, eG, kc, kg, rc.history.restarts, rg.history.restarts, eS,
              st_cpu.fine_applications, st_gpu.fine_applications);
  const bool ok = eF < 1e-10 && eG < 1e-10 && eS < 1e-10 && kc == kg &&
                  rc.history.restarts == rg.history.restarts &&
                  st_cpu.fine_applications == st_gpu.fine_applications;
  // the reference's own desk presets (build_context, runner.cpp:75-88),
  // 2D backward Euler with CG / BiCGStab inner solves, N = 8
  bool ok2 = true;
  for (const CaseName cn : {CaseName::Diffusion, CaseName::DiffusionReaction,
                            CaseName::AdvectionDiffusionReaction}) {
    const BlockOperatorContext c2 = build_context(make_preset(cn, Scale::Desk), 8);
    gpu::Backend g2(c2);
    BlockVector X = c2.zero_vector();
    for (int n = 0; n < c2.block_count(); ++n)
      for (size_t i = 0; i < X[n].size(); ++i) X[n][i] = std::cos(0.37 * n + 0.011 * i);
    const double f2 = rel(g2.apply_F(X, exec), apply_F(c2, X, exec));
    const double g2e = rel(g2.apply_G_inverse(X), apply_G_inverse(c2, X));
    SolverConfig c8;  // default tolerance 1e-8, as run_experiment
    const BlockVector ref = sequential_fine_solve(c2);
    SolveOptions o;
    o.reference = &ref;
    const SolveResult r1 = pitsbicg_solve(c2, c8, exec, o);
    const SolveResult r2 = g2.pitsbicg_solve(c8, exec, o);
    const double s2 = relmax(r2.solution, r1.solution);
    const auto &a = r1.history.records.back(), &b = r2.history.records.back();
    const bool e_ok = b.error_vs_reference.has_value() &&
                      std::fabs(*b.error_vs_reference - *a.error_vs_reference) <=
                          1e-4 * *a.error_vs_reference + 1e-11;
    std::printf("%s desk N=8: apply_F rel %.3e, G^-1 rel %.3e, pitsbicg k %d/%d, lambda relmax %.3e, "
                "error_vs_reference %.6e/%.6e\n",
                to_string(cn).c_str(), f2, g2e, a.k, b.k, s2, *a.error_vs_reference,
                b.error_vs_reference ? *b.error_vs_reference : -1.0);
    ok2 = ok2 && f2 < 1e-9 && g2e < 1e-9 && a.k == b.k && s2 < 1e-8 && e_ok &&
          r1.history.restarts == r2.history.restarts;
  }
  // iterate_observer (solvers.hpp:54): the same rows, each with its iterate
  bool ok3 = true;
  {
    std::vector<std::pair<IterationRecord, BlockVector>> seen_cpu, seen_gpu;
    SolveOptions oc, og;
    oc.iterate_observer = [&](const IterationRecord& r, const BlockVector& v) {
      seen_cpu.emplace_back(r, v);
    };
    og.iterate_observer = [&](const IterationRecord& r, const BlockVector& v) {
      seen_gpu.emplace_back(r, v);
    };
    const SolveResult a = pitsbicg_solve(ctx, cfg, exec, oc);
    const SolveResult b = gpu.pitsbicg_solve(cfg, exec, og);
    ok3 = seen_cpu.size() == seen_gpu.size() && seen_gpu.size() == b.history.records.size() &&
          !seen_gpu.empty() && rel(seen_gpu.back().second, b.solution) == 0.0;
    for (size_t i = 0; ok3 && i < seen_cpu.size(); ++i)
      ok3 = seen_cpu[i].first.k == seen_gpu[i].first.k &&
            seen_cpu[i].first.fine_applications == seen_gpu[i].first.fine_applications &&
            rel(seen_gpu[i].second, seen_cpu[i].second) < 1e-9;
    std::printf("iterate_observer: %zu rows cpu, %zu rows gpu: %s\n", seen_cpu.size(),
                seen_gpu.size(), ok3 ? "same" : "DIFFERENT");
  }
  // InnerSolveError payload (errors.hpp:15-21): a NaN right-hand side through
  // the desk preset's coarse sweep, on both paths
  bool ok4 = false;
  {
    const BlockOperatorContext c2 = build_context(make_preset(CaseName::Diffusion, Scale::Desk), 4);
    gpu::Backend g2(c2);
    BlockVector X = c2.zero_vector();
    for (int n = 0; n < c2.block_count(); ++n)
      for (size_t i = 0; i < X[n].size(); ++i) X[n][i] = std::cos(0.1 * n + 0.02 * i);
    X[1][5] = std::nan("");
    double rc_rel = 0, rg_rel = 0;
    int rc_it = -1, rg_it = -2;
    std::string wc, wg;
    try {
      apply_G_inverse(c2, X);
    } catch (const InnerSolveError& e) {
      rc_rel = e.achieved_relative_residual, rc_it = e.iterations, wc = e.what();
    }
    try {
      g2.apply_G_inverse(X);
    } catch (const InnerSolveError& e) {
      rg_rel = e.achieved_relative_residual, rg_it = e.iterations, wg = e.what();
    }
    auto unsign = [](std::string w) {  // the sign of a NaN is not part of the contract
      for (size_t k; (k = w.find("-nan")) != std::string::npos;) w.erase(k, 1);
      return w;
    };
    ok4 = !wc.empty() && rc_it == rg_it && std::isnan(rc_rel) == std::isnan(rg_rel) &&
          unsign(wc) == unsign(wg);
    std::printf("InnerSolveError cpu {%g, %d, \"%s\"} gpu {%g, %d, \"%s\"}\n", rc_rel, rc_it,
                wc.c_str(), rg_rel, rg_it, wg.c_str());
  }
  // a coarse propagator on another operator is rejected at construction
  bool ok5 = false;
  {
    PDECoefficients c3;
    c3.diffusion = 2.0;
    const SpatialOperator op2 = assemble_spatial_operator(c3, g);
    BlockOperatorContext bad(Propagator(op, part, 100, PropagatorRole::Fine),
                             Propagator(op2, part, 1, PropagatorRole::Coarse), ScalarField(g, y0));
    try {
      gpu::Backend gb(bad);
    } catch (const std::invalid_argument&) {
      ok5 = true;
    }
    std::printf("different coarse operator rejected: %s\n", ok5 ? "yes" : "NO");
  }
  // pinned staging: N >= 32 takes pit_apply_F's overlapped copy path
  bool ok6 = false;
  {
    const int M2 = 256, N2 = 40;
    const GridPtr g2 = SpatialGrid::make(1, 0.0, 1.0, M2 + 2);
    const SpatialOperator op3 = assemble_spatial_operator(c, g2);
    const TimeSlabPartition part2(N2 / 1024.0, N2);
    std::vector<double> z0(M2);
    for (int i = 0; i < M2; ++i) z0[i] = std::sin(3 * M_PI * g2->interior_coord(i));
    BlockOperatorContext c4(Propagator(op3, part2, 50, PropagatorRole::Fine),
                            Propagator(op3, part2, 1, PropagatorRole::Coarse), ScalarField(g2, z0));
    gpu::Backend g4(c4);
    BlockVector X = c4.zero_vector();
    for (int n = 0; n < N2; ++n)
      for (int i = 0; i < M2; ++i) X[n][i] = std::cos(0.3 * n + 0.05 * i);
    RunStats sg;
    double e = 0;
    for (int rep = 0; rep < 3; ++rep) e = std::fmax(e, rel(g4.apply_F(X, exec, &sg), apply_F(c4, X, exec)));
    ok6 = e < 1e-10 && g4.worker_count() > 0 && sg.fine_busy_ms > 0.0 &&
          sg.fine_applications == 3L * (N2 - 1);
    std::printf("pinned-staging apply_F rel %.3e, device slots %d, fine busy %.3f ms / wall %.3f ms\n",
                e, g4.worker_count(), sg.fine_busy_ms, sg.fine_parallel_ms);
  }
  // a general (non-separable) SourceFn: the context is built with it, the
  // backend samples the same function into the C ABI's source tables
  bool ok7 = false;
  {
    const SourceFn f = [](double t, std::span<const double> x) {
      return 2.0 * ((1.0 + t) * x[0] * (1.0 - x[0]) + std::sin(3.0 * t) * std::cos(2.0 * M_PI * x[0]));
    };
    BlockOperatorContext cs(Propagator(op, part, 100, PropagatorRole::Fine, f),
                            Propagator(op, part, 1, PropagatorRole::Coarse, f), ScalarField(g, y0));
    gpu::Backend gs(cs, f);
    const double eB = rel(gs.assemble_rhs(exec), assemble_rhs(cs, exec));
    const SolveResult sc = pitsbicg_solve(cs, cfg, exec);
    const SolveResult sg = gs.pitsbicg_solve(cfg, exec);
    const double eL = relmax(sg.solution, sc.solution);
    ok7 = eB < 1e-10 && eL < 1e-10 && sc.history.records.back().k == sg.history.records.back().k;
    std::printf("general SourceFn: assemble_rhs rel %.3e, pitsbicg k cpu %d gpu %d, lambda rel %.3e\n",
                eB, sc.history.records.back().k, sg.history.records.back().k, eL);
  }
  // a variable-coefficient operator through the CSR constructor (pde.hpp:36-37)
  bool ok8 = false;
  {
    const int Mv = 150, Nv = 8;
    const GridPtr gv = SpatialGrid::make(1, 0.0, 1.0, Mv + 2);
    const double h = gv->spacing();
    CsrMatrix a;
    a.n = Mv;
    a.row_ptr.push_back(0);
    for (int i = 0; i < Mv; ++i) {
      const double x = gv->interior_coord(i);
      const double mm = 1.0 + 0.5 * std::sin(2 * M_PI * (x - h / 2));
      const double mp = 1.0 + 0.5 * std::sin(2 * M_PI * (x + h / 2));
      const double adv = 20.0 * (1.0 + x);
      if (i > 0) {
        a.col.push_back(i - 1);
        a.val.push_back(-mm / (h * h) - adv / (2 * h));
      }
      a.col.push_back(i);
      a.val.push_back((mm + mp) / (h * h) + 0.5);
      if (i < Mv - 1) {
        a.col.push_back(i + 1);
        a.val.push_back(-mp / (h * h) + adv / (2 * h));
      }
      a.row_ptr.push_back(static_cast<int>(a.col.size()));
    }
    const SpatialOperator opv(std::move(a), gv, false);
    const TimeSlabPartition pv(0.05, Nv);
    std::vector<double> yv(Mv);
    for (int i = 0; i < Mv; ++i) yv[i] = std::sin(M_PI * gv->interior_coord(i));
    BlockOperatorContext cv(Propagator(opv, pv, 20, PropagatorRole::Fine),
                            Propagator(opv, pv, 1, PropagatorRole::Coarse), ScalarField(gv, yv));
    gpu::Backend bv(cv);
    SolverConfig c9;
    c9.tolerance = 1e-9;
    const SolveResult sc = pitsbicg_solve(cv, c9, exec);
    const SolveResult sg = bv.pitsbicg_solve(c9, exec);
    const double eL = relmax(sg.solution, sc.solution);
    ok8 = eL < 1e-8 && std::abs(sc.history.records.back().k - sg.history.records.back().k) <= 1;
    std::printf("variable-coefficient operator: pitsbicg k cpu %d gpu %d, lambda rel %.3e\n",
                sc.history.records.back().k, sg.history.records.back().k, eL);
  }
  // a source on a 2D grid (propagator.cpp:36-44 samples it node by node)
  bool ok9 = false;
  {
    const GridPtr g2 = SpatialGrid::make_unit(2, 19);
    PDECoefficients pc;
    pc.velocity = VelocityField::Rotation;
    pc.diffusion = 0.1;
    pc.reaction = 0.5;
    const SourceFn f2 = [](double t, std::span<const double> x) {
      return (1.0 + t) * std::exp(-8.0 * (x[0] * x[0] + x[1] * x[1])) + std::sin(3.0 * t) * x[0] * x[1];
    };
    const SpatialOperator o2 = assemble_spatial_operator(pc, g2);
    const TimeSlabPartition p2(0.4, 4);
    const int m2 = g2->interior_per_axis();
    std::vector<double> y2(static_cast<size_t>(m2) * m2);
    for (int j = 0; j < m2; ++j)
      for (int i = 0; i < m2; ++i) {
        const double xx = g2->interior_coord(i), yy = g2->interior_coord(j);
        y2[g2->flat_index(i, j)] = std::exp(-20.0 * (xx * xx + yy * yy));
      }
    BlockOperatorContext c2s(Propagator(o2, p2, 10, PropagatorRole::Fine, f2),
                             Propagator(o2, p2, 1, PropagatorRole::Coarse, f2), ScalarField(g2, y2));
    gpu::Backend b2(c2s, f2);
    SolverConfig c8;
    const double eB = relmax(b2.assemble_rhs(exec), assemble_rhs(c2s, exec));
    const SolveResult sc = pitsbicg_solve(c2s, c8, exec);
    const SolveResult sg = b2.pitsbicg_solve(c8, exec);
    const double eL = relmax(sg.solution, sc.solution);
    ok9 = eB < 1e-9 && eL < 1e-7 && sc.history.records.back().k == sg.history.records.back().k;
    std::printf("2D source: assemble_rhs rel %.3e, pitsbicg k cpu %d gpu %d, lambda rel %.3e\n", eB,
                sc.history.records.back().k, sg.history.records.back().k, eL);
  }
  const bool all = ok && ok2 && ok3 && ok4 && ok5 && ok6 && ok7 && ok8 && ok9;
  std::printf("%s\n", all ? "ADAPTER OK" : "ADAPTER FAIL");
  return all ? 0 : 1;
}
