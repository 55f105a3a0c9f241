// test_adapter.cpp — the reference's own API driving the B200 path through
// integration/pit_gpu_backend.hpp, checked against the reference's CPU path
// on c1 (1D heat, M=100, N=16, 100/1 BE steps, tol 1e-10).  Built by
// oracle/Makefile (needs the reference headers; runs on the GPU box).
#include <cmath>
#include <cstdio>

#include "pit/block_system.hpp"
#include "pit/pde.hpp"
#include "pit/propagator.hpp"
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
  std::printf("%s\n", ok ? "ADAPTER OK" : "ADAPTER FAIL");
  return ok ? 0 : 1;
}
