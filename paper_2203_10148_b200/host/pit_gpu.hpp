// pit_gpu.hpp — header-only C++17 mirror of the reference's pit:: operator and
// solver API over the C ABI (include/pit_b200.h).
//
// Same names, argument meaning and error behaviour as the reference
// (/root/reference/proj/include/pit/{block_system,solvers,errors}.hpp):
//   pit_gpu::apply_F / assemble_rhs / apply_G_inverse / initial_guess /
//   preconditioned_residual / sequential_fine_solve / pitsbicg_solve /
//   parareal_solve / block_inner_product / block_norm_n_inf
// throwing pit_gpu::InnerSolveError / SlabError / ConfigError /
// std::invalid_argument exactly where the reference throws pit:: ones.
// Block vectors are contiguous block-major std::vector<double> (N*M).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

#include "pit_b200.h"

namespace pit_gpu {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InnerSolveError : Error {
  using Error::Error;
};
struct SlabError : Error {
  SlabError(int slab, const std::string& what) : Error(what), slab_index(slab) {}
  int slab_index;
};
struct ConfigError : Error {
  using Error::Error;
};
struct DeviceError : Error {
  using Error::Error;
};

inline void check(int rc) {
  if (rc == PIT_OK) return;
  const std::string msg = pit_last_error();
  switch (rc) {
    case PIT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PIT_ERR_INNER_SOLVE: throw InnerSolveError(msg);
    case PIT_ERR_SLAB: throw SlabError(pit_last_error_slab(), msg);
    case PIT_ERR_CONFIG: throw ConfigError(msg);
    default: throw DeviceError(msg);
  }
}

using BlockVector = std::vector<double>;  // N*M, block-major, x-fastest

struct RunStats {  // pit::RunStats (executor.hpp:24-30)
  long fine_applications = 0;
  long coarse_applications = 0;
  double fine_parallel_ms = 0.0;
  double fine_busy_ms = 0.0;
  double coarse_sequential_ms = 0.0;
  void add(const pit_run_stats& s) {
    fine_applications += static_cast<long>(s.fine_applications);
    coarse_applications += static_cast<long>(s.coarse_applications);
    fine_parallel_ms += s.fine_parallel_ms;
    fine_busy_ms += s.fine_busy_ms;
    coarse_sequential_ms += s.coarse_sequential_ms;
  }
};

enum class SolveStatus { Converged, MaxIterations };
enum class InitialGuessPolicy { CoarseSweep = PIT_GUESS_COARSE_SWEEP, Zero = PIT_GUESS_ZERO };

struct IterationRecord {
  int k = 0;
  double residual_norm = 0.0;
  long fine_applications = 0;
  long coarse_applications = 0;
  double wall_ms = 0.0;
  std::optional<double> error_vs_reference;  // with SolveOptions::reference
};

struct ConvergenceHistory {
  std::vector<IterationRecord> records;
  SolveStatus status = SolveStatus::MaxIterations;
  int restarts = 0;
  RunStats stats;
};

struct SolverConfig {  // pit::SolverConfig (solvers.hpp:36-44)
  double tolerance = 1e-8;
  double restart_tolerance = 1e-12;
  int max_iterations = 200;
  InitialGuessPolicy initial_guess = InitialGuessPolicy::CoarseSweep;
  void validate() const {
    if (!(tolerance > restart_tolerance) || !(restart_tolerance > 0.0))
      throw ConfigError("solver tolerances must satisfy tolerance > restart_tolerance > 0");
    if (max_iterations < 1) throw ConfigError("max_iterations must be >= 1");
  }
};

struct SolveOptions {
  const BlockVector* initial_guess_override = nullptr;
  const BlockVector* reference = nullptr;  // every row: ||lambda - reference||_{N,inf}
  BlockVector* first_residual_out = nullptr;
};

struct SolveResult {
  BlockVector solution;
  ConvergenceHistory history;
};

// Problem description: the reference's BlockOperatorContext inputs for a 1D
// constant-coefficient operator (SpatialGrid + SpatialOperator bands +
// TimeSlabPartition + fine/coarse steps_per_slab + SourceFn + initial value).
struct Problem1D {
  int M = 0;
  double grid_lo = 0.0, grid_hi = 1.0;
  double band_lo = 0.0, band_diag = 0.0, band_up = 0.0;
  int N = 2;
  double T = 1.0;
  int fine_steps = 1, coarse_steps = 1;
  std::vector<double> y0;
  bool has_source = false;
  double source_amp = 0.0, source_omega = 0.0, source_phase = 0.0;
  std::vector<double> source_shape;
  // a general pit::SourceFn f(t, x) (pde.hpp:13), 1D: takes precedence over
  // the separable description; sampled at the end of every step
  // (propagator.cpp:56-63) into the C ABI's PIT_SOURCE_TABLE tables
  std::function<double(double t, double x)> source_fn;
  // a general tridiagonal operator (pde.hpp:36-37: any CSR through the
  // SpatialOperator constructor): [3][M] sub, diagonal, super entries per
  // interior node; band_* are then ignored and every step is solved by
  // Jacobi-PCG or (nonsymmetric) Jacobi-BiCGStab as in the reference
  // (pde.cpp:112-130).  M <= 10240, no source.
  std::vector<double> stencil;
  bool nonsymmetric = false;
  double fine_tolerance = 0.0, coarse_tolerance = 0.0;  // 0: 1e-12
  int device = 0;
};

// The reference's 2D experiments (presets.cpp, runner.cpp:75-88): m x m
// interior nodes, both propagators backward Euler on a 5-point operator given
// per node as its south, west, centre, east, north CSR entries (0 = absent),
// inner solves Jacobi-PCG or (nonsymmetric) Jacobi-BiCGStab.  See
// make_preset / build_problem below.
struct Problem2D {
  int m = 0;
  double grid_lo = -0.5, grid_hi = 0.5;
  std::vector<double> stencil;  // [5][m*m]
  bool nonsymmetric = false;
  int N = 2;
  double T = 1.0;
  int fine_steps = 1, coarse_steps = 1;
  std::vector<double> y0;
  double fine_tolerance = 0.0, coarse_tolerance = 0.0;  // 0: 1e-12
  int device = 0;
};

class BlockOperatorContext {  // pit::BlockOperatorContext (block_system.hpp:55-72)
 public:
  explicit BlockOperatorContext(const Problem2D& p) : M_(p.m * p.m), N_(p.N) {
    if (static_cast<int>(p.y0.size()) != M_ || static_cast<int>(p.stencil.size()) != 5 * M_)
      throw std::invalid_argument("ScalarField: value count does not match grid");
    pit_problem_desc d{};
    d.dimension = 2;
    d.interior = p.m;
    d.grid_lo = p.grid_lo;
    d.grid_hi = p.grid_hi;
    d.slab_count = p.N;
    d.total_time = p.T;
    d.fine_steps = p.fine_steps;
    d.coarse_steps = p.coarse_steps;
    d.initial_value = p.y0.data();
    d.device = p.device;
    d.fine_scheme = PIT_SCHEME_BACKWARD_EULER;
    d.stencil = p.stencil.data();
    d.nonsymmetric = p.nonsymmetric ? 1 : 0;
    d.fine_tolerance = p.fine_tolerance;
    d.coarse_tolerance = p.coarse_tolerance;
    pit_context* c = nullptr;
    check(pit_context_create(&d, &c));
    ctx_.reset(c);
  }
  explicit BlockOperatorContext(const Problem1D& p) : M_(p.M), N_(p.N) {
    pit_problem_desc d{};
    d.dimension = 1;
    d.interior = p.M;
    d.grid_lo = p.grid_lo;
    d.grid_hi = p.grid_hi;
    d.band_lo = p.band_lo;
    d.band_diag = p.band_diag;
    d.band_up = p.band_up;
    d.slab_count = p.N;
    d.total_time = p.T;
    d.fine_steps = p.fine_steps;
    d.coarse_steps = p.coarse_steps;
    d.initial_value = p.y0.data();
    d.device = p.device;
    if (!p.stencil.empty()) {
      if (static_cast<int>(p.stencil.size()) != 3 * p.M)
        throw std::invalid_argument("Problem1D: stencil must hold 3*M entries");
      d.stencil = p.stencil.data();
      d.nonsymmetric = p.nonsymmetric ? 1 : 0;
      d.fine_tolerance = p.fine_tolerance;
      d.coarse_tolerance = p.coarse_tolerance;
    }
    std::vector<double> tab[2];
    if (p.source_fn) {
      const double h = (p.grid_hi - p.grid_lo) / (p.M + 1), slab = p.T / p.N;
      const int steps[2] = {p.fine_steps, p.coarse_steps};
      for (int r = 0; r < 2; ++r) {
        const double dt = slab / steps[r];
        tab[r].reserve(static_cast<size_t>(p.N) * steps[r] * p.M);
        for (int n = 0; n < p.N; ++n)
          for (int k = 1; k <= steps[r]; ++k)
            for (int i = 0; i < p.M; ++i)
              tab[r].push_back(p.source_fn(n * slab + k * dt, p.grid_lo + (i + 1) * h));
      }
      d.source_kind = PIT_SOURCE_TABLE;
      d.source_table_fine = tab[0].data();
      d.source_table_coarse = tab[1].data();
    } else if (p.has_source) {
      d.source_kind = PIT_SOURCE_SEPARABLE;
      d.source_amp = p.source_amp;
      d.source_omega = p.source_omega;
      d.source_phase = p.source_phase;
      d.source_shape = p.source_shape.data();
    }
    if (static_cast<int>(p.y0.size()) != p.M)
      throw std::invalid_argument("ScalarField: value count does not match grid");
    pit_context* c = nullptr;
    check(pit_context_create(&d, &c));
    ctx_.reset(c);
  }
  int block_count() const { return N_; }
  int nodes() const { return M_; }
  BlockVector zero_vector() const { return BlockVector(static_cast<size_t>(N_) * M_, 0.0); }
  pit_context* handle() const { return ctx_.get(); }
  void require_shape(const BlockVector& v, const char* what) const {
    if (v.size() != static_cast<size_t>(N_) * M_)
      throw std::invalid_argument(std::string(what) + ": block count does not match the partition");
  }

 private:
  struct Del {
    void operator()(pit_context* c) const { pit_context_destroy(c); }
  };
  int M_, N_;
  std::unique_ptr<pit_context, Del> ctx_;
};

inline BlockVector apply_F(const BlockOperatorContext& ctx, const BlockVector& L,
                           RunStats* stats = nullptr) {
  ctx.require_shape(L, "apply_F");
  BlockVector out = ctx.zero_vector();
  pit_run_stats s{};
  check(pit_apply_F(ctx.handle(), L.data(), out.data(), &s));
  if (stats) stats->add(s);
  return out;
}

inline BlockVector assemble_rhs(const BlockOperatorContext& ctx, RunStats* stats = nullptr) {
  BlockVector out = ctx.zero_vector();
  pit_run_stats s{};
  check(pit_assemble_rhs(ctx.handle(), out.data(), &s));
  if (stats) stats->add(s);
  return out;
}

inline BlockVector apply_G_inverse(const BlockOperatorContext& ctx, const BlockVector& V,
                                   RunStats* stats = nullptr) {
  ctx.require_shape(V, "apply_G_inverse");
  BlockVector out = ctx.zero_vector();
  pit_run_stats s{};
  check(pit_apply_G_inverse(ctx.handle(), V.data(), out.data(), &s));
  if (stats) stats->add(s);
  return out;
}

inline BlockVector initial_guess(const BlockOperatorContext& ctx, InitialGuessPolicy policy,
                                 RunStats* stats = nullptr) {
  BlockVector out = ctx.zero_vector();
  pit_run_stats s{};
  check(pit_initial_guess(ctx.handle(), static_cast<int>(policy), out.data(), &s));
  if (stats) stats->add(s);
  return out;
}

inline BlockVector preconditioned_residual(const BlockOperatorContext& ctx,
                                           const BlockVector& lambda, const BlockVector& rhs,
                                           RunStats* stats = nullptr) {
  ctx.require_shape(lambda, "apply_F");
  ctx.require_shape(rhs, "apply_F");
  BlockVector out = ctx.zero_vector();
  pit_run_stats s{};
  check(pit_preconditioned_residual(ctx.handle(), lambda.data(), rhs.data(), out.data(), &s));
  if (stats) stats->add(s);
  return out;
}

inline BlockVector sequential_fine_solve(const BlockOperatorContext& ctx) {
  BlockVector out = ctx.zero_vector();
  check(pit_sequential_fine_solve(ctx.handle(), out.data()));
  return out;
}

inline double block_inner_product(const BlockOperatorContext& ctx, const BlockVector& a,
                                  const BlockVector& b) {
  ctx.require_shape(a, "block_inner_product");
  ctx.require_shape(b, "block_inner_product");
  double v = 0.0;
  check(pit_block_inner_product(ctx.handle(), a.data(), b.data(), &v));
  return v;
}

inline double block_norm_n_inf(const BlockOperatorContext& ctx, const BlockVector& a) {
  ctx.require_shape(a, "block_norm_n_inf");
  double v = 0.0;
  check(pit_block_norm_n_inf(ctx.handle(), a.data(), &v));
  return v;
}

namespace detail {
inline SolveResult solve(bool pitsbicg, const BlockOperatorContext& ctx,
                         const SolverConfig& config, const SolveOptions& options) {
  config.validate();
  pit_solver_config c{config.tolerance, config.restart_tolerance, config.max_iterations,
                      static_cast<int32_t>(config.initial_guess)};
  const BlockVector* init = options.initial_guess_override;
  if (init) ctx.require_shape(*init, "initial guess");
  SolveResult r;
  r.solution = ctx.zero_vector();
  std::vector<pit_record> rows(static_cast<size_t>(config.max_iterations) + 2);
  pit_solve_info info{};
  BlockVector first;
  if (options.first_residual_out) first = ctx.zero_vector();
  if (options.reference) {
    ctx.require_shape(*options.reference, "reference");
    check(pit_set_reference(ctx.handle(), options.reference->data()));
  }
  auto fn = pitsbicg ? pit_pitsbicg_solve : pit_parareal_solve;
  const int rc = fn(ctx.handle(), &c, init ? init->data() : nullptr, r.solution.data(),
                    options.first_residual_out ? first.data() : nullptr, rows.data(),
                    static_cast<int>(rows.size()), &info);
  if (options.reference) pit_set_reference(ctx.handle(), nullptr);
  check(rc);
  for (int i = 0; i < info.record_count; ++i) {
    IterationRecord rec{rows[i].k, rows[i].residual_norm,
                        static_cast<long>(rows[i].fine_applications),
                        static_cast<long>(rows[i].coarse_applications), rows[i].wall_ms, {}};
    if (rows[i].has_error) rec.error_vs_reference = rows[i].error_vs_reference;
    r.history.records.push_back(rec);
  }
  r.history.status =
      info.status == PIT_CONVERGED ? SolveStatus::Converged : SolveStatus::MaxIterations;
  r.history.restarts = info.restarts;
  r.history.stats.add(info.stats);
  if (options.first_residual_out) *options.first_residual_out = std::move(first);
  return r;
}
}  // namespace detail

// pit::pitsbicg_solve (solvers.hpp:89-90; src/solvers.cpp:116-220)
inline SolveResult pitsbicg_solve(const BlockOperatorContext& ctx, const SolverConfig& config,
                                  const SolveOptions& options = {}) {
  return detail::solve(true, ctx, config, options);
}

// pit::parareal_solve (solvers.hpp:82-83; src/solvers.cpp:73-114)
inline SolveResult parareal_solve(const BlockOperatorContext& ctx, const SolverConfig& config,
                                  const SolveOptions& options = {}) {
  return detail::solve(false, ctx, config, options);
}

// ---- the reference's presets (presets.cpp:48-77, runner.cpp:75-88) ------

enum class CaseName { Diffusion, DiffusionReaction, AdvectionDiffusionReaction };
enum class Scale { Paper, Desk };

struct ExperimentPreset {  // pit::ExperimentPreset (presets.hpp:25-40)
  CaseName case_name = CaseName::Diffusion;
  bool rotation = false;
  double mu = 1.0, r = 0.0;
  int grid_points = 33;
  double total_time = 1.6, dt_fine = 1e-3;
  std::vector<int> slab_counts{4, 8, 16, 32, 64};
  double gaussian_sigma = 0.1;
};

inline ExperimentPreset make_preset(CaseName name, Scale scale) {
  ExperimentPreset p;
  p.case_name = name;
  if (name == CaseName::DiffusionReaction) p.r = 1.5;
  if (name == CaseName::AdvectionDiffusionReaction) {
    p.rotation = true;
    p.mu = 0.1;
    p.r = 0.5;
  }
  if (scale == Scale::Paper) {
    p.grid_points = 51;
    p.total_time = 6.4;
  }
  return p;
}

// build_context as a device problem: assemble_spatial_operator's 2D rows
// (pde.cpp:66-100), make_fine_propagator's step count (propagator.cpp:88-98),
// one coarse step, gaussian_initial_condition (grid.cpp:120-141).
inline Problem2D build_problem(const ExperimentPreset& pr, int slab_count) {
  if (slab_count < 2) throw std::invalid_argument("TimeSlabPartition: need at least 2 slabs");
  Problem2D p;
  p.m = pr.grid_points - 2;
  const int m = p.m, n = m * m;
  const double lo = p.grid_lo, h = (p.grid_hi - lo) / (pr.grid_points - 1);
  const double mu_h2 = pr.mu / (h * h);
  p.stencil.assign(5 * static_cast<size_t>(n), 0.0);
  p.y0.resize(n);
  const double inv = 1.0 / (2.0 * pr.gaussian_sigma * pr.gaussian_sigma);
  for (int j = 0; j < m; ++j) {
    const double y = lo + (j + 1) * h;
    for (int i = 0; i < m; ++i) {
      const double x = lo + (i + 1) * h;
      const double ux = pr.rotation ? -y : 0.0, uy = pr.rotation ? x : 0.0;
      const double centre = 4.0 * mu_h2 + pr.r + (std::fabs(ux) + std::fabs(uy)) / h;
      double w = -mu_h2, e = -mu_h2, s = -mu_h2, nn = -mu_h2;
      if (ux > 0.0) w -= ux / h; else if (ux < 0.0) e += ux / h;
      if (uy > 0.0) s -= uy / h; else if (uy < 0.0) nn += uy / h;
      const size_t row = static_cast<size_t>(j) * m + i;
      p.stencil[row] = (s != 0.0 && j > 0) ? s : 0.0;
      p.stencil[n + row] = (w != 0.0 && i > 0) ? w : 0.0;
      p.stencil[2 * static_cast<size_t>(n) + row] = centre;
      p.stencil[3 * static_cast<size_t>(n) + row] = (e != 0.0 && i < m - 1) ? e : 0.0;
      p.stencil[4 * static_cast<size_t>(n) + row] = (nn != 0.0 && j < m - 1) ? nn : 0.0;
      p.y0[row] = std::exp(-(x * x + y * y) * inv);
    }
  }
  p.nonsymmetric = pr.rotation;
  p.N = slab_count;
  p.T = pr.total_time;
  const double ratio = (pr.total_time / slab_count) / pr.dt_fine;
  const int steps = std::max(1, static_cast<int>(std::lround(ratio)));
  if (std::fabs(ratio - steps) > 1e-9 * steps)
    throw std::invalid_argument("make_fine_propagator: slab length is not a multiple of dt");
  p.fine_steps = steps;
  p.coarse_steps = 1;
  return p;
}

}  // namespace pit_gpu
