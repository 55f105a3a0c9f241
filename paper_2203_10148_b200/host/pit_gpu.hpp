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

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
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
  int device = 0;
};

class BlockOperatorContext {  // pit::BlockOperatorContext (block_system.hpp:55-72)
 public:
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
    if (p.has_source) {
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
  auto fn = pitsbicg ? pit_pitsbicg_solve : pit_parareal_solve;
  check(fn(ctx.handle(), &c, init ? init->data() : nullptr, r.solution.data(),
           options.first_residual_out ? first.data() : nullptr, rows.data(),
           static_cast<int>(rows.size()), &info));
  for (int i = 0; i < info.record_count; ++i)
    r.history.records.push_back({rows[i].k, rows[i].residual_norm,
                                 static_cast<long>(rows[i].fine_applications),
                                 static_cast<long>(rows[i].coarse_applications), rows[i].wall_ms});
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

}  // namespace pit_gpu
