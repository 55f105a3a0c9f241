// pit_gpu_backend.hpp — the binding a reference maintainer adds to
// /root/reference/proj/include/pit/ to route the PiT hot path to the B200
// kernels.  It takes the reference's own types (pit::BlockOperatorContext,
// pit::BlockVector, pit::SolverConfig, pit::SolveResult) and calls the C ABI
// (include/pit_b200.h).  Only this header is new; no reference source changes.
//
//   pit::gpu::Backend gpu(ctx);                     // once per context
//   pit::BlockVector f = gpu.apply_F(L, exec, &stats);        // == pit::apply_F
//   pit::SolveResult r = gpu.pitsbicg_solve(cfg, exec, opts); // == pit::pitsbicg_solve
//
// Requirements checked at construction (else std::invalid_argument):
//   * 1D grid: SpatialOperator a tridiagonal CSR.  Constant bands (what
//     assemble_spatial_operator builds for 1D, pde.cpp:55-64, or hand-built
//     central-difference advection) take the direct solve; any other
//     tridiagonal operator (variable coefficients, pde.hpp:36-37) is solved
//     per step by the reference's own inner solvers on the device
//     (M <= 10240, no source);
//   * 2D grid (the desk/paper presets, runner.cpp:75-88): any 5-point CSR
//     (assemble_spatial_operator's 2D rows, pde.cpp:66-100, any velocity),
//     m <= 101 points per axis; both propagators backward Euler with the
//     reference's inner solvers (CG if op().symmetric(), else BiCGStab);
//   * a source, if any: the context's own SourceFn (sampled into tables), or
//     separable f(t,x) = amp*sin(omega*t+phase)*g(x),
//     described by a SeparableSource (the std::function itself is opaque;
//     1D only).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pit/block_system.hpp"
#include "pit/errors.hpp"
#include "pit/solvers.hpp"
#include "pit_b200.h"

namespace pit::gpu {

struct SeparableSource {
  double amp = 0.0, omega = 0.0, phase = 0.0;
  std::vector<double> shape;  // g(x_i) at the interior nodes
};

inline void check(int rc) {
  if (rc == PIT_OK) return;
  const std::string msg = pit_last_error();
  switch (rc) {
    case PIT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PIT_ERR_INNER_SOLVE: {
      // the achieved relative residual and iteration count of the failing
      // inner solve (errors.hpp:15-21)
      double rel = std::nan("");
      int64_t its = 0;
      pit_last_error_detail(&rel, &its);
      throw pit::InnerSolveError(msg, rel, static_cast<int>(its));
    }
    case PIT_ERR_SLAB: throw pit::SlabError(pit_last_error_slab(), msg);
    case PIT_ERR_CONFIG: throw pit::ConfigError(msg);
    default: throw pit::Error(msg);
  }
}

class Backend {
 public:
  // A context built with a general SourceFn (pde.hpp:13): pass the same
  // function; it is sampled where Propagator::run samples it
  // (propagator.cpp:25-47, 56-63) into the C ABI's PIT_SOURCE_TABLE tables
  // (N * steps * M doubles per propagator).  The Propagator keeps its
  // SourceFn private, so the context alone cannot supply it.
  Backend(const BlockOperatorContext& ctx, const SourceFn& source, int device = 0)
      : Backend(ctx, nullptr, device, &source) {}

  explicit Backend(const BlockOperatorContext& ctx, const SeparableSource* source = nullptr,
                   int device = 0, const SourceFn* general = nullptr)
      : ctx_(ctx) {
    const SpatialGrid& g = ctx.fine().op().grid();
    // one spatial operator feeds both device propagators: the reference's
    // context only checks grid, partition and source agreement
    // (block_system.cpp:90-113), so reject a coarse operator that differs
    {
      const SpatialOperator& f = ctx.fine().op();
      const SpatialOperator& c = ctx.coarse().op();
      const CsrMatrix& a = f.matrix();
      const CsrMatrix& b = c.matrix();
      if (a.n != b.n || a.row_ptr != b.row_ptr || a.col != b.col || a.val != b.val ||
          f.symmetric() != c.symmetric())
        throw std::invalid_argument(
            "pit::gpu::Backend: the fine and coarse propagators must share one spatial operator");
    }
    if (g.dimension() == 2) {
      init_2d(ctx, g, device, general);
      return;
    }
    const CsrMatrix& A = ctx.fine().op().matrix();
    double band[3] = {0.0, 0.0, 0.0};  // lo, diag, up
    bool seen[3] = {false, false, false};
    bool constant = true;
    // per-node sub, diagonal, super entries: a general tridiagonal operator
    // (variable coefficients) goes to the device's iterative path
    std::vector<double> tri(3 * static_cast<size_t>(A.n), 0.0);
    for (int i = 0; i < A.n; ++i) {
      for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
        const int off = A.col[k] - i + 1;  // 0 sub, 1 diag, 2 super
        if (off < 0 || off > 2)
          throw std::invalid_argument("pit::gpu::Backend: operator is not tridiagonal");
        tri[static_cast<size_t>(off) * A.n + i] = A.val[k];
        if (!seen[off]) {
          band[off] = A.val[k];
          seen[off] = true;
        } else if (A.val[k] != band[off]) {
          constant = false;
        }
      }
    }
    const double lo = band[0], di = band[1], up = band[2];
    if (ctx.fine().has_source() && !source && !(general && *general))
      throw std::invalid_argument(
          "pit::gpu::Backend: a source needs its SourceFn or a SeparableSource");
    pit_problem_desc d{};
    d.dimension = 1;
    d.interior = g.interior_per_axis();
    d.grid_lo = g.lo();
    d.grid_hi = g.hi();
    d.band_lo = lo;
    d.band_diag = di;
    d.band_up = up;
    d.slab_count = ctx.block_count();
    d.total_time = ctx.partition().total_time();
    d.fine_steps = ctx.fine().steps_per_slab();
    d.coarse_steps = ctx.coarse().steps_per_slab();
    const auto y0 = ctx.initial_value().values();
    d.initial_value = y0.data();
    if (!constant) {
      // Jacobi-PCG / Jacobi-BiCGStab per step, as the reference's
      // ImplicitStepSolver (pde.cpp:112-130); no direct solve, no source
      if (ctx.fine().has_source() && !(general && *general))
        throw std::invalid_argument(
            "pit::gpu::Backend: a source on a variable-coefficient operator needs its SourceFn");
      d.stencil = tri.data();
      d.nonsymmetric = ctx.fine().op().symmetric() ? 0 : 1;
    }
    if (source) {
      d.source_kind = PIT_SOURCE_SEPARABLE;
      d.source_amp = source->amp;
      d.source_omega = source->omega;
      d.source_phase = source->phase;
      d.source_shape = source->shape.data();
    }
    std::vector<double> tab[2];
    if (!source && general && *general && ctx.fine().has_source()) {
      sample_tables(ctx, g, *general, tab);
      d.source_kind = PIT_SOURCE_TABLE;
      d.source_table_fine = tab[0].data();
      d.source_table_coarse = tab[1].data();
    }
    d.device = device;
    pit_context* c = nullptr;
    check(pit_context_create(&d, &c));
    h_.reset(c);
    M_ = d.interior;
    N_ = d.slab_count;
  }

  // 2D: the per-row south/west/centre/east/north entries of A (0 when the
  // CSR row has none) and the operator's symmetry flag go to the device.
  // The context's SourceFn sampled where Propagator::run samples it
  // (propagator.cpp:25-47: every interior node, x fastest; 56-63: the end of
  // every step) into the C ABI's PIT_SOURCE_TABLE tables.
  static void sample_tables(const BlockOperatorContext& ctx, const SpatialGrid& g,
                            const SourceFn& f, std::vector<double> (&tab)[2]) {
    const Propagator* prop[2] = {&ctx.fine(), &ctx.coarse()};
    const int m = g.interior_per_axis(), dim = g.dimension(), N = ctx.block_count();
    const size_t M = dim == 2 ? static_cast<size_t>(m) * m : static_cast<size_t>(m);
    for (int r = 0; r < 2; ++r) {
      const int steps = prop[r]->steps_per_slab();
      const double dt = prop[r]->internal_dt();
      tab[r].resize(static_cast<size_t>(N) * steps * M);
      size_t at = 0;
      for (int n = 0; n < N; ++n) {
        const double t0 = ctx.partition().breakpoint(n);
        for (int k = 1; k <= steps; ++k) {
          const double t = t0 + k * dt;
          if (dim == 1) {
            for (int i = 0; i < m; ++i) {
              const double x[1] = {g.interior_coord(i)};
              tab[r][at++] = f(t, x);
            }
          } else {
            for (int j = 0; j < m; ++j)
              for (int i = 0; i < m; ++i) {
                const double x[2] = {g.interior_coord(i), g.interior_coord(j)};
                tab[r][at++] = f(t, x);
              }
          }
        }
      }
    }
  }

  void init_2d(const BlockOperatorContext& ctx, const SpatialGrid& g, int device,
               const SourceFn* general) {
    if (ctx.fine().has_source() && !(general && *general))
      throw std::invalid_argument("pit::gpu::Backend: a source on a 2D grid needs its SourceFn");
    const SpatialOperator& op = ctx.fine().op();
    const CsrMatrix& A = op.matrix();
    const int m = g.interior_per_axis(), M = m * m;
    std::vector<double> st(5 * static_cast<size_t>(M), 0.0);
    for (int i = 0; i < A.n; ++i)
      for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
        const int d = A.col[k] - i;
        const int slot = d == -m ? 0 : d == -1 ? 1 : d == 0 ? 2 : d == 1 ? 3 : d == m ? 4 : -1;
        if (slot < 0) throw std::invalid_argument("pit::gpu::Backend: operator is not 5-point");
        st[static_cast<size_t>(slot) * M + i] = A.val[k];
      }
    pit_problem_desc d{};
    d.dimension = 2;
    d.interior = m;
    d.grid_lo = g.lo();
    d.grid_hi = g.hi();
    d.slab_count = ctx.block_count();
    d.total_time = ctx.partition().total_time();
    d.fine_steps = ctx.fine().steps_per_slab();
    d.coarse_steps = ctx.coarse().steps_per_slab();
    const auto y0 = ctx.initial_value().values();
    d.initial_value = y0.data();
    d.device = device;
    d.fine_scheme = PIT_SCHEME_BACKWARD_EULER;
    d.stencil = st.data();
    d.nonsymmetric = op.symmetric() ? 0 : 1;
    std::vector<double> tab[2];
    if (ctx.fine().has_source()) {
      sample_tables(ctx, g, *general, tab);
      d.source_kind = PIT_SOURCE_TABLE;
      d.source_table_fine = tab[0].data();
      d.source_table_coarse = tab[1].data();
    }
    pit_context* c = nullptr;
    check(pit_context_create(&d, &c));
    h_.reset(c);
    M_ = M;
    N_ = d.slab_count;
  }

  // pit::apply_F.  The BlockVector's blocks are gathered (host threads) into
  // a page-locked staging buffer, so pit_apply_F takes its overlapped path:
  // chunked H2D copies, K1's slabs starting as their chunk lands, chunked
  // D2H copies of finished output blocks; the result is scattered back.
  BlockVector apply_F(const BlockVector& L, SlabExecutor& /*exec*/,
                      RunStats* stats = nullptr) const {
    check_blocks(L, "apply_F");
    stage();
    gather(L, stage_in_);
    pit_run_stats s{};
    check(pit_apply_F(h_.get(), stage_in_, stage_out_, &s));
    add(stats, s);
    BlockVector v = ctx_.zero_vector();
    scatter(stage_out_, v);
    return v;
  }

  // Fine slabs resident at once on the GPU: the worker count to pass to
  // pit::timing_report (executor.cpp:156-171) for a device run.
  int worker_count() const {
    int slots = 0;
    check(pit_context_slots(h_.get(), &slots));
    return slots;
  }

  BlockVector apply_G_inverse(const BlockVector& V, RunStats* stats = nullptr) const {
    auto x = flat(V, "apply_G_inverse");
    std::vector<double> out(x.size());
    pit_run_stats s{};
    check(pit_apply_G_inverse(h_.get(), x.data(), out.data(), &s));
    add(stats, s);
    return unflat(out);
  }

  BlockVector assemble_rhs(SlabExecutor& /*exec*/, RunStats* stats = nullptr) const {
    std::vector<double> out(static_cast<size_t>(N_) * M_);
    pit_run_stats s{};
    check(pit_assemble_rhs(h_.get(), out.data(), &s));
    add(stats, s);
    return unflat(out);
  }

  SolveResult pitsbicg_solve(const SolverConfig& config, SlabExecutor& /*exec*/,
                             const SolveOptions& options = {}) const {
    return solve(true, config, options);
  }
  SolveResult parareal_solve(const SolverConfig& config, SlabExecutor& /*exec*/,
                             const SolveOptions& options = {}) const {
    return solve(false, config, options);
  }

 private:
  struct Del {
    void operator()(pit_context* c) const { pit_context_destroy(c); }
  };
  struct HostDel {
    void operator()(double* p) const { pit_host_free(p); }
  };

  void check_blocks(const BlockVector& v, const char* what) const {
    if (v.block_count() != N_)
      throw std::invalid_argument(std::string(what) + ": block count does not match the partition");
    for (int n = 0; n < N_; ++n) require_same_grid(v[n], ctx_.initial_value());
  }
  void stage() const {
    if (stage_in_) return;
    const size_t bytes = sizeof(double) * static_cast<size_t>(N_) * M_;
    void *a = nullptr, *b = nullptr;
    check(pit_host_alloc(bytes, &a));
    in_keep_.reset(static_cast<double*>(a));
    check(pit_host_alloc(bytes, &b));
    out_keep_.reset(static_cast<double*>(b));
    stage_in_ = in_keep_.get();
    stage_out_ = out_keep_.get();
  }
  // block copies split over host threads (a single thread's memcpy is far
  // below the host's memory bandwidth)
  template <class F>
  void parallel_blocks(F&& f) const {
    const int nt = std::max(1, std::min<int>(8, static_cast<int>(std::thread::hardware_concurrency())));
    if (nt == 1 || static_cast<size_t>(N_) * M_ < (1u << 18)) {
      for (int n = 0; n < N_; ++n) f(n);
      return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (int n = t * N_ / nt; n < (t + 1) * N_ / nt; ++n) f(n);
      });
    for (auto& x : th) x.join();
  }
  void gather(const BlockVector& v, double* dst) const {
    parallel_blocks([&](int n) {
      std::memcpy(dst + static_cast<size_t>(n) * M_, v[n].values().data(), sizeof(double) * M_);
    });
  }
  void scatter(const double* src, BlockVector& v) const {
    parallel_blocks([&](int n) {
      std::memcpy(v[n].values().data(), src + static_cast<size_t>(n) * M_, sizeof(double) * M_);
    });
  }

  std::vector<double> flat(const BlockVector& v, const char* what) const {
    if (v.block_count() != N_)
      throw std::invalid_argument(std::string(what) + ": block count does not match the partition");
    std::vector<double> x(static_cast<size_t>(N_) * M_);
    for (int n = 0; n < N_; ++n) {
      require_same_grid(v[n], ctx_.initial_value());
      std::memcpy(x.data() + static_cast<size_t>(n) * M_, v[n].values().data(),
                  sizeof(double) * M_);
    }
    return x;
  }
  BlockVector unflat(const std::vector<double>& x) const {
    BlockVector v = ctx_.zero_vector();
    for (int n = 0; n < N_; ++n)
      std::memcpy(v[n].values().data(), x.data() + static_cast<size_t>(n) * M_,
                  sizeof(double) * M_);
    return v;
  }
  static void add(RunStats* st, const pit_run_stats& s) {
    if (!st) return;
    st->fine_applications += static_cast<long>(s.fine_applications);
    st->coarse_applications += static_cast<long>(s.coarse_applications);
    st->fine_parallel_ms += s.fine_parallel_ms;
    st->fine_busy_ms += s.fine_busy_ms;
    st->coarse_sequential_ms += s.coarse_sequential_ms;
  }

  SolveResult solve(bool pitsbicg, const SolverConfig& config, const SolveOptions& options) const {
    config.validate();
    pit_solver_config c{config.tolerance, config.restart_tolerance, config.max_iterations,
                        config.initial_guess == InitialGuessPolicy::Zero ? PIT_GUESS_ZERO
                                                                         : PIT_GUESS_COARSE_SWEEP};
    std::vector<double> init;
    if (options.initial_guess_override) init = flat(*options.initial_guess_override, "initial guess");
    std::vector<double> lam(static_cast<size_t>(N_) * M_), first;
    if (options.first_residual_out) first.resize(lam.size());
    std::vector<pit_record> rows(static_cast<size_t>(config.max_iterations) + 2);
    pit_solve_info info{};
    auto fn = pitsbicg ? pit_pitsbicg_solve : pit_parareal_solve;
    // SolveOptions::iterate_observer (solvers.hpp:54): each row with the
    // iterate it describes, rebuilt as a BlockVector
    struct Obs {
      const Backend* self;
      const std::function<void(const IterationRecord&, const BlockVector&)>* fn;
    } obs{this, &options.iterate_observer};
    if (options.iterate_observer) {
      check(pit_set_iterate_observer(
          h_.get(),
          [](const pit_record* row, const double* lam, int, int, void* user) {
            auto* o = static_cast<Obs*>(user);
            BlockVector v = o->self->ctx_.zero_vector();
            o->self->scatter(lam, v);
            (*o->fn)(to_record(*row), v);
          },
          &obs));
    }
    // SolveOptions::reference: every row carries block_norm_n_inf(lambda - reference)
    if (options.reference) {
      const std::vector<double> ref = flat(*options.reference, "reference");
      check(pit_set_reference(h_.get(), ref.data()));
    }
    const int rc = fn(h_.get(), &c, init.empty() ? nullptr : init.data(), lam.data(),
                      first.empty() ? nullptr : first.data(), rows.data(),
                      static_cast<int>(rows.size()), &info);
    if (options.reference) pit_set_reference(h_.get(), nullptr);
    if (options.iterate_observer) pit_set_iterate_observer(h_.get(), nullptr, nullptr);
    check(rc);
    SolveResult r{unflat(lam), {}};
    for (int i = 0; i < info.record_count; ++i) r.history.records.push_back(to_record(rows[i]));
    r.history.status =
        info.status == PIT_CONVERGED ? SolveStatus::Converged : SolveStatus::MaxIterations;
    r.history.restarts = info.restarts;
    add(&r.history.stats, info.stats);
    if (options.first_residual_out) *options.first_residual_out = unflat(first);
    return r;
  }

  static IterationRecord to_record(const pit_record& row) {
    IterationRecord rec;
    rec.k = row.k;
    rec.residual_norm = row.residual_norm;
    rec.fine_applications = static_cast<long>(row.fine_applications);
    rec.coarse_applications = static_cast<long>(row.coarse_applications);
    rec.wall_ms = row.wall_ms;
    if (row.has_error) rec.error_vs_reference = row.error_vs_reference;
    return rec;
  }

  const BlockOperatorContext& ctx_;
  std::unique_ptr<pit_context, Del> h_;
  int M_ = 0, N_ = 0;
  // page-locked staging of apply_F (allocated on first use)
  mutable std::unique_ptr<double, HostDel> in_keep_, out_keep_;
  mutable double* stage_in_ = nullptr;
  mutable double* stage_out_ = nullptr;
};

}  // namespace pit::gpu
