// ref_driver.cpp — extern "C" driver over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie (/root/reference/proj/src/*.cpp, minus
// cli.cpp which needs the absent CLI11.hpp) into oracle/_ref/libpitref.so.
// It builds BASELINE contexts through the reference's public C++ API
// (SpatialGrid::make, SpatialOperator, Propagator, BlockOperatorContext) and
// exposes apply_F / apply_G_inverse / assemble_rhs / initial_guess /
// sequential_fine_solve / pitsbicg_solve / parareal_solve with flat
// block-major double arrays, so tests and bench.py can call the reference
// itself (golden vectors, the CPU baseline, and the loop pin).
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "pit/block_system.hpp"
#include "pit/errors.hpp"
#include "pit/executor.hpp"
#include "pit/pde.hpp"
#include "pit/presets.hpp"
#include "pit/propagator.hpp"
#include "pit/runner.hpp"
#include "pit/solvers.hpp"

namespace {

thread_local std::string g_err;

struct RefCtx {
  std::unique_ptr<pit::BlockOperatorContext> ctx;
  int M = 0;
  int N = 0;
  std::vector<double> shape;
  pit::SourceFn src;  // the source both propagators were built with
};

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const pit::SlabError*>(&e)) return 3;
  if (dynamic_cast<const pit::InnerSolveError*>(&e)) return 2;
  if (dynamic_cast<const pit::ConfigError*>(&e)) return 4;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  return 5;
}

pit::BlockVector unflat(const RefCtx& r, const double* x) {
  pit::BlockVector v = r.ctx->zero_vector();
  for (int n = 0; n < r.N; ++n) {
    auto vals = v[n].values();
    std::memcpy(vals.data(), x + static_cast<size_t>(n) * r.M, sizeof(double) * r.M);
  }
  return v;
}

void flat(const RefCtx& r, const pit::BlockVector& v, double* x) {
  for (int n = 0; n < r.N; ++n) {
    auto vals = v[n].values();
    std::memcpy(x + static_cast<size_t>(n) * r.M, vals.data(), sizeof(double) * r.M);
  }
}

void copy_history(const pit::ConvergenceHistory& h, int* rec_k, double* rec_res,
                  long* rec_fine, long* rec_coarse, int max_rec, int* nrec, int* restarts,
                  int* converged) {
  const int n = static_cast<int>(h.records.size());
  *nrec = n;
  for (int i = 0; i < n && i < max_rec; ++i) {
    rec_k[i] = h.records[i].k;
    rec_res[i] = h.records[i].residual_norm;
    rec_fine[i] = h.records[i].fine_applications;
    rec_coarse[i] = h.records[i].coarse_applications;
  }
  *restarts = h.restarts;
  *converged = h.status == pit::SolveStatus::Converged ? 1 : 0;
}

}  // namespace

extern "C" {

const char* pitref_last_error() { return g_err.c_str(); }

// 1D context over a general tridiagonal operator given per interior node
// (sub, diag, sup; 0 = absent) through the SpatialOperator CSR constructor
// (pde.hpp:36-37): variable coefficients.  No source.
void* pitref_create_1d_csr(int M, double lo, double hi, const double* sub, const double* diag,
                           const double* sup, int symmetric, int N, double T, int fine_steps,
                           int coarse_steps, const double* y0, int test_source);

// 1D context on [lo, hi] with M interior points.  When use_bands == 0 the
// operator comes from assemble_spatial_operator(diffusion, reaction)
// (pde.cpp:45-64); otherwise a hand-built tridiagonal CSR with the given
// bands (the route c3's central-difference advection needs, pde.hpp:36-37).
// Source (has_source == 1): f(t, x_i) = amp * sin(omega*t + phase) * shape[i];
// has_source == 2: a non-separable test source
//   f(t, x) = amp * ((1 + t) * x * (1 - x) + sin(omega * t) * cos(phase * x))
// (shape unused) for the general-source path (PIT_SOURCE_TABLE).
void* pitref_create_1d(int M, double lo, double hi, double diffusion, double reaction,
                       int use_bands, double band_lo, double band_diag, double band_up,
                       int symmetric, int N, double T, int fine_steps, int coarse_steps,
                       const double* y0, int has_source, const double* shape, double amp,
                       double omega, double phase) {
  try {
    auto r = std::make_unique<RefCtx>();
    r->M = M;
    r->N = N;
    const pit::GridPtr g = pit::SpatialGrid::make(1, lo, hi, M + 2);
    pit::SpatialOperator op = [&]() {
      if (!use_bands) {
        pit::PDECoefficients c;
        c.diffusion = diffusion;
        c.reaction = reaction;
        return pit::assemble_spatial_operator(c, g);
      }
      pit::CsrMatrix a;
      a.n = M;
      a.row_ptr.push_back(0);
      for (int i = 0; i < M; ++i) {
        if (i > 0 && band_lo != 0.0) {
          a.col.push_back(i - 1);
          a.val.push_back(band_lo);
        }
        a.col.push_back(i);
        a.val.push_back(band_diag);
        if (i < M - 1 && band_up != 0.0) {
          a.col.push_back(i + 1);
          a.val.push_back(band_up);
        }
        a.row_ptr.push_back(static_cast<int>(a.col.size()));
      }
      return pit::SpatialOperator(std::move(a), g, symmetric != 0);
    }();
    const pit::TimeSlabPartition part(T, N);
    pit::SourceFn src;
    if (has_source == 2) {
      src = [amp, omega, phase](double t, std::span<const double> x) {
        return amp * ((1.0 + t) * x[0] * (1.0 - x[0]) + std::sin(omega * t) * std::cos(phase * x[0]));
      };
    } else if (has_source) {
      r->shape.assign(shape, shape + M);
      const double h = g->spacing();
      const std::vector<double>* sh = &r->shape;
      src = [sh, lo, h, amp, omega, phase](double t, std::span<const double> x) {
        const long i = std::lround((x[0] - lo) / h) - 1;
        return amp * std::sin(omega * t + phase) * (*sh)[static_cast<size_t>(i)];
      };
    }
    r->src = src;
    pit::Propagator fine(op, part, fine_steps, pit::PropagatorRole::Fine, src);
    pit::Propagator coarse(op, part, coarse_steps, pit::PropagatorRole::Coarse, src);
    pit::ScalarField init(g, std::vector<double>(y0, y0 + M));
    r->ctx = std::make_unique<pit::BlockOperatorContext>(std::move(fine), std::move(coarse),
                                                         std::move(init));
    return r.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// 2D heat on [lo, hi]^2 with m interior points per axis: the reference's
// own 2D operator (assemble_spatial_operator, zero velocity, pde.cpp:66-100)
// and its backward-Euler propagators (CG to kInnerSolveRelTol, pde.hpp:78).
// Blocks are m*m values, x fastest.  Used to pin the 2D coarse CG step.
void* pitref_create_2d(int m, double lo, double hi, double diffusion, double reaction, int N,
                       double T, int fine_steps, int coarse_steps, const double* y0) {
  try {
    auto r = std::make_unique<RefCtx>();
    r->M = m * m;
    r->N = N;
    const pit::GridPtr g = pit::SpatialGrid::make(2, lo, hi, m + 2);
    pit::PDECoefficients c;
    c.diffusion = diffusion;
    c.reaction = reaction;
    pit::SpatialOperator op = pit::assemble_spatial_operator(c, g);
    const pit::TimeSlabPartition part(T, N);
    pit::Propagator fine(op, part, fine_steps, pit::PropagatorRole::Fine);
    pit::Propagator coarse(op, part, coarse_steps, pit::PropagatorRole::Coarse);
    pit::ScalarField init(g, std::vector<double>(y0, y0 + r->M));
    r->ctx = std::make_unique<pit::BlockOperatorContext>(std::move(fine), std::move(coarse),
                                                         std::move(init));
    return r.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// The reference's own experiment contexts: build_context(make_preset(case,
// scale), N) (runner.cpp:75-88, presets.cpp:48-77); case 0 diffusion,
// 1 diffusion_reaction, 2 advection_diffusion_reaction; scale 0 desk, 1 paper.
void* pitref_create_preset(int case_id, int scale, int N) {
  try {
    const pit::CaseName cn = case_id == 0   ? pit::CaseName::Diffusion
                             : case_id == 1 ? pit::CaseName::DiffusionReaction
                                            : pit::CaseName::AdvectionDiffusionReaction;
    const pit::ExperimentPreset preset =
        pit::make_preset(cn, scale == 1 ? pit::Scale::Paper : pit::Scale::Desk);
    auto r = std::make_unique<RefCtx>();
    r->ctx = std::make_unique<pit::BlockOperatorContext>(pit::build_context(preset, N));
    r->M = static_cast<int>(r->ctx->initial_value().values().size());
    r->N = N;
    return r.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// pit::run_experiment (runner.cpp:108-147) on a preset with the given slab
// counts; writes <out_dir>/<case>.csv.  solver: 0 parareal, 1 pitsbicg, 2 both.
int pitref_run_experiment(int case_id, int scale, const int* slabs, int nslabs, int solver,
                          double tol, const char* out_dir) {
  try {
    const pit::CaseName cn = case_id == 0   ? pit::CaseName::Diffusion
                             : case_id == 1 ? pit::CaseName::DiffusionReaction
                                            : pit::CaseName::AdvectionDiffusionReaction;
    pit::RunSpec spec;
    spec.preset = pit::make_preset(cn, scale == 1 ? pit::Scale::Paper : pit::Scale::Desk);
    spec.preset.slab_counts.assign(slabs, slabs + nslabs);
    spec.solver = solver == 0 ? pit::SolverChoice::Parareal
                  : solver == 1 ? pit::SolverChoice::PiTSBiCG
                                : pit::SolverChoice::Both;
    spec.solver_config.tolerance = tol;
    spec.out_dir = out_dir;
    std::ostringstream log;
    pit::run_experiment(spec, log);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pitref_initial_value(void* p, double* out) {
  auto* r = static_cast<RefCtx*>(p);
  auto v = r->ctx->initial_value().values();
  std::memcpy(out, v.data(), sizeof(double) * v.size());
  return 0;
}

void pitref_destroy(void* p) { delete static_cast<RefCtx*>(p); }

double pitref_spacing(void* p) {
  return static_cast<RefCtx*>(p)->ctx->grid_ptr()->spacing();
}

int pitref_apply_F(void* p, const double* L, double* out, int workers) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    pit::SlabExecutor exec(workers);
    flat(r, pit::apply_F(*r.ctx, unflat(r, L), exec), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pitref_apply_G_inverse(void* p, const double* V, double* out) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    flat(r, pit::apply_G_inverse(*r.ctx, unflat(r, V)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pitref_assemble_rhs(void* p, double* out, int workers) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    pit::SlabExecutor exec(workers);
    flat(r, pit::assemble_rhs(*r.ctx, exec), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pitref_initial_guess(void* p, double* out) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    flat(r, pit::initial_guess(*r.ctx, pit::InitialGuessPolicy::CoarseSweep), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pitref_sequential_fine(void* p, double* out) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    flat(r, pit::sequential_fine_solve(*r.ctx), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The values Propagator::sample_source(t) (private; propagator.cpp:25-47)
// hands to rhs.axpy(dt, .): the context's SourceFn at the M interior nodes.
int pitref_sample_source(void* p, double t, double* out) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    const pit::SpatialGrid& g = *r.ctx->grid_ptr();
    for (int i = 0; i < r.M; ++i) {
      const double x[1] = {g.interior_coord(i)};
      out[i] = r.src ? r.src(t, x) : 0.0;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// test_source != 0: the non-separable source of pitref_create_1d (has_source
// == 2) with amp 2, omega 3, phase 2 pi.
void* pitref_create_1d_csr(int M, double lo, double hi, const double* sub, const double* diag,
                           const double* sup, int symmetric, int N, double T, int fine_steps,
                           int coarse_steps, const double* y0, int test_source) {
  try {
    auto r = std::make_unique<RefCtx>();
    r->M = M;
    r->N = N;
    const pit::GridPtr g = pit::SpatialGrid::make(1, lo, hi, M + 2);
    pit::CsrMatrix a;
    a.n = M;
    a.row_ptr.push_back(0);
    for (int i = 0; i < M; ++i) {
      if (i > 0 && sub[i] != 0.0) {
        a.col.push_back(i - 1);
        a.val.push_back(sub[i]);
      }
      a.col.push_back(i);
      a.val.push_back(diag[i]);
      if (i < M - 1 && sup[i] != 0.0) {
        a.col.push_back(i + 1);
        a.val.push_back(sup[i]);
      }
      a.row_ptr.push_back(static_cast<int>(a.col.size()));
    }
    const pit::SpatialOperator op(std::move(a), g, symmetric != 0);
    const pit::TimeSlabPartition part(T, N);
    pit::SourceFn src;
    if (test_source)
      src = [](double t, std::span<const double> x) {
        return 2.0 * ((1.0 + t) * x[0] * (1.0 - x[0]) + std::sin(3.0 * t) * std::cos(2.0 * M_PI * x[0]));
      };
    r->src = src;
    pit::Propagator fine(op, part, fine_steps, pit::PropagatorRole::Fine, src);
    pit::Propagator coarse(op, part, coarse_steps, pit::PropagatorRole::Coarse, src);
    pit::ScalarField init(g, std::vector<double>(y0, y0 + M));
    r->ctx = std::make_unique<pit::BlockOperatorContext>(std::move(fine), std::move(coarse),
                                                          std::move(init));
    return r.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Propagator::propagate / propagate_homogeneous on one field (role 0 fine, 1 coarse).
int pitref_propagate(void* p, int role, int with_source, const double* in, int slab,
                     double* out) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    const pit::Propagator& prop = role == 0 ? r.ctx->fine() : r.ctx->coarse();
    pit::ScalarField f(r.ctx->grid_ptr(), std::vector<double>(in, in + r.M));
    pit::ScalarField y = with_source ? prop.propagate(f, slab) : prop.propagate_homogeneous(f, slab);
    std::memcpy(out, y.values().data(), sizeof(double) * r.M);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Signature-compatible with orc_prop_fn (oracle/pit_oracle.h): lets the
// restated solver loop run on the reference's own propagators.
int pitref_prop_callback(void* user, int role, int with_source, const double* in, int slab,
                         double* out) {
  return pitref_propagate(user, role, with_source, in, slab, out);
}

static int run_solver(int which, void* p, double tol, double eps0, int max_iter, int zero_guess,
                      int workers, const double* lambda_init, double* lambda_out,
                      double* first_residual_out, int* rec_k, double* rec_res, long* rec_fine,
                      long* rec_coarse, int max_rec, int* nrec, int* restarts, int* converged) {
  try {
    auto& r = *static_cast<RefCtx*>(p);
    pit::SlabExecutor exec(workers);
    pit::SolverConfig cfg;
    cfg.tolerance = tol;
    cfg.restart_tolerance = eps0;
    cfg.max_iterations = max_iter;
    cfg.initial_guess =
        zero_guess ? pit::InitialGuessPolicy::Zero : pit::InitialGuessPolicy::CoarseSweep;
    pit::SolveOptions opt;
    pit::BlockVector init = r.ctx->zero_vector();
    if (lambda_init) {
      init = unflat(r, lambda_init);
      opt.initial_guess_override = &init;
    }
    pit::BlockVector first = r.ctx->zero_vector();
    if (first_residual_out) opt.first_residual_out = &first;
    pit::SolveResult res = which == 0 ? pit::pitsbicg_solve(*r.ctx, cfg, exec, opt)
                                      : pit::parareal_solve(*r.ctx, cfg, exec, opt);
    flat(r, res.solution, lambda_out);
    if (first_residual_out) flat(r, first, first_residual_out);
    copy_history(res.history, rec_k, rec_res, rec_fine, rec_coarse, max_rec, nrec, restarts,
                 converged);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pitref_pitsbicg(void* p, double tol, double eps0, int max_iter, int zero_guess, int workers,
                    const double* lambda_init, double* lambda_out, double* first_residual_out,
                    int* rec_k, double* rec_res, long* rec_fine, long* rec_coarse, int max_rec,
                    int* nrec, int* restarts, int* converged) {
  return run_solver(0, p, tol, eps0, max_iter, zero_guess, workers, lambda_init, lambda_out,
                    first_residual_out, rec_k, rec_res, rec_fine, rec_coarse, max_rec, nrec,
                    restarts, converged);
}

int pitref_parareal(void* p, double tol, double eps0, int max_iter, int zero_guess, int workers,
                    const double* lambda_init, double* lambda_out, double* first_residual_out,
                    int* rec_k, double* rec_res, long* rec_fine, long* rec_coarse, int max_rec,
                    int* nrec, int* restarts, int* converged) {
  return run_solver(1, p, tol, eps0, max_iter, zero_guess, workers, lambda_init, lambda_out,
                    first_residual_out, rec_k, rec_res, rec_fine, rec_coarse, max_rec, nrec,
                    restarts, converged);
}

// Seeded inputs with the generator family of the reference's own tests
// (tests/oracles.cpp:108-122): std::mt19937_64 + libstdc++ distributions,
// drawn in order — the same bits as pit_seeded_* in the product library, so
// the bench's reference arm builds BASELINE inputs without loading it.
void pitref_seeded_normal(unsigned long long seed, long n, double mean, double stddev,
                          double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(mean, stddev);
  for (long i = 0; i < n; ++i) out[i] = dist(rng);
}

void pitref_seeded_uniform(unsigned long long seed, long n, double a, double b, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(a, b);
  for (long i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
