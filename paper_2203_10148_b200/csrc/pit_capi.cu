// pit_capi.cu — the C ABI (include/pit_b200.h): device context, the block
// operators, and the device-resident PiTSBiCG / parareal drivers.
//
// The solver drivers restate the reference's control flow op for op
// (pitsbicg_solve, src/solvers.cpp:116-220; parareal_solve, 73-114): the same
// branches, restart rules, history rows and cost counters.  All block
// vectors stay in HBM; per iteration only the per-block reduction partials
// (N doubles per phase) come back to the host, where they are summed in slab
// order exactly as block_inner_product does (block_system.cpp:76-87).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "coeffs.h"
#include "pit_b200.h"
#include "pit_comm.h"
#include "pit_kernels.cuh"
#include "pit_kernels2d.cuh"

using namespace pitb;

namespace {

thread_local std::string g_err;
thread_local int g_err_slab = -1;
// InnerSolveError payload of the last failure (include/pit/errors.hpp:15-21)
thread_local bool g_err_detail = false;
thread_local double g_err_relres = 0.0;
thread_local int64_t g_err_iters = 0;

int set_err(int code, const std::string& msg, int slab = -1) {
  g_err = msg;
  g_err_slab = slab;
  g_err_detail = false;
  return code;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return set_err(PIT_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                                       " at " #expr);                                        \
  } while (0)

#define PIT_TRY(expr)      \
  do {                     \
    int rc_ = (expr);      \
    if (rc_) return rc_;   \
  } while (0)

// Binds the context's device for the duration of an entry point and restores
// the caller's current device on exit (a process may drive several contexts
// on different GPUs, and the caller — e.g. torch — may switch devices
// between calls).  dev < 0: no-op.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (dev < 0) return;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) {
      cudaGetLastError();
      cur = -1;
    }
    if (cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};
#define PIT_DEVICE_SCOPE(ctx) DeviceScope device_scope_((ctx) ? (ctx)->desc.device : -1)

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct Role {
  pit_step_coeffs c{};
  StepParams P{};
  double* d_zc = nullptr;
  double* d_pos = nullptr;  // [3*T]: ppos, qpos, zt
  double* d_ds = nullptr;
  double* d_tab = nullptr;  // PIT_SOURCE_TABLE: [N*steps][M] fl(dt*f)
  int mpt = 0, nsub = 0, nseg = 0, warps = 0;
};

}  // namespace

struct pit_context {
  pit_problem_desc desc{};
  int M = 0, N = 0;
  double h = 0, weight = 0;
  bool has_source = false;
  // 2D (config 5): m points per axis, M = m*m
  int dim = 1, m = 0;
  pit_step_coeffs_2d c2{};
  Layout2D lay2{};
  long long* d_cg_iters = nullptr;
  Role role[2];
  // 2D backward Euler (K6): per role I + dt*A stencil and Jacobi inverse
  bool be2 = false;
  Be2Params bp[2]{};
  double* d_be2[2] = {};  // [6][M]: coef[5][M], minv[M]
  double* d_shape = nullptr;
  double* d_y0 = nullptr;
  std::vector<double> y0;
  DevStatus* d_status = nullptr;
  DevStatus* h_status = nullptr;  // pinned mirror
  // slab-sharded multi-GPU (pit_context_attach_comm): owned blocks, the halo
  // / chain block, the partials all-gather buffers, a high-priority stream
  // for the halo exchange and the boundary slab
  pit_comm* comm = nullptr;
  int shard_first = 0, shard_count = 0;
  double* d_halo = nullptr;
  double* d_gather = nullptr;
  double* h_gather = nullptr;  // pinned
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_comm[2] = {};
  // apply_GF with K2 overlapped on K1 (single GPU): per-block ready flags
  // (epoch-tagged, never reset), the sweep's stream, timing events
  int* d_ready = nullptr;
  int ready_epoch = 0;
  cudaStream_t gf_stream = nullptr;
  cudaEvent_t ev_gf[5] = {};
  int gf_overlap = -1;  // -1 untested, 0 off, 1 on
  // device-resident solver loop (pitsbicg_device_loop): the scalars, the
  // skip flag every launch of an iteration carries, timing events
  SolverScalars* d_sc = nullptr;
  SolverScalars* h_sc = nullptr;  // pinned
  const int* skip = nullptr;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<size_t, int>> ev_spans;  // (first event index, role)
  unsigned long long busy_mark = 0;  // busy_ns already charged to RunStats
  // one BiCGStab iteration of the device loop as a CUDA graph (launch-bound
  // solves): the instantiated graph, the buffers / tolerances it was captured
  // with, timing events around its launches; -1 untested, 0 off, 1 on
  cudaGraphExec_t it_exec = nullptr;
  std::vector<unsigned long long> it_key;
  cudaEvent_t ev_it[2] = {};
  int graph_mode = -1;
  // SolveOptions::iterate_observer (solvers.hpp:54): called after every
  // history row with the iterate the row describes (host copy)
  pit_iterate_observer observer = nullptr;
  void* observer_user = nullptr;
  double* h_observed = nullptr;  // pinned N*M, allocated when an observer is set
  double* h_partials = nullptr;  // pinned, 3*N
  double* d_partials = nullptr;  // 3*N
  cudaStream_t stream = nullptr;
  // solver work buffers (the rank's blocks each), allocated on first solve
  double* buf[10] = {};
  size_t buf_n = 0;
  int sms = 148;
  // K1 piece scheduling (SlabArgs::state): 0 = from occupancy, 1 = off, n = forced
  int pieces = 0;
  double* d_state = nullptr;
  size_t state_n = 0;
  int* d_sched = nullptr;
  size_t sched_n = 0;
  long long* d_trace = nullptr;  // PIT_PHASE_TIMING builds: K1 unit trace
  // host-entry scratch (see to_device)
  double* scratch[3] = {};
  size_t scratch_n[3] = {};
  bool scratch_busy[3] = {};
  // SolveOptions::reference: per-row error_vs_reference (Recorder)
  double* d_ref = nullptr;
  double* d_ref_diff = nullptr;
  // host-buffer pipelining of pit_apply_F (see pipelined_apply_F)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_pipe = nullptr;
  unsigned* d_sync = nullptr;  // [1 + kPipeMaxChunks]: in_ready, out_done[]
  int pipe = -1;               // -1 untested, 0 unavailable/off, 1 ready
  int pipe_chunks = 0;         // PIT_E2E_CHUNKS (0 = auto)
  size_t nm() const { return (size_t)N * (size_t)M; }
};

namespace {

int validate_desc(const pit_problem_desc* d) {
  if (!d) return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: null description");
  if (d->dimension != 1 && d->dimension != 2)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "SpatialGrid: dimension must be 1 or 2");
  if (d->dimension == 1 && d->fine_scheme != PIT_SCHEME_BACKWARD_EULER)
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_create: 1D fine propagators are backward Euler");
  if (d->dimension == 1 && d->stencil) {
    // a general tridiagonal operator: the reference's inner solvers (K6 on a
    // one-row grid)
    if (!be2d_supported(d->interior, 1))
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: general 1D operators need M <= 10240");
    if (d->source_kind != PIT_SOURCE_NONE && d->source_kind != PIT_SOURCE_TABLE)
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: a general 1D operator takes its source as tables "
                     "(PIT_SOURCE_TABLE)");
    if (d->coarse_tolerance < 0.0 || d->fine_tolerance < 0.0)
      return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: negative inner tolerance");
  }
  if (d->dimension == 2 && d->fine_scheme == PIT_SCHEME_BACKWARD_EULER) {
    if (!be2d_supported(d->interior, d->interior))
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: implicit 2D propagators need m <= 101 points per axis");
    if (!d->stencil && d->band_lo != d->band_up)
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: 2D band operators are isotropic (band_lo == band_up)");
    if (d->source_kind != PIT_SOURCE_NONE && d->source_kind != PIT_SOURCE_TABLE)
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: 2D sources are given as tables (PIT_SOURCE_TABLE)");
    if (d->coarse_tolerance < 0.0 || d->fine_tolerance < 0.0)
      return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: negative inner tolerance");
  } else if (d->dimension == 2) {
    if (d->fine_scheme != PIT_SCHEME_EXPLICIT_EULER)
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: unknown 2D fine scheme");
    if (d->band_lo != d->band_up)
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: 2D operators are the isotropic 5-point stencil "
                     "(band_lo == band_up)");
    if (d->source_kind != PIT_SOURCE_NONE)
      return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: no sources in 2D");
    if (d->interior > 256)
      return set_err(PIT_ERR_INVALID_ARGUMENT,
                     "pit_context_create: 2D grids up to 256 interior points per axis");
    if (d->coarse_tolerance < 0.0)
      return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: negative coarse tolerance");
  }
  if (d->interior < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "SpatialGrid: points_per_axis must be >= 3");
  if (!(d->grid_hi > d->grid_lo)) return set_err(PIT_ERR_INVALID_ARGUMENT, "SpatialGrid: empty extent");
  if (!(d->total_time > 0.0))
    return set_err(PIT_ERR_INVALID_ARGUMENT, "TimeSlabPartition: T must be positive");
  if (d->slab_count < 2)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "TimeSlabPartition: need at least 2 slabs");
  if (d->fine_steps < 1 || d->coarse_steps < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "Propagator: steps_per_slab must be >= 1");
  if (!d->initial_value) return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: null initial value");
  if (d->source_kind == PIT_SOURCE_TABLE && (!d->source_table_fine || !d->source_table_coarse))
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_create: a table source needs the fine and the coarse table");
  if (d->source_kind != PIT_SOURCE_NONE && d->source_kind != PIT_SOURCE_SEPARABLE &&
      d->source_kind != PIT_SOURCE_TABLE)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: unknown source kind");
  if (d->source_kind == PIT_SOURCE_SEPARABLE && !d->source_shape)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: separable source needs a shape");
  return PIT_OK;
}

double grid_spacing(const pit_problem_desc* d) {
  // SpatialGrid: spacing = (hi - lo) / (points_per_axis - 1), points = M + 2 (grid.cpp:19)
  return (d->grid_hi - d->grid_lo) / static_cast<double>(d->interior + 2 - 1);
}

// Scaled explicit form (pit_step_coeffs_2d): an = 2^e exactly and
// kappa = ac/an exact; rescale period R keeps |z| <= |y| 2^768.
// oracle/pit_oracle2d.c orc2_coefficients restates this.
void explicit_scaling(double ac, double an, int steps, int32_t* scaled, int32_t* R, double* kappa,
                      double* anR, double* anLast) {
  int e = 0;
  const double mant = std::frexp(an, &e);  // an = mant * 2^e
  *scaled = 0;
  *R = 1;
  *kappa = 0.0;
  *anR = 1.0;
  *anLast = 1.0;
  if (!(an > 0.0) || mant != 0.5 || e - 1 >= 0) return;
  const double k = ac / an;
  if (!std::isfinite(k) || k * an != ac) return;
  const int sh = 1 - e;  // an = 2^-sh, sh >= 1
  int r = 768 / sh;
  if (r < 1) return;
  if (r > steps) r = steps;
  const int j = steps - r * ((steps - 1) / r);  // factors carried after the last fold
  *scaled = 1;
  *R = r;
  *kappa = k;
  *anR = std::ldexp(1.0, -sh * r);
  *anLast = std::ldexp(1.0, -sh * j);
}

// 2D coefficients (pit_step_coeffs_2d); K4 layout and K5 decomposition.
int coeffs_2d(const pit_problem_desc* d, pit_step_coeffs_2d* c) {
  const int m = d->interior;
  const double slab = d->total_time / d->slab_count;
  const double dtf = slab / d->fine_steps;  // Propagator::internal_dt
  const double dtc = slab / d->coarse_steps;
  const double off = d->band_lo, diag = d->band_diag;
  *c = pit_step_coeffs_2d{};
  c->m = m;
  c->fine_steps = d->fine_steps;
  c->coarse_steps = d->coarse_steps;
  c->an = (double)(-(long double)dtf * (long double)off);
  c->ac = (double)(1.0L - (long double)dtf * (long double)diag);
  explicit_scaling(c->ac, c->an, d->fine_steps, &c->scaled, &c->R, &c->kappa, &c->anR,
                   &c->anLast);
  c->O = off * dtc;         // ImplicitStepSolver: val *= dt      (pde.cpp:107)
  c->D = diag * dtc + 1.0;  //                     diagonal += 1   (pde.cpp:108)
  c->minv = c->D != 0.0 ? 1.0 / c->D : 1.0;  // jacobi_inverse_diagonal (sparse.cpp:43-50)
  c->rel_tol = d->coarse_tolerance > 0.0 ? d->coarse_tolerance : 1e-12;
  c->cap = d->coarse_max_iterations > 0 ? d->coarse_max_iterations : 10LL * m * m;
  c->rows = kCgRowsMax;
  c->cluster = (m + c->rows - 1) / c->rows;
  c->rows = (m + c->cluster - 1) / c->cluster;
  c->threads = 32 * ((m + 31) / 32);
  Layout2D L{d->tile_rows, d->tile_cols, d->tile_cluster, d->tile_warps};
  if (L.tr == 0) L = auto_layout_2d(m);
  if (L.tr == 0 || !layout2d_supported(L.tr, L.tc, L.cl, L.warps) || 32 * L.tc < m ||
      L.cl * L.warps * L.tr < m)
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_create: no compiled 2D tile layout covers m=" + std::to_string(m));
  c->tile_rows = L.tr;
  c->tile_cols = L.tc;
  c->tile_cluster = L.cl;
  c->tile_warps = L.warps;
  return PIT_OK;
}

Ex2Params ex2_params(const pit_context* ctx) {
  Ex2Params P{};
  P.m = ctx->m;
  P.steps = ctx->c2.fine_steps;
  P.ac = ctx->c2.ac;
  P.an = ctx->c2.an;
#ifdef PIT_PHASE_TIMING
  P.timing = ctx->role[PIT_FINE].P.timing;
#endif
  P.scaled = ctx->c2.scaled;
  P.R = ctx->c2.R;
  P.kappa = ctx->c2.kappa;
  P.anR = ctx->c2.anR;
  P.anLast = ctx->c2.anLast;
  if (const char* e = std::getenv("PIT_UNSCALED")) {
    if (std::atoi(e)) P.scaled = 0;  // A/B knob: the same bits either way
  }
  return P;
}

Cg2Params cg2_params(const pit_context* ctx) {
  Cg2Params P{};
  P.m = ctx->m;
  P.steps = ctx->c2.coarse_steps;
  P.rows = ctx->c2.rows;
  P.cluster = ctx->c2.cluster;
  P.D = ctx->c2.D;
  P.O = ctx->c2.O;
  P.minv = ctx->c2.minv;
  P.rel_tol = ctx->c2.rel_tol;
  P.cap = ctx->c2.cap;
#ifdef PIT_PHASE_TIMING
  P.timing = ctx->role[PIT_COARSE].P.timing;
#endif
  return P;
}

int role_coeffs(const pit_problem_desc* d, int role, pit_step_coeffs* c, std::vector<double>* zc,
                Layout* lay, std::vector<double>* ppos, std::vector<double>* qpos,
                std::vector<double>* zt) {
  const int M = d->interior;
  const int steps = role == PIT_FINE ? d->fine_steps : d->coarse_steps;
  // TimeSlabPartition::slab_length() = T/N; Propagator::internal_dt() = slab/steps
  const double dt = (d->total_time / d->slab_count) / steps;
  int mpt = role == PIT_FINE ? d->fine_mpt : d->coarse_mpt;
  int nsub = role == PIT_FINE ? d->fine_nsub : d->coarse_nsub;
  int nseg = role == PIT_FINE ? d->fine_nseg : d->coarse_nseg;
  int warps = role == PIT_FINE ? d->fine_warps : d->coarse_warps;
  if (mpt == 0 || warps == 0) {
    Layout l = auto_layout(M, role);
    mpt = l.mpt;
    nsub = l.nsub;
    nseg = l.nseg;
    warps = l.warps;
  }
  if (nseg == 0) nseg = 1;
  if (nsub == 0) nsub = 1;
  if (mpt == 0 || !layout_supported(mpt, nsub, nseg, warps) || 32 * mpt * warps < M)
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_create: no compiled slab layout covers M=" + std::to_string(M));
  lay->mpt = mpt;
  lay->nsub = nsub;
  lay->nseg = nseg;
  lay->warps = warps;
  if (build_step_coeffs(M, mpt, nsub, nseg, warps, steps, d->band_lo, d->band_diag, d->band_up,
                        dt, c, zc, ppos, qpos, zt))
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_create: step matrix I + dt*A is not factorizable with constant "
                   "factors (needs delta^2 > 4*lam*mu)");
  return PIT_OK;
}

void fill_params(const pit_step_coeffs& c, StepParams* P) {
  P->nl = c.nl;
  P->nu = c.nu;
  P->inv = c.inv;
  P->gneg = c.gneg;
  P->invR = c.invR;
  P->invLast = c.invLast;
  const int sub = c.mpt / (c.nsub * c.nseg);
  P->pS = c.pS;
  P->qS = c.qS;
  P->Pseg = c.Pseg;
  P->Qseg = c.Qseg;
  P->narrow = c.narrow;
  for (int u = 0; u < 8; ++u) P->pw[u] = u < c.nsub ? c.pw[u] : 0.0;
  for (int j = 0; j < 32; ++j) {
    P->nlpow[j] = j < sub ? c.nlpow[j] : 0.0;
    P->plane[j] = c.plane[j];
    P->qlane[j] = c.qlane[j];
  }
  for (int s = 0; s < 5; ++s) {
    P->pp[s] = c.pp[s];
    P->qq[s] = c.qq[s];
  }
  P->p32 = c.p32;
  P->q32 = c.q32;
  P->M = c.M;
  P->steps = c.steps;
  P->R = c.R;
  P->K0 = c.K0;
  P->scan_f = c.scan_f;
  P->scan_b = c.scan_b;
}

// The failure (if any) recorded in the host mirror of DevStatus, as the
// reference's exception; the copy and the sync are the caller's.
int eval_status(pit_context* ctx, bool fine_batch) {
  const int bad = fine_batch ? ctx->h_status->slab : ctx->h_status->sweep_slab;
  if (bad != INT_MAX) {
    const double relres = ctx->h_status->fail[0], iters = ctx->h_status->fail[1];
    const int kind = (int)ctx->h_status->fail[2];
    // reset the failure fields (not busy_ns)
    DevStatus* h = ctx->h_status;
    h->slab = INT_MAX;
    h->sweep_slab = INT_MAX;
    h->fail[0] = h->fail[1] = 0.0;
    h->fail[2] = -1.0;
    CUDA_TRY(cudaMemcpyAsync(ctx->d_status, ctx->h_status, offsetof(DevStatus, busy_ns),
                             cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (fine_batch) {
      const std::string what = ctx->be2
                                   ? "implicit step solve did not converge or produced non-finite "
                                     "values"
                                   : "implicit step produced non-finite values";
      return set_err(PIT_ERR_SLAB, "slab " + std::to_string(bad) + ": " + what, bad);
    }
    // InnerSolveError with the reference's message and payload
    // (src/pde.cpp:119-128)
    std::string what;
    if (kind == kFailNotConverged)
      what = "implicit step solve did not converge (relative residual " + std::to_string(relres) +
             " after " + std::to_string((long long)iters) + " iterations)";
    else
      what = "implicit step produced non-finite values";
    const int rc = set_err(PIT_ERR_INNER_SOLVE, what, bad);
    g_err_detail = kind == kFailNotConverged || kind == kFailNonFinite;
    g_err_relres = relres;
    g_err_iters = (int64_t)iters;
    return rc;
  }
  return PIT_OK;
}

int check_status(pit_context* ctx, bool fine_batch) {
  CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return eval_status(ctx, fine_batch);
}

void bind_status(pit_context* ctx, SlabArgs* A) {
  A->status = &ctx->d_status->slab;
  A->busy_ns = &ctx->d_status->busy_ns;
}
void bind_status(pit_context* ctx, SweepArgs* A) {
  A->status = &ctx->d_status->sweep_slab;
  A->fail_info = ctx->d_status->fail;
}

int attach_pieces(pit_context* ctx, SlabArgs* A, int ctas);
// Fine propagation WITH source of a batch of slabs (assemble_rhs): K1's source
// path, or K6 with the source table.
int launch_fine_source(pit_context* ctx, SlabArgs& A, int ctas, cudaStream_t st) {
  if (ctx->be2) {
    CUDA_TRY(launch_be2d_batch(ctx->bp[PIT_FINE], A, ctas, st, true));
    return PIT_OK;
  }
  Role& R = ctx->role[PIT_FINE];
  PIT_TRY(attach_pieces(ctx, &A, ctas));
  CUDA_TRY(launch_slab(R.mpt, R.nsub, R.nseg, R.warps, true, R.P, A, ctas, st));
  return PIT_OK;
}

// State and scheduler buffers for K1 piece scheduling (grow-only; the
// launcher decides whether the batch is cut into pieces at all).
int attach_pieces(pit_context* ctx, SlabArgs* A, int ctas) {
  if (ctx->pieces == 1 || ctas <= 0) return PIT_OK;
  const Role& R = ctx->role[PIT_FINE];  // K1 runs the fine propagator
  const size_t padded = (size_t)R.mpt * 32 * R.warps;  // state in register order
  const size_t ns = (size_t)ctas * padded, nq = 2 + (size_t)(kMaxPieces - 1) * ctas;
  if (ctx->state_n < ns) {
    cudaFree(ctx->d_state);
    ctx->d_state = nullptr;
    ctx->state_n = 0;
    CUDA_TRY(cudaMalloc(&ctx->d_state, ns * sizeof(double)));
    ctx->state_n = ns;
  }
  if (ctx->sched_n < nq) {
    cudaFree(ctx->d_sched);
    ctx->d_sched = nullptr;
    ctx->sched_n = 0;
    CUDA_TRY(cudaMalloc(&ctx->d_sched, nq * sizeof(int)));
    ctx->sched_n = nq;
  }
  A->state = ctx->d_state;
  A->sched = ctx->d_sched;
  A->pieces = ctx->pieces;
  return PIT_OK;
}

// Fine batch over output blocks [first, first+count) (global indices).
int run_slab_batch(pit_context* ctx, int mode, const double* L, const double* halo,
                   const double* rhs, double* out, int first, int count, cudaStream_t st,
                   const unsigned* in_ready = nullptr, unsigned* out_done = nullptr,
                   int chunk_blocks = 0, int* ready = nullptr, int epoch = 0,
                   int reserve_sms = 0, double* host_out = nullptr) {
  Role& R = ctx->role[PIT_FINE];
  SlabArgs A{};
  A.host_out = host_out;
  A.ready = ready;
  A.epoch = epoch;
  A.reserve_sms = reserve_sms;
  A.skip = ctx->skip;
  A.mode = mode;
  A.in_ready = in_ready;
  A.out_done = out_done;
  A.chunk_blocks = chunk_blocks;
  A.block_shift = first == 0 ? 1 : 0;
  bind_status(ctx, &A);
  const size_t M = ctx->M;
  int ctas;
  if (first == 0) {
    ctas = count - 1;
    A.in = L;
    A.in_shift = 0;
    A.Lsub = L + M;
    A.rhs = rhs ? rhs + M : nullptr;
    A.out = out + M;
    A.slab0 = 0;
    A.L0 = L;
    A.rhs0 = rhs;
    A.out0 = out;
    if (ctas == 0) {  // single block: block 0 only
      if (mode == kApplyF)
        CUDA_TRY(cudaMemcpyAsync(out, L, M * sizeof(double), cudaMemcpyDeviceToDevice, st));
      else
        return set_err(PIT_ERR_INVALID_ARGUMENT, "residual over a single block is not supported");
      return PIT_OK;
    }
  } else {
    if (!halo) return set_err(PIT_ERR_INVALID_ARGUMENT, "apply_F: slab range needs the halo block");
    ctas = count;
    A.in = L;
    A.halo = halo;
    A.in_shift = -1;
    A.Lsub = L;
    A.rhs = rhs;
    A.out = out;
    A.slab0 = first - 1;
  }
  if (ctx->be2) {
    CUDA_TRY(launch_be2d_batch(ctx->bp[PIT_FINE], A, ctas, st));
    return PIT_OK;
  }
  if (ctx->dim == 2) {
    CUDA_TRY(launch_explicit2d(ctx->lay2, ex2_params(ctx), A, ctas, st));
    return PIT_OK;
  }
  PIT_TRY(attach_pieces(ctx, &A, ctas));
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
  if (!ctx->d_trace) CUDA_TRY(cudaMalloc(&ctx->d_trace, sizeof(long long) * 8 * kMaxPieces * (size_t)ctx->N));
  CUDA_TRY(cudaMemsetAsync(ctx->d_trace, 0, sizeof(long long) * 8 * kMaxPieces * (size_t)ctx->N, st));
  A.trace = ctx->d_trace;
#endif
  CUDA_TRY(launch_slab(R.mpt, R.nsub, R.nseg, R.warps, false, R.P, A, ctas, st));
  return PIT_OK;
}

// One sequential sweep launch (SweepArgs semantics) for either dimension.
int launch_sweep_any(pit_context* ctx, int role, bool src, const SweepArgs& A, cudaStream_t st) {
  if (ctx->dim == 1 && !ctx->be2) {
    Role& R = ctx->role[role];
    CUDA_TRY(launch_sweep(R.mpt, R.nsub, R.nseg, R.warps, src, R.P, A, st));
    return PIT_OK;
  }
  if (ctx->be2) {
    CUDA_TRY(launch_be2d_sweep(ctx->bp[role], A, st, src));
    return PIT_OK;
  }
  if (role == PIT_COARSE) {
    CUDA_TRY(launch_cg_sweep2d(cg2_params(ctx), A, ctx->d_cg_iters, st));
    return PIT_OK;
  }
  // 2D fine sweep (sequential_fine_solve, Propagator::propagate): one K4
  // cluster launch per slab, chained through W
  if (A.V) return set_err(PIT_ERR_INVALID_ARGUMENT, "internal: fine sweep with an added vector");
  const size_t M = ctx->M;
  for (int s = 0; s < A.count; ++s) {
    SlabArgs S{};
    S.in = s == 0 ? A.start : A.W + (size_t)(s - 1) * M;
    S.in_shift = 0;
    S.out = A.W + (size_t)s * M;
    S.mode = kPropagate;
    S.slab0 = A.slab0 + s;
    S.status = A.status;
    S.skip = A.skip;
    CUDA_TRY(launch_explicit2d(ctx->lay2, ex2_params(ctx), S, 1, st));
  }
  return PIT_OK;
}

// Sequential sweep over output blocks [first, first+count): W_first-1 = W_prev.
int run_sweep(pit_context* ctx, int role, bool with_source, const double* V, const double* W_prev,
              double* W, int first, int count, bool add_v, cudaStream_t st) {
  const size_t M = ctx->M;
  SweepArgs A{};
  bind_status(ctx, &A);
  A.skip = ctx->skip;
  if (first == 0) {
    // block 0: W_0 = V_0 (G^-1) — the caller seeds block 0 otherwise
    if (add_v && V != W)
      CUDA_TRY(cudaMemcpyAsync(W, V, M * sizeof(double), cudaMemcpyDeviceToDevice, st));
    A.start = W;
    A.V = add_v ? V + M : nullptr;
    A.W = W + M;
    A.count = count - 1;
    A.slab0 = 0;
  } else {
    if (!W_prev) return set_err(PIT_ERR_INVALID_ARGUMENT, "coarse sweep: slab range needs W_prev");
    A.start = W_prev;
    A.V = add_v ? V : nullptr;
    A.W = W;
    A.count = count;
    A.slab0 = first - 1;
  }
  const bool src = with_source && ctx->has_source;
  return launch_sweep_any(ctx, role, src, A, st);
}

// Sum per-block partials (np per block, component k) in slab order.
double sum_partials(const double* h, int blocks, int np, int k) {
  double s = 0.0;
  for (int n = 0; n < blocks; ++n) s += h[(size_t)n * np + k];
  return s;
}
double max_sqrt_partials(const double* h, int blocks, int np, int k) {
  double w = 0.0;
  for (int n = 0; n < blocks; ++n) w = std::max(w, std::sqrt(h[(size_t)n * np + k]));
  return w;
}

int fetch_partials(pit_context* ctx, int count) {
  CUDA_TRY(cudaMemcpyAsync(ctx->h_partials, ctx->d_partials, sizeof(double) * (size_t)count,
                           cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return PIT_OK;
}

int ensure_buffers(pit_context* ctx, size_t n) {
  if (ctx->buf[0] && ctx->buf_n >= n) return PIT_OK;
  for (auto& b : ctx->buf) {
    cudaFree(b);
    b = nullptr;
  }
  ctx->buf_n = 0;
  for (auto& b : ctx->buf) CUDA_TRY(cudaMalloc(&b, n * sizeof(double)));
  ctx->buf_n = n;
  return PIT_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

const char* pit_last_error(void) { return g_err.c_str(); }
int pit_last_error_slab(void) { return g_err_slab; }
const char* pit_version(void) { return "pit_b200 0.1 (sm_100a)"; }

int pit_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int pit_step_coefficients(const pit_problem_desc* desc, int role, pit_step_coeffs* out) {
  PIT_TRY(validate_desc(desc));
  if (desc->dimension != 1) return set_err(PIT_ERR_INVALID_ARGUMENT, "not a 1D description");
  std::vector<double> zc, ppos, qpos, zt;
  Layout lay;
  return role_coeffs(desc, role, out, &zc, &lay, &ppos, &qpos, &zt);
}

int pit_step_correction(const pit_problem_desc* desc, int role, double* zc_out) {
  PIT_TRY(validate_desc(desc));
  std::vector<double> zc, ppos, qpos, zt;
  Layout lay;
  pit_step_coeffs c;
  PIT_TRY(role_coeffs(desc, role, &c, &zc, &lay, &ppos, &qpos, &zt));
  std::memcpy(zc_out, zc.data(), zc.size() * sizeof(double));
  return PIT_OK;
}

int pit_step_positions(const pit_problem_desc* desc, int role, double* ppos_out,
                       double* qpos_out, double* zt_out) {
  PIT_TRY(validate_desc(desc));
  std::vector<double> zc, ppos, qpos, zt;
  Layout lay;
  pit_step_coeffs c;
  PIT_TRY(role_coeffs(desc, role, &c, &zc, &lay, &ppos, &qpos, &zt));
  std::memcpy(ppos_out, ppos.data(), ppos.size() * sizeof(double));
  std::memcpy(qpos_out, qpos.data(), qpos.size() * sizeof(double));
  if (zt_out) std::memcpy(zt_out, zt.data(), zt.size() * sizeof(double));
  return PIT_OK;
}

int pit_context_create(const pit_problem_desc* desc, pit_context** out) {
  if (!out) return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: null output");
  *out = nullptr;
  PIT_TRY(validate_desc(desc));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(PIT_ERR_CUDA, "no CUDA device: the PiT kernels require a B200 (sm_100a)");
  if (desc->device < 0 || desc->device >= ndev)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_context_create: bad device ordinal");
  DeviceScope device_scope_(desc->device);  // the caller's device is restored on return
  {
    int cur = -1;
    CUDA_TRY(cudaGetDevice(&cur));
    if (cur != desc->device) return set_err(PIT_ERR_CUDA, "pit_context_create: cannot bind device");
  }
  auto ctx = new pit_context();
  ctx->desc = *desc;
  ctx->desc.source_shape = nullptr;
  ctx->desc.initial_value = nullptr;
  ctx->dim = desc->dimension;
  ctx->m = desc->interior;
  ctx->M = ctx->dim == 2 ? ctx->m * ctx->m : ctx->m;
  ctx->N = desc->slab_count;
  ctx->shard_count = ctx->N;
  ctx->h = grid_spacing(desc);
  // inner_product weight h^d (grid.cpp:113-114)
  ctx->weight = ctx->dim == 2 ? ctx->h * ctx->h : ctx->h;
  ctx->has_source = desc->source_kind != PIT_SOURCE_NONE;
  ctx->y0.assign(desc->initial_value, desc->initial_value + ctx->M);
  auto fail = [&](int rc) {
    pit_context_destroy(ctx);
    return rc;
  };
  ctx->be2 = (ctx->dim == 2 && desc->fine_scheme == PIT_SCHEME_BACKWARD_EULER) ||
             (ctx->dim == 1 && desc->stencil != nullptr);
  if (ctx->be2) {
    // ImplicitStepSolver (pde.cpp:103-110): every entry times dt, then the
    // diagonal + 1; jacobi_inverse_diagonal (sparse.cpp:43-50)
    const int M = ctx->M;
    std::vector<double> st(5 * (size_t)M, 0.0);
    if (ctx->dim == 1) {
      // [3][M] sub, diagonal, super -> west, centre, east of a one-row grid
      for (int i = 0; i < M; ++i) {
        st[(size_t)M + i] = i > 0 ? desc->stencil[i] : 0.0;
        st[2 * (size_t)M + i] = desc->stencil[(size_t)M + i];
        st[3 * (size_t)M + i] = i < M - 1 ? desc->stencil[2 * (size_t)M + i] : 0.0;
      }
    } else if (desc->stencil) {
      st.assign(desc->stencil, desc->stencil + 5 * (size_t)M);
    } else {
      const int m = ctx->m;
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
          const size_t r = (size_t)j * m + i;
          st[r] = j > 0 ? desc->band_lo : 0.0;
          st[M + r] = i > 0 ? desc->band_lo : 0.0;
          st[2 * (size_t)M + r] = desc->band_diag;
          st[3 * (size_t)M + r] = i < m - 1 ? desc->band_lo : 0.0;
          st[4 * (size_t)M + r] = j < m - 1 ? desc->band_lo : 0.0;
        }
    }
    for (int r = 0; r < 2; ++r) {
      const int steps = r == PIT_FINE ? desc->fine_steps : desc->coarse_steps;
      const double dt = (desc->total_time / desc->slab_count) / steps;
      std::vector<double> h(6 * (size_t)M);
      for (size_t k = 0; k < 5 * (size_t)M; ++k) h[k] = st[k] * dt;
      for (int i = 0; i < M; ++i) {
        double& c = h[2 * (size_t)M + i];
        c = c + 1.0;
        h[5 * (size_t)M + i] = c != 0.0 ? 1.0 / c : 1.0;
      }
      if (cudaMalloc(&ctx->d_be2[r], sizeof(double) * h.size()) != cudaSuccess ||
          cudaMemcpy(ctx->d_be2[r], h.data(), sizeof(double) * h.size(),
                     cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
      Be2Params& P = ctx->bp[r];
      P.m = ctx->m;
      P.my = ctx->dim == 2 ? ctx->m : 1;
      P.M = M;
      P.steps = steps;
      P.coef = ctx->d_be2[r];
      P.minv = ctx->d_be2[r] + 5 * (size_t)M;
      const double tol = r == PIT_FINE ? desc->fine_tolerance : desc->coarse_tolerance;
      const long long cap = r == PIT_FINE ? desc->fine_max_iterations : desc->coarse_max_iterations;
      P.rel_tol = tol > 0.0 ? tol : 1e-12;          // kInnerSolveRelTol (pde.hpp:78)
      P.cap = cap > 0 ? (int)std::min<long long>(cap, INT_MAX) : 10 * M;  // pde.hpp:79
      P.symmetric = desc->nonsymmetric ? 0 : 1;
    }
    if (cudaMalloc(&ctx->d_cg_iters, sizeof(long long)) != cudaSuccess ||
        cudaMemset(ctx->d_cg_iters, 0, sizeof(long long)) != cudaSuccess)
      return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
    ctx->bp[PIT_COARSE].iters = ctx->d_cg_iters;
  } else if (ctx->dim == 2) {
    int rc = coeffs_2d(desc, &ctx->c2);
    if (rc) return fail(rc);
    ctx->lay2 = Layout2D{ctx->c2.tile_rows, ctx->c2.tile_cols, ctx->c2.tile_cluster,
                         ctx->c2.tile_warps};
    if (cudaMalloc(&ctx->d_cg_iters, sizeof(long long)) != cudaSuccess ||
        cudaMemset(ctx->d_cg_iters, 0, sizeof(long long)) != cudaSuccess)
      return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
  }
  for (int r = 0; r < (ctx->dim == 1 && !ctx->be2 ? 2 : 0); ++r) {
    std::vector<double> zc, ppos, qpos, zt;
    Layout lay;
    int rc = role_coeffs(desc, r, &ctx->role[r].c, &zc, &lay, &ppos, &qpos, &zt);
    if (rc) return fail(rc);
    Role& R = ctx->role[r];
    R.mpt = lay.mpt;
    R.nsub = lay.nsub;
    R.nseg = lay.nseg;
    R.warps = lay.warps;
    fill_params(R.c, &R.P);
    if (cudaMalloc(&R.d_zc, sizeof(double) * zc.size()) != cudaSuccess ||
        cudaMemcpy(R.d_zc, zc.data(), sizeof(double) * zc.size(), cudaMemcpyHostToDevice) !=
            cudaSuccess)
      return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
    R.P.zc = R.d_zc;
    std::vector<double> pos(ppos);
    pos.insert(pos.end(), qpos.begin(), qpos.end());
    pos.insert(pos.end(), zt.begin(), zt.end());
    if (cudaMalloc(&R.d_pos, sizeof(double) * pos.size()) != cudaSuccess ||
        cudaMemcpy(R.d_pos, pos.data(), sizeof(double) * pos.size(), cudaMemcpyHostToDevice) !=
            cudaSuccess)
      return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
    R.P.ppos = R.d_pos;
    R.P.qpos = R.d_pos + ppos.size();
    R.P.zt = R.d_pos + 2 * ppos.size();
  }
  if (cudaMalloc(&ctx->d_y0, sizeof(double) * ctx->M) != cudaSuccess ||
      cudaMemcpy(ctx->d_y0, ctx->y0.data(), sizeof(double) * ctx->M, cudaMemcpyHostToDevice) !=
          cudaSuccess)
    return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
  if (desc->source_kind == PIT_SOURCE_TABLE) {
    // general source: fl(dt*f) per step and point, as the reference's
    // rhs.axpy(dt, sample_source(t)) forms it (propagator.cpp:60-62)
    const double slab = desc->total_time / desc->slab_count;
    for (int r = 0; r < 2; ++r) {
      Role& R = ctx->role[r];
      const int steps_r = r == PIT_FINE ? desc->fine_steps : desc->coarse_steps;
      const double dt = slab / steps_r;
      const double* f = r == PIT_FINE ? desc->source_table_fine : desc->source_table_coarse;
      const size_t n = (size_t)ctx->N * steps_r * ctx->M;
      std::vector<double> tab(n);
      for (size_t i = 0; i < n; ++i) tab[i] = dt * f[i];
      if (cudaMalloc(&R.d_tab, sizeof(double) * n) != cudaSuccess ||
          cudaMemcpy(R.d_tab, tab.data(), sizeof(double) * n, cudaMemcpyHostToDevice) !=
              cudaSuccess)
        return fail(set_err(PIT_ERR_CUDA, "pit_context_create: the source table does not fit "
                                          "the device (N*steps*M doubles per propagator)"));
      R.P.tab = R.d_tab;
      if (ctx->be2) ctx->bp[r].tab = R.d_tab;
    }
  } else if (ctx->has_source) {
    if (cudaMalloc(&ctx->d_shape, sizeof(double) * ctx->M) != cudaSuccess ||
        cudaMemcpy(ctx->d_shape, desc->source_shape, sizeof(double) * ctx->M,
                   cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
    const double slab = desc->total_time / desc->slab_count;
    for (int r = 0; r < 2; ++r) {
      Role& R = ctx->role[r];
      const int steps = R.c.steps;
      const double dt = slab / steps;
      // source sampled at step END: t = breakpoint(n) + step*dt (propagator.cpp:56-63)
      std::vector<double> ds((size_t)ctx->N * steps);
      for (int n = 0; n < ctx->N; ++n) {
        const double t0 = n * slab;
        for (int k = 1; k <= steps; ++k) {
          const double t = t0 + k * dt;
          const double sv = desc->source_amp * std::sin(desc->source_omega * t + desc->source_phase);
          ds[(size_t)n * steps + (k - 1)] = dt * sv;
        }
      }
      if (cudaMalloc(&R.d_ds, sizeof(double) * ds.size()) != cudaSuccess ||
          cudaMemcpy(R.d_ds, ds.data(), sizeof(double) * ds.size(), cudaMemcpyHostToDevice) !=
              cudaSuccess)
        return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
      R.P.ds = R.d_ds;
      R.P.shape = ctx->d_shape;
    }
  }
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, desc->device);
#ifdef PIT_PHASE_TIMING
  for (int r = 0; r < 2; ++r) {
    cudaMalloc(&ctx->role[r].P.timing, 64 * sizeof(long long));
    cudaMemset(ctx->role[r].P.timing, 0, 64 * sizeof(long long));
  }
#endif
  if (const char* e = std::getenv("PIT_PIECES")) ctx->pieces = std::max(0, std::atoi(e));
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->d_status, sizeof(DevStatus)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_status, sizeof(DevStatus)) != cudaSuccess ||
      cudaMalloc(&ctx->d_partials, sizeof(double) * 3 * (size_t)ctx->N) != cudaSuccess ||
      cudaMallocHost(&ctx->h_partials, sizeof(double) * 3 * (size_t)ctx->N) != cudaSuccess)
    return fail(set_err(PIT_ERR_CUDA, "pit_context_create: device allocation failed"));
  {
    DevStatus init{};
    init.slab = INT_MAX;  // "no failing slab"
    init.sweep_slab = INT_MAX;
    init.fail[2] = -1.0;
    *ctx->h_status = init;
    if (cudaMemcpy(ctx->d_status, &init, sizeof(DevStatus), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_err(PIT_ERR_CUDA, "pit_context_create: status init failed"));
  }
  *out = ctx;
  return PIT_OK;
}

int pit_context_destroy(pit_context* ctx) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return PIT_OK;
  for (auto& R : ctx->role) {
    cudaFree(R.d_zc);
    cudaFree(R.d_pos);
    cudaFree(R.d_ds);
    cudaFree(R.d_tab);
  }
  cudaFree(ctx->d_shape);
  cudaFree(ctx->d_y0);
  cudaFree(ctx->d_status);
  cudaFree(ctx->d_partials);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->h_observed) cudaFreeHost(ctx->h_observed);
  if (ctx->h_partials) cudaFreeHost(ctx->h_partials);
  for (auto& b : ctx->buf) cudaFree(b);
  for (auto& b : ctx->scratch) cudaFree(b);
  cudaFree(ctx->d_state);
  cudaFree(ctx->d_sched);
  cudaFree(ctx->d_trace);
  cudaFree(ctx->d_cg_iters);
  cudaFree(ctx->d_be2[0]);
  cudaFree(ctx->d_be2[1]);
  cudaFree(ctx->d_sync);
  cudaFree(ctx->d_ref);
  cudaFree(ctx->d_ref_diff);
  cudaFree(ctx->d_halo);
  cudaFree(ctx->d_ready);
  cudaFree(ctx->d_sc);
  if (ctx->h_sc) cudaFreeHost(ctx->h_sc);
  if (ctx->it_exec) cudaGraphExecDestroy(ctx->it_exec);
  for (cudaEvent_t e : ctx->ev_it)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->gf_stream) cudaStreamDestroy(ctx->gf_stream);
  for (auto& e : ctx->ev_gf)
    if (e) cudaEventDestroy(e);
  cudaFree(ctx->d_gather);
  if (ctx->h_gather) cudaFreeHost(ctx->h_gather);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  for (auto& e : ctx->ev_comm)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_pipe) cudaEventDestroy(ctx->ev_pipe);
  if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
  if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PIT_OK;
}

int pit_coarse_iterations(const pit_context* ctx, int64_t* out) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "null argument");
  *out = 0;
  if (ctx->d_cg_iters) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    long long v = 0;
    CUDA_TRY(cudaMemcpy(&v, ctx->d_cg_iters, sizeof(long long), cudaMemcpyDeviceToHost));
    *out = v;
  }
  return PIT_OK;
}

int pit_step_coefficients_2d(const pit_problem_desc* desc, pit_step_coeffs_2d* out) {
  PIT_TRY(validate_desc(desc));
  if (!out) return set_err(PIT_ERR_INVALID_ARGUMENT, "null output");
  if (desc->dimension != 2) return set_err(PIT_ERR_INVALID_ARGUMENT, "not a 2D description");
  return coeffs_2d(desc, out);
}

int pit_context_shape(const pit_context* ctx, int* M, int* N, double* spacing) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (M) *M = ctx->M;
  if (N) *N = ctx->N;
  if (spacing) *spacing = ctx->h;
  return PIT_OK;
}

// ---- device-pointer entry points ----------------------------------------

int pit_apply_F_device(pit_context* ctx, const double* L, const double* halo, double* out,
                       int first, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !L || !out || first < 0 || count < 1 || first + count > ctx->N)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "apply_F: block count does not match the partition");
  return run_slab_batch(ctx, kApplyF, L, halo, nullptr, out, first, count,
                        stream ? (cudaStream_t)stream : ctx->stream);
}

int pit_residual_device(pit_context* ctx, const double* lambda, const double* halo,
                        const double* rhs, double* out, int first, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !lambda || !rhs || !out || first < 0 || count < 1 || first + count > ctx->N)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "residual: block count does not match the partition");
  return run_slab_batch(ctx, kResidual, lambda, halo, rhs, out, first, count,
                        stream ? (cudaStream_t)stream : ctx->stream);
}

int pit_coarse_sweep_device(pit_context* ctx, const double* V, const double* W_prev, double* W,
                            int first, int count, int with_source, int add_v, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !W || first < 0 || count < 1 || first + count > ctx->N || (add_v && !V))
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "apply_G_inverse: block count does not match the partition");
  return run_sweep(ctx, PIT_COARSE, with_source != 0, V, W_prev, W, first, count, add_v != 0,
                   stream ? (cudaStream_t)stream : ctx->stream);
}

int pit_block_partials_device(pit_context* ctx, const double* a, const double* b, double* partials,
                              int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !a || !b || !partials || count < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "block partials: bad arguments");
  const double* A[1] = {a};
  const double* B[1] = {b};
  CUDA_TRY(launch_dots(ctx->M, count, ctx->weight, 1, A, B, partials,
                       stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_block_partials2_device(pit_context* ctx, const double* a0, const double* b0,
                               const double* a1, const double* b1, double* partials, int count,
                               void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !a0 || !b0 || !a1 || !b1 || !partials || count < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "block partials: bad arguments");
  const double* A[2] = {a0, a1};
  const double* B[2] = {b0, b1};
  CUDA_TRY(launch_dots(ctx->M, count, ctx->weight, 2, A, B, partials,
                       stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_update_s_device(pit_context* ctx, double alpha, const double* r, const double* d, double* s,
                        double* partials, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !r || !d || !s || !partials || count < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "update_s: bad arguments");
  CUDA_TRY(launch_update_s(ctx->M, count, ctx->weight, alpha, r, d, s, partials,
                           stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_update_lr_device(pit_context* ctx, double alpha, double omega, const double* p,
                         const double* s, const double* t, const double* rs, double* lam, double* r,
                         double* partials, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !p || !s || !t || !rs || !lam || !r || !partials || count < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "update_lr: bad arguments");
  CUDA_TRY(launch_update_lr(ctx->M, count, ctx->weight, alpha, omega, p, s, t, rs, lam, r,
                            partials, stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_update_p_device(pit_context* ctx, double omega, double beta, const double* d,
                        const double* r, double* p, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !d || !r || !p || count < 1)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "update_p: bad arguments");
  CUDA_TRY(launch_update_p((size_t)count * ctx->M, omega, beta, d, r, p,
                           stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_axpy_device(pit_context* ctx, double a, const double* x, double* y, int count,
                    void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !x || !y || count < 1) return set_err(PIT_ERR_INVALID_ARGUMENT, "axpy: bad arguments");
  CUDA_TRY(launch_axpy((size_t)count * ctx->M, a, x, y, stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_add_device(pit_context* ctx, const double* x, double* y, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !x || !y || count < 1) return set_err(PIT_ERR_INVALID_ARGUMENT, "add: bad arguments");
  CUDA_TRY(launch_add((size_t)count * ctx->M, x, y, stream ? (cudaStream_t)stream : ctx->stream));
  return PIT_OK;
}

int pit_fine_source_device(pit_context* ctx, double* out, int first, int count, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !out || first < 0 || count < 1 || first + count > ctx->N)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "assemble_rhs: block count does not match the partition");
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
  CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)count * ctx->M * sizeof(double), st));
  if (!ctx->has_source) return PIT_OK;
  SlabArgs A{};
  A.mode = kPropagate;
  bind_status(ctx, &A);
  const int skip = first == 0 ? 1 : 0;  // block 0 is y0, set by the caller
  A.out = out + (size_t)skip * ctx->M;
  A.slab0 = first + skip - 1;
  PIT_TRY(launch_fine_source(ctx, A, count - skip, st));
  return PIT_OK;
}

int pit_sync_status(pit_context* ctx, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (stream) CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  int rc = check_status(ctx, true);
  if (!rc) rc = check_status(ctx, false);
  ctx->busy_mark = ctx->h_status->busy_ns;  // device-entry batches carry no RunStats
  return rc;
}

// ---- host-pointer entry points -------------------------------------------

namespace {

// Scratch device vectors for the host-pointer entry points: the context keeps
// up to three N*M buffers (allocated on first use) so repeated calls do not
// pay cudaMalloc/cudaFree.
struct DevVec {
  double* p = nullptr;
};

int to_device(pit_context* ctx, const double* h, size_t n, DevVec* d) {
  int slot = -1;
  for (int i = 0; i < 3; ++i)
    if (!ctx->scratch_busy[i]) {
      slot = i;
      break;
    }
  if (slot < 0) return set_err(PIT_ERR_INVALID_ARGUMENT, "internal: scratch exhausted");
  if (ctx->scratch_n[slot] < n) {
    cudaFree(ctx->scratch[slot]);
    ctx->scratch[slot] = nullptr;
    ctx->scratch_n[slot] = 0;
    CUDA_TRY(cudaMalloc(&ctx->scratch[slot], n * sizeof(double)));
    ctx->scratch_n[slot] = n;
  }
  ctx->scratch_busy[slot] = true;
  d->p = ctx->scratch[slot];
  if (h)
    CUDA_TRY(cudaMemcpyAsync(d->p, h, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  return PIT_OK;
}

// Releases all scratch slots when the entry point returns.
struct ScratchScope {
  pit_context* ctx;
  ~ScratchScope() {
    for (auto& b : ctx->scratch_busy) b = false;
  }
};

int to_host(pit_context* ctx, const double* d, size_t n, double* h) {
  CUDA_TRY(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return PIT_OK;
}

// RunStats bookkeeping (executor.hpp:24-30): fine_busy_ms sums the per-slab
// durations the fine kernels measured (DevStatus::busy_ns, read back by the
// check_status that follows every fine batch), as the executor sums its
// per-task times (executor.cpp:124-128).
void add_fine(pit_context* ctx, pit_run_stats* s, double ms) {
  const unsigned long long now = ctx->h_status->busy_ns;
  const double busy = (double)(now - ctx->busy_mark) * 1e-6;
  ctx->busy_mark = now;
  if (!s) return;
  s->fine_applications += ctx->N - 1;
  s->fine_parallel_ms += ms;
  s->fine_busy_ms += busy;
}
void add_coarse(pit_context* ctx, pit_run_stats* s, double ms) {
  if (!s) return;
  s->coarse_applications += ctx->N - 1;
  s->coarse_sequential_ms += ms;
}

}  // namespace

namespace {

constexpr int kPipeMaxChunks = 64;

PFN_cuStreamWriteValue32_v11070 g_write32 = nullptr;
PFN_cuStreamWaitValue32_v11070 g_wait32 = nullptr;

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Lazily sets up the copy streams, the event and the chunk counters, and
// probes stream memory operations once (pipe = 0 when anything is missing:
// pit_apply_F then copies, computes and copies back in sequence).
int pipe_setup(pit_context* ctx) {
  if (ctx->pipe >= 0) return PIT_OK;
  ctx->pipe = 0;
  if (const char* e = std::getenv("PIT_E2E_CHUNKS")) {
    ctx->pipe_chunks = std::atoi(e);
    if (ctx->pipe_chunks < 0) return PIT_OK;  // < 0: pipelining off
  }
  // Under a kernel profiler or sanitizer (ncu / compute-sanitizer inject
  // through the tree launcher, which exports these) kernels are serialised
  // against the copy streams, so K1 would wait on chunks that cannot land.
  for (const char* v : {"NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                        "CUDA_INJECTION64_PATH"})
    if (std::getenv(v) != nullptr) return PIT_OK;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &p, 12000, cudaEnableDefault, &q) !=
          cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    return PIT_OK;
  g_write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
  if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000, cudaEnableDefault, &q) !=
          cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    return PIT_OK;
  g_wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
  CUDA_TRY(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_pipe, cudaEventDisableTiming));
  CUDA_TRY(cudaMalloc(&ctx->d_sync, sizeof(unsigned) * (1 + kPipeMaxChunks)));
  CUDA_TRY(cudaMemsetAsync(ctx->d_sync, 0, sizeof(unsigned) * (1 + kPipeMaxChunks), ctx->stream));
  // probe: a write and an already-satisfied wait
  if (g_write32((CUstream)ctx->stream, (CUdeviceptr)ctx->d_sync, 1u, 0) != CUDA_SUCCESS ||
      g_wait32((CUstream)ctx->stream, (CUdeviceptr)ctx->d_sync, 1u, CU_STREAM_WAIT_VALUE_GEQ) !=
          CUDA_SUCCESS) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return PIT_OK;
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->pipe = 1;
  return PIT_OK;
}

// pit_apply_F over pinned host buffers with the copies overlapped with K1:
// the input goes up in chunks of whole blocks on the h2d stream (each chunk
// followed by a stream write in_ready = k+1); K1's CTAs wait for the chunk
// holding their blocks; each CTA counts its finished output block into
// out_done[chunk]; the d2h stream waits for a chunk's count and copies it
// back.  Same kernel, same arithmetic: the output is bit-identical to the
// sequential path.
int pipelined_apply_F(pit_context* ctx, const double* L, double* out, double* dL, double* dO) {
  const int N = ctx->N;
  const size_t M = ctx->M;
  int nch = ctx->pipe_chunks > 0 ? ctx->pipe_chunks : 16;
  nch = std::min(std::min(nch, kPipeMaxChunks), N);
  const int cb = (N + nch - 1) / nch;  // blocks per chunk
  nch = (N + cb - 1) / cb;
  auto unblock = [&]() {  // release every waiter (error paths)
    for (int k = 0; k <= nch; ++k)
      g_write32((CUstream)ctx->stream, (CUdeviceptr)(ctx->d_sync + k), 0x7fffffffu, 0);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->h2d);
    cudaStreamSynchronize(ctx->d2h);
  };
  CUDA_TRY(cudaMemsetAsync(ctx->d_sync, 0, sizeof(unsigned) * (1 + nch), ctx->stream));
  CUDA_TRY(cudaEventRecord(ctx->ev_pipe, ctx->stream));
  CUDA_TRY(cudaStreamWaitEvent(ctx->h2d, ctx->ev_pipe, 0));
  CUDA_TRY(cudaStreamWaitEvent(ctx->d2h, ctx->ev_pipe, 0));
  for (int k = 0; k < nch; ++k) {
    const size_t b0 = (size_t)k * cb, nb = std::min((size_t)cb, (size_t)N - b0);
    cudaError_t e = cudaMemcpyAsync(dL + b0 * M, L + b0 * M, nb * M * sizeof(double),
                                    cudaMemcpyHostToDevice, ctx->h2d);
    if (e != cudaSuccess || g_write32((CUstream)ctx->h2d, (CUdeviceptr)ctx->d_sync,
                                      (unsigned)(k + 1), 0) != CUDA_SUCCESS) {
      unblock();
      return set_err(PIT_ERR_CUDA, "apply_F: pipelined host-to-device copy failed");
    }
  }
  // One CTA per slab unless PIT_PIECES forces a cut (measured on c2,
  // tools/e2e_probe.py): CTAs start as their chunk lands and so finish
  // staggered, which lets the D2H copies overlap the kernel's tail; piece
  // scheduling packs the kernel tighter (1.78 vs 2.12 ms) but ends every slab
  // at once and leaves the whole D2H after it (2.81 vs 2.48 ms end to end).
  const int saved_pieces = ctx->pieces;
  if (ctx->pieces == 0) ctx->pieces = 1;
  // The output goes back without a copy engine when the caller's buffer is
  // mapped into the device's address space (cudaHostAlloc / torch pinned
  // memory under unified addressing): each CTA streams its finished block to
  // host memory itself (SlabArgs::host_out), so a block is on its way the
  // moment it is done instead of when its whole chunk is (c2: 2.25 -> 2.21 ms).
  // PIT_E2E_DIRECT=0 keeps the D2H stream.
  double* mapped = nullptr;
  const char* direct = std::getenv("PIT_E2E_DIRECT");
  if (!(direct && std::atoi(direct) == 0) &&
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped), out, 0) != cudaSuccess) {
    cudaGetLastError();
    mapped = nullptr;
  }
  if (mapped) {
    int rc = run_slab_batch(ctx, kApplyF, dL, nullptr, nullptr, dO, 0, N, ctx->stream,
                            ctx->d_sync, nullptr, cb, nullptr, 0, 0, mapped);
    ctx->pieces = saved_pieces;
    if (rc) {
      const std::string msg = g_err;
      unblock();
      return set_err(rc, msg);
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return check_status(ctx, true);
  }
  // K1 is launched before the D2H stream's waits are enqueued: with lazy
  // module loading a first launch may wait for outstanding work, and the
  // waits depend on this very kernel.
  int rc = run_slab_batch(ctx, kApplyF, dL, nullptr, nullptr, dO, 0, N, ctx->stream, ctx->d_sync,
                          ctx->d_sync + 1, cb);
  ctx->pieces = saved_pieces;
  if (rc) {
    const std::string msg = g_err;
    unblock();
    return set_err(rc, msg);
  }
  for (int k = 0; k < nch; ++k) {
    const size_t b0 = (size_t)k * cb, nb = std::min((size_t)cb, (size_t)N - b0);
    if (g_wait32((CUstream)ctx->d2h, (CUdeviceptr)(ctx->d_sync + 1 + k), (unsigned)nb,
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS ||
        cudaMemcpyAsync(out + b0 * M, dO + b0 * M, nb * M * sizeof(double),
                        cudaMemcpyDeviceToHost, ctx->d2h) != cudaSuccess) {
      cudaStreamSynchronize(ctx->stream);  // K1 needs only the H2D side
      cudaStreamSynchronize(ctx->d2h);
      return set_err(PIT_ERR_CUDA, "apply_F: pipelined device-to-host copy failed");
    }
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->d2h));
  return check_status(ctx, true);
}

}  // namespace

int pit_apply_F(pit_context* ctx, const double* L, double* out, pit_run_stats* stats) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !L || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "apply_F: null argument");
  ScratchScope scope_{ctx};
  const auto t0 = Clock::now();
  if (ctx->dim == 1 && !ctx->be2 && ctx->N >= 32 && is_pinned(L) && is_pinned(out)) {
    PIT_TRY(pipe_setup(ctx));
    if (ctx->pipe == 1) {
      DevVec dL, dO;
      PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &dL));
      PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &dO));
      PIT_TRY(pipelined_apply_F(ctx, L, out, dL.p, dO.p));
      add_fine(ctx, stats, ms_since(t0));
      return PIT_OK;
    }
  }
  DevVec dL, dO;
  PIT_TRY(to_device(ctx, L, ctx->nm(), &dL));
  PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &dO));
  PIT_TRY(run_slab_batch(ctx, kApplyF, dL.p, nullptr, nullptr, dO.p, 0, ctx->N, ctx->stream));
  PIT_TRY(check_status(ctx, true));
  PIT_TRY(to_host(ctx, dO.p, ctx->nm(), out));
  add_fine(ctx, stats, ms_since(t0));
  return PIT_OK;
}

int pit_assemble_rhs(pit_context* ctx, double* rhs, pit_run_stats* stats) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !rhs) return set_err(PIT_ERR_INVALID_ARGUMENT, "assemble_rhs: null argument");
  ScratchScope scope_{ctx};
  const auto t0 = Clock::now();
  DevVec d;
  PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &d));
  CUDA_TRY(cudaMemsetAsync(d.p, 0, ctx->nm() * sizeof(double), ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(d.p, ctx->d_y0, ctx->M * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  if (ctx->has_source) {
    SlabArgs A{};
    A.mode = kPropagate;
    A.in = nullptr;
    A.out = d.p + ctx->M;
    A.slab0 = 0;
    bind_status(ctx, &A);
    PIT_TRY(launch_fine_source(ctx, A, ctx->N - 1, ctx->stream));
    PIT_TRY(check_status(ctx, true));
    add_fine(ctx, stats, ms_since(t0));
  }
  return to_host(ctx, d.p, ctx->nm(), rhs);
}

int pit_apply_G_inverse(pit_context* ctx, const double* V, double* out, pit_run_stats* stats) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !V || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "apply_G_inverse: null argument");
  ScratchScope scope_{ctx};
  const auto t0 = Clock::now();
  DevVec d;
  PIT_TRY(to_device(ctx, V, ctx->nm(), &d));
  PIT_TRY(run_sweep(ctx, PIT_COARSE, false, d.p, nullptr, d.p, 0, ctx->N, true, ctx->stream));
  PIT_TRY(check_status(ctx, false));
  PIT_TRY(to_host(ctx, d.p, ctx->nm(), out));
  add_coarse(ctx, stats, ms_since(t0));
  return PIT_OK;
}

namespace {
int initial_guess_dev(pit_context* ctx, int policy, double* d, pit_run_stats* stats) {
  const auto t0 = Clock::now();
  CUDA_TRY(cudaMemsetAsync(d, 0, ctx->nm() * sizeof(double), ctx->stream));
  if (policy == PIT_GUESS_ZERO) return PIT_OK;
  CUDA_TRY(cudaMemcpyAsync(d, ctx->d_y0, ctx->M * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  PIT_TRY(run_sweep(ctx, PIT_COARSE, true, nullptr, nullptr, d, 0, ctx->N, false, ctx->stream));
  PIT_TRY(check_status(ctx, false));
  add_coarse(ctx, stats, ms_since(t0));
  return PIT_OK;
}
int assemble_rhs_dev(pit_context* ctx, double* d, pit_run_stats* stats) {
  const auto t0 = Clock::now();
  CUDA_TRY(cudaMemsetAsync(d, 0, ctx->nm() * sizeof(double), ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(d, ctx->d_y0, ctx->M * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  if (!ctx->has_source) return PIT_OK;
  SlabArgs A{};
  A.mode = kPropagate;
  A.out = d + ctx->M;
  bind_status(ctx, &A);
  PIT_TRY(launch_fine_source(ctx, A, ctx->N - 1, ctx->stream));
  PIT_TRY(check_status(ctx, true));
  add_fine(ctx, stats, ms_since(t0));
  return PIT_OK;
}
}  // namespace

int pit_initial_guess(pit_context* ctx, int policy, double* out, pit_run_stats* stats) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "initial_guess: null argument");
  ScratchScope scope_{ctx};
  DevVec d;
  PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &d));
  PIT_TRY(initial_guess_dev(ctx, policy, d.p, stats));
  return to_host(ctx, d.p, ctx->nm(), out);
}

int pit_preconditioned_residual(pit_context* ctx, const double* lambda, const double* rhs,
                                double* out, pit_run_stats* stats) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !lambda || !rhs || !out)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "preconditioned_residual: null argument");
  ScratchScope scope_{ctx};
  DevVec dl, db, dr;
  PIT_TRY(to_device(ctx, lambda, ctx->nm(), &dl));
  PIT_TRY(to_device(ctx, rhs, ctx->nm(), &db));
  PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &dr));
  auto t0 = Clock::now();
  PIT_TRY(run_slab_batch(ctx, kResidual, dl.p, nullptr, db.p, dr.p, 0, ctx->N, ctx->stream));
  PIT_TRY(check_status(ctx, true));
  add_fine(ctx, stats, ms_since(t0));
  t0 = Clock::now();
  PIT_TRY(run_sweep(ctx, PIT_COARSE, false, dr.p, nullptr, dr.p, 0, ctx->N, true, ctx->stream));
  PIT_TRY(check_status(ctx, false));
  add_coarse(ctx, stats, ms_since(t0));
  return to_host(ctx, dr.p, ctx->nm(), out);
}

int pit_sequential_fine_solve(pit_context* ctx, double* out) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "sequential_fine_solve: null argument");
  ScratchScope scope_{ctx};
  DevVec d;
  PIT_TRY(to_device(ctx, nullptr, ctx->nm(), &d));
  CUDA_TRY(cudaMemsetAsync(d.p, 0, ctx->nm() * sizeof(double), ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(d.p, ctx->d_y0, ctx->M * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  PIT_TRY(run_sweep(ctx, PIT_FINE, true, nullptr, nullptr, d.p, 0, ctx->N, false, ctx->stream));
  PIT_TRY(check_status(ctx, false));
  return to_host(ctx, d.p, ctx->nm(), out);
}

int pit_propagate(pit_context* ctx, int role, int with_source, const double* in, int slab,
                  double* out) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !out || (role != PIT_FINE && role != PIT_COARSE))
    return set_err(PIT_ERR_INVALID_ARGUMENT, "Propagator: bad argument");
  ScratchScope scope_{ctx};
  if (slab < 0 || slab >= ctx->N)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "Propagator: slab_index out of range");
  const size_t M = ctx->M;
  DevVec di, dout;
  PIT_TRY(to_device(ctx, in, M, &di));
  if (!in) CUDA_TRY(cudaMemsetAsync(di.p, 0, M * sizeof(double), ctx->stream));
  PIT_TRY(to_device(ctx, nullptr, M, &dout));
  SweepArgs A{};
  A.start = di.p;
  A.W = dout.p;
  A.count = 1;
  A.slab0 = slab;
  bind_status(ctx, &A);
  const bool src = with_source && ctx->has_source;
  if (!in && !src) {
    // source_contribution with f == 0 is exactly zero (propagator.cpp:78)
    CUDA_TRY(cudaMemsetAsync(dout.p, 0, M * sizeof(double), ctx->stream));
  } else {
    PIT_TRY(launch_sweep_any(ctx, role, src, A, ctx->stream));
    PIT_TRY(check_status(ctx, false));
  }
  return to_host(ctx, dout.p, M, out);
}

int pit_block_inner_product(pit_context* ctx, const double* a, const double* b, double* out) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !a || !b || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "block_inner_product: null");
  ScratchScope scope_{ctx};
  DevVec da, db;
  PIT_TRY(to_device(ctx, a, ctx->nm(), &da));
  PIT_TRY(to_device(ctx, b, ctx->nm(), &db));
  const double* A[1] = {da.p};
  const double* B[1] = {db.p};
  CUDA_TRY(launch_dots(ctx->M, ctx->N, ctx->weight, 1, A, B, ctx->d_partials, ctx->stream));
  PIT_TRY(fetch_partials(ctx, ctx->N));
  *out = sum_partials(ctx->h_partials, ctx->N, 1, 0);
  return PIT_OK;
}

int pit_block_norm_n_inf(pit_context* ctx, const double* a, double* out) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !a || !out) return set_err(PIT_ERR_INVALID_ARGUMENT, "block_norm_n_inf: null");
  ScratchScope scope_{ctx};
  DevVec da;
  PIT_TRY(to_device(ctx, a, ctx->nm(), &da));
  const double* A[1] = {da.p};
  CUDA_TRY(launch_dots(ctx->M, ctx->N, ctx->weight, 1, A, A, ctx->d_partials, ctx->stream));
  PIT_TRY(fetch_partials(ctx, ctx->N));
  *out = max_sqrt_partials(ctx->h_partials, ctx->N, 1, 0);
  return PIT_OK;
}

// ---------------------------------------------------------------------------
// Solvers (device-resident iterates)
// ---------------------------------------------------------------------------

namespace {

// ---------------------------------------------------------------------------
// The solvers on a rank's blocks.  One GPU: the rank owns every block and no
// communicator is attached.  Sharded (pit_context_attach_comm): the rank owns
// blocks [first, first+count) and the halo, the coarse chain and the
// reductions go through the communicator; the arithmetic of
// every block is the same kernel's, and the partials are summed in global
// slab order, so every world size gives the one-GPU bits.
// ---------------------------------------------------------------------------

// fine.source_contribution of blocks [first, first+count) (block 0, y0, is
// the caller's): the K1 source propagation from the zero field
int fine_source(pit_context* ctx, double* out, int first, int count, cudaStream_t st) {
  const int skip = first == 0 ? 1 : 0;
  if (count - skip <= 0) return PIT_OK;
  SlabArgs A{};
  A.mode = kPropagate;
  bind_status(ctx, &A);
  A.out = out + (size_t)skip * ctx->M;
  A.slab0 = first + skip - 1;
  PIT_TRY(launch_fine_source(ctx, A, count - skip, st));
  return PIT_OK;
}

struct Run {
  pit_context* ctx;
  pit_comm* comm;  // nullptr: one GPU
  int first, count;
  cudaStream_t st;
  size_t nl() const { return (size_t)count * ctx->M; }
  bool has_prev() const { return comm && comm->rank > 0; }
  bool has_next() const { return comm && comm->rank + 1 < comm->world; }
};

Run make_run(pit_context* ctx, bool sharded) {
  if (sharded && ctx->comm) return Run{ctx, ctx->comm, ctx->shard_first, ctx->shard_count, ctx->stream};
  return Run{ctx, nullptr, 0, ctx->N, ctx->stream};
}

int comm_err(int rc, const char* what) {
  return set_err(rc ? rc : PIT_ERR_CUDA, what ? what : "communication failed");
}
#define COMM_TRY(expr)                       \
  do {                                       \
    const char* what_ = nullptr;             \
    int rc_ = (expr);                        \
    if (rc_) return comm_err(rc_, what_);    \
  } while (0)

// Status checks: one GPU after every phase (as the reference throws at the
// failing call); sharded at the next reduction, where every rank learns the
// lowest failing slab of all ranks and raises the same error (a rank that
// stopped early would leave its peers waiting in the chain).
int run_check(Run& R, bool fine_batch) {
  if (R.comm) return PIT_OK;
  return check_status(R.ctx, fine_batch);
}

// fine batch (apply_F or the preconditioned residual's rhs - F lam) over the
// rank's blocks; sharded: the blocks after the first start at once, the
// first waits for the halo block first-1 from rank-1 (on the comm stream)
int run_fine(Run& R, int mode, const double* x, const double* rhs, double* out,
             pit_run_stats* stats) {
  pit_context* ctx = R.ctx;
  const size_t M = ctx->M;
  const auto t0 = Clock::now();
  if (!R.has_prev() && !R.has_next()) {
    PIT_TRY(run_slab_batch(ctx, mode, x, nullptr, rhs, out, 0, R.count, R.st));
  } else {
    cudaStream_t cs = ctx->comm_stream;
    CUDA_TRY(cudaEventRecord(ctx->ev_comm[0], R.st));  // x ready
    if (R.first == 0) {
      PIT_TRY(run_slab_batch(ctx, mode, x, nullptr, rhs, out, 0, R.count, R.st));
      CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev_comm[0], 0));
      COMM_TRY(pitcomm::send(R.comm, x + (R.count - 1) * M, M, R.comm->rank + 1, cs, &what_));
    } else {
      if (R.count > 1)
        PIT_TRY(run_slab_batch(ctx, mode, x + M, x, rhs ? rhs + M : nullptr, out + M, R.first + 1,
                               R.count - 1, R.st));
      CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev_comm[0], 0));
      COMM_TRY(pitcomm::shift(R.comm, x + (R.count - 1) * M, ctx->d_halo, M, cs, &what_));
      PIT_TRY(run_slab_batch(ctx, mode, x, ctx->d_halo, rhs, out, R.first, 1, cs));
    }
    CUDA_TRY(cudaEventRecord(ctx->ev_comm[1], cs));
    CUDA_TRY(cudaStreamWaitEvent(R.st, ctx->ev_comm[1], 0));
  }
  PIT_TRY(run_check(R, true));
  add_fine(ctx, stats, ms_since(t0));
  return PIT_OK;
}

// the sequential chain W_n = G(W_{n-1}) (+ V_n) over the rank's blocks;
// sharded: W_{first-1} comes from rank-1, W_{last} goes to rank+1
int run_chain(Run& R, int role, bool with_source, const double* V, double* W, bool add_v,
              pit_run_stats* stats) {
  pit_context* ctx = R.ctx;
  const size_t M = ctx->M;
  const auto t0 = Clock::now();
  if (R.first == 0) {
    PIT_TRY(run_sweep(ctx, role, with_source, V, nullptr, W, 0, R.count, add_v, R.st));
  } else {
    COMM_TRY(pitcomm::recv(R.comm, ctx->d_halo, M, R.comm->rank - 1, R.st, &what_));
    PIT_TRY(run_sweep(ctx, role, with_source, V, ctx->d_halo, W, R.first, R.count, add_v, R.st));
  }
  if (R.has_next())
    COMM_TRY(pitcomm::send(R.comm, W + (R.count - 1) * M, M, R.comm->rank + 1, R.st, &what_));
  PIT_TRY(run_check(R, false));
  if (role == PIT_COARSE) add_coarse(ctx, stats, ms_since(t0));
  return PIT_OK;
}

// ctx->h_partials[N*np] (global slab order) from the rank's local partials
// in ctx->d_partials[count*np]
int run_reduce(Run& R, int np) {
  pit_context* ctx = R.ctx;
  if (!R.comm) return fetch_partials(ctx, R.count * np);
  const int world = R.comm->world, N = ctx->N;
  const int maxc = (N + world - 1) / world;
  const size_t per = (size_t)maxc * 3 + 4;  // partials, then DevStatus' slab fields + fail[3]
  double* send = ctx->d_gather;
  double* recv = ctx->d_gather + per;
  CUDA_TRY(cudaMemcpyAsync(send, ctx->d_partials, sizeof(double) * (size_t)R.count * np,
                           cudaMemcpyDeviceToDevice, R.st));
  CUDA_TRY(cudaMemcpyAsync(send + (size_t)maxc * 3, ctx->d_status, offsetof(DevStatus, busy_ns),
                           cudaMemcpyDeviceToDevice, R.st));
  COMM_TRY(pitcomm::allgather(R.comm, send, per, recv, R.st, &what_));
  CUDA_TRY(cudaMemcpyAsync(ctx->h_gather, recv, sizeof(double) * per * world,
                           cudaMemcpyDeviceToHost, R.st));
  CUDA_TRY(cudaStreamSynchronize(R.st));
  int bad_fine = INT_MAX, bad_sweep = INT_MAX, sweep_rank = -1;
  for (int r = 0; r < world; ++r) {
    const int base = N / world, extra = N % world;
    const int fr = r * base + std::min(r, extra), cr = base + (r < extra ? 1 : 0);
    const double* g = ctx->h_gather + (size_t)r * per;
    std::memcpy(ctx->h_partials + (size_t)fr * np, g, sizeof(double) * (size_t)cr * np);
    DevStatus s{};
    std::memcpy(&s, g + (size_t)maxc * 3, offsetof(DevStatus, busy_ns));
    bad_fine = std::min(bad_fine, s.slab);
    if (s.sweep_slab < bad_sweep) {
      bad_sweep = s.sweep_slab;
      sweep_rank = r;
    }
  }
  if (bad_fine == INT_MAX && bad_sweep == INT_MAX) return PIT_OK;
  // every rank raises the same error; the local status is cleared as
  // check_status would
  const bool local_failed = ctx->h_status->slab != INT_MAX || ctx->h_status->sweep_slab != INT_MAX;
  (void)local_failed;
  CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                           R.st));
  CUDA_TRY(cudaStreamSynchronize(R.st));
  DevStatus* h = ctx->h_status;
  h->slab = h->sweep_slab = INT_MAX;
  h->fail[0] = h->fail[1] = 0.0;
  h->fail[2] = -1.0;
  CUDA_TRY(cudaMemcpyAsync(ctx->d_status, ctx->h_status, offsetof(DevStatus, busy_ns),
                           cudaMemcpyHostToDevice, R.st));
  CUDA_TRY(cudaStreamSynchronize(R.st));
  if (bad_sweep != INT_MAX) {
    DevStatus s{};
    std::memcpy(&s, ctx->h_gather + (size_t)sweep_rank * per + (size_t)maxc * 3,
                offsetof(DevStatus, busy_ns));
    const int kind = (int)s.fail[2];
    const std::string what =
        kind == kFailNotConverged
            ? "implicit step solve did not converge (relative residual " +
                  std::to_string(s.fail[0]) + " after " + std::to_string((long long)s.fail[1]) +
                  " iterations)"
            : "implicit step produced non-finite values";
    const int rc = set_err(PIT_ERR_INNER_SOLVE, what, bad_sweep);
    g_err_detail = kind == kFailNotConverged || kind == kFailNonFinite;
    g_err_relres = s.fail[0];
    g_err_iters = (int64_t)s.fail[1];
    return rc;
  }
  return set_err(PIT_ERR_SLAB,
                 "slab " + std::to_string(bad_fine) + ": implicit step produced non-finite values",
                 bad_fine);
}

// per-block h<a_k, b_k> of the rank's blocks, reduced: ctx->h_partials
int run_dots(Run& R, int np, const double* const* a, const double* const* b) {
  CUDA_TRY(launch_dots(R.ctx->M, R.count, R.ctx->weight, np, a, b, R.ctx->d_partials, R.st));
  return run_reduce(R, np);
}

int run_copy(Run& R, double* dst, const double* src) {
  CUDA_TRY(cudaMemcpyAsync(dst, src, R.nl() * sizeof(double), cudaMemcpyDeviceToDevice, R.st));
  return PIT_OK;
}

// initial_guess (solvers.cpp:49-64) over the rank's blocks
int run_initial_guess(Run& R, int policy, double* d, pit_run_stats* stats) {
  pit_context* ctx = R.ctx;
  CUDA_TRY(cudaMemsetAsync(d, 0, R.nl() * sizeof(double), R.st));
  if (policy == PIT_GUESS_ZERO) return PIT_OK;
  if (R.first == 0)
    CUDA_TRY(cudaMemcpyAsync(d, ctx->d_y0, ctx->M * sizeof(double), cudaMemcpyDeviceToDevice,
                             R.st));
  return run_chain(R, PIT_COARSE, true, nullptr, d, false, stats);
}

// assemble_rhs (block_system.cpp:149-172) over the rank's blocks
int run_rhs(Run& R, double* d, pit_run_stats* stats) {
  pit_context* ctx = R.ctx;
  const auto t0 = Clock::now();
  CUDA_TRY(cudaMemsetAsync(d, 0, R.nl() * sizeof(double), R.st));
  if (R.first == 0)
    CUDA_TRY(cudaMemcpyAsync(d, ctx->d_y0, ctx->M * sizeof(double), cudaMemcpyDeviceToDevice,
                             R.st));
  if (!ctx->has_source) return PIT_OK;
  PIT_TRY(fine_source(ctx, d, R.first, R.count, R.st));
  PIT_TRY(run_check(R, true));
  add_fine(ctx, stats, ms_since(t0));
  return PIT_OK;
}

// block_norm_n_inf(lambda - reference) (solvers.cpp:131), on the device:
// diff = fma(-1, ref, lambda) = lambda - ref exactly rounded.
double error_vs_reference(Run& R, const double* lam) {
  pit_context* ctx = R.ctx;
  const size_t nl = R.nl();
  if (cudaMemcpyAsync(ctx->d_ref_diff, lam, nl * sizeof(double), cudaMemcpyDeviceToDevice,
                      R.st) != cudaSuccess ||
      launch_axpy(nl, -1.0, ctx->d_ref + (size_t)R.first * ctx->M, ctx->d_ref_diff, R.st) !=
          cudaSuccess)
    return NAN;
  const double* A[1] = {ctx->d_ref_diff};
  if (run_dots(R, 1, A, A)) return NAN;
  return max_sqrt_partials(ctx->h_partials, ctx->N, 1, 0);
}

struct Recorder {
  pit_record* rows;
  int cap;
  int n = 0;
  pit_run_stats* stats;
  Clock::time_point t0;
  Run* run = nullptr;           // with a reference set: error_vs_reference of *lam
  const double* lam = nullptr;
  int rc = PIT_OK;              // first failure of an observer's copy
  void operator()(int k, double res) {
    pit_context* ctx = run->ctx;
    pit_record row{};
    row.k = k;
    row.residual_norm = res;
    row.fine_applications = stats->fine_applications;
    row.coarse_applications = stats->coarse_applications;
    if (ctx->d_ref && lam) {
      row.error_vs_reference = error_vs_reference(*run, lam);
      row.has_error = 1;
    }
    row.wall_ms = ms_since(t0);
    if (n < cap && rows) rows[n] = row;
    ++n;
    // SolveOptions::iterate_observer: after the row is recorded, with the
    // iterate it describes (solvers.cpp:101, 136); sharded: the rank's blocks
    if (ctx->observer && lam) {
      if (cudaMemcpyAsync(ctx->h_observed, lam, run->nl() * sizeof(double),
                          cudaMemcpyDeviceToHost, run->st) != cudaSuccess ||
          cudaStreamSynchronize(run->st) != cudaSuccess) {
        if (!rc) rc = set_err(PIT_ERR_CUDA, "iterate_observer: device-to-host copy failed");
        return;
      }
      ctx->observer(&row, ctx->h_observed, run->count, ctx->M, ctx->observer_user);
    }
  }
};

int validate_cfg(const pit_solver_config* cfg) {
  if (!cfg) return set_err(PIT_ERR_INVALID_ARGUMENT, "null solver config");
  if (!(cfg->tolerance > cfg->restart_tolerance) || !(cfg->restart_tolerance > 0.0))
    return set_err(PIT_ERR_CONFIG,
                   "solver tolerances must satisfy tolerance > restart_tolerance > 0");
  if (cfg->max_iterations < 1) return set_err(PIT_ERR_CONFIG, "max_iterations must be >= 1");
  return PIT_OK;
}

// G^-1 F x with the coarse sweep (K2) running concurrently with the fine
// batch (K1): K1's CTAs publish each finished block of F x, K2 (launched on
// its own high-priority stream, one SM left free by K1's persistent grid)
// waits for block n before it adds it to W_n.  The dependency is one-way
// (K1 never waits on K2), so whatever the scheduling, both finish; the
// arithmetic is the serial path's.  1D single-GPU, TMA sweep layouts.
bool gf_overlap_ok(pit_context* ctx) {
  if (ctx->gf_overlap < 0) {
    const char* e = std::getenv("PIT_GF_OVERLAP");
    if (ctx->dim == 2 && !ctx->be2) {
      // config 5 (K4 clusters in slab order, many waves; K5 on its own
      // cluster): worth it once the batch is more than two waves of clusters
      const int sms = ctx->sms;
      const int forced = e ? std::atoi(e) : -1;
      ctx->gf_overlap = ctx->N >= 3 && forced != 0 &&
                        (forced == 1 || (long long)(ctx->N - 1) * ctx->lay2.cl > 2LL * sms);
      return ctx->gf_overlap == 1;
    }
    ctx->gf_overlap = ctx->dim == 1 && !ctx->be2 && ctx->M % 16 == 0 && ctx->M >= 1024 &&
                      ctx->N >= 3 && ctx->role[PIT_COARSE].nseg == 1 &&
                      ctx->role[PIT_COARSE].mpt % 2 == 0 && !(e && std::atoi(e) == 0);
    // only a batch of more than one wave gains: its first wave's blocks are
    // out while the rest still runs (one wave ends all at once)
    int slots = 0;
    const Role& R = ctx->role[PIT_FINE];
    if (ctx->gf_overlap &&
        (slab_slots(R.mpt, R.nsub, R.nseg, R.warps, false, R.P, &slots) != cudaSuccess ||
         ctx->N - 1 <= slots))
      ctx->gf_overlap = 0;
    cudaGetLastError();
    if (e && std::atoi(e) == 1 && ctx->dim == 1 && !ctx->be2 && ctx->M % 16 == 0 &&
        ctx->M >= 1024 && ctx->N >= 3)
      ctx->gf_overlap = 1;  // forced on (A/B runs)
  }
  return ctx->gf_overlap == 1;
}

// timing spans of a deferred (device-loop) iteration, read after its sync
cudaEvent_t ev_take(pit_context* ctx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_used++];
}
int span_begin(pit_context* ctx, int role, cudaStream_t st) {
  ctx->ev_spans.emplace_back(ctx->ev_used, role);
  cudaEvent_t e = ev_take(ctx);
  if (!e) return set_err(PIT_ERR_CUDA, "event pool");
  CUDA_TRY(cudaEventRecord(e, st));
  return PIT_OK;
}
int span_end(pit_context* ctx, cudaStream_t st) {
  cudaEvent_t e = ev_take(ctx);
  if (!e) return set_err(PIT_ERR_CUDA, "event pool");
  CUDA_TRY(cudaEventRecord(e, st));
  return PIT_OK;
}
void spans_collect(pit_context* ctx, pit_run_stats* st) {
  for (const auto& sp : ctx->ev_spans) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev_pool[sp.first], ctx->ev_pool[sp.first + 1]);
    if (sp.second == PIT_FINE)
      st->fine_parallel_ms += ms;
    else
      st->coarse_sequential_ms += ms;
  }
  cudaGetLastError();
  ctx->ev_spans.clear();
  ctx->ev_used = 0;
}

// mode kApplyF: out = G^-1 (F x), F x staged in tmp; mode kResidual:
// out = G^-1 (rhs - F x) (preconditioned_residual), in place when tmp == out.
int apply_GF_overlapped(Run& R, const double* x, double* tmp, double* out, pit_run_stats* st,
                        bool deferred = false, int mode = kApplyF, const double* rhs = nullptr) {
  pit_context* ctx = R.ctx;
  const size_t M = ctx->M;
  if (!ctx->d_ready) {
    CUDA_TRY(cudaMalloc(&ctx->d_ready, sizeof(int) * (size_t)ctx->N));
    CUDA_TRY(cudaMemsetAsync(ctx->d_ready, 0, sizeof(int) * (size_t)ctx->N, R.st));
    CUDA_TRY(cudaStreamCreateWithPriority(&ctx->gf_stream, cudaStreamNonBlocking, -1));
    for (int i = 0; i < 5; ++i)
      CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_gf[i], i == 0 ? cudaEventDisableTiming
                                                               : cudaEventDefault));
  }
  if (++ctx->ready_epoch <= 0) ctx->ready_epoch = 1;
  const int epoch = ctx->ready_epoch;
  const auto t0 = Clock::now();
  CUDA_TRY(cudaEventRecord(ctx->ev_gf[0], R.st));  // x ready, tmp and out free
  CUDA_TRY(cudaStreamWaitEvent(ctx->gf_stream, ctx->ev_gf[0], 0));
  SweepArgs A{};
  bind_status(ctx, &A);
  A.start = tmp;  // V_0
  A.W0 = tmp == out ? nullptr : out;  // W_0 = V_0
  A.V = tmp + M;
  A.W = out + M;
  A.count = R.count - 1;
  A.slab0 = 0;
  A.ready = ctx->d_ready;
  A.epoch = epoch;
  A.ready_shift = 1;
  A.skip = ctx->skip;
  auto launch_coarse = [&]() -> int {
    if (deferred)
      PIT_TRY(span_begin(ctx, PIT_COARSE, ctx->gf_stream));
    else
      CUDA_TRY(cudaEventRecord(ctx->ev_gf[3], ctx->gf_stream));
    if (ctx->dim == 2) {
      CUDA_TRY(launch_cg_sweep2d(cg2_params(ctx), A, ctx->d_cg_iters, ctx->gf_stream));
      return deferred ? span_end(ctx, ctx->gf_stream) : PIT_OK;
    }
    const Role& Rc = ctx->role[PIT_COARSE];
    const cudaError_t le = launch_sweep(Rc.mpt, Rc.nsub, Rc.nseg, Rc.warps, false, Rc.P, A,
                                        ctx->gf_stream);
    if (le == cudaErrorNotSupported) {
      // this layout / alignment has no I/O-warp sweep: serial from now on
      cudaGetLastError();
      ctx->gf_overlap = 0;
      CUDA_TRY(cudaStreamWaitEvent(ctx->gf_stream, ctx->ev_gf[2], 0));
      PIT_TRY(run_sweep(ctx, PIT_COARSE, false, tmp, nullptr, out, 0, R.count, true,
                        ctx->gf_stream));
    } else {
      CUDA_TRY(le);
    }
    return deferred ? span_end(ctx, ctx->gf_stream) : PIT_OK;
  };
  if (deferred)
    PIT_TRY(span_begin(ctx, PIT_FINE, R.st));
  else
    CUDA_TRY(cudaEventRecord(ctx->ev_gf[1], R.st));
  // one CTA per slab in launch order, not piece scheduling: the first wave's
  // blocks are then out after one slab's latency, while pieces would hold
  // every block back to the last piece round (c2 TTT 39.0 vs 42.4 ms)
  const int saved_pieces = ctx->pieces;
  if (ctx->pieces == 0) ctx->pieces = 1;
  const int rc1 = run_slab_batch(ctx, mode, x, nullptr, rhs, tmp, 0, R.count, R.st,
                                 nullptr, nullptr, 0, ctx->d_ready, epoch, 1);
  ctx->pieces = saved_pieces;
  PIT_TRY(rc1);
  if (deferred) PIT_TRY(span_end(ctx, R.st));
  CUDA_TRY(cudaEventRecord(ctx->ev_gf[2], R.st));
  // The sweep is launched after the fine batch in 1D and 2D alike: a first
  // launch of a kernel may wait for outstanding work (lazy module loading),
  // and the batch never waits on the sweep, so this order cannot deadlock.
  // Config 5: K5's cluster (high-priority stream) gets its SMs as K4's first
  // wave of clusters retires, then follows K4 block by block (it needs V_b
  // only after slab b's CG solves).
  PIT_TRY(launch_coarse());
  CUDA_TRY(cudaEventRecord(ctx->ev_gf[4], ctx->gf_stream));
  CUDA_TRY(cudaStreamWaitEvent(R.st, ctx->ev_gf[4], 0));
  if (deferred) return PIT_OK;
  PIT_TRY(check_status(ctx, true));
  PIT_TRY(check_status(ctx, false));
  float k1 = 0.f, k2 = 0.f;
  cudaEventElapsedTime(&k1, ctx->ev_gf[1], ctx->ev_gf[2]);
  cudaEventElapsedTime(&k2, ctx->ev_gf[3], ctx->ev_gf[4]);
  const double wall = ms_since(t0);
  // RunStats: the fine batch's own span, the sweep's own span (they overlap)
  add_fine(ctx, st, std::min<double>(k1, wall));
  add_coarse(ctx, st, std::min<double>(k2, wall));
  return PIT_OK;
}

// G^-1 F x  ->  out   (F into tmp, then the in-place sweep)
int apply_GF(Run& R, const double* x, double* tmp, double* out, pit_run_stats* st) {
  if (!R.comm && gf_overlap_ok(R.ctx)) return apply_GF_overlapped(R, x, tmp, out, st);
  PIT_TRY(run_fine(R, kApplyF, x, nullptr, tmp, st));
  return run_chain(R, PIT_COARSE, false, tmp, out, true, st);
}

// preconditioned_residual (solvers.cpp:66-71): G^-1 (rhs - F lam)
int precond_residual(Run& R, const double* lam, const double* rhs, double* out,
                     pit_run_stats* st) {
  if (!R.comm && gf_overlap_ok(R.ctx))
    return apply_GF_overlapped(R, lam, out, out, st, false, kResidual, rhs);
  PIT_TRY(run_fine(R, kResidual, lam, rhs, out, st));
  return run_chain(R, PIT_COARSE, false, out, out, true, st);
}

// pitsbicg_solve, src/solvers.cpp:116-220.  lam (device) holds the rank's
// blocks of the iterate.
int pitsbicg_dev(Run& R, const pit_solver_config* cfg, bool have_init, double* lam,
                 double* first_residual_dev, pit_record* rows, int cap, pit_solve_info* info) {
  pit_context* ctx = R.ctx;
  PIT_TRY(ensure_buffers(ctx, R.nl()));
  const int N = ctx->N, M = ctx->M, nb = R.count;
  const size_t nl = R.nl();
  double *rhs = ctx->buf[1], *r = ctx->buf[2], *rs = ctx->buf[3], *p = ctx->buf[4],
         *d = ctx->buf[5], *s = ctx->buf[6], *t = ctx->buf[7], *f = ctx->buf[8];
  pit_solve_info inf{};
  inf.min_restart_margin = INFINITY;
  pit_run_stats& st = inf.stats;
  Recorder rec{rows, cap, 0, &st, Clock::now(), &R, lam};
  auto finish = [&](int status) -> int {
    if (rec.rc) return rec.rc;
    inf.status = status;
    inf.total_records = rec.n;
    inf.record_count = std::min(rec.n, cap);
    if (info) *info = inf;
    return PIT_OK;
  };
  if (!have_init) PIT_TRY(run_initial_guess(R, cfg->initial_guess, lam, &st));
  PIT_TRY(run_rhs(R, rhs, &st));
  PIT_TRY(precond_residual(R, lam, rhs, r, &st));
  if (first_residual_dev) PIT_TRY(run_copy(R, first_residual_dev, r));
  // ||r|| and <r,r> (= rho of iteration 1, r~ = r) from one partials pass
  {
    const double* A[1] = {r};
    PIT_TRY(run_dots(R, 1, A, A));
  }
  double r_norm = max_sqrt_partials(ctx->h_partials, N, 1, 0);
  double rr_shadow = sum_partials(ctx->h_partials, N, 1, 0);  // <r, r~> with r~ = r
  rec(0, r_norm);
  if (r_norm <= cfg->tolerance) return finish(PIT_CONVERGED);
  PIT_TRY(run_copy(R, rs, r));
  PIT_TRY(run_copy(R, p, r));

  for (int k = 1; k <= cfg->max_iterations; ++k) {
    auto restart = [&]() -> int {
      PIT_TRY(run_copy(R, rs, r));
      PIT_TRY(run_copy(R, p, r));
      ++inf.restarts;
      rec(k, r_norm);
      // r~ = r: <r, r~> becomes <r, r>
      const double* A[1] = {r};
      PIT_TRY(run_dots(R, 1, A, A));
      rr_shadow = sum_partials(ctx->h_partials, N, 1, 0);
      return PIT_OK;
    };
    // rho = <r, r~>: the value computed when r (or r~) last changed
    const double rho = rr_shadow;
    PIT_TRY(apply_GF(R, p, f, d, &st));
    {
      const double* A[1] = {d};
      const double* B[1] = {rs};
      PIT_TRY(run_dots(R, 1, A, B));
    }
    const double d_dot = sum_partials(ctx->h_partials, N, 1, 0);
    if (std::abs(d_dot) < 1e-300) {
      PIT_TRY(restart());
      continue;
    }
    const double alpha = rho / d_dot;
    CUDA_TRY(launch_update_s(M, nb, ctx->weight, alpha, r, d, s, ctx->d_partials, R.st));
    PIT_TRY(run_reduce(R, 1));
    const double s_norm = max_sqrt_partials(ctx->h_partials, N, 1, 0);
    if (s_norm <= cfg->tolerance) {
      CUDA_TRY(launch_axpy(nl, alpha, p, lam, R.st));
      std::swap(ctx->buf[2], ctx->buf[6]);  // r = move(s)
      rec(k, s_norm);
      CUDA_TRY(cudaStreamSynchronize(R.st));
      return finish(PIT_CONVERGED);
    }
    PIT_TRY(apply_GF(R, s, f, t, &st));
    {
      const double* A[2] = {t, t};
      const double* B[2] = {t, s};
      PIT_TRY(run_dots(R, 2, A, B));
    }
    const double tt = sum_partials(ctx->h_partials, N, 2, 0);
    if (tt < 1e-300) {
      PIT_TRY(restart());
      continue;
    }
    const double omega = sum_partials(ctx->h_partials, N, 2, 1) / tt;
    if (std::abs(omega) < 1e-300) {
      PIT_TRY(restart());
      continue;
    }
    // lambda += alpha p; lambda += omega s; s -= omega t; r = move(s)
    CUDA_TRY(launch_update_lr(M, nb, ctx->weight, alpha, omega, p, s, t, rs, lam, r,
                              ctx->d_partials, R.st));
    PIT_TRY(run_reduce(R, 2));
    r_norm = max_sqrt_partials(ctx->h_partials, N, 2, 0);
    const double rr = sum_partials(ctx->h_partials, N, 2, 0);
    const double r_dot = sum_partials(ctx->h_partials, N, 2, 1);
    rec(k, r_norm);
    if (r_norm <= cfg->tolerance) return finish(PIT_CONVERGED);
    inf.min_restart_margin = std::min(inf.min_restart_margin, std::abs(r_dot) / cfg->restart_tolerance);
    if (std::abs(r_dot) <= cfg->restart_tolerance) {
      PIT_TRY(run_copy(R, rs, r));
      PIT_TRY(run_copy(R, p, r));
      ++inf.restarts;
      rr_shadow = rr;
    } else {
      const double beta = (alpha / omega) * (r_dot / rho);
      CUDA_TRY(launch_update_p(nl, omega, beta, d, r, p, R.st));
      rr_shadow = r_dot;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(R.st));
  return finish(PIT_MAX_ITERATIONS);
}

// G^-1 F x of a device-loop iteration: no status read, timing spans
// (spans = false inside a stream capture: no event records)
int apply_GF_deferred(Run& R, const double* x, double* tmp, double* out, bool spans = true) {
  pit_context* ctx = R.ctx;
  if (gf_overlap_ok(ctx)) return apply_GF_overlapped(R, x, tmp, out, nullptr, true);
  if (spans) PIT_TRY(span_begin(ctx, PIT_FINE, R.st));
  PIT_TRY(run_slab_batch(ctx, kApplyF, x, nullptr, nullptr, tmp, 0, R.count, R.st));
  if (spans) PIT_TRY(span_end(ctx, R.st));
  if (spans) PIT_TRY(span_begin(ctx, PIT_COARSE, R.st));
  PIT_TRY(run_sweep(ctx, PIT_COARSE, false, tmp, nullptr, out, 0, R.count, true, R.st));
  return spans ? span_end(ctx, R.st) : PIT_OK;
}

// An iteration of the device loop runs as one CUDA graph launch from the
// second iteration on, where the fine batch and the coarse sweep run back to
// back on one stream (no K2-on-K1 overlap: that path forks streams), i.e. on
// the launch-bound solves the device loop serves.  PIT_NO_GRAPH=1 disables it.
bool iteration_graph_ok(pit_context* ctx) {
  if (ctx->graph_mode < 0) {
    const char* e = std::getenv("PIT_NO_GRAPH");
    ctx->graph_mode = (e && std::atoi(e) != 0) || gf_overlap_ok(ctx) ? 0 : 1;
  }
  return ctx->graph_mode == 1;
}

// pitsbicg_solve (src/solvers.cpp:116-220) with the scalar recurrence on the
// device (single GPU): an iteration's launches are enqueued without waiting
// — scalars_kernel sums the partials in slab order and takes the reference's
// branches, setting SolverScalars::stop so that the remaining launches of
// the iteration skip their work — and the host reads the scalars, the status
// and the branch once per iteration (instead of after every phase).  The
// arithmetic, branches and history are those of pitsbicg_dev.
int pitsbicg_device_loop(Run& R, const pit_solver_config* cfg, bool have_init, double* lam,
                         double* first_residual_dev, pit_record* rows, int cap,
                         pit_solve_info* info) {
  pit_context* ctx = R.ctx;
  PIT_TRY(ensure_buffers(ctx, R.nl()));
  if (!ctx->d_sc) {
    CUDA_TRY(cudaMalloc(&ctx->d_sc, sizeof(SolverScalars)));
    CUDA_TRY(cudaMallocHost(&ctx->h_sc, sizeof(SolverScalars)));
  }
  const int N = ctx->N, M = ctx->M, nb = R.count;
  const size_t nl = R.nl();
  double *rhs = ctx->buf[1], *r = ctx->buf[2], *rs = ctx->buf[3], *p = ctx->buf[4],
         *d = ctx->buf[5], *s = ctx->buf[6], *t = ctx->buf[7], *f = ctx->buf[8];
  SolverScalars* sc = ctx->d_sc;
  SolverScalars& hs = *ctx->h_sc;
  pit_solve_info inf{};
  inf.min_restart_margin = INFINITY;
  pit_run_stats& st = inf.stats;
  Recorder rec{rows, cap, 0, &st, Clock::now(), &R, lam};
  auto finish = [&](int status) -> int {
    if (rec.rc) return rec.rc;
    inf.status = status;
    inf.total_records = rec.n;
    inf.record_count = std::min(rec.n, cap);
    if (info) *info = inf;
    return PIT_OK;
  };
  // the start is pitsbicg_dev's (one host read of ||r|| there)
  if (!have_init) PIT_TRY(run_initial_guess(R, cfg->initial_guess, lam, &st));
  PIT_TRY(run_rhs(R, rhs, &st));
  PIT_TRY(precond_residual(R, lam, rhs, r, &st));
  if (first_residual_dev) PIT_TRY(run_copy(R, first_residual_dev, r));
  {
    const double* A[1] = {r};
    PIT_TRY(run_dots(R, 1, A, A));
  }
  double r_norm = max_sqrt_partials(ctx->h_partials, N, 1, 0);
  // <r, r~> with r~ = r, read before rec() (whose error_vs_reference reuses
  // the partials)
  const double rho0 = sum_partials(ctx->h_partials, N, 1, 0);
  rec(0, r_norm);
  if (r_norm <= cfg->tolerance) return finish(PIT_CONVERGED);
  PIT_TRY(run_copy(R, rs, r));
  PIT_TRY(run_copy(R, p, r));
  {
    SolverScalars z{};
    z.rho = rho0;
    z.margin = INFINITY;
    CUDA_TRY(cudaMemcpyAsync(sc, &z, sizeof(z), cudaMemcpyHostToDevice, R.st));
  }
  const double tol = cfg->tolerance, eps0 = cfg->restart_tolerance;
  const long n1 = N - 1;
  ctx->skip = &sc->stop;
  struct SkipReset {
    pit_context* c;
    ~SkipReset() { c->skip = nullptr; }
  } skip_reset{ctx};
  // the launches of one iteration (every pointer and scalar argument is the
  // same in every iteration, so the sequence can be captured once)
  auto enqueue_iteration = [&](bool spans) -> int {
    CUDA_TRY(cudaMemsetAsync(&sc->flag, 0, 2 * sizeof(int), R.st));  // flag, stop
    PIT_TRY(apply_GF_deferred(R, p, f, d, spans));
    {
      const double* A[1] = {d};
      const double* B[1] = {rs};
      CUDA_TRY(launch_dots(M, nb, ctx->weight, 1, A, B, ctx->d_partials, R.st, sc));
    }
    CUDA_TRY(launch_scalars(sc, ctx->d_partials, N, kScAlpha, tol, eps0, R.st));
    CUDA_TRY(launch_update_s(M, nb, ctx->weight, 0.0, r, d, s, ctx->d_partials, R.st, sc));
    CUDA_TRY(launch_scalars(sc, ctx->d_partials, N, kScSnorm, tol, eps0, R.st));
    PIT_TRY(apply_GF_deferred(R, s, f, t, spans));
    {
      const double* A[2] = {t, t};
      const double* B[2] = {t, s};
      CUDA_TRY(launch_dots(M, nb, ctx->weight, 2, A, B, ctx->d_partials, R.st, sc));
    }
    CUDA_TRY(launch_scalars(sc, ctx->d_partials, N, kScOmega, tol, eps0, R.st));
    CUDA_TRY(launch_update_lr(M, nb, ctx->weight, 0.0, 0.0, p, s, t, rs, lam, r, ctx->d_partials,
                              R.st, sc));
    CUDA_TRY(launch_scalars(sc, ctx->d_partials, N, kScR, tol, eps0, R.st));
    CUDA_TRY(launch_update_p(nl, 0.0, 0.0, d, r, p, R.st, sc));
    CUDA_TRY(cudaMemcpyAsync(ctx->h_sc, sc, sizeof(SolverScalars), cudaMemcpyDeviceToHost, R.st));
    return PIT_OK;
  };
  // graph of an iteration, (re)captured when the buffers or tolerances differ
  // from the cached instance's; any failure falls back to plain launches
  auto iteration_graph = [&]() -> cudaGraphExec_t {
    unsigned long long bits[2];
    std::memcpy(&bits[0], &tol, 8);
    std::memcpy(&bits[1], &eps0, 8);
    const std::vector<unsigned long long> key = {
        (unsigned long long)(uintptr_t)lam, (unsigned long long)(uintptr_t)r,
        (unsigned long long)(uintptr_t)rs,  (unsigned long long)(uintptr_t)p,
        (unsigned long long)(uintptr_t)d,   (unsigned long long)(uintptr_t)s,
        (unsigned long long)(uintptr_t)t,   (unsigned long long)(uintptr_t)f,
        (unsigned long long)(uintptr_t)R.st, bits[0], bits[1], (unsigned long long)nb};
    if (ctx->it_exec && key == ctx->it_key) return ctx->it_exec;
    if (ctx->it_exec) {
      cudaGraphExecDestroy(ctx->it_exec);
      ctx->it_exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(R.st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    int rc = enqueue_iteration(false);
    if (rc == PIT_OK &&
        cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                        R.st) != cudaSuccess)
      rc = PIT_ERR_CUDA;
    const cudaError_t ce = cudaStreamEndCapture(R.st, &g);
    if (rc != PIT_OK || ce != cudaSuccess || !g ||
        cudaGraphInstantiate(&ctx->it_exec, g, 0) != cudaSuccess)
      ctx->it_exec = nullptr;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    if (ctx->it_exec) ctx->it_key = key;
    return ctx->it_exec;
  };
  double fine_share = 0.5;  // of an iteration's device time (first, eager iteration)
  for (int k = 1; k <= cfg->max_iterations; ++k) {
    cudaGraphExec_t graph = nullptr;
    if (k > 1 && iteration_graph_ok(ctx)) {
      graph = iteration_graph();
      if (!graph) ctx->graph_mode = 0;  // not capturable here: plain launches from now on
    }
    if (graph) {
      if (!ctx->ev_it[0]) {
        CUDA_TRY(cudaEventCreate(&ctx->ev_it[0]));
        CUDA_TRY(cudaEventCreate(&ctx->ev_it[1]));
      }
      CUDA_TRY(cudaEventRecord(ctx->ev_it[0], R.st));
      CUDA_TRY(cudaGraphLaunch(graph, R.st));
      CUDA_TRY(cudaEventRecord(ctx->ev_it[1], R.st));
      // one wait per iteration: the scalars and the status came with the graph
      CUDA_TRY(cudaStreamSynchronize(R.st));
      PIT_TRY(eval_status(ctx, true));
      PIT_TRY(eval_status(ctx, false));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev_it[0], ctx->ev_it[1]);
      st.fine_parallel_ms += fine_share * ms;
      st.coarse_sequential_ms += (1.0 - fine_share) * ms;
    } else {
      const double f0 = st.fine_parallel_ms, c0 = st.coarse_sequential_ms;
      PIT_TRY(enqueue_iteration(true));
      // one read per iteration: the scalars and the failing-slab status
      PIT_TRY(check_status(ctx, true));
      PIT_TRY(eval_status(ctx, false));
      spans_collect(ctx, &st);
      const double df = st.fine_parallel_ms - f0, dc = st.coarse_sequential_ms - c0;
      if (df + dc > 0.0) fine_share = df / (df + dc);
    }
    {
      const unsigned long long now = ctx->h_status->busy_ns;
      st.fine_busy_ms += (double)(now - ctx->busy_mark) * 1e-6;
      ctx->busy_mark = now;
    }
    // counters of the applications the iteration actually ran
    const int flag = hs.flag;
    const int applies = (flag == kFlagRestartD || flag == kFlagHalf) ? 1 : 2;
    st.fine_applications += applies * n1;
    st.coarse_applications += applies * n1;
    inf.min_restart_margin = std::min(inf.min_restart_margin, hs.margin);
    auto restart = [&]() -> int {
      PIT_TRY(run_copy(R, rs, r));
      PIT_TRY(run_copy(R, p, r));
      ++inf.restarts;
      rec(k, r_norm);
      // r~ = r: <r, r~> becomes <r, r>
      const double* A[1] = {r};
      CUDA_TRY(launch_dots(M, nb, ctx->weight, 1, A, A, ctx->d_partials, R.st));
      CUDA_TRY(cudaMemsetAsync(&sc->flag, 0, 2 * sizeof(int), R.st));
      CUDA_TRY(launch_scalars(sc, ctx->d_partials, N, kScRho, tol, eps0, R.st));
      return PIT_OK;
    };
    switch (flag) {
      case kFlagRestartD:
      case kFlagRestartT:
      case kFlagRestartW:
        PIT_TRY(restart());
        continue;
      case kFlagHalf:
        CUDA_TRY(launch_axpy(nl, 0.0, p, lam, R.st, &sc->alpha));
        std::swap(ctx->buf[2], ctx->buf[6]);  // r = move(s)
        rec(k, hs.s_norm);
        CUDA_TRY(cudaStreamSynchronize(R.st));
        return finish(PIT_CONVERGED);
      default:
        break;
    }
    r_norm = hs.r_norm;
    rec(k, r_norm);
    if (flag == kFlagConverged) return finish(PIT_CONVERGED);
    if (flag == kFlagRestartR) {  // the device already set rho = <r, r>
      PIT_TRY(run_copy(R, rs, r));
      PIT_TRY(run_copy(R, p, r));
      ++inf.restarts;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(R.st));
  return finish(PIT_MAX_ITERATIONS);
}

// parareal_solve, src/solvers.cpp:73-114.
int parareal_dev(Run& R, const pit_solver_config* cfg, bool have_init, double* lam,
                 double* first_residual_dev, pit_record* rows, int cap, pit_solve_info* info) {
  pit_context* ctx = R.ctx;
  PIT_TRY(ensure_buffers(ctx, R.nl()));
  const int N = ctx->N;
  double *rhs = ctx->buf[1], *corr = ctx->buf[2];
  pit_solve_info inf{};
  inf.min_restart_margin = INFINITY;
  pit_run_stats& st = inf.stats;
  Recorder rec{rows, cap, 0, &st, Clock::now(), &R, lam};
  if (!have_init) PIT_TRY(run_initial_guess(R, cfg->initial_guess, lam, &st));
  PIT_TRY(run_rhs(R, rhs, &st));
  int status = PIT_MAX_ITERATIONS;
  for (int k = 0;; ++k) {
    const pit_run_stats before = st;
    PIT_TRY(precond_residual(R, lam, rhs, corr, &st));
    if (k == 0 && first_residual_dev) PIT_TRY(run_copy(R, first_residual_dev, corr));
    const double* A[1] = {corr};
    PIT_TRY(run_dots(R, 1, A, A));
    const double res = max_sqrt_partials(ctx->h_partials, N, 1, 0);
    const pit_run_stats after = st;
    st = before;  // the row charges the work spent reaching the current iterate
    rec(k, res);
    st = after;
    if (res <= cfg->tolerance) {
      status = PIT_CONVERGED;
      break;
    }
    if (k == cfg->max_iterations) break;
    CUDA_TRY(launch_add(R.nl(), corr, lam, R.st));
  }
  CUDA_TRY(cudaStreamSynchronize(R.st));
  if (rec.rc) return rec.rc;
  inf.status = status;
  inf.total_records = rec.n;
  inf.record_count = std::min(rec.n, cap);
  if (info) *info = inf;
  return PIT_OK;
}

// The device-resident loop on one GPU, where it is measured to pay: launch-
// bound solves (c1 1.52 -> 1.39 ms); with K2 overlapped on K1 the host loop
// is faster (c2 36.0 vs 37.3 ms, profiles/r2p_device_loop.txt), so the large
// overlapped configs keep it.  PIT_HOST_SCALARS=1/0 forces either.
bool device_loop_ok(const Run& R) {
  static const int forced = [] {
    const char* e = std::getenv("PIT_HOST_SCALARS");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : -1;
  }();
  if (R.comm || forced == 1) return false;
  if (forced == 0) return true;
  return !gf_overlap_ok(R.ctx);
}

int solve_host(int which, pit_context* ctx, const pit_solver_config* cfg, const double* lambda_init,
               double* lambda_out, double* first_residual_out, pit_record* records,
               int max_records, pit_solve_info* info) {
  if (!ctx || !lambda_out) return set_err(PIT_ERR_INVALID_ARGUMENT, "solve: null argument");
  PIT_TRY(validate_cfg(cfg));
  Run R = make_run(ctx, false);
  PIT_TRY(ensure_buffers(ctx, R.nl()));
  double* lam = ctx->buf[0];
  double* first = first_residual_out ? ctx->buf[9] : nullptr;
  if (lambda_init)
    CUDA_TRY(cudaMemcpyAsync(lam, lambda_init, ctx->nm() * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
  if (which == 0 && device_loop_ok(R))
    PIT_TRY(pitsbicg_device_loop(R, cfg, lambda_init != nullptr, lam, first, records, max_records,
                                 info));
  else if (which == 0)
    PIT_TRY(pitsbicg_dev(R, cfg, lambda_init != nullptr, lam, first, records, max_records, info));
  else
    PIT_TRY(parareal_dev(R, cfg, lambda_init != nullptr, lam, first, records, max_records, info));
  PIT_TRY(to_host(ctx, ctx->buf[0], ctx->nm(), lambda_out));
  if (first_residual_out) PIT_TRY(to_host(ctx, first, ctx->nm(), first_residual_out));
  return PIT_OK;
}

// the *_solve_device entry points: lambda (and the optional initial guess)
// are the caller's device arrays of the rank's blocks
int solve_device(int which, bool sharded, pit_context* ctx, const pit_solver_config* cfg,
                 const double* lambda_init_dev, double* lambda_dev, pit_record* records,
                 int max_records, pit_solve_info* info, void* stream) {
  if (!ctx || !lambda_dev) return set_err(PIT_ERR_INVALID_ARGUMENT, "solve: null argument");
  if (sharded && !ctx->comm)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "sharded solve: no communicator attached");
  PIT_TRY(validate_cfg(cfg));
  Run R = make_run(ctx, sharded);
  if (stream) CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  if (lambda_init_dev && lambda_init_dev != lambda_dev)
    CUDA_TRY(cudaMemcpyAsync(lambda_dev, lambda_init_dev, R.nl() * sizeof(double),
                             cudaMemcpyDeviceToDevice, R.st));
  if (which == 0 && device_loop_ok(R))
    PIT_TRY(pitsbicg_device_loop(R, cfg, lambda_init_dev != nullptr, lambda_dev, nullptr, records,
                                 max_records, info));
  else if (which == 0)
    PIT_TRY(pitsbicg_dev(R, cfg, lambda_init_dev != nullptr, lambda_dev, nullptr, records,
                         max_records, info));
  else
    PIT_TRY(parareal_dev(R, cfg, lambda_init_dev != nullptr, lambda_dev, nullptr, records,
                         max_records, info));
  CUDA_TRY(cudaStreamSynchronize(R.st));
  return PIT_OK;
}

}  // namespace

int pit_context_slots(const pit_context* ctx, int* slots) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !slots) return set_err(PIT_ERR_INVALID_ARGUMENT, "null argument");
  if (ctx->dim == 1 && !ctx->be2) {
    const Role& R = ctx->role[PIT_FINE];
    CUDA_TRY(slab_slots(R.mpt, R.nsub, R.nseg, R.warps, false, R.P, slots));
  } else if (ctx->be2) {
    *slots = ctx->sms;  // K6: one 512-thread CTA per SM
  } else {
    *slots = ctx->sms / std::max(1, ctx->lay2.cl);  // K4: one cluster per slab, 1 CTA per SM
  }
  return PIT_OK;
}

int pit_host_alloc(size_t bytes, void** out) {
  if (!out) return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_host_alloc: null output");
  *out = nullptr;
  CUDA_TRY(cudaMallocHost(out, bytes));
  return PIT_OK;
}

int pit_host_free(void* p) {
  if (p) CUDA_TRY(cudaFreeHost(p));
  return PIT_OK;
}

int pit_last_error_detail(double* achieved_relative_residual, int64_t* iterations) {
  if (!g_err_detail) return PIT_ERR_INVALID_ARGUMENT;
  if (achieved_relative_residual) *achieved_relative_residual = g_err_relres;
  if (iterations) *iterations = g_err_iters;
  return PIT_OK;
}

int pit_set_iterate_observer(pit_context* ctx, pit_iterate_observer fn, void* user) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (fn && !ctx->h_observed)
    CUDA_TRY(cudaMallocHost(&ctx->h_observed, ctx->nm() * sizeof(double)));
  ctx->observer = fn;
  ctx->observer_user = user;
  return PIT_OK;
}

int pit_set_reference(pit_context* ctx, const double* reference) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (!reference) {
    cudaFree(ctx->d_ref);
    cudaFree(ctx->d_ref_diff);
    ctx->d_ref = ctx->d_ref_diff = nullptr;
    return PIT_OK;
  }
  if (!ctx->d_ref) {
    CUDA_TRY(cudaMalloc(&ctx->d_ref, ctx->nm() * sizeof(double)));
    CUDA_TRY(cudaMalloc(&ctx->d_ref_diff, ctx->nm() * sizeof(double)));
  }
  CUDA_TRY(cudaMemcpyAsync(ctx->d_ref, reference, ctx->nm() * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return PIT_OK;
}

int pit_pitsbicg_solve(pit_context* ctx, const pit_solver_config* cfg, const double* lambda_init,
                       double* lambda_out, double* first_residual_out, pit_record* records,
                       int max_records, pit_solve_info* info) {
  PIT_DEVICE_SCOPE(ctx);
  return solve_host(0, ctx, cfg, lambda_init, lambda_out, first_residual_out, records,
                    max_records, info);
}

int pit_parareal_solve(pit_context* ctx, const pit_solver_config* cfg, const double* lambda_init,
                       double* lambda_out, double* first_residual_out, pit_record* records,
                       int max_records, pit_solve_info* info) {
  PIT_DEVICE_SCOPE(ctx);
  return solve_host(1, ctx, cfg, lambda_init, lambda_out, first_residual_out, records,
                    max_records, info);
}

int pit_pitsbicg_solve_device(pit_context* ctx, const pit_solver_config* cfg,
                              const double* lambda_init_dev, double* lambda_dev,
                              pit_record* records, int max_records, pit_solve_info* info,
                              void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  return solve_device(0, false, ctx, cfg, lambda_init_dev, lambda_dev, records, max_records, info,
                      stream);
}

// ---- slab-sharded multi-GPU ------------------------------------------------

int pit_comm_nccl_unique_id(unsigned char* id) {
  if (!id) return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_comm_nccl_unique_id: null output");
  COMM_TRY(pitcomm::unique_id(id, &what_));
  return PIT_OK;
}

int pit_comm_create_nccl(const unsigned char* id, int rank, int world, int device,
                         pit_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_comm_create_nccl: bad arguments");
  *out = nullptr;
  COMM_TRY(pitcomm::create_nccl(id, rank, world, device, out, &what_));
  return PIT_OK;
}

int pit_comm_create_host(const pit_comm_ops* ops, int rank, int world, pit_comm** out) {
  if (!ops || !out || !ops->send || !ops->recv || !ops->allgather || world < 1 || rank < 0 ||
      rank >= world)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "pit_comm_create_host: bad arguments");
  auto c = new pit_comm();
  c->rank = rank;
  c->world = world;
  c->kind = 1;
  c->ops = *ops;
  *out = c;
  return PIT_OK;
}

int pit_comm_destroy(pit_comm* comm) {
  pitcomm::destroy(comm);
  return PIT_OK;
}

int pit_context_attach_comm(pit_context* ctx, pit_comm* comm) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (!comm) {
    ctx->comm = nullptr;
    ctx->shard_first = 0;
    ctx->shard_count = ctx->N;
    return PIT_OK;
  }
  if (comm->world > ctx->N)
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_attach_comm: more ranks than slabs (every rank must own a block)");
  if (comm->kind == 0 && comm->device != ctx->desc.device)
    return set_err(PIT_ERR_INVALID_ARGUMENT,
                   "pit_context_attach_comm: the communicator's device is not the context's");
  const int base = ctx->N / comm->world, extra = ctx->N % comm->world;
  ctx->shard_first = comm->rank * base + std::min(comm->rank, extra);
  ctx->shard_count = base + (comm->rank < extra ? 1 : 0);
  const int maxc = base + (extra ? 1 : 0);
  const size_t per = (size_t)maxc * 3 + 4;
  cudaFree(ctx->d_gather);
  ctx->d_gather = nullptr;
  if (ctx->h_gather) cudaFreeHost(ctx->h_gather);
  ctx->h_gather = nullptr;
  CUDA_TRY(cudaMalloc(&ctx->d_gather, sizeof(double) * per * (comm->world + 1)));
  CUDA_TRY(cudaMallocHost(&ctx->h_gather, sizeof(double) * per * comm->world));
  if (!ctx->d_halo) CUDA_TRY(cudaMalloc(&ctx->d_halo, sizeof(double) * ctx->M));
  if (!ctx->comm_stream)
    CUDA_TRY(cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, -1));
  for (auto& e : ctx->ev_comm)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ctx->comm = comm;
  return PIT_OK;
}

int pit_context_shard(const pit_context* ctx, int* first, int* count) {
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (first) *first = ctx->shard_first;
  if (count) *count = ctx->shard_count;
  return PIT_OK;
}

int pit_sharded_apply_F_device(pit_context* ctx, const double* L_local, double* out_local,
                               void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx || !L_local || !out_local)
    return set_err(PIT_ERR_INVALID_ARGUMENT, "sharded apply_F: null argument");
  if (!ctx->comm) return set_err(PIT_ERR_INVALID_ARGUMENT, "sharded apply_F: no communicator");
  Run R = make_run(ctx, true);
  if (stream) R.st = (cudaStream_t)stream;
  // no status read here (stream-ordered, as pit_apply_F_device):
  // pit_sync_status reports a failing slab
  return run_fine(R, kApplyF, L_local, nullptr, out_local, nullptr);
}

int pit_sharded_sync_status(pit_context* ctx, void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  if (!ctx) return set_err(PIT_ERR_INVALID_ARGUMENT, "null context");
  if (!ctx->comm) return pit_sync_status(ctx, stream);
  Run R = make_run(ctx, true);
  if (stream) R.st = (cudaStream_t)stream;
  const int rc = run_reduce(R, 0);  // every rank's status, nothing else
  CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(DevStatus),
                           cudaMemcpyDeviceToHost, R.st));
  CUDA_TRY(cudaStreamSynchronize(R.st));
  ctx->busy_mark = ctx->h_status->busy_ns;
  return rc;
}

int pit_sharded_pitsbicg_solve_device(pit_context* ctx, const pit_solver_config* cfg,
                                      const double* lambda_init_local, double* lambda_local,
                                      pit_record* records, int max_records, pit_solve_info* info,
                                      void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  return solve_device(0, true, ctx, cfg, lambda_init_local, lambda_local, records, max_records,
                      info, stream);
}

int pit_sharded_parareal_solve_device(pit_context* ctx, const pit_solver_config* cfg,
                                      const double* lambda_init_local, double* lambda_local,
                                      pit_record* records, int max_records, pit_solve_info* info,
                                      void* stream) {
  PIT_DEVICE_SCOPE(ctx);
  return solve_device(1, true, ctx, cfg, lambda_init_local, lambda_local, records, max_records,
                      info, stream);
}

// instrumented builds only: per-phase cycle totals of CTA 0 (warps 0, 1)
extern "C" int pit_debug_phase_timing(pit_context* ctx, int role, long long* out32) {
  PIT_DEVICE_SCOPE(ctx);
#ifdef PIT_PHASE_TIMING
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(out32, ctx->role[role].P.timing, 64 * sizeof(long long),
                      cudaMemcpyDeviceToHost));
  return PIT_OK;
#else
  (void)ctx;
  (void)role;
  (void)out32;
  return set_err(PIT_ERR_INVALID_ARGUMENT, "not an instrumented build");
#endif
}

// K1 unit trace of the last fine batch: n rows of {smid, block, t0, t_end,
// t_loaded, t_computed, 0, 0} (ns).
extern "C" int pit_debug_trace(pit_context* ctx, long long* out, int n) {
  PIT_DEVICE_SCOPE(ctx);
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
  if (n > kMaxPieces * ctx->N) n = kMaxPieces * ctx->N;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(out, ctx->d_trace, sizeof(long long) * 8 * (size_t)n, cudaMemcpyDeviceToHost));
  return PIT_OK;
#else
  (void)ctx;
  (void)out;
  (void)n;
  return set_err(PIT_ERR_INVALID_ARGUMENT, "not an instrumented build");
#endif
}

int pit_measure_fp64_peak(int device, double* tflops) {
  if (!tflops) return set_err(PIT_ERR_INVALID_ARGUMENT, "null output");
  DeviceScope device_scope_(device);
  CUDA_TRY(measure_fp64_peak(tflops));
  return PIT_OK;
}

// ---- seeded inputs ---------------------------------------------------------

void pit_seeded_uniform(uint64_t seed, int64_t n, double a, double b, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(a, b);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void pit_seeded_normal(uint64_t seed, int64_t n, double mean, double stddev, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(mean, stddev);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
