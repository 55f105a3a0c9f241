/*
 * pit_b200.h — C ABI of the B200-native PiTSBiCG hot path.
 *
 * The reference (/root/reference/proj) exposes this path only as a C++
 * library API in namespace pit; it has no FFI.  Each entry point below is the
 * flat-array, status-code replacement of one reference function, so a C++
 * shim (paper_2203_10148_b200/host/pit_gpu.hpp, shown in INTEGRATION.md) or a
 * ctypes binding can keep the reference's signatures:
 *
 *   pit_apply_F            <- pit::apply_F              include/pit/block_system.hpp:77-78
 *   pit_assemble_rhs       <- pit::assemble_rhs         include/pit/block_system.hpp:82-83
 *   pit_apply_G_inverse    <- pit::apply_G_inverse      include/pit/block_system.hpp:88-89
 *   pit_initial_guess      <- pit::initial_guess        include/pit/solvers.hpp:69-70
 *   pit_preconditioned_residual
 *                          <- pit::preconditioned_residual include/pit/solvers.hpp:74-75
 *   pit_sequential_fine_solve
 *                          <- pit::sequential_fine_solve include/pit/solvers.hpp:64
 *   pit_propagate          <- pit::Propagator::propagate / propagate_homogeneous /
 *                             source_contribution       include/pit/propagator.hpp:38-44
 *   pit_pitsbicg_solve     <- pit::pitsbicg_solve       include/pit/solvers.hpp:89-90
 *   pit_parareal_solve     <- pit::parareal_solve       include/pit/solvers.hpp:82-83
 *   pit_block_inner_product / pit_block_norm_n_inf
 *                          <- pit::block_inner_product / block_norm_n_inf
 *                                                       include/pit/block_system.hpp:37-40
 *   pit_set_reference      <- pit::SolveOptions::reference  include/pit/solvers.hpp:50-52
 *   pit_context_create     <- pit::BlockOperatorContext ctor (block_system.hpp:55-72)
 *                             + Propagator ctors (propagator.hpp:31-36) + SpatialOperator
 *
 * Data layout: a block vector is caller-owned contiguous double[N*M],
 * block-major, x-fastest (the reference's flat convention,
 * src/dense_oracle.cpp:153-177, src/grid.cpp:35-38).  Host entry points take
 * host pointers and copy; the *_device variants take device pointers
 * (cudaMalloc'd, N*M doubles) and a cudaStream_t passed as void*.
 *
 * Errors (reference exceptions -> status codes, include/pit/errors.hpp):
 *   PIT_ERR_INVALID_ARGUMENT  std::invalid_argument (shapes, slab index)
 *   PIT_ERR_INNER_SOLVE       pit::InnerSolveError (non-finite implicit step)
 *   PIT_ERR_SLAB              pit::SlabError (lowest failing slab of a fine
 *                             batch; pit_last_error_slab() gives the index)
 *   PIT_ERR_CONFIG            pit::ConfigError (solver tolerances)
 *   PIT_ERR_CUDA              CUDA runtime failure / no device
 * pit_last_error() returns the message of the last failure on this thread.
 */
#ifndef PIT_B200_H
#define PIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PIT_OK = 0,
  PIT_ERR_INVALID_ARGUMENT = 1,
  PIT_ERR_INNER_SOLVE = 2,
  PIT_ERR_SLAB = 3,
  PIT_ERR_CONFIG = 4,
  PIT_ERR_CUDA = 5
};

enum { PIT_FINE = 0, PIT_COARSE = 1 };
/* PIT_SOURCE_SEPARABLE: f(t, x_i) = amp sin(omega t + phase) shape[i].
 * PIT_SOURCE_TABLE: a general SourceFn (include/pit/pde.hpp:13) sampled by the
 * caller exactly where Propagator::run samples it (src/propagator.cpp:56-63,
 * the END of every step): source_table_fine[(n*fine_steps + k-1)*M + i] =
 * f(breakpoint(n) + k*dt_fine, x_i), n < N, k = 1..fine_steps, and
 * source_table_coarse likewise with the coarse steps (host arrays, copied;
 * N*steps*M doubles each, so meant for moderate problems).  Each step adds
 * fl(dt*f) to the state, the reference's rhs.axpy(dt, sample_source(t)). */
enum { PIT_SOURCE_NONE = 0, PIT_SOURCE_SEPARABLE = 1, PIT_SOURCE_TABLE = 2 };
enum { PIT_GUESS_COARSE_SWEEP = 0, PIT_GUESS_ZERO = 1 };
enum { PIT_CONVERGED = 0, PIT_MAX_ITERATIONS = 1 };
/* fine propagator scheme: backward Euler (the reference's Propagator,
 * src/propagator.cpp:50-71) or explicit Euler (config 5; not in the
 * reference, which has implicit propagators only) */
enum { PIT_SCHEME_BACKWARD_EULER = 0, PIT_SCHEME_EXPLICIT_EULER = 1 };

/* Problem description: the 1D operator A (dy/dt = -A y + f) as constant
 * tridiagonal bands on M interior nodes of [grid_lo, grid_hi] with Dirichlet
 * walls (assemble_spatial_operator, src/pde.cpp:55-64: lo = -mu/h^2,
 * diag = 2mu/h^2 + r, up = -mu/h^2; any constant bands are accepted, e.g.
 * central-difference advection), the partition (T, N), steps per slab for
 * the fine and coarse propagators, and an optional source sampled at step
 * ends (src/propagator.cpp:61-65): separable, f(t, x_i) = amp * sin(omega*t +
 * phase) * shape[i], or a general SourceFn given as tables (PIT_SOURCE_TABLE).
 * A general tridiagonal operator (variable coefficients) is given per node
 * through `stencil` and solved iteratively, as the reference does. */
typedef struct pit_problem_desc {
  int32_t dimension;      /* 1 */
  int32_t interior;       /* M */
  double grid_lo, grid_hi;
  double band_lo, band_diag, band_up;
  int32_t slab_count;     /* N >= 2 */
  double total_time;      /* T > 0 */
  int32_t fine_steps;     /* >= 1 */
  int32_t coarse_steps;   /* >= 1 */
  int32_t source_kind;    /* PIT_SOURCE_* */
  double source_amp, source_omega, source_phase;
  const double* source_shape; /* [M] host, copied; NULL when no source */
  const double* initial_value;/* [M] host y0, copied */
  int32_t device;         /* CUDA ordinal */
  /* kernel layout per role: points per thread, contiguous sub-chunks per
   * thread chunk, strided segments per slab, warps per slab CTA
   * (sub-chunk length = mpt / (nsub*nseg)); all 0 = auto */
  int32_t fine_mpt, fine_nsub, fine_nseg, fine_warps;
  int32_t coarse_mpt, coarse_nsub, coarse_nseg, coarse_warps;
  /* dimension 2 (config 5): interior = m points per axis on [grid_lo,
   * grid_hi]^2, blocks of M = m*m values (x fastest); the operator is the
   * 5-point stencil band_diag (centre) / band_lo (= band_up, each of the four
   * neighbours), i.e. the reference's 2D assemble_spatial_operator with zero
   * velocity (src/pde.cpp:66-100).  Fine: fine_scheme must be
   * PIT_SCHEME_EXPLICIT_EULER; coarse: backward Euler solved by Jacobi-PCG
   * (solve_cg, src/sparse.cpp:60-114) to coarse_tolerance (0: 1e-12,
   * kInnerSolveRelTol, pde.hpp:78) within coarse_max_iterations (0: 10*M,
   * pde.hpp:79).  No sources in 2D. */
  int32_t fine_scheme;
  double coarse_tolerance;
  int64_t coarse_max_iterations;
  /* K4 layout (tile rows, tile columns, CTAs per cluster, warps per CTA);
   * all 0 = auto */
  int32_t tile_rows, tile_cols, tile_cluster, tile_warps;
  /* dimension 2 with fine_scheme == PIT_SCHEME_BACKWARD_EULER: the
   * reference's desk/paper presets (src/presets.cpp, runner.cpp:75-88).  Both
   * propagators step backward Euler on the general 5-point operator
   * `stencil` (host, [5][M]: the south, west, centre, east, north entries of
   * A per interior node as assemble_spatial_operator emits them,
   * src/pde.cpp:66-100, 0 where a row has no such entry; NULL = the
   * isotropic band_diag / band_lo stencil) and solve every step with
   * Jacobi-PCG, or Jacobi-BiCGStab when `nonsymmetric` (ImplicitStepSolver,
   * src/pde.cpp:112-130), to fine/coarse_tolerance (0: 1e-12) within
   * fine/coarse_max_iterations (0: 10*M).  m <= 101 (grid_points <= 103);
   * a source as PIT_SOURCE_TABLE. */
  /* dimension 1 with `stencil` set: a general tridiagonal operator (any
   * pit::SpatialOperator the reference's 1D propagators accept through the
   * CSR constructor, include/pit/pde.hpp:36-37, e.g. variable coefficients):
   * stencil is [3][M], the sub-diagonal, diagonal and super-diagonal entry of
   * A per interior node (0 where absent; band_* are ignored).  Every step is
   * then solved as the reference solves it, Jacobi-PCG or (nonsymmetric)
   * Jacobi-BiCGStab to fine/coarse_tolerance (K6 on a one-row grid);
   * M <= 10240; a source as PIT_SOURCE_TABLE. */
  const double* stencil;
  int32_t nonsymmetric;
  double fine_tolerance;
  int64_t fine_max_iterations;
  /* PIT_SOURCE_TABLE (1D): see the enum above */
  const double* source_table_fine;
  const double* source_table_coarse;
} pit_problem_desc;

typedef struct pit_context pit_context;

/* Mirrors pit::RunStats (include/pit/executor.hpp:24-30), accumulated. */
typedef struct pit_run_stats {
  int64_t fine_applications;
  int64_t coarse_applications;
  double fine_parallel_ms;
  double fine_busy_ms;
  double coarse_sequential_ms;
} pit_run_stats;

/* One convergence-history row (include/pit/solvers.hpp:17-24).
 * error_vs_reference = block_norm_n_inf(lambda - reference) when a reference
 * is set (pit_set_reference; SolveOptions::reference), has_error = 1. */
typedef struct pit_record {
  int32_t k;
  double residual_norm;
  int64_t fine_applications;
  int64_t coarse_applications;
  double wall_ms;
  double error_vs_reference;
  int32_t has_error;
} pit_record;

/* Solver configuration (include/pit/solvers.hpp:36-44). */
typedef struct pit_solver_config {
  double tolerance;          /* default 1e-8 */
  double restart_tolerance;  /* default 1e-12 */
  int32_t max_iterations;    /* default 200 */
  int32_t initial_guess;     /* PIT_GUESS_* */
} pit_solver_config;

typedef struct pit_solve_info {
  int32_t status;            /* PIT_CONVERGED / PIT_MAX_ITERATIONS */
  int32_t restarts;
  int32_t record_count;      /* rows written (<= max_records) */
  int32_t total_records;     /* rows produced */
  double min_restart_margin; /* min |<r,r~>|/eps0 at the restart test */
  pit_run_stats stats;
} pit_solve_info;

/* Per-role step coefficients of the chunked constant-factor backward-Euler
 * solve, exported so tests can check that the oracle's own
 * recipe produces identical bits. */
typedef struct pit_step_coeffs {
  int32_t M, mpt, nsub, nseg, warps, steps;
  double delta, lam, mu;
  double dstar, nl, nu, inv, gneg;
  int32_t K0, R;
  double invR, invLast;
  double pS, qS;          /* nl^sub, nu^sub, sub = mpt/(nsub*nseg) */
  double Pseg, Qseg;      /* nl^lseg, nu^lseg, lseg = 32*warps*nsub*sub */
  double nlpow[32];       /* nl^j, j < sub  (narrow corner) */
  double pw[8];           /* nl^(u*sub), u < nsub (narrow corner) */
  int32_t narrow;         /* corner correction in geometric form */
  double pp[5], qq[5], p32, q32;
  double plane[32], qlane[32];
  /* Kogge-Stone stages per direction: terms whose weight (nl^ch)^d, d > 2^s,
   * is <= 2^-70 are dropped (the same rule as K0): 5 = exact warp scan */
  int32_t scan_f, scan_b;
} pit_step_coeffs;

const char* pit_last_error(void);
int pit_last_error_slab(void);
/* The payload of the last PIT_ERR_INNER_SOLVE on this thread
 * (pit::InnerSolveError::achieved_relative_residual / iterations,
 * include/pit/errors.hpp:15-21, thrown at src/pde.cpp:119-128): the inner
 * Krylov solve's relative true residual and iteration count of the failing
 * step (2D propagators; the 1D direct solve reports NaN and 0).  Returns
 * PIT_ERR_INVALID_ARGUMENT when the last error carried no payload. */
int pit_last_error_detail(double* achieved_relative_residual, int64_t* iterations);
const char* pit_version(void);
int pit_device_count(void);

int pit_context_create(const pit_problem_desc* desc, pit_context** out);
int pit_context_destroy(pit_context* ctx);
int pit_context_shape(const pit_context* ctx, int* M, int* N, double* spacing);
/* cumulative inner CG iterations of the 2D coarse sweeps (0 in 1D, where
 * the coarse step is a direct tridiagonal solve) */
int pit_coarse_iterations(const pit_context* ctx, int64_t* out);
/* Fine slabs resident at once on the context's GPU (K1 occupancy x SMs):
 * the device's worker count for pit::timing_report (src/executor.cpp:156-171),
 * whose parallel_efficiency = fine_busy_ms / (slots * fine_parallel_ms). */
int pit_context_slots(const pit_context* ctx, int* slots);
/* Page-locked host buffers (cudaMallocHost): host block vectors here take
 * pit_apply_F's overlapped path — the input goes up in chunks while the
 * kernel already runs, the output is stored into the (device-mapped) buffer
 * by the kernel itself (staging for C++ bindings whose own storage is
 * pageable, e.g. the reference's BlockVector). */
int pit_host_alloc(size_t bytes, void** out);
int pit_host_free(void* p);
/* Coefficients for role PIT_FINE / PIT_COARSE (no device needed). */
int pit_step_coefficients(const pit_problem_desc* desc, int role, pit_step_coeffs* out);

/* 2D (config 5) step coefficients, as used by the kernels:
 *   fine explicit Euler y' = fma(ac, y, an*((yW + yE) + (yN + yS))),
 *     ac = 1 - dt_f*diag, an = -dt_f*off (long double, rounded once);
 *   coarse BE matrix I + dt_c*A: centre D = diag*dt_c + 1, neighbour
 *     O = off*dt_c (ImplicitStepSolver, src/pde.cpp:106-109), minv = 1/D;
 *   K5 decomposition: cluster CTAs of `threads` threads, `rows` rows each
 *     (sets the CG reduction order). */
typedef struct pit_step_coeffs_2d {
  int32_t m, fine_steps, coarse_steps;
  double ac, an;
  /* scaled form (an a power of two, kappa = ac/an exact): the kernel carries
   * z = y / an^j and steps z' = fma(kappa, z, (zW + zE) + (zN + zS)), folding
   * an^R back every R steps and an^(steps mod R) at the end — the same bits
   * as the unscaled form wherever no value is subnormal */
  int32_t scaled, R;
  double kappa, anR, anLast;
  double D, O, minv;
  double rel_tol;
  int64_t cap;
  int32_t rows, cluster, threads;
  int32_t tile_rows, tile_cols, tile_cluster, tile_warps;
} pit_step_coeffs_2d;
int pit_step_coefficients_2d(const pit_problem_desc* desc, pit_step_coeffs_2d* out);
/* zc correction vector (first K0 entries used), length M (no device needed). */
int pit_step_correction(const pit_problem_desc* desc, int role, double* zc_out);
/* per-thread weights, length 32*warps each (no device needed): segment-carry
 * weights nl^(t*ch), nu^((T-1-t)*ch) and narrow-corner weights zc_0 nl^(t*ch). */
int pit_step_positions(const pit_problem_desc* desc, int role, double* ppos_out, double* qpos_out,
                       double* zt_out);

/* ---- host-pointer entry points (copy in, compute, copy out) ---------- */
/* pit_apply_F with page-locked L and out (cudaHostAlloc / cudaHostRegister /
 * torch pin_memory) overlaps the copies with the fine batch: the input goes
 * up in chunks of blocks, K1's slabs start as their chunk lands and their
 * output chunks go back as they complete (same kernel, same bits).  Pageable
 * buffers take the sequential copy-compute-copy path. */
int pit_apply_F(pit_context* ctx, const double* L, double* out, pit_run_stats* stats);
int pit_assemble_rhs(pit_context* ctx, double* rhs, pit_run_stats* stats);
int pit_apply_G_inverse(pit_context* ctx, const double* V, double* out, pit_run_stats* stats);
int pit_initial_guess(pit_context* ctx, int policy, double* out, pit_run_stats* stats);
int pit_preconditioned_residual(pit_context* ctx, const double* lambda, const double* rhs,
                                double* out, pit_run_stats* stats);
int pit_sequential_fine_solve(pit_context* ctx, double* out);
/* role PIT_FINE/PIT_COARSE; with_source 1 = propagate, 0 = propagate_homogeneous;
 * in == NULL means the zero field (source_contribution). */
int pit_propagate(pit_context* ctx, int role, int with_source, const double* in, int slab,
                  double* out);
int pit_block_inner_product(pit_context* ctx, const double* a, const double* b, double* out);
int pit_block_norm_n_inf(pit_context* ctx, const double* a, double* out);

/* SolveOptions::iterate_observer (include/pit/solvers.hpp:54, called at
 * src/solvers.cpp:101,136): after each history row of the following solves
 * the observer receives the row and the iterate it describes as a host array
 * lambda[N*M] (valid for the duration of the call).  NULL clears it.  While
 * an observer is set every row costs one device-to-host copy of lambda. */
typedef void (*pit_iterate_observer)(const pit_record* row, const double* lambda, int N, int M,
                                     void* user);
int pit_set_iterate_observer(pit_context* ctx, pit_iterate_observer fn, void* user);

/* SolveOptions::reference (solvers.hpp:50-52): a host block vector [N*M]
 * kept on the device; every history row of the following solves carries
 * block_norm_n_inf(lambda - reference).  NULL clears it. */
int pit_set_reference(pit_context* ctx, const double* reference);

/* Full solve.  lambda_out [N*M]; lambda_init optional override [N*M];
 * first_residual_out optional [N*M]; records optional [max_records]. */
int pit_pitsbicg_solve(pit_context* ctx, const pit_solver_config* cfg, const double* lambda_init,
                       double* lambda_out, double* first_residual_out, pit_record* records,
                       int max_records, pit_solve_info* info);
int pit_parareal_solve(pit_context* ctx, const pit_solver_config* cfg, const double* lambda_init,
                       double* lambda_out, double* first_residual_out, pit_record* records,
                       int max_records, pit_solve_info* info);

/* ---- device-pointer entry points (stream = cudaStream_t or NULL) ----- */
/* Slab-range forms for slab-sharded multi-GPU drivers: blocks are indexed
 * globally; the device arrays hold blocks [first, first+count) at offset 0,
 * halo = block first-1 (NULL when first == 0). */
int pit_apply_F_device(pit_context* ctx, const double* L, const double* halo, double* out,
                       int first, int count, void* stream);
int pit_residual_device(pit_context* ctx, const double* lambda, const double* halo,
                        const double* rhs, double* out, int first, int count, void* stream);
int pit_coarse_sweep_device(pit_context* ctx, const double* V, const double* W_prev, double* W,
                            int first, int count, int with_source, int add_v, void* stream);
int pit_block_partials_device(pit_context* ctx, const double* a, const double* b, double* partials,
                              int count, void* stream);
/* Two fused partials per block: partials[2b] = h<a0,b0>, partials[2b+1] = h<a1,b1>. */
int pit_block_partials2_device(pit_context* ctx, const double* a0, const double* b0,
                               const double* a1, const double* b1, double* partials, int count,
                               void* stream);
/* BiCGStab vector phases (pitsbicg_solve's op order, src/solvers.cpp:168-214),
 * on `count` blocks of M doubles, fused with their reductions:
 *   update_s:  s = r - alpha d;                    partials[b] = h<s,s>
 *   update_lr: lam += alpha p; lam += omega s; r = s - omega t;
 *              partials[2b] = h<r,r>, partials[2b+1] = h<r,rs>
 *   update_p:  p = (p - omega d) * beta + r
 *   axpy:      y = y + a x          add: y = y + x */
int pit_update_s_device(pit_context* ctx, double alpha, const double* r, const double* d, double* s,
                        double* partials, int count, void* stream);
int pit_update_lr_device(pit_context* ctx, double alpha, double omega, const double* p,
                         const double* s, const double* t, const double* rs, double* lam, double* r,
                         double* partials, int count, void* stream);
int pit_update_p_device(pit_context* ctx, double omega, double beta, const double* d,
                        const double* r, double* p, int count, void* stream);
int pit_axpy_device(pit_context* ctx, double a, const double* x, double* y, int count, void* stream);
int pit_add_device(pit_context* ctx, const double* x, double* y, int count, void* stream);
/* assemble_rhs blocks [first, first+count) without block 0's y0:
 * out_n = fine.source_contribution(n-1) for n >= 1, zero for n = 0 and when
 * the problem has no source (block_system.cpp:149-172). */
int pit_fine_source_device(pit_context* ctx, double* out, int first, int count, void* stream);
int pit_sync_status(pit_context* ctx, void* stream);
int pit_pitsbicg_solve_device(pit_context* ctx, const pit_solver_config* cfg,
                              const double* lambda_init_dev, double* lambda_dev,
                              pit_record* records, int max_records, pit_solve_info* info,
                              void* stream);

/* ---- slab-sharded multi-GPU (one rank per GPU) -------- */
/* Replaces the reference's slab fan-out (block_system.cpp:123-132,
 * executor.cpp:105-154) across GPUs.  Every rank creates a context for the
 * whole problem (N = all slabs) on its own GPU, and attaches a communicator;
 * it then owns the contiguous slab range (first, count) = the first N % world
 * ranks get ceil(N/world) blocks, the others floor(N/world).  Traffic: one
 * halo block per rank pair per fine batch, the coarse chain's W block per
 * rank pair per sweep, and an all-gather of per-block reduction partials,
 * summed in global slab order on every rank, so histories are bit-identical
 * to one GPU's for any world size.
 * Transports: NCCL (rank 0 makes the id with pit_comm_nccl_unique_id, the
 * caller distributes it) or host callbacks (blocking, on host buffers). */
typedef struct pit_comm pit_comm;
typedef struct pit_comm_ops {
  int (*send)(const double* buf, size_t n, int peer, void* user);
  int (*recv)(double* buf, size_t n, int peer, void* user);
  int (*allgather)(const double* in, size_t n, double* out /* [world*n] */, void* user);
  void* user;
} pit_comm_ops;
int pit_comm_nccl_unique_id(unsigned char* id /* [128] */);
int pit_comm_create_nccl(const unsigned char* id /* [128] */, int rank, int world, int device,
                         pit_comm** out);
int pit_comm_create_host(const pit_comm_ops* ops, int rank, int world, pit_comm** out);
int pit_comm_destroy(pit_comm* comm);
/* NULL detaches (the context is single-GPU again); the comm must outlive its
 * use by the context */
int pit_context_attach_comm(pit_context* ctx, pit_comm* comm);
int pit_context_shard(const pit_context* ctx, int* first, int* count);
/* Sharded operators and solvers on the rank's local blocks (device arrays of
 * count*M doubles, block `first` at offset 0).  apply_F overlaps the halo
 * exchange with the interior slabs: the rank's first block waits for the
 * halo, every other block starts at once. */
int pit_sharded_apply_F_device(pit_context* ctx, const double* L_local, double* out_local,
                               void* stream);
/* Collective pit_sync_status: every rank returns the error of the lowest
 * failing slab of any rank (a SlabError for a fine batch, InnerSolveError
 * with its payload for a sweep). */
int pit_sharded_sync_status(pit_context* ctx, void* stream);
int pit_sharded_pitsbicg_solve_device(pit_context* ctx, const pit_solver_config* cfg,
                                      const double* lambda_init_local, double* lambda_local,
                                      pit_record* records, int max_records, pit_solve_info* info,
                                      void* stream);
int pit_sharded_parareal_solve_device(pit_context* ctx, const pit_solver_config* cfg,
                                      const double* lambda_init_local, double* lambda_local,
                                      pit_record* records, int max_records, pit_solve_info* info,
                                      void* stream);

/* Measured FP64 FMA throughput of `device` in TFLOP/s (2 flops per DFMA):
 * the roofline denominator for the FP64-pipe-bound fine propagator. */
int pit_measure_fp64_peak(int device, double* tflops);

/* Seeded inputs (the libstdc++ generators of the reference's tests,
 * tests/oracles.cpp:108-122): std::mt19937_64 + uniform_real_distribution /
 * normal_distribution, drawn in order. */
void pit_seeded_uniform(uint64_t seed, int64_t n, double a, double b, double* out);
void pit_seeded_normal(uint64_t seed, int64_t n, double mean, double stddev, double* out);

#ifdef __cplusplus
}
#endif
#endif
