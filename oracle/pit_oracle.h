/*
 * pit_oracle.h — CPU restatement of the reference PiTSBiCG hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is linked into, loaded by,
 * or called from the product (paper_2203_10148_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker.
 *
 * What it restates (reference = /root/reference/proj):
 *   - the solver control flow and op order of pitsbicg_solve
 *     (src/solvers.cpp:116-220), parareal_solve (73-114), initial_guess
 *     (49-64), preconditioned_residual (66-71), sequential_fine_solve (40-47);
 *   - apply_F / assemble_rhs / apply_G_inverse (src/block_system.cpp:115-195);
 *   - block_inner_product / block_norm_n_inf (block_system.cpp:76-87) and
 *     inner_product / l2_norm (src/grid.cpp:107-118);
 *   - Propagator::run (src/propagator.cpp:50-71): steps_per_slab backward
 *     Euler steps, source sampled at the step END.
 *
 * Two arithmetic modes for the block-vector algebra:
 *   ORC_MODE_REFERENCE  the reference's own op order (sequential per-block
 *                       sums, y += a*x as a separate multiply and add);
 *                       driven by the reference's Propagator (oracle/_ref)
 *                       it reproduces pit::pitsbicg_solve bit for bit.
 *   ORC_MODE_DEVICE     the op order of the CUDA kernels (fixed-tree block
 *                       reductions, fused multiply-adds); driven by the
 *                       mirrored propagator below it is the parity oracle
 *                       for the GPU path, bit for bit.
 *
 * Two propagators:
 *   orc_stepper_*       CPU copy of the CUDA chunked tridiagonal algorithm
 *                       (same coefficient recipe, same chunking, same scans).
 *   orc_thomas_*        plain sequential Thomas elimination, an
 *                       algorithm-independent cross-check.
 */
#ifndef PIT_ORACLE_H
#define PIT_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_M 64

enum { ORC_MODE_REFERENCE = 0, ORC_MODE_DEVICE = 1 };
enum { ORC_FINE = 0, ORC_COARSE = 1 };

/* Coefficients of the chunked constant-factor backward-Euler step.  Mirrors
 * pit_step_coeffs in include/pit_b200.h field for field. */
typedef struct orc_stepper {
  int M;          /* interior points */
  int m;          /* points per thread */
  int nsub;       /* contiguous sub-chunks per thread chunk */
  int nseg;       /* strided segments; sub = m / (nsub*nseg) */
  int warps;      /* warps per slab CTA */
  int Mp;         /* padded length = 32*warps*m */
  int steps;      /* BE steps per slab */
  double delta, lam, mu;   /* I + dt*A: diagonal, sub, super */
  double dstar, nl, nu, inv;
  double gneg;             /* -gamma' of the corner rank-1 correction */
  int K0;                  /* correction extent */
  double pS, qS;           /* nl^sub, nu^sub */
  double Pseg, Qseg;       /* nl^lseg, nu^lseg, lseg = 32*warps*nsub*sub */
  double nlpow[32];        /* nl^j, j < sub (narrow corner) */
  double pw[8];            /* nl^(u*sub), u < nsub (narrow corner) */
  int narrow;              /* corner in geometric form */
  double pp[5], qq[5], p32, q32;
  double plane[32], qlane[32];
  int R;                   /* rescale period, homogeneous propagation */
  double invR, invLast;    /* inv^R, inv^(steps % R) */
  double* zc;              /* [M] correction vector z' (entries >= K0 unused) */
  double* ppos;            /* [32*warps] nl^(t*ch), ch = nsub*sub */
  double* qpos;            /* [32*warps] nu^((T-1-t)*ch) */
  double* zt;              /* [32*warps] zc_0 nl^(t*ch) */
  int scan_f, scan_b;      /* warp-scan stages kept per direction: the first
                              dropped term has weight (nl^ch)^(2^s) <= 2^-70 */
} orc_stepper;

int orc_stepper_init(orc_stepper* s, int M, int m, int nsub, int nseg, int warps, int steps,
                     double band_lo, double band_diag, double band_up, double dt);
void orc_stepper_free(orc_stepper* s);

/* Propagate one slab: in[M] -> out[M].  ds (length steps) is dt*s(t_k) for
 * the separable source f = s(t) g(x) sampled at step ends, or NULL for the
 * homogeneous map; g[M] is the spatial shape. */
void orc_stepper_propagate(const orc_stepper* s, const double* in, const double* ds,
                           const double* g, double* out);

/* ... with a general source: tab[k*M + i] = fl(dt*f(t_k, x_i)) */
void orc_stepper_propagate_table(const orc_stepper* s, const double* in, const double* tab,
                                 double* out);

/* Plain Thomas, the textbook algorithm (no chunking, no deferred scaling).
 * ds == NULL and g != NULL: g is a general-source table [steps][M] of fl(dt*f). */
void orc_thomas_propagate(int M, int steps, double band_lo, double band_diag, double band_up,
                          double dt, const double* in, const double* ds, const double* g,
                          double* out);

/* Propagator callback: role ORC_FINE / ORC_COARSE, with_source 0/1. */
typedef int (*orc_prop_fn)(void* user, int role, int with_source, const double* in, int slab,
                           double* out);

typedef struct orc_problem {
  int M;            /* values per block */
  int N;            /* slab count = block count */
  double weight;    /* h^d of inner_product (grid.cpp:113-114) */
  int has_source;
  int mode;         /* ORC_MODE_* */
  const double* y0; /* [M] */
  orc_prop_fn prop;
  void* user;
  /* 1: the fine propagator is re-entrant, so the independent slabs of
   * apply_F / assemble_rhs run on OpenMP threads (the per-slab arithmetic is
   * unchanged, so results are bitwise independent of the thread count);
   * 0 (callback problems, e.g. the reference's Propagator through Python):
   * slabs run in order on the calling thread */
  int parallel;
} orc_problem;

typedef struct orc_record {
  int k;
  double residual;
  long fine_applications;
  long coarse_applications;
} orc_record;

typedef struct orc_history {
  orc_record* records; /* caller-provided, capacity max_records */
  int max_records;
  int count;
  int converged;       /* 1 Converged, 0 MaxIterations */
  int restarts;
  long fine_applications, coarse_applications;
  double min_restart_margin; /* min |<r,r~>| / eps0 seen at the restart test */
} orc_history;

/* Block-vector primitives in the selected mode. */
double orc_block_dot(const orc_problem* p, const double* a, const double* b);
double orc_block_norm(const orc_problem* p, const double* a);
double orc_block_partial(const orc_problem* p, const double* a, const double* b); /* one block */

int orc_apply_F(const orc_problem* p, const double* L, double* out, orc_history* h);
int orc_assemble_rhs(const orc_problem* p, double* rhs, orc_history* h);
int orc_apply_G_inverse(const orc_problem* p, const double* V, double* out, orc_history* h);
int orc_initial_guess(const orc_problem* p, int zero, double* out, orc_history* h);
int orc_sequential_fine(const orc_problem* p, double* out);
int orc_preconditioned_residual(const orc_problem* p, const double* lambda, const double* rhs,
                                double* out, orc_history* h);

/* pitsbicg_solve: lambda [N*M] out; lambda_init optional override; first_residual optional. */
int orc_pitsbicg(const orc_problem* p, double tol, double eps0, int max_iter, int zero_guess,
                 const double* lambda_init, double* lambda, double* first_residual,
                 orc_history* h);
int orc_parareal(const orc_problem* p, double tol, double eps0, int max_iter, int zero_guess,
                 const double* lambda_init, double* lambda, double* first_residual,
                 orc_history* h);

orc_problem* orc_problem_new(int M, int N, double weight, int has_source, int mode,
                             const double* y0, orc_prop_fn prop, void* user);
void orc_problem_delete(orc_problem* p);
/* one propagation through the problem's callback (tests) */
int orc_problem_propagate(const orc_problem* p, int role, int with_source, const double* in,
                          int slab, double* out);

/* Elementwise BiCGStab phases in the device op order (tests of sharded drivers). */
void orc_vec_update_s(long n, double alpha, const double* r, const double* d, double* s);
void orc_vec_update_lr(long n, double alpha, double omega, const double* p, const double* s,
                       const double* t, double* lam, double* r);
void orc_vec_update_p(long n, double omega, double beta, const double* d, const double* r,
                      double* p);
void orc_vec_axpy(long n, double a, const double* x, double* y);

/* Convenience: a 1D problem whose propagators are orc_stepper (mirrored) or
 * plain Thomas.  Owns its steppers and source tables. */
typedef struct orc_1d orc_1d;
orc_1d* orc_1d_create(int M, double h, double band_lo, double band_diag, double band_up, int N,
                      double total_time, int fine_steps, int coarse_steps, int fine_m,
                      int fine_nsub, int fine_nseg, int fine_warps, int coarse_m,
                      int coarse_nsub, int coarse_nseg, int coarse_warps, const double* y0,
                      int has_source, const double* src_shape, double src_amp,
                      double src_omega, double src_phase, int use_thomas, int mode);
void orc_1d_destroy(orc_1d* o);
/* general source (PIT_SOURCE_TABLE): f(t_k, x_i) per role, [N][steps][M] */
int orc_1d_set_source_tables(orc_1d* o, const double* fine, const double* coarse);
const orc_problem* orc_1d_problem(orc_1d* o);
const orc_stepper* orc_1d_stepper(orc_1d* o, int role);
/* ds table for slab n: dt*amp*sin(omega*t_k + phase), t_k = n*(T/N) + k*dt, k = 1..steps */
const double* orc_1d_ds(orc_1d* o, int role, int slab);

#ifdef __cplusplus
}
#endif
#endif
