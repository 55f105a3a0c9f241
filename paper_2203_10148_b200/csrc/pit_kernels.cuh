// pit_kernels.cuh — kernel entry points and host launchers (internal).
#pragma once

#include <cuda_runtime.h>

#include "pit_step.cuh"

namespace pitb {

enum SlabMode { kApplyF = 0, kResidual = 1, kPropagate = 2 };

// Per-context device status (pinned host mirror), read back in one copy
// after each operator:
//   slab, sweep_slab  lowest failing slab (INT_MAX = none) of the fine
//            batches (SlabError) and of the sequential sweeps (InnerSolveError)
//   fail[3]  sequential-sweep failure payload of InnerSolveError
//            (include/pit/errors.hpp:15-21): achieved relative residual,
//            inner iterations, kind (0 = the Krylov solve missed its
//            tolerance at the cap or stalled, 1 = non-finite values)
//   busy_ns  summed per-slab durations of the fine batches (cumulative): the
//            device analogue of the executor's per-task busy time
//            (executor.cpp:124-128), feeding RunStats::fine_busy_ms
struct DevStatus {
  int slab;        // fine batches (SlabError)
  int sweep_slab;  // sequential sweeps (InnerSolveError)
  double fail[3];
  unsigned long long busy_ns;
};
constexpr int kFailNotConverged = 0, kFailNonFinite = 1;

// K1: one CTA per slab, all slabs of the batch in parallel.
struct SlabArgs {
  const double* in;    // CTA b reads field in + (b + in_shift)*M (nullptr: zero field)
  const double* halo;  // field used when b + in_shift < 0
  int in_shift;
  const double* Lsub;  // kApplyF / kResidual: CTA b subtracts from Lsub + b*M
  const double* rhs;   // kResidual: rhs + b*M
  double* out;         // out + b*M
  int slab0;           // propagation slab index of CTA 0
  int mode;
  int* status;         // atomicMin of the first slab with a non-finite result
  const double* L0;    // block 0 (done by CTA 0 when non-null):
  const double* rhs0;  //   kApplyF:   out0 = L0
  double* out0;        //   kResidual: out0 = rhs0 - L0
  // Piece scheduling (launch_slab fills pieces/nblk): when the batch exceeds
  // one wave of resident CTAs, each slab's steps are cut into `pieces`
  // consecutive step ranges and a persistent grid pops (piece, slab) units
  // from a queue: the first pieces in slab order, then each later piece as
  // soon as the CTA running its predecessor pushes it.  The state between
  // pieces goes through state + b*M.
  // state == nullptr: one CTA per slab, one launch wave (or more).
  double* state;
  int* sched;   // {head, tail, queue[(pieces-1)*nblk]}, zeroed by the launcher
  int pieces;   // 0 = choose from occupancy (launcher), else forced
  int nblk;     // slabs in the batch (set by the launcher)
  long long* trace;  // PIT_PHASE_TIMING builds: per unit {smid, block, t_start, t_end} (ns)
  // Host-buffer pipelining (pit_apply_F with pinned buffers; nullptr = the
  // input is resident): the input arrives in chunks of chunk_blocks global
  // blocks; the copy stream writes in_ready = k+1 after chunk k.  CTA b
  // (global output block g = b + block_shift) waits for chunk(g) before it
  // loads, and after its output is stored bumps out_done[chunk(g)] (block 0,
  // written by CTA 0, counts in chunk 0), on which the D2H stream waits.
  const unsigned* in_ready;
  unsigned* out_done;
  // host_out != nullptr (the caller's pinned output, mapped): instead of a
  // D2H copy each CTA re-reads its finished block from L2 and streams it to
  // host memory in coalesced 16-byte stores (host_out is block 0's address)
  double* host_out;
  int chunk_blocks;
  int block_shift;
  unsigned long long* busy_ns;  // DevStatus::busy_ns (nullptr: not measured)
  // Overlap with the coarse sweep (apply_GF): after its output block g
  // (global; block 0 too, written by CTA 0) is stored, a CTA publishes
  // ready[g] = epoch (release), which the concurrently running K2 acquires
  // before it reads V_g.  reserve_sms: the persistent grid leaves that many
  // SMs' worth of slots free for K2.
  int* ready;
  int epoch;
  int reserve_sms;
  // device-resident solver loop: the batch is skipped when *skip != 0 (a
  // branch of the iteration was taken by an earlier scalar kernel)
  const int* skip;
};

// K2: one persistent CTA running the sequential sweep
//   W_b = Prop(W_{b-1}) (+ V_b),  W_{-1} = start
struct SweepArgs {
  const double* start;
  const double* V;  // nullptr: no add
  double* W;
  int count;
  int slab0;
  int* status;
  double* fail_info;  // DevStatus::fail, written with the failing slab
  // Overlap with the fine batch producing V (apply_GF, TMA sweep only):
  // V_b (global block b + ready_shift) and `start` (block ready_shift - 1)
  // are read only once ready[...] == epoch; W0 != nullptr: the start block is
  // also copied to W0 (W_0 = V_0, block_system.cpp:181)
  const int* ready;
  int epoch;
  int ready_shift;
  double* W0;
  const int* skip;  // as SlabArgs::skip
};

constexpr int kMaxPieces = 64;

// K2 TMA path: V and W viewed as [rows][16] doubles (128-byte rows),
// 128-byte swizzled boxes of `box_rows` rows (host-encoded tensor maps).
struct __align__(64) SweepTma {
  unsigned char v[128];  // CUtensorMap of V (unused when V == nullptr)
  unsigned char w[128];  // CUtensorMap of W
  int rows;              // rows per slab = M / 16
  int box_rows;          // rows per TMA box (divides rows, <= 256)
  int nbuf;              // slab buffers (3 when shared memory allows, else 2)
};

// The BiCGStab scalars of pitsbicg_solve (src/solvers.cpp:151-214) kept on
// the device: one thread sums the per-block partials in slab order, exactly
// as the host loop does, and sets the branch the reference would take.
struct SolverScalars {
  double rho, d_dot, alpha, s_norm, tt, ts, omega, r_norm, rr, r_dot, beta, margin;
  int flag;  // ScalarFlag
  int stop;  // != 0: the rest of the iteration's kernels skip their work
};
enum ScalarPhase { kScRho = 0, kScAlpha = 1, kScSnorm = 2, kScOmega = 3, kScR = 4 };
enum ScalarFlag {
  kFlagNone = 0,
  kFlagRestartD = 1,    // |<d, r~>| < 1e-300        (solvers.cpp:161-165)
  kFlagHalf = 2,        // ||s|| <= tol: half step   (171-178)
  kFlagRestartT = 3,    // <t, t> < 1e-300           (181-185)
  kFlagRestartW = 4,    // |omega| < 1e-300          (187-190)
  kFlagConverged = 5,   // ||r|| <= tol              (198-201)
  kFlagRestartR = 6     // |<r, r~>| <= eps0         (203-209)
};
cudaError_t launch_scalars(SolverScalars* sc, const double* partials, int N, int phase, double tol,
                           double eps0, cudaStream_t st);

// Launchers; return cudaErrorInvalidConfiguration for an uncompiled layout.
cudaError_t launch_slab(int mpt, int nsub, int nseg, int warps, bool src, const StepParams& P,
                        const SlabArgs& A, int ctas, cudaStream_t st);
cudaError_t launch_sweep(int mpt, int nsub, int nseg, int warps, bool src, const StepParams& P,
                         const SweepArgs& A, cudaStream_t st);
// resident K1 CTAs per wave for the layout (occupancy x SMs)
cudaError_t slab_slots(int mpt, int nsub, int nseg, int warps, bool src, const StepParams& P,
                       int* slots);

// K3: block-vector algebra, one CTA (kVecThreads) per block, fixed reduction
// order (oracle/pit_oracle.c orc_block_partial, ORC_MODE_DEVICE).
constexpr int kVecThreads = 256;
// partials[b*np + k] = weight * <a_k, b_k> over block b, k < np (np <= 3)
cudaError_t launch_dots(int M, int blocks, double weight, int np, const double* const* a,
                        const double* const* b, double* partials, cudaStream_t st,
                        const SolverScalars* sc = nullptr);
// s = r - alpha*d (fma), partials[b] = weight*<s,s>
// sc != nullptr: alpha (omega, beta) are read from sc and the kernel is
// skipped when sc->stop is set
cudaError_t launch_update_s(int M, int blocks, double weight, double alpha, const double* r,
                            const double* d, double* s, double* partials, cudaStream_t st,
                            const SolverScalars* sc = nullptr);
// lam = fma(alpha,p,lam); lam = fma(omega,s,lam); r = fma(-omega,t,s);
// partials[2b] = weight*<r,r>, partials[2b+1] = weight*<r,rs>
cudaError_t launch_update_lr(int M, int blocks, double weight, double alpha, double omega,
                             const double* p, const double* s, const double* t, const double* rs,
                             double* lam, double* r, double* partials, cudaStream_t st,
                             const SolverScalars* sc = nullptr);
// p = fma(fma(-omega, d, p), beta, r)
cudaError_t launch_update_p(size_t n, double omega, double beta, const double* d, const double* r,
                            double* p, cudaStream_t st, const SolverScalars* sc = nullptr);
// y = fma(a, x, y)
cudaError_t launch_axpy(size_t n, double a, const double* x, double* y, cudaStream_t st,
                        const double* a_dev = nullptr);
// y = y + x
cudaError_t launch_add(size_t n, const double* x, double* y, cudaStream_t st);
// measured FP64 DFMA throughput of the current device (TFLOP/s)
cudaError_t measure_fp64_peak(double* tflops);

}  // namespace pitb
