// pit_step.cuh — one backward-Euler step (I + dt*A) y' = y for a slab whose
// M-point state lives in registers across a CTA of 32*WARPS threads.  Each
// thread owns MPT = NSUB*SUB contiguous points, split into NSUB sub-chunks
// of SUB points whose sweeps run interleaved (instruction-level parallelism
// across the sub-chunk chains).  DESIGN.md §3.
//
// Replaces, per slab and step, the reference's ImplicitStepSolver::solve
// (src/pde.cpp:112-130 -> solve_cg/solve_bicgstab, src/sparse.cpp:60-206)
// with a direct tridiagonal solve:
//   y <- U^-1 L^-1 y            constant unit-bidiagonal factors nl, nu,
//        chunked: per-sub-chunk sweeps with zero carry, the thread's end
//        value combined from its sub-chunks, a Kogge-Stone warp scan plus a
//        sequential cross-warp combine for the true thread carries, the
//        sub-chunk carries, and a fix-up y_j += w_j * carry
//   y <- y + (gneg*y_0) zc      corner rank-1 (Sherman-Morrison) correction
// and the diagonal scale inv is deferred: applied as inv^R every R steps
// (homogeneous propagation) or every step when a source is added.
// Every multiply-add is an explicit fma(); oracle/pit_oracle.c
// (chunked_solve) performs the identical operation sequence.
#pragma once

#include <cuda_runtime.h>

namespace pitb {

constexpr unsigned kFull = 0xffffffffu;

struct StepParams {
  double nl, nu, inv, gneg, invR, invLast;
  double pS, qS;            // nl^SUB, nu^SUB (sub-chunk carry weights)
  double fl[32], fu[32];    // fix-up weights nl^(j+1), nu^(SUB-j), j < SUB
  double pp[5], qq[5], p32, q32;  // Kogge-Stone weights, powers of nl^MPT / nu^MPT
  double plane[32], qlane[32];
  int M, steps, R, K0;
  const double* zc;     // [K0] correction vector (device)
  const double* shape;  // [M] source shape g(x_i) (device) or nullptr
  const double* ds;     // [slabs*steps] dt*s(t_k) table (device) or nullptr
};

// Shared memory of one slab CTA: cross-warp carries, broadcast scalar and the
// per-lane carry weights (read with LDS: an indexed constant load would
// serialise across lanes).  The correction vector follows the struct.
template <int WARPS>
struct StepShared {
  double fw[WARPS > 1 ? WARPS : 1];
  double bw[WARPS > 1 ? WARPS : 1];
  double b;
  double pad;
  double plane[32], qlane[32];  // p^lane, q^(31-lane)
};

template <int WARPS>
__device__ __forceinline__ void init_step_shared(const StepParams& P, StepShared<WARPS>& sh,
                                                 int tid) {
  for (int i = tid; i < 32; i += 32 * WARPS) {
    sh.plane[i] = P.plane[i];
    sh.qlane[i] = P.qlane[i];
  }
}

// Kogge-Stone stage: I += c * I[lane -/+ d] on lanes whose source lane exists
// (shfl's in-range predicate guards the DFMA; other lanes keep I).
__device__ __forceinline__ void scan_stage_up(double& I, double c, int d) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, slo, shi;\n\t.reg .f64 t;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "shfl.sync.up.b32 slo|p, lo, %2, 0, -1;\n\t"
      "shfl.sync.up.b32 shi, hi, %2, 0, -1;\n\t"
      "mov.b64 t, {slo, shi};\n\t"
      "@p fma.rn.f64 %0, %1, t, %0;\n\t}"
      : "+d"(I)
      : "d"(c), "r"(d));
}
__device__ __forceinline__ void scan_stage_down(double& J, double c, int d) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, slo, shi;\n\t.reg .f64 t;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "shfl.sync.down.b32 slo|p, lo, %2, 31, -1;\n\t"
      "shfl.sync.down.b32 shi, hi, %2, 31, -1;\n\t"
      "mov.b64 t, {slo, shi};\n\t"
      "@p fma.rn.f64 %0, %1, t, %0;\n\t}"
      : "+d"(J)
      : "d"(c), "r"(d));
}

// s_zc holds the correction vector zero-padded to 32*MPT entries (narrow
// path, K0 <= 32*MPT: only warp 0 touches it) or to the padded slab length
// (wide path); fma(c, 0, y) == y, so padding does not change any bit.
// The lane-0 / lane-31 carry uses weight 1 on a zeroed neighbour value:
// fma(1, W, 0) == W.
template <int SUB, int NSUB, int WARPS>
__device__ __forceinline__ void be_solve(double (&y)[NSUB][SUB], const StepParams& P,
                                         StepShared<WARPS>& sh,
                                         const double* __restrict__ s_zc, int lane, int warp,
                                         int g0, bool ghosts, bool wide) {
  // ---- forward: L^-1 ----
#pragma unroll
  for (int j = 1; j < SUB; ++j)
#pragma unroll
    for (int s = 0; s < NSUB; ++s) y[s][j] = fma(P.nl, y[s][j - 1], y[s][j]);
  double I = y[0][SUB - 1];
#pragma unroll
  for (int s = 1; s < NSUB; ++s) I = fma(P.pS, I, y[s][SUB - 1]);
#pragma unroll
  for (int s = 0; s < 5; ++s) scan_stage_up(I, P.pp[s], 1 << s);
  double Ip = __shfl_up_sync(kFull, I, 1);
  Ip = lane == 0 ? 0.0 : Ip;
  double Wc = 0.0;
  if (WARPS > 1) {
    if (lane == 31) sh.fw[warp] = I;
    __syncthreads();
    for (int v = 0; v < warp; ++v) Wc = fma(P.p32, Wc, sh.fw[v]);
  }
  double Cs[NSUB];
  Cs[0] = fma(sh.plane[lane], Wc, Ip);
#pragma unroll
  for (int s = 1; s < NSUB; ++s) Cs[s] = fma(P.pS, Cs[s - 1], y[s - 1][SUB - 1]);
#pragma unroll
  for (int j = SUB - 1; j >= 0; --j)
#pragma unroll
    for (int s = 0; s < NSUB; ++s) y[s][j] = fma(P.fl[j], Cs[s], y[s][j]);
  if (ghosts) {
#pragma unroll
    for (int s = 0; s < NSUB; ++s)
#pragma unroll
      for (int j = 0; j < SUB; ++j)
        y[s][j] = (g0 + s * SUB + j < P.M) ? y[s][j] : 0.0;  // Dirichlet padding
  }
  // ---- backward: U^-1 ----
#pragma unroll
  for (int j = SUB - 2; j >= 0; --j)
#pragma unroll
    for (int s = 0; s < NSUB; ++s) y[s][j] = fma(P.nu, y[s][j + 1], y[s][j]);
  double J = y[NSUB - 1][0];
#pragma unroll
  for (int s = NSUB - 2; s >= 0; --s) J = fma(P.qS, J, y[s][0]);
#pragma unroll
  for (int s = 0; s < 5; ++s) scan_stage_down(J, P.qq[s], 1 << s);
  double Jn = __shfl_down_sync(kFull, J, 1);
  Jn = lane == 31 ? 0.0 : Jn;
  double Vc = 0.0;
  if (WARPS > 1) {
    if (lane == 0) sh.bw[warp] = J;
    __syncthreads();
    for (int v = WARPS - 1; v > warp; --v) Vc = fma(P.q32, Vc, sh.bw[v]);
  }
  double Rs[NSUB];
  Rs[NSUB - 1] = fma(sh.qlane[lane], Vc, Jn);
#pragma unroll
  for (int s = NSUB - 2; s >= 0; --s) Rs[s] = fma(P.qS, Rs[s + 1], y[s + 1][0]);
#pragma unroll
  for (int j = 0; j < SUB; ++j)
#pragma unroll
    for (int s = 0; s < NSUB; ++s) y[s][j] = fma(P.fu[j], Rs[s], y[s][j]);
  // ---- corner rank-1 correction ----
  if (!wide) {
    if (warp == 0) {
      const double c = P.gneg * __shfl_sync(kFull, y[0][0], 0);
#pragma unroll
      for (int s = 0; s < NSUB; ++s)
#pragma unroll
        for (int j = 0; j < SUB; ++j) y[s][j] = fma(c, s_zc[g0 + s * SUB + j], y[s][j]);
    }
  } else {
    if (warp == 0 && lane == 0) sh.b = y[0][0];
    __syncthreads();
    const double c = P.gneg * sh.b;
#pragma unroll
    for (int s = 0; s < NSUB; ++s)
#pragma unroll
      for (int j = 0; j < SUB; ++j) y[s][j] = fma(c, s_zc[g0 + s * SUB + j], y[s][j]);
  }
}

}  // namespace pitb
