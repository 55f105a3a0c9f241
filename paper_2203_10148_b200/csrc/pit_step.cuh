// pit_step.cuh — one backward-Euler step (I + dt*A) y' = y for a slab whose
// M-point state lives in registers across a CTA of 32*WARPS threads, MPT
// contiguous points per thread.
//
// Replaces, per slab and step, the reference's ImplicitStepSolver::solve
// (src/pde.cpp:112-130 -> solve_cg/solve_bicgstab, src/sparse.cpp:60-206)
// with a direct tridiagonal solve:
//   y <- U^-1 L^-1 y            constant unit-bidiagonal factors nl, nu
//        (chunked: per-thread sweep with zero carry, Kogge-Stone warp scan of
//         the chunk end values plus a sequential cross-warp combine for the
//         true carries, and a fix-up y_j += w_j * carry)
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
  double fl[32], fu[32];
  double pp[5], qq[5], p32, q32;
  double plane[32], qlane[32];
  int M, steps, R, K0;
  const double* zc;     // [K0] correction vector (device)
  const double* shape;  // [M] source shape g(x_i) (device) or nullptr
  const double* ds;     // [slabs*steps] dt*s(t_k) table (device) or nullptr
};

// Shared memory of one slab CTA: cross-warp carries, broadcast scalar, and
// the step's coefficient tables (read with LDS instead of indexed constant
// loads, which serialise across lanes).  The correction vector follows.
template <int MPT, int WARPS>
struct StepShared {
  double fw[WARPS > 1 ? WARPS : 1];
  double bw[WARPS > 1 ? WARPS : 1];
  double b;
  double pad;
  double plane[32], qlane[32]; // per-lane carry weights p^lane, q^(31-lane)
};

template <int MPT, int WARPS>
__device__ __forceinline__ void init_step_shared(const StepParams& P, StepShared<MPT, WARPS>& sh,
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
template <int MPT, int WARPS>
__device__ __forceinline__ void be_solve(double (&y)[MPT], const StepParams& P,
                                         StepShared<MPT, WARPS>& sh,
                                         const double* __restrict__ s_zc, int lane, int warp,
                                         int g0, bool ghosts, bool wide) {
  // ---- forward: L^-1 ----
#pragma unroll
  for (int j = 1; j < MPT; ++j) y[j] = fma(P.nl, y[j - 1], y[j]);
  double I = y[MPT - 1];
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
  const double Cc = fma(sh.plane[lane], Wc, Ip);
#pragma unroll
  for (int j = MPT - 1; j >= 0; --j) y[j] = fma(P.fl[j], Cc, y[j]);
  if (ghosts) {
#pragma unroll
    for (int j = 0; j < MPT; ++j) y[j] = (g0 + j < P.M) ? y[j] : 0.0;  // Dirichlet padding
  }
  // ---- backward: U^-1 ----
#pragma unroll
  for (int j = MPT - 2; j >= 0; --j) y[j] = fma(P.nu, y[j + 1], y[j]);
  double J = y[0];
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
  const double Rc = fma(sh.qlane[lane], Vc, Jn);
#pragma unroll
  for (int j = 0; j < MPT; ++j) y[j] = fma(P.fu[j], Rc, y[j]);
  // ---- corner rank-1 correction ----
  if (!wide) {
    if (warp == 0) {
      const double c = P.gneg * __shfl_sync(kFull, y[0], 0);
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = fma(c, s_zc[g0 + j], y[j]);
    }
  } else {
    if (warp == 0 && lane == 0) sh.b = y[0];
    __syncthreads();
    const double c = P.gneg * sh.b;
#pragma unroll
    for (int j = 0; j < MPT; ++j) y[j] = fma(c, s_zc[g0 + j], y[j]);
  }
}

// Full slab propagation: steps BE steps, homogeneous (deferred scaling) or
// with the separable source sampled at each step end.  ds points at this
// slab's row of the dt*s(t_k) table; g holds the thread's source shape.
template <int MPT, int WARPS, bool SRC>
__device__ __forceinline__ void propagate_slab(double (&y)[MPT], const StepParams& P,
                                               StepShared<MPT, WARPS>& sh,
                                               const double* __restrict__ s_zc, int lane,
                                               int warp, int g0, const double* __restrict__ ds,
                                               const double (&g)[MPT]) {
  const bool ghosts = P.M < 32 * WARPS * MPT;
  const bool wide = P.K0 > 32 * MPT;
  if (SRC) {
    double dsk = ds[0];
    for (int k = 0; k < P.steps; ++k) {
      const double dsn = (k + 1 < P.steps) ? ds[k + 1] : 0.0;
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = fma(dsk, g[j], y[j]);
      be_solve<MPT, WARPS>(y, P, sh, s_zc, lane, warp, g0, ghosts, wide);
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = y[j] * P.inv;
      dsk = dsn;
    }
  } else {
    int cnt = 0;
    for (int k = 0; k < P.steps; ++k) {
      be_solve<MPT, WARPS>(y, P, sh, s_zc, lane, warp, g0, ghosts, wide);
      if (++cnt == P.R) {
        cnt = 0;
#pragma unroll
        for (int j = 0; j < MPT; ++j) y[j] = y[j] * P.invR;
      }
    }
    if (cnt) {
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = y[j] * P.invLast;
    }
  }
}

}  // namespace pitb
