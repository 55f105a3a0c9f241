// pit_step.cuh — one backward-Euler step (I + dt*A) y' = y for a slab whose
// M-point state lives in registers across a CTA of 32*WARPS threads, MPT
// contiguous points per thread.
//
// Replaces, per slab and step, the reference's ImplicitStepSolver::solve
// (src/pde.cpp:112-130 -> solve_cg/solve_bicgstab, src/sparse.cpp:60-206)
// with a direct tridiagonal solve:
//   y <- U^-1 L^-1 y            constant unit-bidiagonal factors nl, nu
//        (chunked: per-thread sweep, Kogge-Stone warp scan of the chunk
//         carries, sequential cross-warp carry, fix-up)
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

// Shared-memory layout used by the step: s_fw[WARPS], s_bw[WARPS], s_b[1]
// (broadcast), s_zc[K0] (correction vector).
template <int WARPS>
struct StepShared {
  double fw[WARPS > 1 ? WARPS : 1];
  double bw[WARPS > 1 ? WARPS : 1];
  double b;
};

template <int MPT, int WARPS>
__device__ __forceinline__ void be_solve(double (&y)[MPT], const StepParams& P, double plane,
                                         double qlane, StepShared<WARPS>& sh,
                                         const double* __restrict__ s_zc, int lane, int warp,
                                         int g0) {
  // ---- forward: L^-1 ----
#pragma unroll
  for (int j = 1; j < MPT; ++j) y[j] = fma(P.nl, y[j - 1], y[j]);
  double I = y[MPT - 1];
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const double t = __shfl_up_sync(kFull, I, 1 << s);
    if (lane >= (1 << s)) I = fma(P.pp[s], t, I);
  }
  const double Ip = __shfl_up_sync(kFull, I, 1);
  double Wc = 0.0;
  if (WARPS > 1) {
    if (lane == 31) sh.fw[warp] = I;
    __syncthreads();
    for (int v = 0; v < warp; ++v) Wc = fma(P.p32, Wc, sh.fw[v]);
  }
  const double Cc = lane == 0 ? Wc : fma(plane, Wc, Ip);
#pragma unroll
  for (int j = 0; j < MPT; ++j) y[j] = fma(P.fl[j], Cc, y[j]);
  if (g0 + MPT > P.M) {
#pragma unroll
    for (int j = 0; j < MPT; ++j)
      if (g0 + j >= P.M) y[j] = 0.0;  // Dirichlet: padded nodes decouple
  }
  // ---- backward: U^-1 ----
#pragma unroll
  for (int j = MPT - 2; j >= 0; --j) y[j] = fma(P.nu, y[j + 1], y[j]);
  double J = y[0];
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const double t = __shfl_down_sync(kFull, J, 1 << s);
    if (lane < 32 - (1 << s)) J = fma(P.qq[s], t, J);
  }
  const double Jn = __shfl_down_sync(kFull, J, 1);
  double Vc = 0.0;
  if (WARPS > 1) {
    if (lane == 0) sh.bw[warp] = J;
    __syncthreads();
    for (int v = WARPS - 1; v > warp; --v) Vc = fma(P.q32, Vc, sh.bw[v]);
  }
  const double Rc = lane == 31 ? Vc : fma(qlane, Vc, Jn);
#pragma unroll
  for (int j = 0; j < MPT; ++j) y[j] = fma(P.fu[j], Rc, y[j]);
  // ---- corner rank-1 correction ----
  if (P.K0 <= 32 * MPT) {
    if (warp == 0) {
      const double c = P.gneg * __shfl_sync(kFull, y[0], 0);
      if (g0 < P.K0) {
#pragma unroll
        for (int j = 0; j < MPT; ++j)
          if (g0 + j < P.K0) y[j] = fma(c, s_zc[g0 + j], y[j]);
      }
    }
  } else {
    if (warp == 0 && lane == 0) sh.b = y[0];
    __syncthreads();
    const double c = P.gneg * sh.b;
    if (g0 < P.K0) {
#pragma unroll
      for (int j = 0; j < MPT; ++j)
        if (g0 + j < P.K0) y[j] = fma(c, s_zc[g0 + j], y[j]);
    }
  }
}

// Full slab propagation: steps BE steps, homogeneous (deferred scaling) or
// with the separable source sampled at each step end.  ds points at this
// slab's row of the dt*s(t_k) table; g holds the thread's source shape.
template <int MPT, int WARPS, bool SRC>
__device__ __forceinline__ void propagate_slab(double (&y)[MPT], const StepParams& P,
                                               double plane, double qlane,
                                               StepShared<WARPS>& sh,
                                               const double* __restrict__ s_zc, int lane,
                                               int warp, int g0, const double* __restrict__ ds,
                                               const double (&g)[MPT]) {
  if (SRC) {
    double dsk = ds[0];
    for (int k = 0; k < P.steps; ++k) {
      const double dsn = (k + 1 < P.steps) ? ds[k + 1] : 0.0;
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = fma(dsk, g[j], y[j]);
      be_solve<MPT, WARPS>(y, P, plane, qlane, sh, s_zc, lane, warp, g0);
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = y[j] * P.inv;
      dsk = dsn;
    }
  } else {
    int cnt = 0;
    for (int k = 0; k < P.steps; ++k) {
      be_solve<MPT, WARPS>(y, P, plane, qlane, sh, s_zc, lane, warp, g0);
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
