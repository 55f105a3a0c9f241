// pit_step.cuh — one backward-Euler step (I + dt*A) y' = y for a slab whose
// M-point state lives in registers across a CTA of 32*WARPS threads, MPT
// contiguous points per thread.
//
// Replaces, per slab and step, the reference's ImplicitStepSolver::solve
// (src/pde.cpp:112-130 -> solve_cg/solve_bicgstab, src/sparse.cpp:60-206)
// with a direct tridiagonal solve:
//   y <- U^-1 L^-1 y            constant unit-bidiagonal factors nl, nu
//        (chunked, two passes per direction: a per-thread sweep with zero
//         carry gives the chunk's end value, a Kogge-Stone warp scan plus a
//         sequential cross-warp combine gives every chunk its true carry,
//         and the sweep is rerun from that carry)
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

// d = fma(a, b, d) when p, else d unchanged: one predicated DFMA (no selects).
__device__ __forceinline__ void fma_if(bool p, double& d, double a, double b) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q fma.rn.f64 %0, %1, %2, %0;\n\t}"
      : "+d"(d)
      : "d"(a), "d"(b), "r"((unsigned)p));
}

// s_zc holds the correction vector zero-padded to 32*MPT entries (narrow
// path, K0 <= 32*MPT: only warp 0 touches it) or to the padded slab length
// (wide path); fma(c, 0, y) == y, so padding does not change any bit.
template <int MPT, int WARPS>
__device__ __forceinline__ void be_solve(double (&y)[MPT], const StepParams& P, double plane,
                                         double qlane, StepShared<WARPS>& sh,
                                         const double* __restrict__ s_zc, int lane, int warp,
                                         int g0, bool ghosts, bool wide) {
  // ---- forward: L^-1 (pass 1: chunk end with zero carry-in) ----
  double z = y[0];
#pragma unroll
  for (int j = 1; j < MPT; ++j) z = fma(P.nl, z, y[j]);
  double I = z;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const double t = __shfl_up_sync(kFull, I, 1 << s);
    fma_if(lane >= (1 << s), I, P.pp[s], t);
  }
  const double Ip = __shfl_up_sync(kFull, I, 1);
  double Wc = 0.0;
  if (WARPS > 1) {
    if (lane == 31) sh.fw[warp] = I;
    __syncthreads();
#pragma unroll
    for (int v = 0; v < WARPS - 1; ++v) fma_if(v < warp, Wc, P.p32, sh.fw[v]);
  }
  double Cc = Wc;
  if (lane != 0) Cc = fma(plane, Wc, Ip);
  // pass 2: the chunk's sweep again, from the true carry
  y[0] = fma(P.nl, Cc, y[0]);
#pragma unroll
  for (int j = 1; j < MPT; ++j) y[j] = fma(P.nl, y[j - 1], y[j]);
  if (ghosts) {
#pragma unroll
    for (int j = 0; j < MPT; ++j) y[j] = (g0 + j < P.M) ? y[j] : 0.0;  // Dirichlet padding
  }
  // ---- backward: U^-1 (pass 1: chunk start with zero carry from the right) ----
  double h = y[MPT - 1];
#pragma unroll
  for (int j = MPT - 2; j >= 0; --j) h = fma(P.nu, h, y[j]);
  double J = h;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const double t = __shfl_down_sync(kFull, J, 1 << s);
    fma_if(lane < 32 - (1 << s), J, P.qq[s], t);
  }
  const double Jn = __shfl_down_sync(kFull, J, 1);
  double Vc = 0.0;
  if (WARPS > 1) {
    if (lane == 0) sh.bw[warp] = J;
    __syncthreads();
#pragma unroll
    for (int v = WARPS - 1; v > 0; --v) fma_if(v > warp, Vc, P.q32, sh.bw[v]);
  }
  double Rc = Vc;
  if (lane != 31) Rc = fma(qlane, Vc, Jn);
  // pass 2
  y[MPT - 1] = fma(P.nu, Rc, y[MPT - 1]);
#pragma unroll
  for (int j = MPT - 2; j >= 0; --j) y[j] = fma(P.nu, y[j + 1], y[j]);
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
                                               double plane, double qlane,
                                               StepShared<WARPS>& sh,
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
      be_solve<MPT, WARPS>(y, P, plane, qlane, sh, s_zc, lane, warp, g0, ghosts, wide);
#pragma unroll
      for (int j = 0; j < MPT; ++j) y[j] = y[j] * P.inv;
      dsk = dsn;
    }
  } else {
    int cnt = 0;
    for (int k = 0; k < P.steps; ++k) {
      be_solve<MPT, WARPS>(y, P, plane, qlane, sh, s_zc, lane, warp, g0, ghosts, wide);
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
