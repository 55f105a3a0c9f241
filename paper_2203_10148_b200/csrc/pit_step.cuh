// pit_step.cuh — one backward-Euler step (I + dt*A) y' = y for a slab whose
// M-point state lives in registers across a CTA of T = 32*WARPS threads.
// DESIGN.md §3.
//
// Layout: the (padded) slab is split into NSEG super-segments of
// Lseg = T*SUB points; thread t owns chunk t (SUB contiguous points) of every
// segment: point s*Lseg + t*SUB + j sits in y[s][j].  The NSEG segments are
// swept, scanned and fixed up side by side, so every phase has NSEG-way
// instruction-level parallelism, and the corner correction touches only
// segment 0.
//
// Replaces, per slab and step, the reference's ImplicitStepSolver::solve
// (src/pde.cpp:112-130 -> solve_cg/solve_bicgstab, src/sparse.cpp:60-206)
// with a direct tridiagonal solve:
//   y <- U^-1 L^-1 y     constant unit-bidiagonal factors nl, nu; per
//        direction: chunk sweeps with zero carry (end value only); Kogge-Stone
//        warp scans and a sequential cross-warp combine give each chunk its
//        carry within its segment; the segment totals are chained segment to
//        segment; the chunk carry adds the segment carry-in (weight
//        nl^(t*SUB)); the chunk sweep is rerun from that carry
//   y <- y + (gneg*y_0) zc   corner rank-1 (Sherman-Morrison) correction
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
  double Pseg, Qseg;        // nl^Lseg, nu^Lseg (segment-to-segment carry weights)
  double fl[32], fu[32];    // fix-up weights nl^(j+1), nu^(SUB-j), j < SUB
  double pp[5], qq[5], p32, q32;  // Kogge-Stone weights: powers of nl^SUB / nu^SUB
  double plane[32], qlane[32];
  int M, steps, R, K0;
  const double* zc;     // [K0] correction vector (device)
  const double* ppos;   // [T] nl^(t*SUB)  (device)
  const double* qpos;   // [T] nu^((T-1-t)*SUB)  (device)
  const double* shape;  // [M] source shape g(x_i) (device) or nullptr
  const double* ds;     // [slabs*steps] dt*s(t_k) table (device) or nullptr
  long long* timing;    // PIT_PHASE_TIMING builds only: [2 warps][16 phases] cycles
};

#ifdef PIT_PHASE_TIMING
#define PIT_PHASE(k)                          \
  do {                                        \
    const long long now_ = clock64();         \
    ph_acc[k] += now_ - ph_t;                 \
    ph_t = now_;                              \
  } while (0)
#else
#define PIT_PHASE(k) \
  do {               \
  } while (0)
#endif

// Shared memory of one slab CTA: per-segment cross-warp totals, broadcast
// scalar and the per-lane carry weights (read with LDS: an indexed constant
// load would serialise across lanes).  The correction vector follows.
template <int NSEG, int WARPS>
struct StepShared {
  double fw[NSEG][WARPS > 1 ? WARPS : 1];
  double bw[NSEG][WARPS > 1 ? WARPS : 1];
  double b;
  double pad;
  double plane[32], qlane[32];  // p^lane, q^(31-lane)
  double cf[5][32], cb[5][32];  // Kogge-Stone weights, 0 where a lane has no source lane
};

template <int NSEG, int WARPS>
__device__ __forceinline__ void init_step_shared(const StepParams& P,
                                                 StepShared<NSEG, WARPS>& sh, int tid) {
  for (int i = tid; i < 32; i += 32 * WARPS) {
    sh.plane[i] = P.plane[i];
    sh.qlane[i] = P.qlane[i];
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      sh.cf[st][i] = i >= (1 << st) ? P.pp[st] : 0.0;
      sh.cb[st][i] = i < 32 - (1 << st) ? P.qq[st] : 0.0;
    }
  }
}

// Per-thread constants of the step (registers, loaded once per kernel).
struct StepLane {
  double plane, qlane, ppos, qpos;
};

// One step.  Per direction: pass 1 runs each chunk's sweep with zero carry
// (only the end value is kept); Kogge-Stone warp scans (per-lane weights
// from shared memory, zero where a lane has no source lane: fma(0, t, I) ==
// I) and the cross-warp combine give each chunk its carry within the
// segment; the segment totals are chained segment to segment; pass 2 reruns
// each chunk's sweep from its true carry.  No per-point constants are
// needed, and the NSEG chunk sweeps of a thread interleave.
// s_zc holds the correction vector zero-padded to 32*SUB entries (narrow
// path, K0 <= 32*SUB: warp 0 of segment 0 only) or to the padded slab length
// (wide path); fma(c, 0, y) == y, so padding does not change any bit.  The
// lane-0 / lane-31 carry uses weight 1 on a zeroed neighbour value, and
// segment 0 (NSEG-1 backward) adds a zero segment carry-in: both exact.
template <int SUB, int NSEG, int WARPS>
__device__ __forceinline__ void be_solve(double (&y)[NSEG][SUB], const StepParams& P,
                                         const StepLane& L, StepShared<NSEG, WARPS>& sh,
                                         const double* __restrict__ s_zc, int lane, int warp,
                                         int g0, bool ghosts, bool wide
#ifdef PIT_PHASE_TIMING
                                         , long long (&ph_acc)[16], long long& ph_t
#endif
) {
  constexpr int LSEG = 32 * WARPS * SUB;
  double I[NSEG], Ip[NSEG], Wc[NSEG], Tot[NSEG];
  // ---- forward: L^-1 ----
#pragma unroll
  for (int s = 0; s < NSEG; ++s) I[s] = y[s][0];
#pragma unroll
  for (int j = 1; j < SUB; ++j)
#pragma unroll
    for (int s = 0; s < NSEG; ++s) I[s] = fma(P.nl, I[s], y[s][j]);
  PIT_PHASE(0);
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const double c = sh.cf[st][lane];
#pragma unroll
    for (int s = 0; s < NSEG; ++s) I[s] = fma(c, __shfl_up_sync(kFull, I[s], 1 << st), I[s]);
  }
#pragma unroll
  for (int s = 0; s < NSEG; ++s) {
    Ip[s] = __shfl_up_sync(kFull, I[s], 1);
    Ip[s] = lane == 0 ? 0.0 : Ip[s];
    Wc[s] = 0.0;
  }
  PIT_PHASE(1);
  if (WARPS > 1) {
    if (lane == 31) {
#pragma unroll
      for (int s = 0; s < NSEG; ++s) sh.fw[s][warp] = I[s];
    }
    __syncthreads();
    for (int v = 0; v < warp; ++v)
#pragma unroll
      for (int s = 0; s < NSEG; ++s) Wc[s] = fma(P.p32, Wc[s], sh.fw[s][v]);
    if (NSEG > 1) {
#pragma unroll
      for (int s = 0; s < NSEG - 1; ++s) Tot[s] = 0.0;
#pragma unroll
      for (int v = 0; v < WARPS; ++v)
#pragma unroll
        for (int s = 0; s < NSEG - 1; ++s) Tot[s] = fma(P.p32, Tot[s], sh.fw[s][v]);
    }
  } else if (NSEG > 1) {
#pragma unroll
    for (int s = 0; s < NSEG - 1; ++s) Tot[s] = __shfl_sync(kFull, I[s], 31);
  }
  PIT_PHASE(2);
  {
    double S = 0.0;  // segment carry-in
#pragma unroll
    for (int s = 0; s < NSEG; ++s) {
      if (s > 0) S = fma(P.Pseg, S, Tot[s - 1]);
      double C = fma(L.plane, Wc[s], Ip[s]);
      C = fma(L.ppos, S, C);
      y[s][0] = fma(P.nl, C, y[s][0]);
    }
  }
#pragma unroll
  for (int j = 1; j < SUB; ++j)
#pragma unroll
    for (int s = 0; s < NSEG; ++s) y[s][j] = fma(P.nl, y[s][j - 1], y[s][j]);
  if (ghosts) {
#pragma unroll
    for (int s = 0; s < NSEG; ++s)
#pragma unroll
      for (int j = 0; j < SUB; ++j)
        y[s][j] = (s * LSEG + g0 + j < P.M) ? y[s][j] : 0.0;  // Dirichlet padding
  }
  PIT_PHASE(3);
  // ---- backward: U^-1 ----
#pragma unroll
  for (int s = 0; s < NSEG; ++s) I[s] = y[s][SUB - 1];
#pragma unroll
  for (int j = SUB - 2; j >= 0; --j)
#pragma unroll
    for (int s = 0; s < NSEG; ++s) I[s] = fma(P.nu, I[s], y[s][j]);
  PIT_PHASE(4);
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const double c = sh.cb[st][lane];
#pragma unroll
    for (int s = 0; s < NSEG; ++s) I[s] = fma(c, __shfl_down_sync(kFull, I[s], 1 << st), I[s]);
  }
#pragma unroll
  for (int s = 0; s < NSEG; ++s) {
    Ip[s] = __shfl_down_sync(kFull, I[s], 1);
    Ip[s] = lane == 31 ? 0.0 : Ip[s];
    Wc[s] = 0.0;
  }
  PIT_PHASE(5);
  if (WARPS > 1) {
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < NSEG; ++s) sh.bw[s][warp] = I[s];
    }
    __syncthreads();
    for (int v = WARPS - 1; v > warp; --v)
#pragma unroll
      for (int s = 0; s < NSEG; ++s) Wc[s] = fma(P.q32, Wc[s], sh.bw[s][v]);
    if (NSEG > 1) {
#pragma unroll
      for (int s = 1; s < NSEG; ++s) Tot[s] = 0.0;
#pragma unroll
      for (int v = WARPS - 1; v >= 0; --v)
#pragma unroll
        for (int s = 1; s < NSEG; ++s) Tot[s] = fma(P.q32, Tot[s], sh.bw[s][v]);
    }
  } else if (NSEG > 1) {
#pragma unroll
    for (int s = 1; s < NSEG; ++s) Tot[s] = __shfl_sync(kFull, I[s], 0);
  }
  PIT_PHASE(6);
  {
    double S = 0.0;  // segment carry from the right
#pragma unroll
    for (int s = NSEG - 1; s >= 0; --s) {
      if (s < NSEG - 1) S = fma(P.Qseg, S, Tot[s + 1]);
      double R = fma(L.qlane, Wc[s], Ip[s]);
      R = fma(L.qpos, S, R);
      y[s][SUB - 1] = fma(P.nu, R, y[s][SUB - 1]);
    }
  }
#pragma unroll
  for (int j = SUB - 2; j >= 0; --j)
#pragma unroll
    for (int s = 0; s < NSEG; ++s) y[s][j] = fma(P.nu, y[s][j + 1], y[s][j]);
  PIT_PHASE(7);
  // ---- corner rank-1 correction ----
  if (!wide) {
    if (warp == 0) {
      const double c = P.gneg * __shfl_sync(kFull, y[0][0], 0);
      if (g0 < P.K0) {
#pragma unroll
        for (int j = 0; j < SUB; ++j) y[0][j] = fma(c, s_zc[g0 + j], y[0][j]);
      }
    }
  } else {
    if (warp == 0 && lane == 0) sh.b = y[0][0];
    __syncthreads();
    const double c = P.gneg * sh.b;
#pragma unroll
    for (int s = 0; s < NSEG; ++s)
      if (s * LSEG + g0 < P.K0) {
#pragma unroll
        for (int j = 0; j < SUB; ++j) y[s][j] = fma(c, s_zc[s * LSEG + g0 + j], y[s][j]);
      }
  }
  PIT_PHASE(8);
}

}  // namespace pitb
