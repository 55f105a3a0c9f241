// pit_step.cuh — one backward-Euler step (I + dt*A) y' = y for a slab whose
// M-point state lives in registers across a CTA of T = 32*WARPS threads.
// DESIGN.md §3.
//
// Layout (Shape<SUB, NSUB, NSEG, WARPS>): the padded slab is NSEG strided
// segments of LSEG = T*NSUB*SUB points; in every segment thread t owns the
// contiguous chunk [t*NSUB*SUB, (t+1)*NSUB*SUB), split into NSUB sub-chunks
// of SUB points.  Register y[c][j], c = s*NSUB + u, holds point
//     s*LSEG + t*NSUB*SUB + u*SUB + j.
// The NSEG*NSUB sub-chunk sweeps of a thread run interleaved (ILP); each
// segment needs one warp scan per direction (its sub-chunks are combined
// inside the thread first), so NSEG trades shuffles for shorter chains.
//
// Replaces, per slab and step, the reference's ImplicitStepSolver::solve
// (src/pde.cpp:112-130 -> solve_cg/solve_bicgstab, src/sparse.cpp:60-206)
// with a direct tridiagonal solve:
//   y <- U^-1 L^-1 y     constant unit-bidiagonal factors nl, nu.  Per
//        direction: pass 1 sweeps every sub-chunk with zero carry (end value
//        only); the thread's chunk end combines its sub-chunks; Kogge-Stone
//        warp scans and a sequential cross-warp combine give each chunk its
//        carry within its segment; segment totals are chained segment to
//        segment; sub-chunk carries follow; pass 2 reruns every sub-chunk's
//        sweep from its true carry.
//        The warp scans keep only the Kogge-Stone stages whose terms can
//        matter: with chunk multiplier w = nl^ch, a chunk's carry from the
//        chunk d positions back has weight w^(d-1), so stages stop at the
//        first s with w^(2^s) <= 2^-70 (scan_f / scan_b; the same threshold
//        as the corner extent K0).  c2 keeps 2 of 5 stages, c3 none.
//   y <- y + (gneg*y_0) zc   corner rank-1 (Sherman-Morrison) correction:
//        narrow form zc_i = zc_0 nl^i on the chunks of segment 0 that start
//        below K0, sub-chunks starting below K0 only (fine propagators),
//        table form otherwise (coarse).
// and the diagonal scale inv is deferred: applied as inv^R every R steps
// (homogeneous propagation) or every step when a source is added.
// Every multiply-add is an explicit fma(); oracle/pit_oracle.c
// (chunked_solve) performs the identical operation sequence.
#pragma once

#include <cuda_runtime.h>

namespace pitb {

constexpr unsigned kFull = 0xffffffffu;

// Barrier among the slab's T compute threads only (named barrier 1): the
// coarse sweep adds I/O warps that never enter the step.
template <int T>
__device__ __forceinline__ void step_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(T) : "memory");
}

struct StepParams {
  double nl, nu, inv, gneg, invR, invLast;
  double pS, qS;            // nl^SUB, nu^SUB        (sub-chunk carry weights)
  double Pseg, Qseg;        // nl^LSEG, nu^LSEG      (segment carry weights)
  double nlpow[32];         // nl^j, j < SUB         (narrow corner)
  double pw[8];             // nl^(u*SUB), u < NSUB  (narrow corner)
  double pp[5], qq[5], p32, q32;  // Kogge-Stone weights: powers of nl^(NSUB*SUB)
  double plane[32], qlane[32];
  int M, steps, R, K0;
  int scan_f, scan_b;       // Kogge-Stone stages kept (pit_step_coeffs)
  int narrow;               // corner in geometric form on segment 0 only
  const double* zc;     // [K0] correction vector (device), table form
  const double* zt;     // [T] zc_0 * nl^(t*NSUB*SUB), narrow form
  const double* ppos;   // [T] nl^(t*NSUB*SUB)  (device)
  const double* qpos;   // [T] nu^((T-1-t)*NSUB*SUB)  (device)
  const double* shape;  // [M] source shape g(x_i) (device) or nullptr
  const double* ds;     // [slabs*steps] dt*s(t_k) table (device) or nullptr
  const double* tab;    // [slabs*steps][M] fl(dt*f(t_k, x_i)) general source (device) or nullptr
  long long* timing;    // PIT_PHASE_TIMING builds only: [2 warps][16 phases] cycles
};

#ifdef PIT_PHASE_TIMING
#define PIT_PHASE(k)                  \
  do {                                \
    const long long now_ = clock64(); \
    ph_acc[k] += now_ - ph_t;         \
    ph_t = now_;                      \
  } while (0)
#else
#define PIT_PHASE(k) \
  do {               \
  } while (0)
#endif

// KS_ in 0..5: the warp scans keep exactly KS_ Kogge-Stone stages
// (compile-time specialisation for StepParams::scan_f == scan_b == KS_);
// KS_ < 0: the stage counts are read from StepParams at run time.
template <int SUB_, int NSUB_, int NSEG_, int WARPS_, int KS_ = -1>
struct Shape {
  static constexpr int SUB = SUB_, NSUB = NSUB_, NSEG = NSEG_, WARPS = WARPS_, KS = KS_;
  static constexpr int T = 32 * WARPS;
  static constexpr int NC = NSUB * NSEG;  // sub-chunks per thread
  static constexpr int CH = NSUB * SUB;   // thread chunk length within a segment
  static constexpr int MPT = NC * SUB;    // points per thread
  static constexpr int LSEG = T * CH;     // segment length
  // global point of register y[c][j] for thread t
  __host__ __device__ static constexpr int point(int t, int c, int j) {
    return (c / NSUB) * LSEG + t * CH + (c % NSUB) * SUB + j;
  }
  // shared-memory slot of the same point: thread-major, odd pitch MPT+1
  __host__ __device__ static constexpr int slot(int t, int c, int j) {
    return t * (MPT + 1) + c * SUB + j;
  }
  __host__ __device__ static int slot_of_point(int i) {
    const int s = i / LSEG, r = i - s * LSEG;
    const int t = r / CH, q = r - t * CH;
    return t * (MPT + 1) + s * CH + q;
  }
};

// Shared memory of one slab CTA: per-segment cross-warp totals, broadcast
// scalar and per-lane weights (read with LDS; an indexed constant load would
// serialise across lanes).  The table-form correction vector follows.
template <int NSEG, int WARPS>
struct StepShared {
  double fw[NSEG][WARPS > 1 ? WARPS : 1];
  double bw[NSEG][WARPS > 1 ? WARPS : 1];
  double b;
  double pad;
  // replicated corner (REPL): thread 0's backward-carry inputs (Ip, the
  // sub-chunk end values E[1..NSUB-1], its first sub-chunk before pass 2)
  double corner[48];
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
// The HOIST variant of be_solve (the sequential sweeps, one CTA whose step
// latency is the whole story) also keeps the lane's Kogge-Stone weights and
// carry weights here instead of re-reading them from shared memory each step.
struct StepLane {
  double ppos, qpos;
  double zt;  // narrow corner: zc_0 nl^(t*CH) of this thread (0 outside warp 0 / beyond K0)
  double cf[5], cb[5], plane, qlane;
};

// One step (see the file comment).  The lane-0 / lane-31 carry uses weight 1
// on a zeroed neighbour value, the Kogge-Stone weight is 0 on lanes without a source
// lane, and the table-form correction vector is zero-padded: every such
// extra term is an exact no-op (fma(w, 0, x) == x, fma(0, t, x) == x).
template <class S, bool HOIST = false, bool ZREG = false>
__device__ __forceinline__ void be_solve(double (&y)[S::NC][S::SUB], const StepParams& P,
                                         const StepLane& L, StepShared<S::NSEG, S::WARPS>& sh,
                                         const double* __restrict__ s_zc, int tid, bool ghosts,
                                         const double (*zreg)[S::SUB]
#ifdef PIT_PHASE_TIMING
                                         , long long (&ph_acc)[16], long long& ph_t
#endif
) {
  constexpr int SUB = S::SUB, NSUB = S::NSUB, NSEG = S::NSEG, WARPS = S::WARPS, NC = S::NC;
  const int lane = tid & 31, warp = tid >> 5;
  double E[NC];
  double I[NSEG], Ip[NSEG], Wc[NSEG], Tot[NSEG];
  // ---- forward: L^-1, pass 1 ----
#pragma unroll
  for (int c = 0; c < NC; ++c) E[c] = y[c][0];
#pragma unroll
  for (int j = 1; j < SUB; ++j)
#pragma unroll
    for (int c = 0; c < NC; ++c) E[c] = fma(P.nl, E[c], y[c][j]);
#pragma unroll
  for (int s = 0; s < NSEG; ++s) {
    I[s] = E[s * NSUB];
#pragma unroll
    for (int u = 1; u < NSUB; ++u) I[s] = fma(P.pS, I[s], E[s * NSUB + u]);
  }
  PIT_PHASE(0);
#pragma unroll
  for (int st = 0; st < (S::KS < 0 ? 5 : S::KS); ++st) {
    if (S::KS < 0 && st >= P.scan_f) break;  // warp-uniform
    const double cw = HOIST ? L.cf[st] : sh.cf[st][lane];
#pragma unroll
    for (int s = 0; s < NSEG; ++s) I[s] = fma(cw, __shfl_up_sync(kFull, I[s], 1 << st), I[s]);
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
    step_sync<S::T>();
    // unrolled with a predicate (not a warp-dependent trip count), so the
    // loads of all warp totals issue ahead of the fma chain; the same chain
#pragma unroll
    for (int v = 0; v < WARPS - 1; ++v)
      if (v < warp) {
#pragma unroll
        for (int s = 0; s < NSEG; ++s) Wc[s] = fma(P.p32, Wc[s], sh.fw[s][v]);
      }
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
    double Sg = 0.0;  // segment carry-in
#pragma unroll
    for (int s = 0; s < NSEG; ++s) {
      double C = fma(HOIST ? L.plane : sh.plane[lane], Wc[s], Ip[s]);
      if (s > 0) {  // segment 0 has no segment carry-in
        Sg = fma(P.Pseg, Sg, Tot[s - 1]);
        C = fma(L.ppos, Sg, C);
      }
#pragma unroll
      for (int u = 0; u < NSUB; ++u) {
        const int c = s * NSUB + u;
        const double Cu = C;
        if (u + 1 < NSUB) C = fma(P.pS, C, E[c]);
        y[c][0] = fma(P.nl, Cu, y[c][0]);
      }
    }
  }
#pragma unroll
  for (int j = 1; j < SUB; ++j)
#pragma unroll
    for (int c = 0; c < NC; ++c) y[c][j] = fma(P.nl, y[c][j - 1], y[c][j]);
  if (ghosts) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int j = 0; j < SUB; ++j) y[c][j] = (S::point(tid, c, j) < P.M) ? y[c][j] : 0.0;
  }
  PIT_PHASE(3);
  // ---- backward: U^-1, pass 1 ----
#pragma unroll
  for (int c = 0; c < NC; ++c) E[c] = y[c][SUB - 1];
#pragma unroll
  for (int j = SUB - 2; j >= 0; --j)
#pragma unroll
    for (int c = 0; c < NC; ++c) E[c] = fma(P.nu, E[c], y[c][j]);
#pragma unroll
  for (int s = 0; s < NSEG; ++s) {
    I[s] = E[s * NSUB + NSUB - 1];
#pragma unroll
    for (int u = NSUB - 2; u >= 0; --u) I[s] = fma(P.qS, I[s], E[s * NSUB + u]);
  }
  PIT_PHASE(4);
#pragma unroll
  for (int st = 0; st < (S::KS < 0 ? 5 : S::KS); ++st) {
    if (S::KS < 0 && st >= P.scan_b) break;  // warp-uniform
    const double cw = HOIST ? L.cb[st] : sh.cb[st][lane];
#pragma unroll
    for (int s = 0; s < NSEG; ++s) I[s] = fma(cw, __shfl_down_sync(kFull, I[s], 1 << st), I[s]);
  }
#pragma unroll
  for (int s = 0; s < NSEG; ++s) {
    Ip[s] = __shfl_down_sync(kFull, I[s], 1);
    Ip[s] = lane == 31 ? 0.0 : Ip[s];
    Wc[s] = 0.0;
  }
  PIT_PHASE(5);
  // REPL (table-form corner in registers, one segment): instead of thread 0
  // broadcasting y_0 behind a third barrier, every thread recomputes thread
  // 0's backward pass-2 chain for its first point from inputs thread 0
  // publishes before the backward barrier — the same fma sequence, so the
  // same bits, with no barrier and no wait on warp 0
  constexpr bool REPL = ZREG && NSEG == 1 && WARPS > 1 && NSUB - 1 + SUB + 1 <= 48;
  if (WARPS > 1) {
    if (REPL && tid == 0) {
      sh.corner[0] = Ip[0];
#pragma unroll
      for (int u = 1; u < NSUB; ++u) sh.corner[u] = E[u];
#pragma unroll
      for (int j = 0; j < SUB; ++j) sh.corner[NSUB + j] = y[0][j];
    }
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < NSEG; ++s) sh.bw[s][warp] = I[s];
    }
    step_sync<S::T>();
#pragma unroll
    for (int v = WARPS - 1; v >= 1; --v)
      if (v > warp) {
#pragma unroll
        for (int s = 0; s < NSEG; ++s) Wc[s] = fma(P.q32, Wc[s], sh.bw[s][v]);
      }
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
    double Sg = 0.0;  // segment carry from the right
#pragma unroll
    for (int s = NSEG - 1; s >= 0; --s) {
      double R = fma(HOIST ? L.qlane : sh.qlane[lane], Wc[s], Ip[s]);
      if (s < NSEG - 1) {  // the last segment has no carry from the right
        Sg = fma(P.Qseg, Sg, Tot[s + 1]);
        R = fma(L.qpos, Sg, R);
      }
#pragma unroll
      for (int u = NSUB - 1; u >= 0; --u) {
        const int c = s * NSUB + u;
        const double Ru = R;
        if (u > 0) R = fma(P.qS, R, E[c]);
        y[c][SUB - 1] = fma(P.nu, Ru, y[c][SUB - 1]);
      }
    }
  }
#pragma unroll
  for (int j = SUB - 2; j >= 0; --j)
#pragma unroll
    for (int c = 0; c < NC; ++c) y[c][j] = fma(P.nu, y[c][j + 1], y[c][j]);
  PIT_PHASE(7);
  // ---- corner rank-1 correction ----
  if (P.narrow) {
    if (warp == 0) {
      const double cc = P.gneg * __shfl_sync(kFull, y[0][0], 0);
      if (tid * S::CH < P.K0) {
        const double a = cc * L.zt;  // P.zt[tid], loaded once per kernel
#pragma unroll
        for (int u = 0; u < NSUB; ++u) {
          if (u * SUB >= P.K0) break;  // warp-uniform: lane 0 has the lowest points
          const double au = a * P.pw[u];
#pragma unroll
          for (int j = 0; j < SUB; ++j) y[u][j] = fma(au, P.nlpow[j], y[u][j]);
        }
      }
    }
  } else {
    double y0;
    if (REPL) {
      double w0 = 0.0;  // warp 0's Wc
#pragma unroll
      for (int v = WARPS - 1; v >= 1; --v) w0 = fma(P.q32, w0, sh.bw[0][v]);
      double R0 = fma(sh.qlane[0], w0, sh.corner[0]);
#pragma unroll
      for (int u = NSUB - 1; u >= 1; --u) R0 = fma(P.qS, R0, sh.corner[u]);
      y0 = fma(P.nu, R0, sh.corner[NSUB + SUB - 1]);
#pragma unroll
      for (int j = SUB - 2; j >= 0; --j) y0 = fma(P.nu, y0, sh.corner[NSUB + j]);
    } else if (WARPS == 1) {
      y0 = __shfl_sync(kFull, y[0][0], 0);  // one warp: no shared-memory round trip
    } else {
      if (tid == 0) sh.b = y[0][0];
      step_sync<S::T>();
      y0 = sh.b;
    }
    const double cc = P.gneg * y0;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if ((c / NSUB) * S::LSEG + tid * S::CH < P.K0) {
#pragma unroll
        for (int j = 0; j < SUB; ++j)
          y[c][j] = fma(cc, ZREG ? zreg[c][j] : s_zc[S::slot(tid, c, j)], y[c][j]);
      }
  }
  PIT_PHASE(8);
}

}  // namespace pitb
