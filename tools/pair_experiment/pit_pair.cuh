// pit_pair.cuh — paired backward-Euler steps for the fine propagator (K1 and
// the sequential fine solve): two consecutive steps share their sweeps.
// DESIGN.md §3.3.1.
//
// The step matrix T = I + dt*A (constant bands) has two constant-factor
// forms (pit_step.cuh uses the first only):
//   type 1:  T = (1/inv) (I - nl S)(I - nu S^T) + sigma e_0 e_0^T
//            x' = inv * (U^-1 L^-1 x + gneg  y_0     z')   (F, B, corner at 0)
//   type 2:  T = (1/inv) (I - nu S^T)(I - nl S) + sigma e_L e_L^T,  L = M-1
//            x' = inv * (L^-1 U^-1 x + gnegM y_{M-1} z'')  (B, F, corner at M-1)
// Both are the same direct solve of the reference's ImplicitStepSolver system
// (src/pde.cpp:103-130).  Alternating them, consecutive steps put two
// backward sweeps, then two forward sweeps, back to back:
//   F | B c0 B | F cM F | B c0 B | ... | closing sweep + its corner
// and a doubled sweep runs as ONE chunked pass over a two-level cascade
//   x_j = y_j + a x_(j-1),   z_j = x_j + a z_(j-1)
// (pass 1: both levels' zero-carry end values, carries as 2-vectors through
// the triangular transfer [w 0; n w, w]; pass 2: both levels from their true
// carries), with the corner between the two sweeps folded through the second
// one by linearity: B(x + c z') = B x + c (B z'), and B z' is again geometric
// in nl.  Per point and step that is the same 4 DFMA as pit_step.cuh, but
// half the scans and barriers, eight independent chains per thread instead
// of four, and the corner work alternates between the first and last warp.
//
// A group of s steps (s = G <= R, the rescale period of the plain path; the
// last group of a slab may be shorter) is
//   phase 0: F (one level); phases 1..s-1: doubled, B on odd, F on even
//   phases; phase s: one level, B + plain corner (s odd) or F + plain corner
//   at M-1 (s even); then the deferred scale inv^s.
// The folded corner of a doubled phase is applied lazily: the next phase's
// pass 1 runs on the uncorrected values and fixes its end values up by
// linearity (the correction is geometric in the sweep's own multiplier), and
// the 64-instruction point update runs after the warp has published its
// total, so no warp waits for another warp's corner; the warps meet on an
// mbarrier (arrive early, wait late) instead of bar.sync.
// Used when the slab fills its layout exactly (no ghost points), NSEG == 1,
// no source, both corners narrow (coeffs.cpp build_pair_coeffs).
// oracle/pit_oracle.c (pair_group) performs the identical operation sequence.
// Measured (tools/exp_pair.cu, B200): c2 one wave of 888 slabs 1.42 -> 1.33 ms,
// steady state 2.86e12 -> 3.04e12 gridpoint-steps/s; c4 3.10 -> 3.00 ms.
#pragma once

#include "pit_step.cuh"  // paper_2203_10148_b200/csrc
#include <type_traits>

#include "pit_sync.cuh"

namespace pitb {

// Paired-step parameters; the harness passes a struct derived from StepParams
// with a member `pair` of this type (template parameter SP below).
struct PairParams {
  int enabled;
  int K0M;               // extent of the corner at M-1 (points from the right end)
  int G;                 // steps per group
  double invG, invGlast;  // inv^G, inv^(steps mod G)
  double pS2, qS2;       // SUB nl^SUB, SUB nu^SUB
  double p32_2, q32_2;   // (32 CH) nl^(32 CH), ...
  double pp2[5], qq2[5];  // (CH 2^st) nl^(CH 2^st), ...
  double plane2[32], qlane2[32];  // (l CH) nl^(l CH), ((31-l) CH) nu^((31-l) CH)
  double nupow[32];      // nu^j, j < SUB
  // deferred corner folded into the next sweep's pass 1 (E-fix):
  // kap[d][0] = SUB a^(SUB-1), kap[d][1] = a^(SUB-1) SUB (SUB+1)/2, a = nl (d=0), nu (d=1)
  double kap[2][2];
  // corner gains [end][folded][u][lane] (device, 2*2*8*32): au = x_edge * gain
  const double* gain;
};

template <int WARPS>
struct PairShared {
  unsigned long long bar;                 // mbarrier, one arrival per warp and phase
  double w[2][2][WARPS > 1 ? WARPS : 1];  // [phase parity][level][warp] warp totals
  double lane[2][2][32];                  // [dir][level][lane] carry weights
  double ks[2][2][5][32];                 // [dir][level][stage][lane], 0 where no source lane
  double gain[2][2][8][32];               // PairParams::gain
};
struct PairSharedNone {};
template <class S, bool PAIR>
using PairSharedFor = typename std::conditional<PAIR, PairShared<S::WARPS>, PairSharedNone>::type;

template <class SP, int WARPS>
__device__ __forceinline__ void init_pair_shared(const SP& P, PairShared<WARPS>& sh,
                                                 int tid) {
  const PairParams& Q = P.pair;
  if (!Q.enabled) return;
  if (tid == 0) mbar_init(reinterpret_cast<uint64_t*>(&sh.bar), WARPS);
  for (int i = tid; i < 32; i += 32 * WARPS) {
    sh.lane[0][0][i] = P.plane[i];
    sh.lane[0][1][i] = Q.plane2[i];
    sh.lane[1][0][i] = P.qlane[i];
    sh.lane[1][1][i] = Q.qlane2[i];
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const bool f = i >= (1 << st), b = i < 32 - (1 << st);
      sh.ks[0][0][st][i] = f ? P.pp[st] : 0.0;
      sh.ks[0][1][st][i] = f ? Q.pp2[st] : 0.0;
      sh.ks[1][0][st][i] = b ? P.qq[st] : 0.0;
      sh.ks[1][1][st][i] = b ? Q.qq2[st] : 0.0;
    }
  }
  for (int i = tid; i < 2 * 2 * 8 * 32; i += 32 * WARPS) (&sh.gain[0][0][0][0])[i] = Q.gain[i];
}

// One chunked sweep of LV cascade levels in direction FWD (a = nl, low to
// high points) or backward (a = nu).
//   PEND (1 yes, 0 no, 2 = the run-time flag `pend`): the folded corner of
//   the previous phase (at this sweep's upstream end, held by warp
//   `FWD ? 0 : WARPS-1`) is still to be applied: y[u][k] += xs * gain[u] * a^k
//   in sweep coordinates.  Pass 1 runs on the uncorrected values and its end
//   values are fixed up by linearity; the point update itself runs after the
//   warp has published its total, off the other warps' critical path.
// Returns the level-1 value at the last point in sweep order of the edge
// thread of each warp (thread T-1's point M-1 for FWD, thread 0's point 0
// for backward): the next corner's source value xs.
template <class SP, class S, bool FWD, int LV, int PEND>
__device__ __forceinline__ double pair_sweep(double (&y)[S::NC][S::SUB], const SP& P,
                                             PairShared<S::WARPS>& sh, int tid, int& par,
                                             bool pend, double xs) {
  static_assert(S::NSEG == 1, "paired steps: one segment");
  constexpr int SUB = S::SUB, NSUB = S::NSUB, WARPS = S::WARPS;
  constexpr int D = FWD ? 0 : 1;
  const PairParams& Q = P.pair;
#define PJ(k) (FWD ? (k) : SUB - 1 - (k))
#define PU(k) (FWD ? (k) : NSUB - 1 - (k))
  const int lane = tid & 31, warp = tid >> 5;
  const double a = FWD ? P.nl : P.nu;
  const double aS = FWD ? P.pS : P.qS, aS2 = FWD ? Q.pS2 : Q.qS2;
  // warp-uniform: this warp holds the pending corner
  const bool hold = (PEND == 1 || (PEND == 2 && pend)) && warp == (FWD ? 0 : WARPS - 1);
  const int kext = FWD ? P.K0 : Q.K0M;
  double E1[NSUB], E2[NSUB];
  // ---- pass 1: zero-carry end values of every sub-chunk ----
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    E1[u] = y[PU(u)][PJ(0)];
    E2[u] = E1[u];
  }
#pragma unroll
  for (int k = 1; k < SUB; ++k) {
#pragma unroll
    for (int u = 0; u < NSUB; ++u) E1[u] = fma(a, E1[u], y[PU(u)][PJ(k)]);
    if (LV == 2) {
#pragma unroll
      for (int u = 0; u < NSUB; ++u) E2[u] = fma(a, E2[u], E1[u]);
    }
  }
  if (PEND && hold) {
#pragma unroll
    for (int u = 0; u < NSUB; ++u) {
      const double au = xs * sh.gain[D][1][u][lane];
      if (LV == 2) E2[u] = fma(au, Q.kap[D][1], E2[u]);
      E1[u] = fma(au, Q.kap[D][0], E1[u]);
    }
  }
  double I1 = E1[0], I2 = E2[0];
#pragma unroll
  for (int u = 1; u < NSUB; ++u) {
    if (LV == 2) I2 = fma(aS, I2, fma(aS2, I1, E2[u]));
    I1 = fma(aS, I1, E1[u]);
  }
  // ---- warp scan (decay-truncated Kogge-Stone), carries from upstream ----
#pragma unroll
  for (int st = 0; st < (S::KS < 0 ? 5 : S::KS); ++st) {
    if (S::KS < 0 && st >= (FWD ? P.scan_f : P.scan_b)) break;  // warp-uniform
    const double cw = sh.ks[D][0][st][lane];
    const double s1 = FWD ? __shfl_up_sync(kFull, I1, 1 << st) : __shfl_down_sync(kFull, I1, 1 << st);
    if (LV == 2) {
      const double cw2 = sh.ks[D][1][st][lane];
      const double s2 =
          FWD ? __shfl_up_sync(kFull, I2, 1 << st) : __shfl_down_sync(kFull, I2, 1 << st);
      I2 = fma(cw, s2, fma(cw2, s1, I2));
    }
    I1 = fma(cw, s1, I1);
  }
  if (WARPS > 1) {
    if (lane == (FWD ? 31 : 0)) {
      sh.w[par][0][warp] = I1;
      if (LV == 2) sh.w[par][1][warp] = I2;
      mbar_arrive(reinterpret_cast<uint64_t*>(&sh.bar));
    }
  }
  double C1 = FWD ? __shfl_up_sync(kFull, I1, 1) : __shfl_down_sync(kFull, I1, 1);
  double C2 = 0.0;
  if (LV == 2) C2 = FWD ? __shfl_up_sync(kFull, I2, 1) : __shfl_down_sync(kFull, I2, 1);
  if (lane == (FWD ? 0 : 31)) {
    C1 = 0.0;
    C2 = 0.0;
  }
  // ---- the pending corner's point update (this warp only) ----
  if (PEND && hold) {
#pragma unroll
    for (int u = 0; u < NSUB; ++u) {
      if (u * SUB >= kext) break;  // warp-uniform
      const double au = xs * sh.gain[D][1][u][lane];
#pragma unroll
      for (int k = 0; k < SUB; ++k)
        y[PU(u)][PJ(k)] = fma(au, FWD ? P.nlpow[k] : Q.nupow[k], y[PU(u)][PJ(k)]);
    }
  }
  if (WARPS > 1) {
    mbar_wait(reinterpret_cast<uint64_t*>(&sh.bar), (unsigned)par);
    const double a32 = FWD ? P.p32 : P.q32, a32_2 = FWD ? Q.p32_2 : Q.q32_2;
    double W1 = 0.0, W2 = 0.0;
#pragma unroll
    for (int k = 0; k < WARPS - 1; ++k) {
      const int v = FWD ? k : WARPS - 1 - k;
      if (FWD ? v < warp : v > warp) {
        if (LV == 2) W2 = fma(a32, W2, fma(a32_2, W1, sh.w[par][1][v]));
        W1 = fma(a32, W1, sh.w[par][0][v]);
      }
    }
    const double lw = sh.lane[D][0][lane];
    if (LV == 2) C2 = fma(lw, W2, fma(sh.lane[D][1][lane], W1, C2));
    C1 = fma(lw, W1, C1);
  }
  par ^= 1;
  // ---- sub-chunk carries, then pass 2 from the true carries ----
  double X[NSUB], Z[NSUB];
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    X[u] = C1;
    Z[u] = C2;
    if (u + 1 < NSUB) {
      if (LV == 2) C2 = fma(aS, C2, fma(aS2, C1, E2[u]));
      C1 = fma(aS, C1, E1[u]);
    }
  }
#pragma unroll
  for (int k = 0; k < SUB; ++k) {
#pragma unroll
    for (int u = 0; u < NSUB; ++u) X[u] = fma(a, X[u], y[PU(u)][PJ(k)]);
#pragma unroll
    for (int u = 0; u < NSUB; ++u) {
      if (LV == 2) {
        Z[u] = fma(a, Z[u], X[u]);
        y[PU(u)][PJ(k)] = Z[u];
      } else {
        y[PU(u)][PJ(k)] = X[u];
      }
    }
  }
  return __shfl_sync(kFull, X[NSUB - 1], FWD ? 31 : 0);
#undef PJ
#undef PU
}

// A closing corner, applied at once: y[u][k] += xs * gain[end][0][u] * a^k
// (END = 0: points from the left, a = nl; END = 1: from the right, a = nu).
template <class SP, class S, int END>
__device__ __forceinline__ void pair_corner_now(double (&y)[S::NC][S::SUB], const SP& P,
                                                PairShared<S::WARPS>& sh, double xs, int tid) {
  constexpr int SUB = S::SUB, NSUB = S::NSUB;
  if ((tid >> 5) != (END ? S::WARPS - 1 : 0)) return;
  const int kext = END ? P.pair.K0M : P.K0;
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    if (u * SUB >= kext) break;  // warp-uniform
    const double au = xs * sh.gain[END][0][u][tid & 31];
#pragma unroll
    for (int k = 0; k < SUB; ++k) {
      double& v = END ? y[NSUB - 1 - u][SUB - 1 - k] : y[u][k];
      v = fma(au, END ? P.pair.nupow[k] : P.nlpow[k], v);
    }
  }
}

// Steps [k0, k1) in groups of G steps; k0 is a multiple of G (piece cuts fall
// on group boundaries), so a piece sequence is the identical operation
// sequence.  par: the mbarrier phase parity, carried across calls.
template <class SP, class S>
__device__ __forceinline__ void run_slab_paired(double (&y)[S::NC][S::SUB], const SP& P,
                                                PairShared<S::WARPS>& sh, int tid, int k0, int k1,
                                                int& par) {
  for (int k = k0; k < k1;) {
    const int s = k1 - k < P.pair.G ? k1 - k : P.pair.G;
    // phase 0: F; phases 1..s-1 doubled (B on odd, F on even phases), each
    // leaving its folded corner to the next phase; phase s closes the group
    double xs = pair_sweep<SP, S, true, 1, 2>(y, P, sh, tid, par, false, 0.0);
    for (int ph = 1; ph < s; ph += 2) {
      xs = pair_sweep<SP, S, false, 2, 2>(y, P, sh, tid, par, ph > 1, xs);
      if (ph + 1 < s) xs = pair_sweep<SP, S, true, 2, 1>(y, P, sh, tid, par, true, xs);
    }
    if (s & 1) {
      xs = pair_sweep<SP, S, false, 1, 2>(y, P, sh, tid, par, s >= 2, xs);
      pair_corner_now<SP, S, 0>(y, P, sh, xs, tid);
    } else {
      xs = pair_sweep<SP, S, true, 1, 2>(y, P, sh, tid, par, true, xs);
      pair_corner_now<SP, S, 1>(y, P, sh, xs, tid);
    }
    const double sc = s == P.pair.G ? P.pair.invG : P.pair.invGlast;
#pragma unroll
    for (int c = 0; c < S::NC; ++c)
#pragma unroll
      for (int j = 0; j < S::SUB; ++j) y[c][j] = y[c][j] * sc;
    k += s;
  }
}

}  // namespace pitb
