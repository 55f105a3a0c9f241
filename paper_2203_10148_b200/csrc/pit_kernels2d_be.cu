// pit_kernels2d_be.cu — K6: 2D backward-Euler propagators with the
// reference's general 5-point operator.
//
// The reference's desk/paper presets (src/presets.cpp:47-77, built by
// runner.cpp:75-88) propagate with backward Euler on the 2D operator of
// assemble_spatial_operator (src/pde.cpp:66-100: 5-point diffusion, reaction,
// first-order upwind rotation).  Every step solves (I + dt*A) x = y with the
// reference's inner solver (ImplicitStepSolver::solve, pde.cpp:112-130):
// Jacobi-PCG when the operator is symmetric (solve_cg, sparse.cpp:60-114),
// Jacobi-BiCGStab otherwise (solve_bicgstab, sparse.cpp:116-206), with the
// same control flow: x0 = 0, tol = rel_tol*||b||, stall / breakdown
// restarts, half-step exit and true-residual confirmation, the 10n cap.
//
// One CTA of kBe2Threads threads per slab (fine batch), or one CTA sweeping
// the slabs in order (coarse sweep, sequential fine solve).  Thread t owns
// interior points t, t+T, ... (PPT of them) and keeps their solver vectors
// in registers; only the stencil's operands (x, p or p^, s^) go through
// zero-padded (m+2)^2 shared-memory buffers, so the stencil reads its
// neighbours without bounds tests.  Stencil rows and the Jacobi inverse stay
// in registers up to 3 points per thread, in shared memory beyond.
// Reductions: per-thread fma chain over its points in
// order, xor butterfly, warp totals summed in order by every thread (one
// block barrier).  oracle/pit_oracle2d_be.c performs the identical
// operation sequence.
#include "pit_kernels2d.cuh"

#include <cmath>

namespace pitb {
namespace {

constexpr int kT = kBe2Threads, kNW = kBe2Threads / 32;

// Per-thread context: owned points (padded indices), stencil rows (in
// registers up to 3 points per thread, else read from shared memory),
// reduction slots and the three operand buffers the stencil reads.
template <int PPT>
struct Be2Ctx {
  static constexpr bool kRegCoef = PPT <= 3;
  static constexpr bool kBig = PPT > 5;  // stencil rows in global memory, two operand buffers
  int m, M, pitch;
  int ip[PPT];        // padded index of owned point k (or -1)
  int ir[PPT];        // index the stencil reads for slot k: ip, or a real point's for an empty
                      // slot (its values are selected to 0: every slot computes, no branches)
  int gi[PPT];        // interior index of owned point k
  double cr[6][kRegCoef ? PPT : 1];  // S, W, C, E, N, minv (kRegCoef)
  const double* cf;   // [6][M] shared memory (!kRegCoef), global memory (kBig)
  double* red;        // [2][2][kNW]
  int par;            // reduction slot set
  double *opx, *opp, *ops;  // padded operand buffers (x, p or p^, s^)
  __device__ __forceinline__ bool ok(int k) const { return ip[k] >= 0; }
  // v for an owned point, exact 0 for an empty slot (so the slot's vectors
  // stay 0 through every linear update and add fma(0, 0, s) == s to the sums)
  __device__ __forceinline__ double keep(int k, double v) const { return ip[k] >= 0 ? v : 0.0; }
  __device__ __forceinline__ double coef(int j, int k) const {
    if constexpr (kRegCoef) return cr[j][k];
    return cf[(size_t)j * M + gi[k]];
  }
};

template <int PPT>
__device__ __forceinline__ double2 block_sum2(Be2Ctx<PPT>& c, double a, double b) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    a = a + __shfl_xor_sync(0xffffffffu, a, off);
    b = b + __shfl_xor_sync(0xffffffffu, b, off);
  }
  double* slot = c.red + c.par * 2 * kNW;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    slot[w] = a;
    slot[kNW + w] = b;
  }
  __syncthreads();
  double sa = slot[0], sb = slot[kNW];
#pragma unroll
  for (int v = 1; v < kNW; ++v) {
    sa = sa + slot[v];
    sb = sb + slot[kNW + v];
  }
  c.par ^= 1;  // the other set is rewritten only after the next barrier
  return make_double2(sa, sb);
}

// Solver vectors of the owned points, in registers.
template <int PPT>
using Vec = double[PPT];

// <a,b> (and <e,f>): per-thread fma chains in point order
template <int PPT>
__device__ __forceinline__ double dot1(Be2Ctx<PPT>& c, const Vec<PPT>& a, const Vec<PPT>& b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) s = fma(a[k], b[k], s);
  return block_sum2(c, s, 0.0).x;
}
template <int PPT>
__device__ __forceinline__ double2 dot2(Be2Ctx<PPT>& c, const Vec<PPT>& a, const Vec<PPT>& b,
                                        const Vec<PPT>& e, const Vec<PPT>& f) {
  double s = 0.0, t = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    s = fma(a[k], b[k], s);
    t = fma(e[k], f[k], t);
  }
  return block_sum2(c, s, t);
}

// (A op)_i in CSR column order south, west, centre, east, north
// (assemble_spatial_operator's row order); op complete (barrier).
template <int PPT>
__device__ __forceinline__ double stencil(const Be2Ctx<PPT>& c, int k, const double* op) {
  const int i = c.ir[k];
  double s = 0.0;
  s = fma(c.coef(0, k), op[i - c.pitch], s);
  s = fma(c.coef(1, k), op[i - 1], s);
  s = fma(c.coef(2, k), op[i], s);
  s = fma(c.coef(3, k), op[i + 1], s);
  s = fma(c.coef(4, k), op[i + c.pitch], s);
  return s;
}

template <int PPT>
__device__ __forceinline__ void publish(const Be2Ctx<PPT>& c, double* op, const Vec<PPT>& v) {
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) op[c.ip[k]] = v[k];
}

// r = b - A x (true_residual, sparse.cpp:53-58); returns ||r||
template <int PPT>
__device__ __forceinline__ double true_residual(Be2Ctx<PPT>& c, const Vec<PPT>& b,
                                                const Vec<PPT>& x, Vec<PPT>& r) {
  publish(c, c.opx, x);
  __syncthreads();  // x complete
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    r[k] = c.keep(k, b[k] - stencil(c, k, c.opx));
    s = fma(r[k], r[k], s);
  }
  return sqrt(block_sum2(c, s, 0.0).x);
}

// Jacobi-PCG, control flow of solve_cg (sparse.cpp:60-114).
template <int PPT>
__device__ bool cg_solve(Be2Ctx<PPT>& c, const Vec<PPT>& b, Vec<PPT>& x, double rel_tol, int cap,
                         int* iters, double* relres) {
  Vec<PPT> r, z, p, q;
#pragma unroll
  for (int k = 0; k < PPT; ++k) x[k] = r[k] = z[k] = p[k] = q[k] = 0.0;
  const double norm_b = sqrt(dot1(c, b, b));
  *iters = 0;
  *relres = 0.0;
  if (norm_b == 0.0) return true;
  const double tol = rel_tol * norm_b;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    r[k] = b[k];
    z[k] = c.coef(5, k) * r[k];
    p[k] = z[k];
  }
  publish(c, c.opp, p);
  double2 d = dot2(c, r, z, r, r);
  double rz = d.x, res = sqrt(d.y);
  int it = 0;
  bool stalled = false;
  for (;;) {
    while (res > tol && it < cap && !stalled) {
      __syncthreads();  // p complete
      double pq = 0.0;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        q[k] = c.keep(k, stencil(c, k, c.opp));
        pq = fma(p[k], q[k], pq);
      }
      pq = block_sum2(c, pq, 0.0).x;
      if (pq == 0.0 || !isfinite(pq)) {
        stalled = true;
        break;
      }
      const double alpha = rz / pq;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        x[k] = fma(alpha, p[k], x[k]);
        r[k] = fma(-alpha, q[k], r[k]);
        z[k] = c.coef(5, k) * r[k];
      }
      ++it;
      d = dot2(c, r, r, r, z);
      res = sqrt(d.x);
      if (!isfinite(res) || res <= tol) break;
      const double beta = d.y / rz;
#pragma unroll
      for (int k = 0; k < PPT; ++k) p[k] = fma(beta, p[k], z[k]);
      publish(c, c.opp, p);  // read by the next stencil after its barrier
      rz = d.y;
    }
    // confirm against the exact residual (sparse.cpp:97-110)
    res = true_residual(c, b, x, r);
    *iters = it;
    *relres = res / norm_b;
    if (res <= tol) return true;
    if (it >= cap || stalled || !isfinite(res)) return false;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      z[k] = c.coef(5, k) * r[k];
      p[k] = z[k];
    }
    publish(c, c.opp, p);
    rz = dot1(c, r, z);
  }
}

// Jacobi-BiCGStab, control flow of solve_bicgstab (sparse.cpp:116-206).
template <int PPT>
__device__ bool bicgstab_solve(Be2Ctx<PPT>& c, const Vec<PPT>& b, Vec<PPT>& x, double rel_tol,
                               int cap, int* iters, double* relres) {
  // p^ and s^ live only in their operand buffers (own values read back)
  Vec<PPT> r, rt, p, v, s, t;
#pragma unroll
  for (int k = 0; k < PPT; ++k) x[k] = r[k] = rt[k] = p[k] = v[k] = s[k] = t[k] = 0.0;
  double* const ph = c.opp;
  double* const sh = c.ops;
  const double norm_b = sqrt(dot1(c, b, b));
  *iters = 0;
  *relres = 0.0;
  if (norm_b == 0.0) return true;
  const double tol = rel_tol * norm_b;
  double rho_prev = 1.0, alpha = 1.0, omega = 1.0, res = 0.0;
  int it = 0;
  bool restart = true, first = true;
  while (it < cap) {
    if (restart) {
      res = true_residual(c, b, x, r);
      if (res <= tol) {
        *iters = it;
        return true;
      }
      if (!isfinite(res)) {
        *iters = it;
        *relres = res / norm_b;
        return false;
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) rt[k] = r[k];
      first = true;
      restart = false;
      rho_prev = 1.0;
      alpha = 1.0;
      omega = 1.0;
    }
    const double rho = dot1(c, rt, r);
    if (rho == 0.0 || !isfinite(rho)) {
      restart = true;
      ++it;
      continue;
    }
    if (first) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) p[k] = r[k];
      first = false;
    } else {
      const double beta = (rho / rho_prev) * (alpha / omega);
#pragma unroll
      for (int k = 0; k < PPT; ++k) p[k] = fma(beta, fma(-omega, v[k], p[k]), r[k]);
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) ph[c.ip[k]] = c.coef(5, k) * p[k];
    __syncthreads();  // ph complete
    double rv = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      v[k] = c.keep(k, stencil(c, k, c.opp));
      rv = fma(rt[k], v[k], rv);
    }
    rv = block_sum2(c, rv, 0.0).x;
    if (rv == 0.0 || !isfinite(rv)) {
      restart = true;
      ++it;
      continue;
    }
    alpha = rho / rv;
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      s[k] = fma(-alpha, v[k], r[k]);
      ss = fma(s[k], s[k], ss);
    }
    if (sqrt(block_sum2(c, ss, 0.0).x) <= tol) {
      // half-iteration exit; keep going from the exact residual if spurious
#pragma unroll
      for (int k = 0; k < PPT; ++k) x[k] = fma(alpha, c.keep(k, ph[c.ir[k]]), x[k]);
      ++it;
      res = true_residual(c, b, x, r);
      if (res <= tol) {
        *iters = it;
        return true;
      }
      if (!isfinite(res)) {
        *iters = it;
        *relres = res / norm_b;
        return false;
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) rt[k] = r[k];
      first = true;
      rho_prev = 1.0;
      alpha = 1.0;
      omega = 1.0;
      continue;
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) sh[c.ip[k]] = c.coef(5, k) * s[k];
    __syncthreads();  // sh complete
    double tt = 0.0, ts = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      t[k] = c.keep(k, stencil(c, k, c.ops));
      tt = fma(t[k], t[k], tt);
      ts = fma(t[k], s[k], ts);
    }
    const double2 d = block_sum2(c, tt, ts);
    omega = d.x == 0.0 ? 0.0 : d.y / d.x;
    double rr = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      x[k] = fma(omega, c.keep(k, sh[c.ir[k]]), fma(alpha, c.keep(k, ph[c.ir[k]]), x[k]));
      r[k] = fma(-omega, t[k], s[k]);
      rr = fma(r[k], r[k], rr);
    }
    ++it;
    res = sqrt(block_sum2(c, rr, 0.0).x);
    if (!isfinite(res)) {
      restart = true;
      continue;
    }
    if (res <= tol) {
      res = true_residual(c, b, x, r);
      if (res <= tol) {
        *iters = it;
        return true;
      }
    }
    if (omega == 0.0) restart = true;
    rho_prev = rho;
  }
  res = true_residual(c, b, x, r);
  *iters = it;
  *relres = res / norm_b;
  return res <= tol;
}

// `steps` backward-Euler steps of the state y (registers).  Returns false at
// the first step whose solve fails or is non-finite (InnerSolveError,
// pde.cpp:119-128).
template <int PPT>
__device__ bool propagate(Be2Ctx<PPT>& c, Vec<PPT>& y, const Be2Params& P, long long* iters,
                          double* fail_info = nullptr, const double* tab = nullptr) {
  Vec<PPT> x;
  for (int step = 0; step < P.steps; ++step) {
    if (tab != nullptr) {  // rhs = y + dt*f(t_step) (propagator.cpp:60-62)
      const double* tk = tab + (size_t)step * P.M;
#pragma unroll
      for (int k = 0; k < PPT; ++k) y[k] = y[k] + c.keep(k, tk[c.gi[k]]);
    }
    int it = 0;
    double relres = 0.0;
    const bool ok = P.symmetric ? cg_solve(c, y, x, P.rel_tol, P.cap, &it, &relres)
                                : bicgstab_solve(c, y, x, P.rel_tol, P.cap, &it, &relres);
    if (iters && threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(iters),
                                             (unsigned long long)it);
    bool bad = !ok;
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0 && !isfinite(x[k])) bad = true;
    if (__syncthreads_or(bad)) {
      if (fail_info != nullptr && threadIdx.x == 0) {  // InnerSolveError payload
        fail_info[0] = relres;
        fail_info[1] = (double)it;
        fail_info[2] = ok ? kFailNonFinite : kFailNotConverged;
      }
      return false;
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) y[k] = x[k];  // the solution is the next right-hand side
  }
  return true;
}

template <int PPT>
__device__ void setup(Be2Ctx<PPT>& c, const Be2Params& P, unsigned char* smem) {
  c.m = P.m;
  c.M = P.M;
  // one-row grids (general 1D operators) need no ghost rows: their south /
  // north coefficients are exact zeros, so pitch 0 makes those operands the
  // point itself (fma(0, finite, s) == s)
  c.pitch = P.my == 1 ? 0 : P.m + 2;
  const int np = P.my == 1 ? P.m + 2 : c.pitch * (P.my + 2);
  double* base = reinterpret_cast<double*>(smem);
  // big grids: x and s^ share a buffer (each operand is published right
  // before the stencil that reads it, never two of them at once)
  constexpr int kBufs = Be2Ctx<PPT>::kBig ? 2 : 3;
  c.opx = base;
  c.opp = base + np;
  c.ops = Be2Ctx<PPT>::kBig ? base : base + 2 * (size_t)np;
  c.red = base + kBufs * (size_t)np;
  double* cf = c.red + 4 * kNW;
  c.par = 0;
  for (int i = threadIdx.x; i < kBufs * np; i += kT) base[i] = 0.0;  // ghost rings stay 0
  if constexpr (Be2Ctx<PPT>::kBig) {
    c.cf = P.coef;  // [5][M] then minv[M], contiguous (pit_context_create)
  } else if constexpr (!Be2Ctx<PPT>::kRegCoef) {
    for (int i = threadIdx.x; i < 5 * P.M; i += kT) cf[i] = P.coef[i];
    for (int i = threadIdx.x; i < P.M; i += kT) cf[5 * P.M + i] = P.minv[i];
    c.cf = cf;
  } else {
    c.cf = nullptr;
  }
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = threadIdx.x + k * kT;
    c.gi[k] = i < P.M ? i : 0;
    if (i < P.M) {
      const int ix = i % P.m, iy = i / P.m;
      c.ip[k] = (iy + 1) * c.pitch + ix + 1;
      c.ir[k] = c.ip[k];
    } else {
      c.ip[k] = -1;
      c.ir[k] = c.pitch + 1;  // point 0: in bounds with all its neighbours
    }
    if constexpr (Be2Ctx<PPT>::kRegCoef) {
#pragma unroll
      for (int j = 0; j < 5; ++j) c.cr[j][k] = i < P.M ? P.coef[(size_t)j * P.M + i] : 0.0;
      c.cr[5][k] = i < P.M ? P.minv[i] : 0.0;
    }
  }
  __syncthreads();
}

template <int PPT>
__device__ __forceinline__ void load_block(const Be2Ctx<PPT>& c, Vec<PPT>& dst, const double* src) {
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    dst[k] = (src && c.ip[k] >= 0) ? src[threadIdx.x + k * kT] : 0.0;
}

// Fine batch (SlabArgs semantics of K1): CTA b propagates its input block and
// writes out + b*M (apply_F / residual / propagate epilogues).
template <int PPT>
__global__ void __launch_bounds__(kBe2Threads, 1)
    be2d_batch_kernel(const __grid_constant__ Be2Params P, const __grid_constant__ SlabArgs A,
                      const int with_source) {
  if (A.skip != nullptr && *A.skip) return;  // device solver loop: branch taken
  extern __shared__ __align__(16) unsigned char smem_raw[];
  long long tb0 = 0;  // busy time of the slab (DevStatus::busy_ns)
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb0));
  Be2Ctx<PPT> c;
  setup<PPT>(c, P, smem_raw);
  const int b = blockIdx.x, slab = A.slab0 + b;
  const int M = P.M;
  const double* src = b + A.in_shift >= 0 ? (A.in ? A.in + (size_t)(b + A.in_shift) * M : nullptr)
                                          : A.halo;
  Vec<PPT> y;
  load_block(c, y, src);
  const double* tab =
      with_source && P.tab != nullptr ? P.tab + (size_t)slab * P.steps * (size_t)M : nullptr;
  const bool ok = propagate(c, y, P, nullptr, nullptr, tab);
  if (!ok && threadIdx.x == 0) atomicMin(A.status, slab);
  const size_t off = (size_t)b * M;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = threadIdx.x + k * kT;
    if (i < M) {
      if (A.mode == kApplyF) {
        A.out[off + i] = A.Lsub[off + i] - y[k];
      } else if (A.mode == kResidual) {
        const double a = A.Lsub[off + i] - y[k];
        A.out[off + i] = A.rhs[off + i] - a;
      } else {
        A.out[off + i] = y[k];
      }
    }
  }
  if (b == 0 && A.out0 != nullptr) {
    for (int i = threadIdx.x; i < M; i += kT) {
      if (A.mode == kApplyF)
        A.out0[i] = A.L0[i];
      else if (A.mode == kResidual)
        A.out0[i] = A.rhs0[i] - A.L0[i];
    }
  }
  if (A.busy_ns != nullptr && threadIdx.x == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    atomicAdd(A.busy_ns, (unsigned long long)(t1 - tb0));
  }
}

// Sequential sweep (SweepArgs semantics of K2): W_b = Prop(W_{b-1}) (+ V_b).
template <int PPT>
__global__ void __launch_bounds__(kBe2Threads, 1)
    be2d_sweep_kernel(const __grid_constant__ Be2Params P, const __grid_constant__ SweepArgs A,
                      const int with_source) {
  if (A.skip != nullptr && *A.skip) return;  // device solver loop: branch taken
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Be2Ctx<PPT> c;
  setup<PPT>(c, P, smem_raw);
  const int M = P.M;
  Vec<PPT> y;
  load_block(c, y, A.start);
  for (int b = 0; b < A.count; ++b) {
    const double* tab = with_source && P.tab != nullptr
                            ? P.tab + (size_t)(A.slab0 + b) * P.steps * (size_t)M
                            : nullptr;
    if (!propagate(c, y, P, P.iters, A.fail_info, tab)) {
      if (threadIdx.x == 0) atomicMin(A.status, A.slab0 + b);
      return;
    }
    double* W = A.W + (size_t)b * M;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int i = threadIdx.x + k * kT;
      if (i < M) {
        if (A.V) y[k] = y[k] + A.V[(size_t)b * M + i];  // W_n = G(W_{n-1}) + V_n (block_system.cpp:187-188)
        W[i] = y[k];
      }
    }
  }
}

}  // namespace

size_t be2d_smem_bytes(int m, int my) {
  // three padded operand buffers, reduction slots, and (more than 3 points
  // per thread) the stencil rows and Jacobi inverse
  const size_t np = my == 1 ? (size_t)(m + 2) : (size_t)(m + 2) * (my + 2), M = (size_t)m * my;
  const size_t ppt = (M + kBe2Threads - 1) / kBe2Threads;
  if (ppt > 5) return sizeof(double) * (2 * np + 4 * kNW);
  const bool reg_coef = ppt <= 3;
  return sizeof(double) * (3 * np + 4 * kNW + (reg_coef ? 0 : 6 * M));
}

bool be2d_supported(int m, int my) {
  return m >= 1 && my >= 1 && (long long)m * my <= kBe2MaxPPT * kBe2Threads &&
         be2d_smem_bytes(m, my) <= 227 * 1024;
}

#define PIT_BE2_PPT(X) X(1) X(2) X(3) X(4) X(5) X(8) X(12) X(16) X(20)
// compiled point count for a grid: exact up to 5, then the next of 8, 12, 16, 20
static int be2d_ppt(int M) {
  const int ppt = (M + kBe2Threads - 1) / kBe2Threads;
  return ppt <= 5 ? ppt : 4 * ((ppt + 3) / 4);
}

cudaError_t launch_be2d_batch(const Be2Params& P, const SlabArgs& A, int slabs, cudaStream_t st,
                              bool src) {
  if (slabs <= 0) return cudaSuccess;
  if (!be2d_supported(P.m, P.my)) return cudaErrorInvalidValue;
  const int ppt = be2d_ppt(P.M);
  if (ppt > 5 && P.minv != P.coef + 5 * (size_t)P.M) return cudaErrorInvalidValue;
  const size_t smem = be2d_smem_bytes(P.m, P.my);
#define X(N)                                                                              \
  if (ppt == N) {                                                                         \
    auto k = be2d_batch_kernel<N>;                                                        \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                         (int)smem);                                      \
    if (e != cudaSuccess) return e;                                                       \
    k<<<slabs, kBe2Threads, smem, st>>>(P, A, src ? 1 : 0);                                            \
    return cudaGetLastError();                                                            \
  }
  PIT_BE2_PPT(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_be2d_sweep(const Be2Params& P, const SweepArgs& A, cudaStream_t st, bool src) {
  if (A.count <= 0) return cudaSuccess;
  if (!be2d_supported(P.m, P.my)) return cudaErrorInvalidValue;
  const int ppt = be2d_ppt(P.M);
  if (ppt > 5 && P.minv != P.coef + 5 * (size_t)P.M) return cudaErrorInvalidValue;
  const size_t smem = be2d_smem_bytes(P.m, P.my);
#define X(N)                                                                              \
  if (ppt == N) {                                                                         \
    auto k = be2d_sweep_kernel<N>;                                                        \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                         (int)smem);                                      \
    if (e != cudaSuccess) return e;                                                       \
    k<<<1, kBe2Threads, smem, st>>>(P, A, src ? 1 : 0);                                                \
    return cudaGetLastError();                                                            \
  }
  PIT_BE2_PPT(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

}  // namespace pitb
