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
// the slabs in order (coarse sweep, sequential fine solve).  All solver
// vectors live in shared memory in a zero-padded (m+2)^2 layout, so the
// stencil reads its neighbours without bounds tests; thread t owns interior
// points t, t+T, ... (PPT of them), whose stencil rows and Jacobi inverse
// stay in registers.  Reductions: per-thread fma chain over its points in
// order, xor butterfly, warp totals summed in order by every thread (one
// block barrier).  oracle/pit_oracle2d_be.c performs the identical
// operation sequence.
#include "pit_kernels2d.cuh"

#include <cmath>

namespace pitb {
namespace {

constexpr int kT = kBe2Threads, kNW = kBe2Threads / 32;

template <int PPT>
struct Be2Ctx {
  int m, M, pitch;
  int ip[PPT];        // padded index of owned point k (or -1)
  double cs[PPT], cw[PPT], cc[PPT], ce[PPT], cn[PPT], mi[PPT];
  double* red;        // [2][2][kNW]
  int par;            // reduction slot set
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

// <a,b> (and <c,d>) over the interior: per-thread fma chains in point order
template <int PPT>
__device__ __forceinline__ double dot1(Be2Ctx<PPT>& c, const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) s = fma(a[c.ip[k]], b[c.ip[k]], s);
  return block_sum2(c, s, 0.0).x;
}
template <int PPT>
__device__ __forceinline__ double2 dot2(Be2Ctx<PPT>& c, const double* a, const double* b,
                                        const double* e, const double* f) {
  double s = 0.0, t = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) {
      s = fma(a[c.ip[k]], b[c.ip[k]], s);
      t = fma(e[c.ip[k]], f[c.ip[k]], t);
    }
  return block_sum2(c, s, t);
}

// (A x)_i in CSR column order south, west, centre, east, north
// (assemble_spatial_operator's row order); x must be visible (barrier).
template <int PPT>
__device__ __forceinline__ double stencil(const Be2Ctx<PPT>& c, int k, const double* x) {
  const int i = c.ip[k];
  double s = 0.0;
  s = fma(c.cs[k], x[i - c.pitch], s);
  s = fma(c.cw[k], x[i - 1], s);
  s = fma(c.cc[k], x[i], s);
  s = fma(c.ce[k], x[i + 1], s);
  s = fma(c.cn[k], x[i + c.pitch], s);
  return s;
}

// r = b - A x (true_residual, sparse.cpp:53-58); returns ||r||
template <int PPT>
__device__ __forceinline__ double true_residual(Be2Ctx<PPT>& c, const double* b, const double* x,
                                                double* r) {
  __syncthreads();  // x complete
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) {
      const int i = c.ip[k];
      r[i] = b[i] - stencil(c, k, x);
      s = fma(r[i], r[i], s);
    }
  return sqrt(block_sum2(c, s, 0.0).x);
}

// Vectors of one solve (padded, in shared memory).
struct Be2Vec {
  double *x, *b, *r, *rt, *p, *ph, *v, *s, *sh, *t;
};

// Jacobi-PCG, control flow of solve_cg (sparse.cpp:60-114).  Uses x, b, r,
// and p (padded operand), v (z), t (q).  Returns true when converged.
template <int PPT>
__device__ bool cg_solve(Be2Ctx<PPT>& c, const Be2Vec& V, double rel_tol, int cap, int* iters) {
  double *x = V.x, *b = V.b, *r = V.r, *p = V.p, *z = V.v, *q = V.t;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) x[c.ip[k]] = 0.0;
  const double norm_b = sqrt(dot1(c, b, b));
  *iters = 0;
  if (norm_b == 0.0) return true;
  const double tol = rel_tol * norm_b;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) {
      const int i = c.ip[k];
      r[i] = b[i];
      z[i] = c.mi[k] * r[i];
      p[i] = z[i];
    }
  double2 d = dot2(c, r, z, r, r);
  double rz = d.x, res = sqrt(d.y);
  int it = 0;
  bool stalled = false;
  for (;;) {
    while (res > tol && it < cap && !stalled) {
      __syncthreads();  // p complete
      double pq = 0.0;
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (c.ip[k] >= 0) {
          const int i = c.ip[k];
          q[i] = stencil(c, k, p);
          pq = fma(p[i], q[i], pq);
        }
      pq = block_sum2(c, pq, 0.0).x;
      if (pq == 0.0 || !isfinite(pq)) {
        stalled = true;
        break;
      }
      const double alpha = rz / pq;
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (c.ip[k] >= 0) {
          const int i = c.ip[k];
          x[i] = fma(alpha, p[i], x[i]);
          r[i] = fma(-alpha, q[i], r[i]);
          z[i] = c.mi[k] * r[i];
        }
      ++it;
      d = dot2(c, r, r, r, z);
      res = sqrt(d.x);
      if (!isfinite(res) || res <= tol) break;
      const double beta = d.y / rz;
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (c.ip[k] >= 0) {
          const int i = c.ip[k];
          p[i] = fma(beta, p[i], z[i]);
        }
      rz = d.y;
    }
    // confirm against the exact residual (sparse.cpp:97-110)
    res = true_residual(c, b, x, r);
    *iters = it;
    if (res <= tol) return true;
    if (it >= cap || stalled || !isfinite(res)) return false;
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) {
        const int i = c.ip[k];
        z[i] = c.mi[k] * r[i];
        p[i] = z[i];
      }
    rz = dot1(c, r, z);
  }
}

// Jacobi-BiCGStab, control flow of solve_bicgstab (sparse.cpp:116-206).
template <int PPT>
__device__ bool bicgstab_solve(Be2Ctx<PPT>& c, const Be2Vec& V, double rel_tol, int cap,
                               int* iters) {
  double *x = V.x, *b = V.b, *r = V.r, *rt = V.rt, *p = V.p, *ph = V.ph, *v = V.v, *s = V.s,
         *sh = V.sh, *t = V.t;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) x[c.ip[k]] = 0.0;
  const double norm_b = sqrt(dot1(c, b, b));
  *iters = 0;
  if (norm_b == 0.0) return true;
  const double tol = rel_tol * norm_b;
  double rho_prev = 1.0, alpha = 1.0, omega = 1.0, res = 0.0;
  int it = 0;
  bool restart = true, first = true;
  auto set_rt = [&]() {
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) rt[c.ip[k]] = r[c.ip[k]];
  };
  while (it < cap) {
    if (restart) {
      res = true_residual(c, b, x, r);
      if (res <= tol) {
        *iters = it;
        return true;
      }
      if (!isfinite(res)) {
        *iters = it;
        return false;
      }
      set_rt();
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
      for (int k = 0; k < PPT; ++k)
        if (c.ip[k] >= 0) p[c.ip[k]] = r[c.ip[k]];
      first = false;
    } else {
      const double beta = (rho / rho_prev) * (alpha / omega);
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (c.ip[k] >= 0) {
          const int i = c.ip[k];
          p[i] = fma(beta, fma(-omega, v[i], p[i]), r[i]);
        }
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) ph[c.ip[k]] = c.mi[k] * p[c.ip[k]];
    __syncthreads();  // ph complete
    double rv = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) {
        const int i = c.ip[k];
        v[i] = stencil(c, k, ph);
        rv = fma(rt[i], v[i], rv);
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
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) {
        const int i = c.ip[k];
        s[i] = fma(-alpha, v[i], r[i]);
        ss = fma(s[i], s[i], ss);
      }
    if (sqrt(block_sum2(c, ss, 0.0).x) <= tol) {
      // half-iteration exit; keep going from the exact residual if spurious
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (c.ip[k] >= 0) x[c.ip[k]] = fma(alpha, ph[c.ip[k]], x[c.ip[k]]);
      ++it;
      res = true_residual(c, b, x, r);
      if (res <= tol) {
        *iters = it;
        return true;
      }
      if (!isfinite(res)) {
        *iters = it;
        return false;
      }
      set_rt();
      first = true;
      rho_prev = 1.0;
      alpha = 1.0;
      omega = 1.0;
      continue;
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) sh[c.ip[k]] = c.mi[k] * s[c.ip[k]];
    __syncthreads();  // sh complete
    double tt = 0.0, ts = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) {
        const int i = c.ip[k];
        t[i] = stencil(c, k, sh);
        tt = fma(t[i], t[i], tt);
        ts = fma(t[i], s[i], ts);
      }
    const double2 d = block_sum2(c, tt, ts);
    omega = d.x == 0.0 ? 0.0 : d.y / d.x;
    double rr = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0) {
        const int i = c.ip[k];
        x[i] = fma(omega, sh[i], fma(alpha, ph[i], x[i]));
        r[i] = fma(-omega, t[i], s[i]);
        rr = fma(r[i], r[i], rr);
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
  return res <= tol;
}

// `steps` backward-Euler steps of the state in V.b (padded), result in V.b.
// Returns false at the first step whose solve fails or is non-finite
// (InnerSolveError, pde.cpp:119-128).
template <int PPT>
__device__ bool propagate(Be2Ctx<PPT>& c, Be2Vec& V, const Be2Params& P, long long* iters) {
  for (int step = 0; step < P.steps; ++step) {
    int it = 0;
    const bool ok = P.symmetric ? cg_solve(c, V, P.rel_tol, P.cap, &it)
                                : bicgstab_solve(c, V, P.rel_tol, P.cap, &it);
    if (iters && threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(iters),
                                             (unsigned long long)it);
    bool bad = !ok;
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (c.ip[k] >= 0 && !isfinite(V.x[c.ip[k]])) bad = true;
    if (__syncthreads_or(bad)) return false;
    double* nb = V.x;  // the solution is the next right-hand side
    V.x = V.b;
    V.b = nb;
  }
  return true;
}

template <int PPT>
__device__ void setup(Be2Ctx<PPT>& c, Be2Vec& V, const Be2Params& P, unsigned char* smem) {
  c.m = P.m;
  c.M = P.M;
  c.pitch = P.m + 2;
  const int np = c.pitch * c.pitch;
  double* base = reinterpret_cast<double*>(smem);
  double* vec[10];
  for (int v = 0; v < 10; ++v) vec[v] = base + (size_t)v * np;
  V = Be2Vec{vec[0], vec[1], vec[2], vec[3], vec[4], vec[5], vec[6], vec[7], vec[8], vec[9]};
  c.red = base + (size_t)10 * np;
  c.par = 0;
  for (int i = threadIdx.x; i < 10 * np; i += kT) base[i] = 0.0;  // ghost rings stay 0
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = threadIdx.x + k * kT;
    if (i < P.M) {
      const int ix = i % P.m, iy = i / P.m;
      c.ip[k] = (iy + 1) * c.pitch + ix + 1;
      c.cs[k] = P.coef[i];
      c.cw[k] = P.coef[P.M + i];
      c.cc[k] = P.coef[2 * P.M + i];
      c.ce[k] = P.coef[3 * P.M + i];
      c.cn[k] = P.coef[4 * P.M + i];
      c.mi[k] = P.minv[i];
    } else {
      c.ip[k] = -1;
      c.cs[k] = c.cw[k] = c.cc[k] = c.ce[k] = c.cn[k] = c.mi[k] = 0.0;
    }
  }
  __syncthreads();
}

template <int PPT>
__device__ __forceinline__ void load_block(const Be2Ctx<PPT>& c, double* dst, const double* src) {
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (c.ip[k] >= 0) dst[c.ip[k]] = src ? src[threadIdx.x + k * kT] : 0.0;
}

// Fine batch (SlabArgs semantics of K1): CTA b propagates its input block and
// writes out + b*M (apply_F / residual / propagate epilogues).
template <int PPT>
__global__ void __launch_bounds__(kBe2Threads, 1)
    be2d_batch_kernel(const __grid_constant__ Be2Params P, const __grid_constant__ SlabArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Be2Ctx<PPT> c;
  Be2Vec V;
  setup<PPT>(c, V, P, smem_raw);
  const int b = blockIdx.x, slab = A.slab0 + b;
  const int M = P.M;
  const double* src = b + A.in_shift >= 0 ? (A.in ? A.in + (size_t)(b + A.in_shift) * M : nullptr)
                                          : A.halo;
  load_block(c, V.b, src);
  const bool ok = propagate(c, V, P, nullptr);
  if (!ok && threadIdx.x == 0) atomicMin(A.status, slab);
  const size_t off = (size_t)b * M;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = threadIdx.x + k * kT;
    if (i < M) {
      const double y = V.b[c.ip[k]];
      if (A.mode == kApplyF) {
        A.out[off + i] = A.Lsub[off + i] - y;
      } else if (A.mode == kResidual) {
        const double a = A.Lsub[off + i] - y;
        A.out[off + i] = A.rhs[off + i] - a;
      } else {
        A.out[off + i] = y;
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
}

// Sequential sweep (SweepArgs semantics of K2): W_b = Prop(W_{b-1}) (+ V_b).
template <int PPT>
__global__ void __launch_bounds__(kBe2Threads, 1)
    be2d_sweep_kernel(const __grid_constant__ Be2Params P, const __grid_constant__ SweepArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Be2Ctx<PPT> c;
  Be2Vec V;
  setup<PPT>(c, V, P, smem_raw);
  const int M = P.M;
  load_block(c, V.b, A.start);
  for (int b = 0; b < A.count; ++b) {
    if (!propagate(c, V, P, P.iters)) {
      if (threadIdx.x == 0) atomicMin(A.status, A.slab0 + b);
      return;
    }
    double* W = A.W + (size_t)b * M;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int i = threadIdx.x + k * kT;
      if (i < M) {
        double y = V.b[c.ip[k]];
        if (A.V) {
          y = y + A.V[(size_t)b * M + i];  // W_n = G(W_{n-1}) + V_n (block_system.cpp:187-188)
          V.b[c.ip[k]] = y;
        }
        W[i] = y;
      }
    }
  }
}

template <class K>
cudaError_t launch_be2(K k, int grid, size_t smem, const Be2Params& P, const void* args,
                       cudaStream_t st);

}  // namespace

size_t be2d_smem_bytes(int m) {
  const size_t np = (size_t)(m + 2) * (m + 2);
  return sizeof(double) * (10 * np + 4 * kNW);
}

bool be2d_supported(int m) {
  return m >= 1 && m * m <= kBe2MaxPPT * kBe2Threads && be2d_smem_bytes(m) <= 227 * 1024;
}

#define PIT_BE2_PPT(X) X(1) X(2) X(3) X(4) X(5)

cudaError_t launch_be2d_batch(const Be2Params& P, const SlabArgs& A, int slabs, cudaStream_t st) {
  if (slabs <= 0) return cudaSuccess;
  if (!be2d_supported(P.m)) return cudaErrorInvalidValue;
  const int ppt = (P.M + kBe2Threads - 1) / kBe2Threads;
  const size_t smem = be2d_smem_bytes(P.m);
#define X(N)                                                                              \
  if (ppt == N) {                                                                         \
    auto k = be2d_batch_kernel<N>;                                                        \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                         (int)smem);                                      \
    if (e != cudaSuccess) return e;                                                       \
    k<<<slabs, kBe2Threads, smem, st>>>(P, A);                                            \
    return cudaGetLastError();                                                            \
  }
  PIT_BE2_PPT(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_be2d_sweep(const Be2Params& P, const SweepArgs& A, cudaStream_t st) {
  if (A.count <= 0) return cudaSuccess;
  if (!be2d_supported(P.m)) return cudaErrorInvalidValue;
  const int ppt = (P.M + kBe2Threads - 1) / kBe2Threads;
  const size_t smem = be2d_smem_bytes(P.m);
#define X(N)                                                                              \
  if (ppt == N) {                                                                         \
    auto k = be2d_sweep_kernel<N>;                                                        \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                         (int)smem);                                      \
    if (e != cudaSuccess) return e;                                                       \
    k<<<1, kBe2Threads, smem, st>>>(P, A);                                                \
    return cudaGetLastError();                                                            \
  }
  PIT_BE2_PPT(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

}  // namespace pitb
