// pit_kernels.cu — K3, the BiCGStab block algebra (block_system.cpp:31-87,
// solvers.cpp:159-215) fused into four passes with fixed-order per-block
// reductions; the device-resident solver loop's scalar kernel; the FP64 pipe
// probe.  K1 (slab_kernel) and K2 (the coarse sweeps) are in
// pit_kernels_impl.cuh, instantiated by pit_k1.cu and pit_k2.cu.
#include <cstdint>

#include "pit_kernels.cuh"
#include "pit_sync.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

namespace pitb {

namespace {

// ---------------------------------------------------------------------------
// K3 vector kernels
// ---------------------------------------------------------------------------

// Warp butterfly (shfl_xor 16..1) then warp totals summed in warp order by
// thread 0.  ws holds kVecThreads/32 doubles.  Result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* ws) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(kFull, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    s = ws[0];
#pragma unroll
    for (int w = 1; w < kVecThreads / 32; ++w) s = s + ws[w];
  }
  return s;
}

struct DotPtrs {
  const double* a[3];
  const double* b[3];
};

template <int NP>
__global__ void __launch_bounds__(kVecThreads) dots_kernel(int M, double weight, DotPtrs ptr,
                                                           double* __restrict__ partials,
                                                           const SolverScalars* sc) {
  if (sc != nullptr && sc->stop) return;
  __shared__ double ws[NP][kVecThreads / 32];
  const size_t off = (size_t)blockIdx.x * M;
  double acc[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = 0.0;
  for (int i = threadIdx.x; i < M; i += kVecThreads) {
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[k] = fma(ptr.a[k][off + i], ptr.b[k][off + i], acc[k]);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const double s = block_sum(acc[k], ws[k]);
    if (threadIdx.x == 0) partials[(size_t)blockIdx.x * NP + k] = weight * s;
  }
}

__global__ void __launch_bounds__(kVecThreads)
    update_s_kernel(int M, double weight, double alpha, const double* __restrict__ r,
                    const double* __restrict__ d, double* __restrict__ s,
                    double* __restrict__ partials, const SolverScalars* sc) {
  if (sc != nullptr) {
    if (sc->stop) return;
    alpha = sc->alpha;
  }
  __shared__ double ws[kVecThreads / 32];
  const size_t off = (size_t)blockIdx.x * M;
  const double na = -alpha;
  double acc = 0.0;
  for (int i = threadIdx.x; i < M; i += kVecThreads) {
    const double v = fma(na, d[off + i], r[off + i]);
    s[off + i] = v;
    acc = fma(v, v, acc);
  }
  const double t = block_sum(acc, ws);
  if (threadIdx.x == 0) partials[blockIdx.x] = weight * t;
}

__global__ void __launch_bounds__(kVecThreads)
    update_lr_kernel(int M, double weight, double alpha, double omega,
                     const double* __restrict__ p, const double* __restrict__ s,
                     const double* __restrict__ t, const double* __restrict__ rs,
                     double* __restrict__ lam, double* __restrict__ r,
                     double* __restrict__ partials, const SolverScalars* sc) {
  if (sc != nullptr) {
    if (sc->stop) return;
    alpha = sc->alpha;
    omega = sc->omega;
  }
  __shared__ double ws[2][kVecThreads / 32];
  const size_t off = (size_t)blockIdx.x * M;
  const double nw = -omega;
  double acc0 = 0.0, acc1 = 0.0;
  for (int i = threadIdx.x; i < M; i += kVecThreads) {
    const double sv = s[off + i];
    double l = lam[off + i];
    l = fma(alpha, p[off + i], l);
    l = fma(omega, sv, l);
    lam[off + i] = l;
    const double rv = fma(nw, t[off + i], sv);
    r[off + i] = rv;
    acc0 = fma(rv, rv, acc0);
    acc1 = fma(rv, rs[off + i], acc1);
  }
  const double a = block_sum(acc0, ws[0]);
  const double c = block_sum(acc1, ws[1]);
  if (threadIdx.x == 0) {
    partials[2 * (size_t)blockIdx.x] = weight * a;
    partials[2 * (size_t)blockIdx.x + 1] = weight * c;
  }
}

__global__ void update_p_kernel(size_t n, double omega, double beta, const double* __restrict__ d,
                                const double* __restrict__ r, double* __restrict__ p,
                                const SolverScalars* sc) {
  if (sc != nullptr) {
    if (sc->stop) return;
    omega = sc->omega;
    beta = sc->beta;
  }
  const double nw = -omega;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = fma(fma(nw, d[i], p[i]), beta, r[i]);
}

__global__ void axpy_kernel(size_t n, double a, const double* __restrict__ x,
                            double* __restrict__ y, const double* a_dev) {
  if (a_dev != nullptr) a = *a_dev;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void add_kernel(size_t n, const double* __restrict__ x, double* __restrict__ y) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = y[i] + x[i];
}

// The sums and branch tests of pitsbicg_solve's scalar recurrence in the
// host loop's exact order (sum_partials / max_sqrt_partials in pit_capi.cu,
// i.e. block_inner_product / block_norm_n_inf): the CTA stages the partials
// (and their square roots) in shared memory in chunks, thread 0 runs the
// sequential sums over them.
constexpr int kScChunk = 2048;  // blocks per staged chunk
__global__ void __launch_bounds__(256) scalars_kernel(SolverScalars* sc, const double* __restrict__ h,
                                                      int N, int phase, double tol, double eps0) {
  if (sc->stop) return;
  __shared__ double a0[kScChunk], a1[kScChunk], rt[kScChunk];
  const int np = (phase == kScOmega || phase == kScR) ? 2 : 1;
  double s0 = 0.0, s1 = 0.0, w = 0.0;
  for (int c0 = 0; c0 < N; c0 += kScChunk) {
    const int n = N - c0 < kScChunk ? N - c0 : kScChunk;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double a = h[(size_t)(c0 + i) * np];
      a0[i] = a;
      rt[i] = sqrt(a);
      if (np == 2) a1[i] = h[(size_t)(c0 + i) * np + 1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < n; ++i) {
        s0 += a0[i];
        const double v = rt[i];
        w = (w < v) ? v : w;  // std::max(w, v)
        if (np == 2) s1 += a1[i];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  switch (phase) {
    case kScRho:
      sc->rho = s0;
      break;
    case kScAlpha:
      sc->d_dot = s0;
      if (fabs(s0) < 1e-300) {
        sc->flag = kFlagRestartD;
        sc->stop = 1;
      } else {
        sc->alpha = sc->rho / s0;
      }
      break;
    case kScSnorm:
      sc->s_norm = w;
      if (w <= tol) {
        sc->flag = kFlagHalf;
        sc->stop = 1;
      }
      break;
    case kScOmega:
      sc->tt = s0;
      sc->ts = s1;
      if (s0 < 1e-300) {
        sc->flag = kFlagRestartT;
        sc->stop = 1;
      } else {
        sc->omega = s1 / s0;
        if (fabs(sc->omega) < 1e-300) {
          sc->flag = kFlagRestartW;
          sc->stop = 1;
        }
      }
      break;
    case kScR: {
      sc->r_norm = w;
      sc->rr = s0;
      sc->r_dot = s1;
      if (w <= tol) {
        sc->flag = kFlagConverged;
        sc->stop = 1;
        break;
      }
      const double m = fabs(s1) / eps0;
      sc->margin = sc->margin < m ? sc->margin : m;
      if (fabs(s1) <= eps0) {
        sc->flag = kFlagRestartR;
        sc->stop = 1;
        sc->rho = s0;
      } else {
        sc->beta = (sc->alpha / sc->omega) * (s1 / sc->rho);
        sc->rho = s1;
      }
      break;
    }
  }
}

int ew_grid(size_t n) {
  size_t g = (n + 255) / 256;
  const size_t cap = 148 * 16;
  return (int)(g < cap ? (g ? g : 1) : cap);
}

}  // namespace

// FP64 pipe probe for the roofline denominator: 8 independent DFMA chains per
// thread, 8 x 256-thread CTAs per SM.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, double a) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fma(v[k], a, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 1.2345) out[0] = s;
}

cudaError_t measure_fp64_peak(double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 64);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = sms * 8, iters = 40000;
  fp64_probe_kernel<<<grid, 256>>>(d, 100, 1.0000001);
  cudaEventRecord(e0);
  fp64_probe_kernel<<<grid, 256>>>(d, iters, 1.0000001);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *tflops = 2.0 * 8 * iters * (double)grid * 256 / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return e;
}

cudaError_t launch_dots(int M, int blocks, double weight, int np, const double* const* a,
                        const double* const* b, double* partials, cudaStream_t st,
                        const SolverScalars* sc) {
  if (blocks <= 0) return cudaSuccess;
  DotPtrs p{};
  for (int k = 0; k < np; ++k) {
    p.a[k] = a[k];
    p.b[k] = b[k];
  }
  switch (np) {
    case 1: dots_kernel<1><<<blocks, kVecThreads, 0, st>>>(M, weight, p, partials, sc); break;
    case 2: dots_kernel<2><<<blocks, kVecThreads, 0, st>>>(M, weight, p, partials, sc); break;
    case 3: dots_kernel<3><<<blocks, kVecThreads, 0, st>>>(M, weight, p, partials, sc); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_update_s(int M, int blocks, double weight, double alpha, const double* r,
                            const double* d, double* s, double* partials, cudaStream_t st,
                            const SolverScalars* sc) {
  if (blocks <= 0) return cudaSuccess;
  update_s_kernel<<<blocks, kVecThreads, 0, st>>>(M, weight, alpha, r, d, s, partials, sc);
  return cudaGetLastError();
}

cudaError_t launch_update_lr(int M, int blocks, double weight, double alpha, double omega,
                             const double* p, const double* s, const double* t, const double* rs,
                             double* lam, double* r, double* partials, cudaStream_t st,
                             const SolverScalars* sc) {
  if (blocks <= 0) return cudaSuccess;
  update_lr_kernel<<<blocks, kVecThreads, 0, st>>>(M, weight, alpha, omega, p, s, t, rs, lam, r,
                                                   partials, sc);
  return cudaGetLastError();
}

cudaError_t launch_update_p(size_t n, double omega, double beta, const double* d, const double* r,
                            double* p, cudaStream_t st, const SolverScalars* sc) {
  if (!n) return cudaSuccess;
  update_p_kernel<<<ew_grid(n), 256, 0, st>>>(n, omega, beta, d, r, p, sc);
  return cudaGetLastError();
}

cudaError_t launch_axpy(size_t n, double a, const double* x, double* y, cudaStream_t st,
                        const double* a_dev) {
  if (!n) return cudaSuccess;
  axpy_kernel<<<ew_grid(n), 256, 0, st>>>(n, a, x, y, a_dev);
  return cudaGetLastError();
}

cudaError_t launch_scalars(SolverScalars* sc, const double* partials, int N, int phase, double tol,
                           double eps0, cudaStream_t st) {
  scalars_kernel<<<1, 256, 0, st>>>(sc, partials, N, phase, tol, eps0);
  return cudaGetLastError();
}

cudaError_t launch_add(size_t n, const double* x, double* y, cudaStream_t st) {
  if (!n) return cudaSuccess;
  add_kernel<<<ew_grid(n), 256, 0, st>>>(n, x, y);
  return cudaGetLastError();
}

}  // namespace pitb
