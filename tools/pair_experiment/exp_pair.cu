// A/B timing of the plain step loop (pit_step.cuh be_solve) against the
// paired steps (pit_pair.cuh) on c2-like slabs, with a numerical comparison.
// An experiment, not product code (DESIGN.md §6 "Paired steps"): measured
// 6-7 % faster than the plain loop for one wave of c2 slabs, but not in the
// product's piece-scheduled batches, so it is not built into libpit_b200.so.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -lineinfo \
//        -I include -I paper_2203_10148_b200/csrc -I tools/pair_experiment \
//        tools/pair_experiment/exp_pair.cu paper_2203_10148_b200/csrc/coeffs.cpp \
//        -o tools/_bin/exp_pair
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "coeffs.h"
#include "pit_pair.cuh"

struct StepParamsX : pitb::StepParams {
  pitb::PairParams pair;
};

// Host recipe of the paired-step extras (long double, rounded once): the
// corner at M-1 (z'' = L^-1 U^-1 e_(M-1)), the folded corners B z' and F z'',
// second-level carry weights, pass-1 fix-up constants, per-lane corner gains.
struct PairCoeffs {
  int enabled = 0, K0M = 0, G = 0;
  double invG = 0, invGlast = 0, gnegM = 0, pS2 = 0, qS2 = 0, p32_2 = 0, q32_2 = 0;
  double pp2[5] = {}, qq2[5] = {}, plane2[32] = {}, qlane2[32] = {}, nupow[32] = {}, kap[2][2] = {};
  std::vector<double> gain;
};
static void build_pair_coeffs(const pit_step_coeffs& c, PairCoeffs* q) {
  typedef long double ld;
  *q = PairCoeffs();
  const int M = c.M, sub = c.mpt / (c.nsub * c.nseg), ch = c.nsub * sub, T = 32 * c.warps;
  q->gain.assign(2 * 2 * 8 * 32, 0.0);
  if (c.nseg != 1 || T * c.mpt != M || !c.narrow || c.steps < 2 || c.nsub > 8) return;
  const ld nl = c.nl, nu = c.nu, invd = c.inv;
  const ld thr = 8.470329472543003e-22L;  // 2^-70
  std::vector<ld> z((size_t)M), v((size_t)M);
  z[0] = 1.0L;
  for (int i = 1; i < M; ++i) z[i] = nl * z[i - 1];
  for (int i = M - 2; i >= 0; --i) z[i] = z[i] + nu * z[i + 1];
  v = z;
  for (int i = M - 2; i >= 0; --i) v[i] = v[i] + nu * v[i + 1];
  const ld z00 = z[0], v00 = v[0];
  z.assign((size_t)M, 0.0L);
  z[M - 1] = 1.0L;
  for (int i = M - 2; i >= 0; --i) z[i] = nu * z[i + 1];
  for (int i = 1; i < M; ++i) z[i] = z[i] + nl * z[i - 1];
  v = z;
  for (int i = 1; i < M; ++i) v[i] = v[i] + nl * v[i - 1];
  const ld zL = z[M - 1], vL = v[M - 1];
  int k0m = 1;
  for (int i = 0; i < M - 1; ++i)
    if (fabsl(z[(size_t)i]) > fabsl(zL) * thr) {
      k0m = M - i;
      break;
    }
  if (!(k0m <= 32 * ch && powl(fabsl(nl * nu), (ld)(M - k0m)) < 7.7e-34L)) return;
  q->K0M = k0m;
  const ld sa = ((ld)c.delta - 1.0L / invd) * invd;
  const ld gM = -(sa / (1.0L + sa * zL)), g0 = (ld)c.gneg;
  q->gnegM = (double)gM;
  for (int l = 0; l < 32; ++l)
    for (int u = 0; u < c.nsub; ++u) {
      const int d0 = l * ch + u * sub, dM = (31 - l) * ch + u * sub;
      if (d0 < c.K0) {
        q->gain[((0 * 2 + 0) * 8 + u) * 32 + l] = (double)(g0 * z00 * powl(nl, (ld)d0));
        q->gain[((0 * 2 + 1) * 8 + u) * 32 + l] = (double)(g0 * v00 * powl(nl, (ld)d0));
      }
      if (dM < k0m) {
        q->gain[((1 * 2 + 0) * 8 + u) * 32 + l] = (double)(gM * zL * powl(nu, (ld)dM));
        q->gain[((1 * 2 + 1) * 8 + u) * 32 + l] = (double)(gM * vL * powl(nu, (ld)dM));
      }
    }
  ld nlp[65], nup[65];
  nlp[0] = nup[0] = 1.0L;
  for (int k = 1; k <= 64; ++k) nlp[k] = nlp[k - 1] * nl, nup[k] = nup[k - 1] * nu;
  for (int j = 0; j < sub; ++j) q->nupow[j] = (double)nup[j];
  q->pS2 = (double)((ld)sub * nlp[sub]);
  q->qS2 = (double)((ld)sub * nup[sub]);
  q->kap[0][0] = (double)((ld)sub * nlp[sub - 1]);
  q->kap[0][1] = (double)((ld)(sub * (sub + 1) / 2) * nlp[sub - 1]);
  q->kap[1][0] = (double)((ld)sub * nup[sub - 1]);
  q->kap[1][1] = (double)((ld)(sub * (sub + 1) / 2) * nup[sub - 1]);
  ld pk = nlp[ch], qk = nup[ch], len = (ld)ch;
  for (int k = 0; k < 5; ++k) {
    q->pp2[k] = (double)(len * pk);
    q->qq2[k] = (double)(len * qk);
    pk = pk * pk, qk = qk * qk, len = len * 2.0L;
  }
  q->p32_2 = (double)(len * pk);
  q->q32_2 = (double)(len * qk);
  ld pl = 1.0L, ql = 1.0L;
  for (int l = 0; l < 32; ++l) {
    q->plane2[l] = (double)((ld)(l * ch) * pl);
    q->qlane2[31 - l] = (double)((ld)(l * ch) * ql);
    pl = pl * nlp[ch], ql = ql * nup[ch];
  }
  q->G = c.R;
  q->invG = c.invR;
  q->invGlast = c.invLast;
  q->enabled = 1;
}

using namespace pitb;

#ifndef PAIR_REGS
#define PAIR_REGS 168
#endif
template <class S>
__global__ void __launch_bounds__(S::T, 65536 / (S::T * (S::MPT > 32 ? 168 : PAIR_REGS)))
    plain_kernel(const __grid_constant__ StepParams P, const double* in, double* out) {
  __shared__ StepShared<S::NSEG, S::WARPS> sh;
  const int tid = threadIdx.x;
  init_step_shared<S::NSEG, S::WARPS>(P, sh, tid);
  double y[S::NC][S::SUB];
  const double* src = in + (size_t)blockIdx.x * P.M;
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) y[c][j] = src[S::point(tid, c, j)];
  __syncthreads();
  StepLane L{};
  L.zt = (P.narrow && tid < 32 && tid * S::CH < P.K0) ? P.zt[tid] : 0.0;
  int cnt = 0;
#ifdef PIT_PHASE_TIMING
  long long ph_acc[16] = {};
  long long ph_t = clock64();
#endif
  for (int k = 0; k < P.steps; ++k) {
#ifdef PIT_PHASE_TIMING
    be_solve<S, false, false>(y, P, L, sh, nullptr, tid, false, nullptr, ph_acc, ph_t);
#else
    be_solve<S, false, false>(y, P, L, sh, nullptr, tid, false, nullptr);
#endif
    if (++cnt == P.R) {
      cnt = 0;
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int j = 0; j < S::SUB; ++j) y[c][j] = y[c][j] * P.invR;
    }
  }
#ifdef PIT_PHASE_TIMING
  if (P.timing && blockIdx.x == 0 && (tid & 31) == 0 && (tid >> 5) < 2)
    for (int k = 0; k < 10; ++k) P.timing[(tid >> 5) * 16 + k] += ph_acc[k];
#endif
  if (cnt) {
#pragma unroll
    for (int c = 0; c < S::NC; ++c)
#pragma unroll
      for (int j = 0; j < S::SUB; ++j) y[c][j] = y[c][j] * P.invLast;
  }
  double* dst = out + (size_t)blockIdx.x * P.M;
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) dst[S::point(tid, c, j)] = y[c][j];
}

template <class S, int D>
#ifndef PAIR_REGS
#define PAIR_REGS 168
#endif
__global__ void __launch_bounds__(S::T, 65536 / (S::T * (S::MPT > 32 ? 168 : PAIR_REGS)))
    pair_kernel(const __grid_constant__ StepParamsX P, const double* in, double* out) {
  __shared__ PairShared<S::WARPS> sh;
  const int tid = threadIdx.x;
  init_pair_shared<StepParamsX, S::WARPS>(P, sh, tid);
  double y[S::NC][S::SUB];
  const double* src = in + (size_t)blockIdx.x * P.M;
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) y[c][j] = src[S::point(tid, c, j)];
  __syncthreads();
  int par = 0;
  run_slab_paired<StepParamsX, S>(y, P, sh, tid, 0, P.steps, par);
  double* dst = out + (size_t)blockIdx.x * P.M;
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) dst[S::point(tid, c, j)] = y[c][j];
}

static double* upload(const std::vector<double>& v) {
  double* d;
  cudaMalloc(&d, v.size() * sizeof(double));
  cudaMemcpy(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice);
  return d;
}

template <class S, int D>
void run(const char* name, int M, int slabs, int steps, double lo, double dg, double up, double dt) {
  pit_step_coeffs c;
  std::vector<double> zc, ppos, qpos, zt;
  if (build_step_coeffs(M, S::MPT, S::NSUB, S::NSEG, S::WARPS, steps, lo, dg, up, dt, &c, &zc, &ppos,
                        &qpos, &zt) != 0) {
    printf("%s: coeffs failed\n", name);
    return;
  }
  PairCoeffs q;
  build_pair_coeffs(c, &q);
  printf("%s: nl %.4f nu %.4f K0 %d K0M %d R %d scan %d/%d narrow %d pair %d (KS %d)\n", name, c.nl,
         c.nu, c.K0, q.K0M, c.R, c.scan_f, c.scan_b, c.narrow, q.enabled, S::KS);
  if (!q.enabled) return;
  StepParamsX P{};
  P.nl = c.nl, P.nu = c.nu, P.inv = c.inv, P.gneg = c.gneg, P.invR = c.invR, P.invLast = c.invLast;
  P.pS = c.pS, P.qS = c.qS, P.Pseg = c.Pseg, P.Qseg = c.Qseg, P.narrow = c.narrow;
  const int sub = S::SUB;
  for (int u = 0; u < 8; ++u) P.pw[u] = u < c.nsub ? c.pw[u] : 0.0;
  for (int j = 0; j < 32; ++j) {
    P.nlpow[j] = j < sub ? c.nlpow[j] : 0.0;
    P.plane[j] = c.plane[j], P.qlane[j] = c.qlane[j];
  }
  for (int s = 0; s < 5; ++s) P.pp[s] = c.pp[s], P.qq[s] = c.qq[s];
  P.p32 = c.p32, P.q32 = c.q32, P.M = M, P.steps = steps, P.R = c.R, P.K0 = c.K0;
  P.scan_f = c.scan_f, P.scan_b = c.scan_b;
  P.zt = upload(zt);
  PairParams& Q = P.pair;
  Q.enabled = 1, Q.K0M = q.K0M, Q.G = q.G, Q.invG = q.invG, Q.invGlast = q.invGlast;
  Q.pS2 = q.pS2, Q.qS2 = q.qS2, Q.p32_2 = q.p32_2, Q.q32_2 = q.q32_2;
  for (int s = 0; s < 5; ++s) Q.pp2[s] = q.pp2[s], Q.qq2[s] = q.qq2[s];
  for (int j = 0; j < 32; ++j) {
    Q.plane2[j] = q.plane2[j], Q.qlane2[j] = q.qlane2[j];
    Q.nupow[j] = j < sub ? q.nupow[j] : 0.0;
  }
  for (int d = 0; d < 2; ++d) Q.kap[d][0] = q.kap[d][0], Q.kap[d][1] = q.kap[d][1];
  Q.gain = upload(q.gain);

  std::vector<double> h((size_t)slabs * M);
  srand(1);
  for (auto& v : h) v = rand() / (double)RAND_MAX * 2 - 1;
  // smooth component so the result is not pure decay
  for (int b = 0; b < slabs; ++b)
    for (int i = 0; i < M; ++i) h[(size_t)b * M + i] += 3.0 * sin(3.14159265358979 * (i + 1) / (M + 1.0));
  double* din = upload(h);
  double *o1, *o2;
  cudaMalloc(&o1, h.size() * 8);
  cudaMalloc(&o2, h.size() * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  float best1 = 1e9, best2 = 1e9;
#ifdef PIT_PHASE_TIMING
  long long* dtim;
  cudaMalloc(&dtim, 32 * 8);
  P.timing = dtim;
  for (int which = 0; which < 2; ++which) {
    cudaMemset(dtim, 0, 32 * 8);
    if (which == 0) plain_kernel<S><<<slabs, S::T>>>(static_cast<const StepParams&>(P), din, o1);
    else pair_kernel<S, D><<<slabs, S::T>>>(P, din, o2);
    long long ht[32];
    cudaMemcpy(ht, dtim, 32 * 8, cudaMemcpyDeviceToHost);
    for (int w = 0; w < 2; ++w) {
      printf("%s %s warp %d cycles/step by phase:", name, which ? "paired" : "plain", w);
      long long tot = 0;
      for (int k = 0; k < 10; ++k) printf(" %lld", ht[w * 16 + k] / steps), tot += ht[w * 16 + k];
      printf("  total %lld\n", tot / steps);
    }
  }
#endif
  for (int it = 0; it < 5; ++it) {
    float ms;
    cudaEventRecord(e0);
    plain_kernel<S><<<slabs, S::T>>>(static_cast<const StepParams&>(P), din, o1);
    cudaEventRecord(e1), cudaEventSynchronize(e1), cudaEventElapsedTime(&ms, e0, e1);
    best1 = fminf(best1, ms);
    cudaEventRecord(e0);
    pair_kernel<S, D><<<slabs, S::T>>>(P, din, o2);
    cudaEventRecord(e1), cudaEventSynchronize(e1), cudaEventElapsedTime(&ms, e0, e1);
    best2 = fminf(best2, ms);
  }
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<double> a(h.size()), b(h.size());
  cudaMemcpy(a.data(), o1, a.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), o2, b.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (size_t i = 0; i < a.size(); ++i) md = fmax(md, fabs(a[i] - b[i])), mx = fmax(mx, fabs(a[i]));
  const double gp = (double)slabs * M * steps;
  printf("%s: slabs %d  plain %.3f ms (%.3fe12 gp/s)  paired %.3f ms (%.3fe12 gp/s)  max|diff| %.3e (max|y| %.3e) %s\n",
         name, slabs, best1, gp / best1 / 1e9, best2, gp / best2 / 1e9, md, mx, cudaGetErrorString(err));
  int occ1 = 0, occ2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, plain_kernel<S>, S::T, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, pair_kernel<S, D>, S::T, 0);
  cudaFuncAttributes f1, f2;
  cudaFuncGetAttributes(&f1, plain_kernel<S>);
  cudaFuncGetAttributes(&f2, pair_kernel<S, D>);
  printf("%s: regs %d/%d  CTAs per SM %d/%d  local %zu/%zu\n", name, f1.numRegs, f2.numRegs, occ1, occ2,
         (size_t)f1.localSizeBytes, (size_t)f2.localSizeBytes);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // one c2 case with the given slab count (for ncu)
    const int M = 4096;
    const double h = 1.0 / (M + 1), dt = 1.0 / 1024 / 1000;
    const double o = -1.0 / (h * h), d = 2.0 / (h * h);
    run<Shape<16, 4, 1, 2, 2>, 4>("c2 n", M, atoi(argv[1]), 1000, o, d, o, dt);
    return 0;
  }
  {  // c2: heat, M = 4096, 1000 steps per slab of length 1/1024
    const int M = 4096;
    const double h = 1.0 / (M + 1), dt = 1.0 / 1024 / 1000;
    const double o = -1.0 / (h * h), d = 2.0 / (h * h);
    run<Shape<16, 4, 1, 2, 2>, 4>("c2", M, 1023, 1000, o, d, o, dt);
    run<Shape<16, 4, 1, 2, 2>, 4>("c2 one wave", M, 888, 1000, o, d, o, dt);
    run<Shape<16, 4, 1, 2, 2>, 4>("c2 1/SM", M, 148, 1000, o, d, o, dt);
    run<Shape<16, 4, 1, 2, 2>, 4>("c2 2/SM", M, 296, 1000, o, d, o, dt);
    run<Shape<16, 4, 1, 2, 2>, 4>("c2 4/SM", M, 592, 1000, o, d, o, dt);
  }
  {  // c4: reaction-diffusion r = 5, M = 8192, 500 steps per slab of 1/2048
    const int M = 8192;
    const double h = 1.0 / (M + 1), dt = 1.0 / 2048 / 500;
    const double o = -1.0 / (h * h), d = 2.0 / (h * h) + 5.0;
    run<Shape<16, 4, 1, 4, 3>, 8>("c4", M, 2047, 500, o, d, o, dt);
  }
  {  // c3: advection-diffusion nu = 1e-2, a = 1 central, M = 2048, 2000 steps per slab of 1/512
    const int M = 2048;
    const double h = 1.0 / (M + 1), dt = 1.0 / 512 / 2000, nu = 1e-2;
    const double lo = -nu / (h * h) - 1.0 / (2 * h), up = -nu / (h * h) + 1.0 / (2 * h);
    run<Shape<16, 4, 1, 1, 0>, 1>("c3", M, 511, 2000, lo, 2 * nu / (h * h), up, dt);
  }
  return 0;
}
