// DFMA throughput vs (independent chains per thread) x (warps per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chains(double* out, int iters, double a) {
  double v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = fma(a, v[k], v[(k + 1) % ILP]);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 1.2345) out[0] = s;
}
template <int ILP>
void run(int warps, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  chains<ILP><<<148, 32 * warps>>>(d, 10, 0.999);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  chains<ILP><<<148, 32 * warps>>>(d, iters, 0.999);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 148.0 * 32 * warps * ILP * iters;
  printf("ILP %d warps/SM %2d: %.2f DFMA/clk/SM (at 1.95GHz)\n", ILP, warps, n / (ms * 1e-3) / 148 / 1.95e9);
}
int main() {
  double* d; cudaMalloc(&d, 64);
  for (int w : {1, 2, 4, 8, 16, 32}) { run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d); }
  return 0;
}
