// SHFL / LDS throughput per SM: independent 32-bit shuffles, varying warps.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void shfl_tput(float* out, int iters) {
  float v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = __shfl_up_sync(0xffffffffu, v[k], 1 + (k & 7));
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 1.2345f) out[0] = s;
}
template <int ILP>
__global__ void lds_tput(double* out, int iters) {
  __shared__ double t[5][32];
  if (threadIdx.x < 32) for (int s = 0; s < 5; ++s) t[s][threadIdx.x] = threadIdx.x * s;
  __syncthreads();
  double v = 0;
  int l = threadIdx.x & 31;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v += t[k % 5][(l + i) & 31];
  }
  if (v == 1.2345) out[0] = v;
}
int main() {
  float* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    int iters = 4000;
    shfl_tput<8><<<148, 32 * w>>>(d, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); shfl_tput<8><<<148, 32 * w>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = 8.0 * iters * w;  // warp-SHFLs per SM
    printf("SHFL ILP8 warps/SM %2d: %.3f warp-SHFL/clk/SM  (%.1f clk per SHFL per warp)\n", w, n / (ms * 1e-3 * 1.95e9), (ms * 1e-3 * 1.95e9) / (8.0 * iters));
  }
  for (int w : {1, 4, 16}) {
    int iters = 4000;
    lds_tput<8><<<148, 32 * w>>>((double*)d, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); lds_tput<8><<<148, 32 * w>>>((double*)d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = 8.0 * iters * w;
    printf("LDS.64 ILP8 warps/SM %2d: %.3f warp-LDS/clk/SM\n", w, n / (ms * 1e-3 * 1.95e9));
  }
  return 0;
}
