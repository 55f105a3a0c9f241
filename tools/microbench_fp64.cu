// FP64 pipe / shuffle / barrier microbenchmarks for the PiT fine-propagator
// roofline (SURVEY.md §8(d) asks for a measured FP64 peak before quoting
// roofline fractions).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = fma(v[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 123.456) out[0] = s;
}

__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v = fma(v, a, b);
  }
  long long t1 = clock64();
  out[0] = v;
  cyc[0] = t1 - t0;
}

__global__ void shfl_lat(double* out, long long* cyc, int iters) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v = __shfl_up_sync(0xffffffffu, v, 1) + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void bar_lat(double* out, long long* cyc, int iters) {
  __shared__ double s[1024];
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[threadIdx.x] = v;
    __syncthreads();
    v = s[(threadIdx.x + 1) % blockDim.x] + 1.0;
    __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d clock(kHz) %d regsPerSM %d smemPerSM %zu\n", p.name, p.multiProcessorCount, p.clockRate, p.regsPerMultiprocessor, p.sharedMemPerMultiprocessor);
  double* d; long long* c; CK(cudaMalloc(&d, 1 << 20)); CK(cudaMalloc(&c, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    for (int blocksPerSM : {1, 2, 4, 8}) {
      if (threads * blocksPerSM > 2048) continue;
      int grid = sms * blocksPerSM;
      dfma_tput<8><<<grid, threads>>>(d, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_tput<8><<<grid, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * (double)grid * threads;
      printf("dfma_tput ILP8 threads %d blocks/SM %d: %.3f ms  %.2f TFLOP/s (%.1f DFMA/clk/SM at %.0f MHz nominal)\n",
             threads, blocksPerSM, ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1e3);
    }
  }
  long long h;
  dfma_lat<<<1, 1>>>(d, c, 1000, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  dfma_lat<<<1, 1>>>(d, c, 1000, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dfma dependent latency: %.2f clk\n", h / 16000.0);
  shfl_lat<<<1, 32>>>(d, c, 1000); CK(cudaDeviceSynchronize());
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("shfl(double)+dadd dependent latency: %.2f clk\n", h / 16000.0);
  for (int t : {64, 128, 256, 512, 1024}) {
    bar_lat<<<1, t>>>(d, c, 1000); CK(cudaDeviceSynchronize());
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("2x syncthreads + sts/lds round, %d threads: %.1f clk\n", t, h / 1000.0);
  }
  return 0;
}
