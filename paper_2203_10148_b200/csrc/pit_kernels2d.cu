// pit_kernels2d.cu — config 5 (2D heat) kernels.  DESIGN.md §3b.
//
// K4 explicit2d_kernel: one thread-block cluster per slab holds the m x m
//   state in registers (TR x TC tile per thread) across all fine steps.
//   West/east neighbours come from the adjacent lanes (warp shuffles; a warp
//   spans the full row width, so lanes 0/31 sit on the Dirichlet boundary);
//   north/south neighbours of a tile's first/last row come from the warp
//   above/below through shared memory, and across CTAs through distributed
//   shared memory.  One cluster barrier per step, split arrive/wait: the
//   tile's interior rows are updated between the arrive of step k-1 and the
//   wait of step k, hiding the barrier latency.
// K5 cg_sweep2d_kernel: one persistent cluster runs the sequential coarse
//   sweep; each slab's backward-Euler step is a Jacobi-PCG solve with the
//   control flow of the reference's solve_cg (src/sparse.cpp:60-114): exit
//   on res <= tol, true-residual confirmation, restart, stall and cap.
//   Reductions: per-thread fma chain over its column strip, warp butterfly,
//   one slot per warp in every CTA of the cluster (DSMEM stores), a cluster
//   barrier, then every thread sums the slots in the same fixed order.
// Every operation order here is mirrored by oracle/pit_oracle2d.c.
#include "pit_kernels2d.cuh"
#include "pit_sync.cuh"

#include <cooperative_groups.h>

#include <cmath>

namespace cg = cooperative_groups;

namespace pitb {
namespace {

__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_sync() {
  cl_arrive();
  cl_wait();
}

// G^-1 F overlap (SlabArgs::ready / SweepArgs::ready): block flags written by
// K4's clusters and read by the concurrently running K5
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// one thread: spin until *flag == epoch; never hang the device on a lost
// producer — give up after 20 s and report the slab as failed
__device__ __noinline__ void wait_block_ready(const int* flag, int epoch, int* status, int slab) {
  long long t0 = -1;
  while (ld_acquire_gpu(flag) != epoch) {
    long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (t0 < 0) t0 = now;
    if (now - t0 > 20000000000LL) {
      atomicMin(status, slab);
      return;
    }
    __nanosleep(256);
  }
}

// y' = fma(ac, y, an * ((w + e) + (n + s)))
__device__ __forceinline__ double ex_point(double ac, double an, double y, double w, double e,
                                           double n, double s) {
  return fma(ac, y, an * ((w + e) + (n + s)));
}

__device__ __forceinline__ void st_async_1(uint32_t raddr, double a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(
                   raddr),
               "d"(a), "r"(rbar)
               : "memory");
}
// TC doubles of a tile row into a peer's row buffer
template <int TC>
__device__ __forceinline__ void send_row(uint32_t raddr, const double (&v)[TC], uint32_t rbar) {
  if constexpr (TC % 2 == 0) {
#pragma unroll
    for (int j = 0; j < TC; j += 2) st_async_v2(raddr + 8 * j, v[j], v[j + 1], rbar);
  } else {
#pragma unroll
    for (int j = 0; j < TC; ++j) st_async_1(raddr + 8 * j, v[j], rbar);
  }
}

template <int TR, int TC, int CL, int WARPS>
struct Tile2 {
  static_assert(TR >= 2, "tile needs a first and a last row");
  static constexpr int T = 32 * WARPS;
  static constexpr int NC = 32 * TC;       // columns covered by a warp row
  static constexpr int ROWS = WARPS * TR;  // rows per CTA
  // top[2][WARPS+1][NC], bot[2][WARPS+1][NC], then mbarriers [WARPS][2]
  static constexpr size_t smem =
      sizeof(double) * 4 * (WARPS + 1) * NC + 2 * WARPS * sizeof(uint64_t);
};

// K4.  Per step k (state y^k in registers, halo rows of y^k in buffer k&1):
//   each warp waits on its own mbarrier for the halo rows of y^k (arrivals
//   of the warps above/below after their shared-memory stores; st.async
//   byte counts from the neighbour CTA for the cluster-edge warps), computes
//   its tiles' first and last rows of y^{k+1}, publishes them (shared-memory
//   stores + arrivals, st.async into the neighbour CTA's buffer (k+1)&1),
//   then computes the interior rows while those stores fly.  Buffer (k+1)&1
//   was last read at step k-1 by a reader that published y^k only after that
//   read, and the writer waited for y^k: no CTA or cluster barrier inside the
//   step loop, and a warp's step is coupled only to its neighbours'.
template <bool SCALED>
__device__ __forceinline__ double ex_update(const Ex2Params& P, double y, double w, double e,
                                            double n, double s) {
  if constexpr (SCALED) return fma(P.kappa, y, (w + e) + (n + s));
  return ex_point(P.ac, P.an, y, w, e, n, s);
}

template <int TR, int TC, int CL, int WARPS, bool SCALED>
__global__ void __launch_bounds__(32 * WARPS, 1)
    explicit2d_kernel(const __grid_constant__ Ex2Params P, const __grid_constant__ SlabArgs A) {
  if (A.skip != nullptr && *A.skip) return;  // device solver loop: branch taken
  using S = Tile2<TR, TC, CL, WARPS>;
  extern __shared__ __align__(16) double sm2[];
  // top(par, w): first row of warp w's tiles (w == WARPS: CTA below's warp 0)
  // bot(par, w): last row of warp w-1's tiles (w == 0: CTA above's last warp)
  double* const top = sm2;
  double* const bot = sm2 + 2 * (WARPS + 1) * S::NC;
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(sm2 + 4 * (WARPS + 1) * S::NC);  // [w][par]
  auto TOP = [&](int par, int w) { return top + ((size_t)par * (WARPS + 1) + w) * S::NC; };
  auto BOT = [&](int par, int w) { return bot + ((size_t)par * (WARPS + 1) + w) * S::NC; };
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int b = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = P.m;
  const int row0 = c * S::ROWS + warp * TR;
  const int col0 = lane * TC;
  const bool ghosts = (CL * S::ROWS > m) || (S::NC > m);
  // halo bytes this warp receives per step from neighbour CTAs
  const bool rx_up = warp == 0 && c > 0, rx_dn = warp == WARPS - 1 && c < CL - 1;
  const unsigned rx_bytes = (unsigned)sizeof(double) * S::NC * (rx_up + rx_dn);
  uint64_t* const my_bar = &mbar[2 * warp];
  long long tb0 = 0;  // busy time of the slab (DevStatus::busy_ns)
  if (c == 0 && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb0));

  for (int i = tid; i < 4 * (WARPS + 1) * S::NC; i += S::T) sm2[i] = 0.0;
  if (tid < WARPS) {
    // own arrive.expect_tx + one arrival per neighbouring warp
    const unsigned cnt = 1 + (tid > 0) + (tid < WARPS - 1);
    mbar_init(&mbar[2 * tid], cnt);
    mbar_init(&mbar[2 * tid + 1], cnt);
  }
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");

  const double* src;
  if (b + A.in_shift >= 0)
    src = A.in ? A.in + (size_t)(b + A.in_shift) * m * m : nullptr;
  else
    src = A.halo;
  double y[TR][TC];
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) {
      const int r = row0 + i, q = col0 + j;
      y[i][j] = (src && r < m && q < m) ? src[(size_t)r * m + q] : 0.0;
    }
  // peer addresses (shared::cluster) of the row buffers this warp feeds
  // (CTA c-1's last warp and CTA c+1's warp 0 consume them)
  constexpr uint32_t kParBytes = (uint32_t)(sizeof(double) * (WARPS + 1) * S::NC);
  const uint32_t up_top = c > 0 ? mapa_u32(smem_u32(TOP(0, WARPS) + col0), c - 1) : 0u;
  const uint32_t up_bar = c > 0 ? mapa_u32(smem_u32(&mbar[2 * (WARPS - 1)]), c - 1) : 0u;
  const uint32_t dn_bot = c < CL - 1 ? mapa_u32(smem_u32(BOT(0, 0) + col0), c + 1) : 0u;
  const uint32_t dn_bar = c < CL - 1 ? mapa_u32(smem_u32(&mbar[0]), c + 1) : 0u;
  cl_sync();  // zeroed buffers and initialised mbarriers cluster-wide

  auto publish = [&](int par, bool remote) {
    double* t0 = TOP(par, warp) + col0;
    double* b0 = BOT(par, warp + 1) + col0;
#pragma unroll
    for (int j = 0; j < TC; ++j) {
      t0[j] = y[0][j];
      b0[j] = y[TR - 1][j];
    }
    __syncwarp();
    if (lane == 0) {  // the warps above and below may read them now
      if (warp > 0) mbar_arrive(&mbar[2 * (warp - 1) + par]);
      if (warp < WARPS - 1) mbar_arrive(&mbar[2 * (warp + 1) + par]);
    }
    if (!remote) return;
    if (warp == 0 && c > 0) send_row<TC>(up_top + par * kParBytes, y[0], up_bar + 8 * par);
    if (warp == WARPS - 1 && c < CL - 1)
      send_row<TC>(dn_bot + par * kParBytes, y[TR - 1], dn_bar + 8 * par);
  };
  // west/east neighbours of row i from the adjacent lanes (a warp spans the
  // full width: lanes 0 and 31 border the Dirichlet walls)
  double Wv[TR], Ev[TR];
  auto shfl_row = [&](int i) {
    const double w = __shfl_up_sync(kFull, y[i][TC - 1], 1);
    const double e = __shfl_down_sync(kFull, y[i][0], 1);
    Wv[i] = lane == 0 ? 0.0 : w;
    Ev[i] = lane == 31 ? 0.0 : e;
  };
  if (lane == 0) mbar_arrive_expect_tx(&my_bar[0], rx_bytes);
  publish(0, true);

  int until_rescale = P.R;
#ifdef PIT_PHASE_TIMING
  long long tacc[6] = {};
  long long tt = clock64();
#define K4_PHASE(i)                     \
  do {                                  \
    const long long now_ = clock64();   \
    tacc[i] += now_ - tt;               \
    tt = now_;                          \
  } while (0)
#else
#define K4_PHASE(i) \
  do {              \
  } while (0)
#endif
  for (int k = 0; k < P.steps; ++k) {
    const int par = k & 1;
    const bool more = k + 1 < P.steps;  // y^{k+1} halos are consumed
    if (lane == 0 && more) mbar_arrive_expect_tx(&my_bar[par ^ 1], rx_bytes);
    bool rs = false;
    if (SCALED) {
      // fold an^R back before step k when k is a positive multiple of R
      if (until_rescale == 0) {
        rs = true;
        until_rescale = P.R;
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) y[i][j] = y[i][j] * P.anR;
      }
      --until_rescale;
    }
#pragma unroll
    for (int i = 0; i < TR; ++i) shfl_row(i);
    K4_PHASE(0);
    mbar_wait(&my_bar[par], (k >> 1) & 1);  // halo rows of y^k
    K4_PHASE(1);
    // new first/last rows into separate registers: y keeps y^k until the
    // interior rows are done
    double n0[TC], nT[TC];
    {
      const double* nb = BOT(par, warp) + col0;
      const double* sb = TOP(par, warp + 1) + col0;
      double Nv[TC], Sv[TC];
#pragma unroll
      for (int j = 0; j < TC; ++j) {
        Nv[j] = nb[j];
        Sv[j] = sb[j];
        if (SCALED && rs) {
          Nv[j] = Nv[j] * P.anR;
          Sv[j] = Sv[j] * P.anR;
        }
      }
#pragma unroll
      for (int j = 0; j < TC; ++j)
        n0[j] = ex_update<SCALED>(P, y[0][j], j > 0 ? y[0][j - 1] : Wv[0],
                                  j < TC - 1 ? y[0][j + 1] : Ev[0], Nv[j], y[1][j]);
#pragma unroll
      for (int j = 0; j < TC; ++j)
        nT[j] = ex_update<SCALED>(P, y[TR - 1][j], j > 0 ? y[TR - 1][j - 1] : Wv[TR - 1],
                                  j < TC - 1 ? y[TR - 1][j + 1] : Ev[TR - 1], y[TR - 2][j], Sv[j]);
    }
    if (ghosts) {
#pragma unroll
      for (int j = 0; j < TC; ++j) {
        if (row0 >= m || col0 + j >= m) n0[j] = 0.0;
        if (row0 + TR - 1 >= m || col0 + j >= m) nT[j] = 0.0;
      }
    }
    K4_PHASE(2);
    {  // publish y^{k+1} first/last rows; their shuffles for step k+1
      double* t0 = TOP(par ^ 1, warp) + col0;
      double* b0 = BOT(par ^ 1, warp + 1) + col0;
#pragma unroll
      for (int j = 0; j < TC; ++j) {
        t0[j] = n0[j];
        b0[j] = nT[j];
      }
      __syncwarp();
      if (lane == 0) {
        if (warp > 0) mbar_arrive(&mbar[2 * (warp - 1) + (par ^ 1)]);
        if (warp < WARPS - 1) mbar_arrive(&mbar[2 * (warp + 1) + (par ^ 1)]);
      }
      if (more) {
        if (warp == 0 && c > 0) send_row<TC>(up_top + (par ^ 1) * kParBytes, n0, up_bar + 8 * (par ^ 1));
        if (warp == WARPS - 1 && c < CL - 1)
          send_row<TC>(dn_bot + (par ^ 1) * kParBytes, nT, dn_bar + 8 * (par ^ 1));
      }
    }
    K4_PHASE(3);
    // interior rows 1..TR-2 of y^{k+1}
    {
      double prev[TC];
#pragma unroll
      for (int j = 0; j < TC; ++j) prev[j] = y[0][j];
#pragma unroll
      for (int i = 1; i < TR - 1; ++i) {
        double cur[TC];
#pragma unroll
        for (int j = 0; j < TC; ++j) cur[j] = y[i][j];
#pragma unroll
        for (int j = 0; j < TC; ++j)
          y[i][j] = ex_update<SCALED>(P, cur[j], j > 0 ? cur[j - 1] : Wv[i],
                                      j < TC - 1 ? cur[j + 1] : Ev[i], prev[j], y[i + 1][j]);
        if (ghosts) {
#pragma unroll
          for (int j = 0; j < TC; ++j)
            if (row0 + i >= m || col0 + j >= m) y[i][j] = 0.0;
        }
#pragma unroll
        for (int j = 0; j < TC; ++j) prev[j] = cur[j];
      }
    }
#pragma unroll
    for (int j = 0; j < TC; ++j) {
      y[0][j] = n0[j];
      y[TR - 1][j] = nT[j];
    }
    K4_PHASE(4);
  }
#ifdef PIT_PHASE_TIMING
  if (P.timing && blockIdx.x == 0 && lane == 0)
    for (int i = 0; i < 5; ++i) P.timing[warp * 8 + i] = tacc[i];
#endif
  if (SCALED) {
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) y[i][j] = y[i][j] * P.anLast;
  }
  cl_sync();  // no CTA leaves while a peer may still address its buffers

  const int slab = A.slab0 + b;
  bool fin = true;
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) fin = fin && isfinite(y[i][j]);
  if (!__all_sync(kFull, fin) && lane == 0) atomicMin(A.status, slab);
  const size_t off = (size_t)b * m * m;
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) {
      const int r = row0 + i, q = col0 + j;
      if (r < m && q < m) {
        const size_t g = off + (size_t)r * m + q;
        if (A.mode == kApplyF) {
          A.out[g] = A.Lsub[g] - y[i][j];
        } else if (A.mode == kResidual) {
          const double a = A.Lsub[g] - y[i][j];
          A.out[g] = A.rhs[g] - a;
        } else {
          A.out[g] = y[i][j];
        }
      }
    }
  if (blockIdx.x == 0 && A.out0 != nullptr) {
    const int n = m * m;
    if (A.mode == kApplyF) {
      for (int i = tid; i < n; i += S::T) A.out0[i] = A.L0[i];
    } else if (A.mode == kResidual) {
      for (int i = tid; i < n; i += S::T) A.out0[i] = A.rhs0[i] - A.L0[i];
    }
  }
  if (A.busy_ns != nullptr && c == 0 && tid == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    atomicAdd(A.busy_ns, (unsigned long long)(t1 - tb0));
  }
  if (A.ready != nullptr) {
    // every CTA's output stores precede the cluster barrier (release /
    // acquire at cluster scope), which precedes thread 0's release at gpu
    // scope (cumulativity): the sweep's acquire of ready[g] sees the block
    __threadfence();
    cl_sync();
    if (c == 0 && tid == 0) {
      __threadfence();
      st_release_gpu(A.ready + b + A.block_shift, A.epoch);
      if (b == 0 && A.out0 != nullptr) st_release_gpu(A.ready, A.epoch);
    }
  }
}

template <class K>
cudaError_t launch_clustered(K kernel, int grid, int block, size_t smem, int cluster,
                             cudaStream_t st, const void* p0, const void* p1) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if (cluster > 8 &&
      (e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) !=
          cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[2] = {const_cast<void*>(p0), const_cast<void*>(p1)};
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(kernel), args);
}

// ---------------------------------------------------------------------------
// K5
// ---------------------------------------------------------------------------

constexpr int kSlotCap = 128;  // warps per cluster: 16 CTAs x 8 warps

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(kFull, v, off);
  return v;
}

// (S f)_k = fma(D, f, O*((w + e) + (n + s))) from the stencil buffer
__device__ __forceinline__ double stencil_S(const double* Ps, int pitch, int k, int t, double D,
                                            double O) {
  const double* row = Ps + (size_t)(k + 1) * pitch + t + 1;
  const double w = row[-1], e = row[1], n = row[-pitch], s = row[pitch];
  return fma(D, row[0], O * ((w + e) + (n + s)));
}

// K5 synchronisation: no cluster barrier inside the solve.  Reductions:
// every warp st.async's its two partials into every CTA's slot array (set
// `pair`, alternating), counted on that CTA's reduction mbarrier; each CTA
// waits for C*W*16 bytes, sums the slots in slot order.  A set is rewritten
// two reductions later, only after every warp of every CTA sent the
// in-between reduction, i.e. after it read this one.  Field publication for
// the stencil: own rows to shared memory (+ __syncthreads), first/last row
// st.async'd into the neighbours' halo rows, counted on their halo mbarrier.
__global__ void __launch_bounds__(256, 1)
    cg_sweep2d_kernel(const __grid_constant__ Cg2Params P, const __grid_constant__ SweepArgs A,
                      long long* iters) {
  if (A.skip != nullptr && *A.skip) return;  // device solver loop: branch taken
  constexpr int RM = kCgRowsMax;
  extern __shared__ __align__(16) double smc[];
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int C = P.cluster;
  const int NT = blockDim.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int W = NT >> 5;
  const int nslot = C * W;
  const int m = P.m, R = P.rows;
  const int pitch = NT + 2;
  double* const Ps = smc;                              // [(RM+2)][pitch], own rows 1..R
  double* const red = smc + (size_t)(RM + 2) * pitch;  // [2][kSlotCap][2]
  double* const Bs = red + 4 * kSlotCap;               // [RM][NT]: the step's right-hand side
  uint64_t* const bars = reinterpret_cast<uint64_t*>(Bs + (size_t)RM * NT);  // rbar[2], hbar
  const double D = P.D, O = P.O, minv = P.minv;
  const unsigned red_bytes = 16u * (unsigned)nslot;
  const unsigned halo_bytes = 8u * (unsigned)NT * ((c > 0) + (c < C - 1));

  for (int i = t; i < (RM + 2) * pitch + 4 * kSlotCap; i += NT) smc[i] = 0.0;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }

  bool valid[RM];
#pragma unroll
  for (int k = 0; k < RM; ++k) valid[k] = t < m && k < R && c * R + k < m;
  auto gidx = [&](int k) { return (size_t)(c * R + k) * m + t; };

  const int tgt = lane < C ? lane : 0;
  const uint32_t red_to = mapa_u32(smem_u32(red), tgt);
  const uint32_t rbar_to = mapa_u32(smem_u32(&bars[0]), tgt);
  const uint32_t up_row = c > 0 ? mapa_u32(smem_u32(Ps + (size_t)(R + 1) * pitch + t + 1), c - 1) : 0u;
  const uint32_t up_bar = c > 0 ? mapa_u32(smem_u32(&bars[2]), c - 1) : 0u;
  const uint32_t dn_row = c < C - 1 ? mapa_u32(smem_u32(Ps + t + 1), c + 1) : 0u;
  const uint32_t dn_bar = c < C - 1 ? mapa_u32(smem_u32(&bars[2]), c + 1) : 0u;
  cl_sync();  // zeroed buffers, initialised barriers cluster-wide
  if (t == 0) {
    mbar_arrive_expect_tx(&bars[0], red_bytes);
    mbar_arrive_expect_tx(&bars[1], red_bytes);
    mbar_arrive_expect_tx(&bars[2], halo_bytes);
  }

  int pair = 0;
  unsigned rph[2] = {0u, 0u}, hph = 0u;
  // cluster-wide sums of a and b (identical bits in every thread)
  auto reduce2 = [&](double a, double b, double& ra, double& rb) {
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane < C)
      st_async_v2(red_to + 16u * (unsigned)((pair * kSlotCap) + c * W + warp), a, b,
                  rbar_to + 8u * pair);
    mbar_wait(&bars[pair], rph[pair]);
    rph[pair] ^= 1u;
    const double* rs = red + 2 * pair * kSlotCap;
    double u = 0.0, v = 0.0;
    for (int i = lane; i < nslot; i += 32) {
      u = u + rs[2 * i];
      v = v + rs[2 * i + 1];
    }
    ra = warp_sum(u);
    rb = warp_sum(v);
    if (t == 0) mbar_arrive_expect_tx(&bars[pair], red_bytes);  // its next use
    pair ^= 1;
  };
  // f: the published field (the stencil's operand) in registers; its own
  // rows also in the stencil buffer (west/east neighbours of other threads)
  // and its first/last row in the neighbours' halo rows
  double f[RM];
  auto put = [&](int k, double v) {
    f[k] = v;
    if (k < R) Ps[(size_t)(k + 1) * pitch + t + 1] = v;
    if (k == 0 && up_row) st_async_1(up_row, v, up_bar);
    if (k == R - 1 && dn_row) st_async_1(dn_row, v, dn_bar);
  };
  // after a full put(): own rows visible CTA-wide, neighbours' rows landed
  auto published = [&]() {
    __syncthreads();
    mbar_wait(&bars[2], hph);
    hph ^= 1u;
    if (t == 0) mbar_arrive_expect_tx(&bars[2], halo_bytes);
  };
  // (S f)_k = fma(D, f, O*((w + e) + (n + s))): north/south from the strip
  // (halo rows at its ends), west/east from the stencil buffer
  auto stencil = [&](int k) {
    const double* row = Ps + (size_t)(k + 1) * pitch + t + 1;
    const double n = k == 0 ? row[-pitch] : f[k > 0 ? k - 1 : 0];
    const double s = k == R - 1 ? row[pitch] : f[k + 1 < RM ? k + 1 : RM - 1];
    return fma(D, f[k], O * ((row[-1] + row[1]) + (n + s)));
  };

  double x[RM], r[RM], q[RM];
  if (A.ready != nullptr) {  // the start block comes from the running fine batch
    if (t == 0) wait_block_ready(A.ready + A.ready_shift - 1, A.epoch, A.status, A.slab0);
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < RM; ++k) {
    const double v = valid[k] ? A.start[gidx(k)] : 0.0;
    Bs[k * NT + t] = v;
    if (A.W0 != nullptr && valid[k]) A.W0[gidx(k)] = v;  // W_0 = V_0 (block_system.cpp:181)
  }

  long long total_it = 0;
#ifdef PIT_PHASE_TIMING
  long long k5acc[8] = {};
  long long k5t = clock64();
#define K5_T(i)                            \
  do {                                     \
    const long long now_ = clock64();      \
    if (i > 0) k5acc[i] += now_ - k5t;     \
    k5t = now_;                            \
  } while (0)
#else
#define K5_T(i) \
  do {          \
  } while (0)
#endif
  for (int s = 0; s < A.count; ++s) {
    const int slab = A.slab0 + s;
    bool ok = true;
    double fail_rel = 0.0, fail_it = 0.0;  // InnerSolveError payload (errors.hpp:15-21)
    for (int cs = 0; cs < P.steps && ok; ++cs) {
      if (cs > 0) {
#pragma unroll
        for (int k = 0; k < RM; ++k) Bs[k * NT + t] = x[k];
      }
#pragma unroll
      for (int k = 0; k < RM; ++k) x[k] = 0.0;
      double nb2, dummy;
      {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < RM; ++k) {
          const double bk = Bs[k * NT + t];
          a = fma(bk, bk, a);
        }
        reduce2(a, 0.0, nb2, dummy);
      }
      const double nb = sqrt(nb2);
      if (nb != 0.0) {
        const double tol = P.rel_tol * nb;
        double rz, rr;
        {
          double a = 0.0, b2 = 0.0;
#pragma unroll
          for (int k = 0; k < RM; ++k) {
            r[k] = Bs[k * NT + t];
            const double z = minv * r[k];  // p = z
            put(k, z);
            a = fma(r[k], z, a);
            b2 = fma(r[k], r[k], b2);
          }
          published();
          reduce2(a, b2, rz, rr);
        }
        double res = sqrt(rr);
        long long it = 0;
        bool stalled = false;
        for (;;) {
          while (res > tol && it < P.cap && !stalled) {
            double pq, d0;
            K5_T(0);
            {
              double a = 0.0;
#pragma unroll
              for (int k = 0; k < RM; ++k) {
                q[k] = valid[k] ? stencil(k) : 0.0;
                a = fma(f[k], q[k], a);
              }
              K5_T(1);
              reduce2(a, 0.0, pq, d0);
              K5_T(2);
            }
            if (pq == 0.0 || !isfinite(pq)) {
              stalled = true;
              break;
            }
            const double alpha = rz / pq;
            double rzn;
            {
              double a = 0.0, b2 = 0.0;
#pragma unroll
              for (int k = 0; k < RM; ++k) {
                x[k] = fma(alpha, f[k], x[k]);
                r[k] = fma(-alpha, q[k], r[k]);
                const double z = minv * r[k];
                a = fma(r[k], r[k], a);
                b2 = fma(r[k], z, b2);
              }
              ++it;
              K5_T(3);
              reduce2(a, b2, rr, rzn);
              K5_T(4);
            }
            res = sqrt(rr);
            if (!isfinite(res) || res <= tol) break;
            const double beta = rzn / rz;
#pragma unroll
            for (int k = 0; k < RM; ++k) put(k, fma(beta, f[k], minv * r[k]));
            K5_T(5);
            published();
            rz = rzn;
            K5_T(6);
          }
          // confirm against the exact residual (sparse.cpp:101-104)
#pragma unroll
          for (int k = 0; k < RM; ++k) put(k, x[k]);
          published();
          {
            double a = 0.0, b2 = 0.0;
#pragma unroll
            for (int k = 0; k < RM; ++k) {
              r[k] = valid[k] ? Bs[k * NT + t] - stencil(k) : 0.0;
              const double z = minv * r[k];
              a = fma(r[k], r[k], a);
              b2 = fma(r[k], z, b2);
            }
            reduce2(a, b2, rr, rz);
          }
          res = sqrt(rr);
          if (res <= tol) break;
          if (it >= P.cap || stalled || !isfinite(res)) {
            ok = false;
            fail_rel = res / nb;
            fail_it = (double)it;
            break;
          }
#pragma unroll
          for (int k = 0; k < RM; ++k) put(k, minv * r[k]);  // restart: p = z
          published();
        }
        total_it += it;
      }
    }  // coarse steps
    bool fin = true;
#pragma unroll
    for (int k = 0; k < RM; ++k) fin = fin && isfinite(x[k]);
    // every thread of the cluster must agree on leaving the sweep
    double bad_l = (ok && fin) ? 0.0 : 1.0, bad_g, d1;
    reduce2(bad_l, 0.0, bad_g, d1);
    if (bad_g != 0.0) {
      if (c == 0 && t == 0) {
        atomicMin(A.status, slab);
        if (A.fail_info != nullptr) {
          A.fail_info[0] = fail_rel;
          A.fail_info[1] = fail_it;
          A.fail_info[2] = ok ? kFailNonFinite : kFailNotConverged;
        }
      }
      break;
    }
    const double* V = A.V ? A.V + (size_t)s * m * m : nullptr;
    double* Wb = A.W + (size_t)s * m * m;
    if (A.ready != nullptr && V != nullptr) {
      // V_s is needed only now, after the slab's CG solves: the wait hides
      // behind them whenever the fine batch is ahead of the sweep
      if (t == 0) wait_block_ready(A.ready + s + A.ready_shift, A.epoch, A.status, slab);
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < RM; ++k) {
      const double v = valid[k] ? (V ? x[k] + V[gidx(k)] : x[k]) : 0.0;
      if (valid[k]) Wb[gidx(k)] = v;
      Bs[k * NT + t] = v;
    }
  }
  if (iters && c == 0 && t == 0) atomicAdd(reinterpret_cast<unsigned long long*>(iters),
                                           (unsigned long long)total_it);
#ifdef PIT_PHASE_TIMING
  if (P.timing && c == 0 && t == 0)
    for (int i = 0; i < 8; ++i) P.timing[i] = k5acc[i];
#endif
  cl_sync();
}

}  // namespace

bool layout2d_supported(int tr, int tc, int cl, int warps) {
#define X(TR, TC, CL, WW) \
  if (tr == TR && tc == TC && cl == CL && warps == WW) return true;
  PIT_LAYOUTS_2D(X)
#undef X
  return false;
}

Layout2D auto_layout_2d(int m) {
  static const Layout2D order[] = {{2, 1, 2, 8}, {4, 2, 2, 8}, {4, 4, 4, 8}, {8, 8, 4, 8}};
  for (const auto& L : order)
    if (32 * L.tc >= m && L.cl * L.warps * L.tr >= m) return L;
  return {0, 0, 0, 0};
}

cudaError_t launch_explicit2d(const Layout2D& L, const Ex2Params& P, const SlabArgs& A, int slabs,
                              cudaStream_t st) {
  if (slabs <= 0) return cudaSuccess;
#define X(TR, TC, CL, WW)                                                                    \
  if (L.tr == TR && L.tc == TC && L.cl == CL && L.warps == WW) {                             \
    using S = Tile2<TR, TC, CL, WW>;                                                         \
    return P.scaled ? launch_clustered(explicit2d_kernel<TR, TC, CL, WW, true>, CL * slabs,  \
                                       S::T, S::smem, CL, st, &P, &A)                        \
                    : launch_clustered(explicit2d_kernel<TR, TC, CL, WW, false>, CL * slabs, \
                                       S::T, S::smem, CL, st, &P, &A);                       \
  }
  PIT_LAYOUTS_2D(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_cg_sweep2d(const Cg2Params& P, const SweepArgs& A, long long* iters,
                              cudaStream_t st) {
  if (A.count <= 0) return cudaSuccess;
  const int nt = 32 * ((P.m + 31) / 32);
  if (nt > 256 || P.rows > kCgRowsMax || P.cluster * (nt / 32) > kSlotCap || P.cluster > 16)
    return cudaErrorInvalidConfiguration;
  const size_t smem = sizeof(double) * ((size_t)(kCgRowsMax + 2) * (nt + 2) + 4 * kSlotCap +
                                        (size_t)kCgRowsMax * nt) +
                      4 * sizeof(uint64_t);
  auto k = cg_sweep2d_kernel;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if (P.cluster > 8 &&
      (e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) !=
          cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.cluster, 1, 1);
  cfg.blockDim = dim3(nt, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P.cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, P, A, iters);
}

}  // namespace pitb
