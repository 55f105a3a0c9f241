// pit_kernels_impl.cuh — device code of K1 (slab_kernel) and K2 (the coarse
// sweeps) and their template launchers, shared by the translation units that
// instantiate them (pit_k1.cu: the fine layouts, pit_k2.cu: the sweeps), so
// the layout instantiations compile in parallel.  Internal.
#pragma once
//
//  K1 slab_kernel   apply_F / preconditioned-residual / propagate over a batch
//                   of slabs, one CTA per slab, state resident in registers
//                   across all fine steps; HBM traffic only at slab boundaries.
//                   Replaces block_system.cpp:115-147 (+ the executor fan-out,
//                   executor.cpp:105-154) and solvers.cpp:66-71's subtraction.
//  K2 sweep_kernel  the sequential coarse sweep (apply_G_inverse,
//                   block_system.cpp:174-195; initial_guess, solvers.cpp:49-64;
//                   sequential_fine_solve, solvers.cpp:40-47) as one persistent
//                   CTA that keeps W_{n-1} in registers from slab to slab.
//  K3 vector kernels the BiCGStab block algebra (block_system.cpp:31-87,
//                   solvers.cpp:159-215) fused into four passes with
//                   fixed-order per-block reductions.
#include <cstdint>

#include "pit_kernels.cuh"
#include "pit_sync.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

namespace pitb {

namespace {

template <class S>
__device__ __forceinline__ void load_field(double (&y)[S::NC][S::SUB],
                                           const double* __restrict__ src, int tid, int M) {
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) {
      const int i = S::point(tid, c, j);
      y[c][j] = (src != nullptr && i < M) ? src[i] : 0.0;
    }
}

template <class S>
__device__ __forceinline__ bool all_finite(const double (&y)[S::NC][S::SUB], int tid, int M) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j)
      if (S::point(tid, c, j) < M && !isfinite(y[c][j])) ok = false;
  return ok;
}

// Table-form correction vector in shared memory (wide path only): slot layout,
// zero beyond K0.
template <class S>
__host__ __device__ inline int zc_smem_len(int narrow) {
  return narrow ? 0 : S::T * (S::MPT + 1);
}
template <class S>
__device__ __forceinline__ void load_zc(const StepParams& P, double* s_zc, int tid) {
  if (P.narrow) return;
  const int n = S::NSEG * S::LSEG;
  for (int i = tid; i < n; i += S::T) s_zc[S::slot_of_point(i)] = i < P.K0 ? P.zc[i] : 0.0;
}

template <int MPT, int WARPS, bool SRC>
struct SlabBounds {
  static constexpr int kThreads = 32 * WARPS;
  static constexpr int kRegs = MPT <= 8 ? 96 : (MPT <= 16 ? 64 : (MPT <= 32 ? 128 : 168));
  static constexpr int kMin0 = 65536 / (kThreads * kRegs);
  static constexpr int kMin = SRC ? 1 : (kMin0 < 1 ? 1 : (kMin0 > 16 ? 16 : kMin0));
};

template <class S>
__device__ __forceinline__ StepLane step_lane(const StepParams& P,
                                              const StepShared<S::NSEG, S::WARPS>& sh, int tid) {
  StepLane L;
  L.ppos = S::NSEG > 1 ? P.ppos[tid] : 0.0;
  L.qpos = S::NSEG > 1 ? P.qpos[tid] : 0.0;
  L.zt = (P.narrow && tid < 32 && tid * S::CH < P.K0) ? P.zt[tid] : 0.0;
  const int lane = tid & 31;
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    L.cf[st] = sh.cf[st][lane];
    L.cb[st] = sh.cb[st][lane];
  }
  L.plane = sh.plane[lane];
  L.qlane = sh.qlane[lane];
  return L;
}

// Steps [k0, k1) of one slab's propagation.  The rescale counter restarts
// from k0 mod R, so cutting a slab into step ranges (piece scheduling) runs
// exactly the same operation sequence as one uninterrupted pass.
template <class S, bool SRC, bool HOIST = false, bool ZREG = false>
__device__ __forceinline__ void run_slab(double (&y)[S::NC][S::SUB], const StepParams& P,
                                         const StepLane& L, StepShared<S::NSEG, S::WARPS>& sh,
                                         const double* s_zc, int tid, int slab, int k0, int k1,
                                         const double (*zreg)[S::SUB] = nullptr) {
  const bool ghosts = P.M < S::NSEG * S::LSEG;
#ifdef PIT_PHASE_TIMING
  long long ph_acc[16] = {};
  long long ph_t = clock64();
#define PIT_TIMING_ARGS , ph_acc, ph_t
#else
#define PIT_TIMING_ARGS
#endif
  if (SRC) {
    // separable source y += dt*s(t_k) g(x): g read through L1 each step (not
    // held in registers, so wide layouts do not spill); or a general source
    // table y += fl(dt*f(t_k, x_i)) (PIT_SOURCE_TABLE)
    const double* ds = P.tab ? nullptr : P.ds + (size_t)slab * P.steps;
    const double* tk = P.tab ? P.tab + ((size_t)slab * P.steps + k0) * P.M : nullptr;
    double dsk = ds ? ds[k0] : 0.0;
    for (int k = k0; k < k1; ++k) {
      const double dsn = (ds && k + 1 < k1) ? ds[k + 1] : 0.0;
      if (tk) {
#pragma unroll
        for (int c = 0; c < S::NC; ++c)
#pragma unroll
          for (int j = 0; j < S::SUB; ++j) {
            const int i = S::point(tid, c, j);
            y[c][j] = y[c][j] + (i < P.M ? __ldg(tk + i) : 0.0);
          }
        tk += P.M;
      } else {
#pragma unroll
        for (int c = 0; c < S::NC; ++c)
#pragma unroll
          for (int j = 0; j < S::SUB; ++j) {
            const int i = S::point(tid, c, j);
            y[c][j] = fma(dsk, i < P.M ? __ldg(P.shape + i) : 0.0, y[c][j]);
          }
      }
      be_solve<S, HOIST, ZREG>(y, P, L, sh, s_zc, tid, ghosts, zreg PIT_TIMING_ARGS);
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int j = 0; j < S::SUB; ++j) y[c][j] = y[c][j] * P.inv;
      dsk = dsn;
    }
  } else {
    int cnt = k0 == 0 ? 0 : k0 % P.R;
    for (int k = k0; k < k1; ++k) {
      be_solve<S, HOIST, ZREG>(y, P, L, sh, s_zc, tid, ghosts, zreg PIT_TIMING_ARGS);
      if (++cnt == P.R) {
        cnt = 0;
#pragma unroll
        for (int c = 0; c < S::NC; ++c)
#pragma unroll
          for (int j = 0; j < S::SUB; ++j) y[c][j] = y[c][j] * P.invR;
      }
      PIT_PHASE(9);
    }
    if (k1 == P.steps && cnt) {
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int j = 0; j < S::SUB; ++j) y[c][j] = y[c][j] * P.invLast;
    }
  }
#ifdef PIT_PHASE_TIMING
  if (P.timing && blockIdx.x == 0 && (tid & 31) == 0 && (tid >> 5) < 2)
    for (int k = 0; k < 10; ++k) P.timing[(tid >> 5) * 16 + k] += ph_acc[k];
#endif
}

// Layouts of few points per thread (the small grids: c1; M <= 1024)
// have registers to spare and are bound by the step's latency: they run the
// HOIST form of the step (scan and carry weights in registers) and keep the
// table-form correction vector in registers too — the same values from
// registers instead of shared memory, so the same bits.
template <class S>
struct SmallLayout {
  static constexpr bool hoist = S::MPT <= 8;
  static constexpr bool zreg = hoist && S::WARPS <= 8;
};
template <class S>
__device__ __forceinline__ void load_zreg(double (&zreg)[SmallLayout<S>::zreg ? S::NC : 1][S::SUB],
                                          const StepParams& P, const double* s_zc, int tid) {
#pragma unroll
  for (int c = 0; c < (SmallLayout<S>::zreg ? S::NC : 1); ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j)
      zreg[c][j] = P.narrow || !SmallLayout<S>::zreg ? 0.0 : s_zc[S::slot(tid, c, j)];
}
template <class S, bool SRC>
__device__ __forceinline__ void run_slab_auto(
    double (&y)[S::NC][S::SUB], const StepParams& P, const StepLane& L,
    StepShared<S::NSEG, S::WARPS>& sh, const double* s_zc, int tid, int slab, int k0, int k1,
    const double (&zreg)[SmallLayout<S>::zreg ? S::NC : 1][S::SUB]) {
  if constexpr (SmallLayout<S>::hoist) {
    if (SmallLayout<S>::zreg && !P.narrow)
      run_slab<S, SRC, true, true>(y, P, L, sh, s_zc, tid, slab, k0, k1, zreg);
    else
      run_slab<S, SRC, true, false>(y, P, L, sh, s_zc, tid, slab, k0, k1, zreg);
  } else {
    run_slab<S, SRC>(y, P, L, sh, s_zc, tid, slab, k0, k1);
  }
}

// Piece state in register order (element (c, j) of thread tid at
// ((c*SUB + j)*T + tid)): one coalesced 256-byte access per warp and element.
template <class S>
__device__ __forceinline__ void load_state(double (&y)[S::NC][S::SUB], const double* st, int tid) {
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) y[c][j] = __ldcg(st + (c * S::SUB + j) * S::T + tid);
}
template <class S>
__device__ __forceinline__ void save_state(const double (&y)[S::NC][S::SUB], double* st, int tid) {
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) __stcg(st + (c * S::SUB + j) * S::T + tid, y[c][j]);
}

template <class S>
__device__ __forceinline__ void slab_epilogue(const double (&y)[S::NC][S::SUB], const SlabArgs& A,
                                              int M, int tid, int b, int slab) {
  if (!all_finite<S>(y, tid, M)) atomicMin(A.status, slab);
  const size_t off = (size_t)b * M;
  double* out = A.out + off;
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) {
      const int i = S::point(tid, c, j);
      if (i < M) {
        if (A.mode == kApplyF) {
          out[i] = A.Lsub[off + i] - y[c][j];
        } else if (A.mode == kResidual) {
          const double a = A.Lsub[off + i] - y[c][j];
          out[i] = A.rhs[off + i] - a;
        } else {
          out[i] = y[c][j];
        }
      }
    }
  if (b == 0 && A.out0 != nullptr) {
    if (A.mode == kApplyF) {
      for (int i = tid; i < M; i += S::T) A.out0[i] = A.L0[i];
    } else if (A.mode == kResidual) {
      for (int i = tid; i < M; i += S::T) A.out0[i] = A.rhs0[i] - A.L0[i];
    }
  }
  if (A.host_out != nullptr) {
    __syncthreads();  // the block's stores above are visible to the whole CTA
    double* h = A.host_out + (size_t)(b + A.block_shift) * M;
    if ((M & 1) == 0) {
      for (int i = 2 * tid; i < M; i += 2 * S::T)
        __stcs(reinterpret_cast<double2*>(h + i), __ldcg(reinterpret_cast<const double2*>(out + i)));
    } else {
      for (int i = tid; i < M; i += S::T) __stcs(h + i, __ldcg(out + i));
    }
    if (b == 0 && A.out0 != nullptr)
      for (int i = tid; i < M; i += S::T) __stcs(A.host_out + i, __ldcg(A.out0 + i));
  }
}

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int sm_id() {
  int v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Overlapped sweep: spin until a producer CTA published ready[g] = epoch;
// never hang the device on a lost producer: after 20 s report the slab as
// failed and go on.
__device__ __noinline__ void wait_ready(const int* flag, int epoch, int* status, int slab) {
  long long t0 = -1;
  while (ld_acquire(flag) != epoch) {
    long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (t0 < 0) t0 = now;
    if (now - t0 > 20000000000LL) {
      atomicMin(status, slab);
      return;
    }
    __nanosleep(128);
  }
}

// Host-buffer pipelining (SlabArgs::in_ready / out_done): wait until the
// chunk holding output block g (and so input blocks g-1, g) has landed.
__device__ __noinline__ void wait_input(const SlabArgs& A, int b, int tid) {
  if (A.in_ready == nullptr) return;
  if (tid == 0) {
    const unsigned need = (unsigned)((b + A.block_shift) / A.chunk_blocks) + 1u;
    long long t0 = -1;
    while (ld_acquire_sys(A.in_ready) < need) {
      // never hang the device on a lost copy: give up after 20 s and report
      // the slab as failed
      long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 < 0) t0 = now;
      if (now - t0 > 20000000000LL) {
        atomicMin(A.status, A.slab0 + b);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}
// ... and publish block g (plus block 0 for CTA 0) once every thread's
// output stores are globally visible.
__device__ __forceinline__ void publish_ready(const SlabArgs& A, int b, int tid) {
  if (A.ready == nullptr) return;
  __syncthreads();  // every thread's output stores precede thread 0's release
  if (tid == 0) {
    __threadfence();
    st_release(A.ready + b + A.block_shift, A.epoch);
    if (b == 0 && A.out0 != nullptr) st_release(A.ready, A.epoch);
  }
}

__device__ __noinline__ void signal_output(const SlabArgs& A, int b, int tid) {
  publish_ready(A, b, tid);
  if (A.out_done == nullptr) return;
  __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    atomicAdd(A.out_done + (b + A.block_shift) / A.chunk_blocks, 1u);
    if (b == 0 && A.out0 != nullptr) atomicAdd(A.out_done, 1u);
  }
}

// K1.  One CTA per slab (A.state == nullptr), or a persistent grid pulling
// (piece, slab) units piece-major (see SlabArgs) so that a batch of
// 1.15 waves does not leave the last wave's SMs one-sixth occupied.
template <class S, bool SRC>
__global__ void __launch_bounds__(S::T, (SlabBounds<S::MPT, S::WARPS, SRC>::kMin))
    slab_kernel(const __grid_constant__ StepParams P, const __grid_constant__ SlabArgs A) {
  if (A.skip != nullptr && *A.skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // static, so every access is a direct shared-window address (a pointer
  // into the dynamic window is converted through SR_CgaCtaId each time)
  __shared__ StepShared<S::NSEG, S::WARPS> sh_s;
  auto* sh = &sh_s;
  double* s_zc = reinterpret_cast<double*>(smem_raw);
  __shared__ int s_unit;
  const int tid = threadIdx.x;
  const int M = P.M;
  load_zc<S>(P, s_zc, tid);
  init_step_shared<S::NSEG, S::WARPS>(P, *sh, tid);
  auto source_of = [&](int b) -> const double* {
    if (b + A.in_shift >= 0) return A.in ? A.in + (size_t)(b + A.in_shift) * M : nullptr;
    return A.halo;
  };
  double y[S::NC][S::SUB];

  if (A.state == nullptr) {
    const int b = blockIdx.x;
    wait_input(A, b, tid);
    const long long tb0 = global_ns();
    load_field<S>(y, source_of(b), tid, M);
    const int slab = A.slab0 + b;
    __syncthreads();
    const StepLane L = step_lane<S>(P, *sh, tid);
    double zreg[SmallLayout<S>::zreg ? S::NC : 1][S::SUB];
    load_zreg<S>(zreg, P, s_zc, tid);
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
    const long long tr0 = global_ns();
#endif
    run_slab_auto<S, SRC>(y, P, L, *sh, s_zc, tid, slab, 0, P.steps, zreg);
    slab_epilogue<S>(y, A, M, tid, b, slab);
    signal_output(A, b, tid);
    if (A.busy_ns != nullptr && tid == 0)
      atomicAdd(A.busy_ns, (unsigned long long)(global_ns() - tb0));
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
    if (A.trace && tid == 0) {
      long long* t = A.trace + 8 * (size_t)b;
      t[0] = sm_id(), t[1] = b, t[2] = tr0, t[3] = global_ns(), t[4] = tr0, t[5] = t[3];
    }
#endif
    return;
  }

  __syncthreads();
  const StepLane L = step_lane<S>(P, *sh, tid);
  double zreg[SmallLayout<S>::zreg ? S::NC : 1][S::SUB];
  load_zreg<S>(zreg, P, s_zc, tid);
  const int units = A.pieces * A.nblk;
  int* head = A.sched;       // next queue position to pop
  int* tail = A.sched + 1;   // next push position
  int* queue = A.sched + 2;  // unit+1 of pushed units (0 = not yet written)
  for (;;) {
    if (tid == 0) {
      // positions < nblk are the first pieces (unit id = position); later
      // positions are filled in completion order by the CTA finishing the
      // previous piece of the same slab
      const int i = atomicAdd(head, 1);
      int u = units;
      if (i < A.nblk) {
        u = i;
      } else if (i < units) {
        int v;
        while ((v = ld_acquire(queue + (i - A.nblk))) == 0) __nanosleep(64);
        u = v - 1;
      }
      s_unit = u;
    }
    __syncthreads();
    const int u = s_unit;
    __syncthreads();  // s_unit is rewritten at the top of the next unit
    if (u >= units) break;
    const int q = u / A.nblk, b = u - q * A.nblk;
    const int slab = A.slab0 + b;
    const int k0 = (int)((long long)P.steps * q / A.pieces);
    const int k1 = (int)((long long)P.steps * (q + 1) / A.pieces);
    double* st = A.state + (size_t)b * (S::NC * S::SUB * S::T);
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
    const long long tr0 = global_ns();
#endif
    if (q == 0) wait_input(A, b, tid);
    const long long tb0 = global_ns();
    if (q == 0) {
      load_field<S>(y, source_of(b), tid, M);
    } else {
      load_state<S>(y, st, tid);
    }
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
    __syncthreads();
    const long long tr1 = global_ns();
#endif
    run_slab_auto<S, SRC>(y, P, L, *sh, s_zc, tid, slab, k0, k1, zreg);
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
    __syncthreads();
    const long long tr2 = global_ns();
#endif
    if (q + 1 < A.pieces) {
      save_state<S>(y, st, tid);
      // bar.sync orders every thread's state stores before thread 0's
      // release (cumulativity); the popping CTA acquires before its bar.sync
      __syncthreads();
      if (tid == 0) st_release(queue + atomicAdd(tail, 1), u + A.nblk + 1);
    } else {
      slab_epilogue<S>(y, A, M, tid, b, slab);
      signal_output(A, b, tid);
    }
    if (A.busy_ns != nullptr && tid == 0)
      atomicAdd(A.busy_ns, (unsigned long long)(global_ns() - tb0));
#if defined(PIT_PHASE_TIMING) || defined(PIT_TRACE)
    if (A.trace && tid == 0) {
      long long* t = A.trace + 8 * (size_t)u;
      t[0] = sm_id(), t[1] = blockIdx.x, t[2] = tr0, t[3] = global_ns(), t[4] = tr1, t[5] = tr2;
    }
#endif
  }
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// K2: one persistent CTA running the sequential chain
//   W_b = Prop(W_{b-1}) (+ V_b).
// TMA (NSEG == 1, M a multiple of 16, even chunks, 16-byte aligned blocks):
// thread 0 streams V_{b+1} into buffer (b+1)&1 with 2D tensor loads (128-byte
// swizzle; completion on an mbarrier) while slab b propagates; after the
// step every thread adds V_b from and writes W_b into its own rows of buffer
// b&1 (conflict-free LDS/STS.128 thanks to the swizzle), and thread 0 issues
// the tensor store of W_b.  A buffer is reloaded only after thread 0's store
// from it has been read out (bulk wait_group.read).
// Otherwise: cp.async V into an odd-pitch slot layout and coalesced W stores.
template <class S>
__device__ __forceinline__ int swz_off(int p) {  // byte offset of point p in a swizzled slab
  const int r = p >> 4, q = p & 15;
  return r * 128 + ((((q >> 1) ^ (r & 7)) << 4) | ((q & 1) << 3));
}

template <class S, bool SRC, bool TMA>
__global__ void __launch_bounds__(S::T, 1)
    sweep_kernel(const __grid_constant__ StepParams P, const __grid_constant__ SweepArgs A,
                 const __grid_constant__ SweepTma X) {
  if (A.skip != nullptr && *A.skip) return;
  constexpr int STAGE_SLOT = S::T * (S::MPT + 1);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ StepShared<S::NSEG, S::WARPS> sh_s;
  auto* sh = &sh_s;
  double* s_zc = reinterpret_cast<double*>(smem_raw);
  unsigned char* after = reinterpret_cast<unsigned char*>(s_zc + zc_smem_len<S>(P.narrow));
  // TMA: two 1024-byte aligned slab buffers of M doubles; slot path: two
  // odd-pitch buffers
  unsigned char* base = TMA ? reinterpret_cast<unsigned char*>(
                                  (reinterpret_cast<uintptr_t>(after) + 1023) & ~uintptr_t(1023))
                            : after;
  const size_t buf_bytes = TMA ? (size_t)P.M * sizeof(double) : (size_t)STAGE_SLOT * sizeof(double);
  const int nbuf = TMA ? X.nbuf : 2;
  uint64_t* vbar = reinterpret_cast<uint64_t*>(base + nbuf * buf_bytes);  // [nbuf]
  const int tid = threadIdx.x;
  const int M = P.M;
  load_zc<S>(P, s_zc, tid);
  init_step_shared<S::NSEG, S::WARPS>(P, *sh, tid);
  double y[S::NC][S::SUB];
  load_field<S>(y, A.start, tid, M);
  if (TMA && tid == 0) {
    for (int i = 0; i < nbuf; ++i) mbar_init(&vbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // slab b uses buffer b % nbuf; V_b is requested D = max(1, nbuf-2) slabs
  // ahead, into a buffer whose last W store was issued >= 1 slab earlier
  // (nbuf >= 3)
  const int D = nbuf > 3 ? nbuf - 2 : 1;
  auto bidx = [&](int b) { return TMA ? b % nbuf : (b & 1); };
  // thread 0: wait until at most `pending` of its bulk store groups are
  // still reading shared memory
  auto wait_reads = [](int pending) {
    switch (pending) {
      case 0: asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); break;
      case 1: asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); break;
      case 2: asm volatile("cp.async.bulk.wait_group.read 2;\n" ::: "memory"); break;
      default: asm volatile("cp.async.bulk.wait_group.read 3;\n" ::: "memory"); break;
    }
  };
  auto bufp = [&](int b) { return base + bidx(b) * buf_bytes; };
  auto prefetch = [&](int b) {
    if (TMA) {
      if (tid == 0) {
        // the store of W_{b-nbuf}, the previous user of this buffer, has
        // read it out; W_{b-nbuf+1} .. W_{b-D-1} may still be pending
        wait_reads(nbuf - D - 1);
        mbar_arrive_expect_tx(&vbar[bidx(b)], (unsigned)(M * sizeof(double)));
        for (int r = 0; r < X.rows; r += X.box_rows)
          tma_load_2d(bufp(b) + r * 128, X.v, 0, b * X.rows + r, &vbar[bidx(b)]);
      }
    } else {
      double* buf = reinterpret_cast<double*>(bufp(b));
      const double* v = A.V + (size_t)b * M;
      for (int i = tid; i < M; i += S::T) cp_async8(buf + S::slot_of_point(i), v + i);
      cp_async_commit();
    }
  };
  __syncthreads();
  if (A.V)
    for (int b = 0; b < (TMA ? D : 1) && b < A.count; ++b) prefetch(b);
  const StepLane L = step_lane<S>(P, *sh, tid);
  double zreg[SmallLayout<S>::zreg ? S::NC : 1][S::SUB];
  load_zreg<S>(zreg, P, s_zc, tid);
  bool ok = true;
  int bad = 0x7fffffff;
  for (int b = 0; b < A.count; ++b) {
    const int slab = A.slab0 + b;
    if (A.V) {
      const int ahead = TMA ? D : 1;
      if (b + ahead < A.count) prefetch(b + ahead);
    }
#ifdef PIT_PHASE_TIMING
    const long long sw0 = clock64();
#endif
    run_slab_auto<S, SRC>(y, P, L, *sh, s_zc, tid, slab, 0, P.steps, zreg);
#ifdef PIT_PHASE_TIMING
    const long long sw1 = clock64();
#endif
    if (ok && !all_finite<S>(y, tid, M)) {
      ok = false;
      bad = slab;
    }
    if (TMA) {
      unsigned char* buf = bufp(b);
      if (A.V) {
        mbar_wait(&vbar[bidx(b)], (unsigned)((b / nbuf) & 1));  // V_b landed
#pragma unroll
        for (int c = 0; c < S::NC; ++c)
#pragma unroll
          for (int j = 0; j < S::SUB; j += 2) {
            const int pnt = S::point(tid, c, j);
            if (pnt < M) {
              const double2 v = *reinterpret_cast<const double2*>(buf + swz_off<S>(pnt));
              y[c][j] = y[c][j] + v.x;
              y[c][j + 1] = y[c][j + 1] + v.y;
            }
          }
      } else if (b >= nbuf) {
        if (tid == 0) wait_reads(nbuf - 1);  // W_{b-nbuf} has left this buffer
        __syncthreads();
      }
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int j = 0; j < S::SUB; j += 2) {
          const int pnt = S::point(tid, c, j);
          if (pnt < M)
            *reinterpret_cast<double2*>(buf + swz_off<S>(pnt)) = make_double2(y[c][j], y[c][j + 1]);
        }
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        for (int r = 0; r < X.rows; r += X.box_rows)
          tma_store_2d(X.w, 0, b * X.rows + r, buf + r * 128);
        bulk_commit();
      }
    } else {
      double* buf = reinterpret_cast<double*>(bufp(b));
      if (A.V) {
        if (b + 1 < A.count)
          cp_async_wait<1>();
        else
          cp_async_wait<0>();
        __syncthreads();
#pragma unroll
        for (int c = 0; c < S::NC; ++c)
#pragma unroll
          for (int j = 0; j < S::SUB; ++j) {
            const double v = S::point(tid, c, j) < M ? buf[S::slot(tid, c, j)] : 0.0;
            y[c][j] = y[c][j] + v;
          }
      }
      // drain W_b through slab b's (consumed) V buffer; each thread
      // overwrites exactly the slots it just read
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int j = 0; j < S::SUB; ++j) buf[S::slot(tid, c, j)] = y[c][j];
      __syncthreads();
      double* W = A.W + (size_t)b * M;
      for (int i = tid; i < M; i += S::T) W[i] = buf[S::slot_of_point(i)];
      __syncthreads();  // the buffer is free for the prefetch of slab b+2
    }
#ifdef PIT_PHASE_TIMING
    if (P.timing && (tid & 31) == 0 && (tid >> 5) < 2) {
      P.timing[(tid >> 5) * 16 + 10] += sw1 - sw0;        // propagation
      P.timing[(tid >> 5) * 16 + 11] += clock64() - sw1;  // V add + W store
    }
#endif
  }
  if (TMA && tid == 0) bulk_wait_all();
  if (!ok) {
    atomicMin(A.status, bad);
    if (A.fail_info != nullptr) {  // direct solve: no Krylov iterations
      A.fail_info[0] = __longlong_as_double(0x7ff8000000000000LL);
      A.fail_info[1] = 0.0;
      A.fail_info[2] = kFailNonFinite;
    }
  }
}

// K2 with a dedicated I/O warp (TMA layouts: NSEG == 1, M a multiple of 16,
// 16-byte aligned blocks).  The T compute threads never meet a CTA-wide
// barrier in the slab loop: their only synchronisation is the step's named
// barrier (step_sync) and two mbarriers per slab buffer, so no compute warp
// waits for the TMA issue or for another warp's I/O.
//   vfull[i]  the I/O thread's arrival (with the V_b bytes when V is added):
//             buffer i holds V_b and its previous W store has drained;
//   wfull[i]  T arrivals: every compute thread has written its rows of W_b
//             (fence.proxy.async first), so the I/O thread may store it.
// The I/O thread (warp WARPS, lane 0): loads V_0 .. V_{nbuf-1}; then per
// slab s: wait wfull, TMA-store W_s, wait for the store to have read the
// buffer, load V_{s+nbuf} into it.  Same arithmetic as sweep_kernel, so the
// same bits.
template <class S, bool SRC>
__global__ void __launch_bounds__(S::T + 32, 1)
    sweep_io_kernel(const __grid_constant__ StepParams P, const __grid_constant__ SweepArgs A,
                    const __grid_constant__ SweepTma X) {
  if (A.skip != nullptr && *A.skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ StepShared<S::NSEG, S::WARPS> sh_s;
  auto* sh = &sh_s;
  double* s_zc = reinterpret_cast<double*>(smem_raw);
  // slab buffers 1024-byte aligned (128-byte swizzle atoms); offsets taken in
  // the shared window so the compiler keeps LDS/STS (not generic LD/ST)
  const unsigned s0 = smem_u32(smem_raw);
  const unsigned after = smem_u32(s_zc + zc_smem_len<S>(P.narrow));
  unsigned char* const base = smem_raw + (((after + 1023u) & ~1023u) - s0);
  const size_t buf_bytes = (size_t)P.M * sizeof(double);
  const int nbuf = X.nbuf;
  uint64_t* vfull = reinterpret_cast<uint64_t*>(base + nbuf * buf_bytes);  // [nbuf]
  uint64_t* wfull = vfull + nbuf;                                           // [nbuf]
  const int tid = threadIdx.x;
  const int M = P.M;
  const bool io = tid >= S::T;
  if (!io) {
    load_zc<S>(P, s_zc, tid);
    init_step_shared<S::NSEG, S::WARPS>(P, *sh, tid);
  } else if (tid == S::T) {
    for (int i = 0; i < nbuf; ++i) {
      mbar_init(&vfull[i], 1);
      mbar_init(&wfull[i], S::T);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // overlapped with the producing fine batch: the start block must be out
  if (tid == 0 && A.ready != nullptr)
    wait_ready(A.ready + A.ready_shift - 1, A.epoch, A.status, A.slab0);
  __syncthreads();  // the only CTA-wide barrier

  if (io) {
    // I/O warp: lane 0 issues the TMA traffic
    const int lane = tid - S::T;
    const unsigned bytes = (unsigned)(M * sizeof(double));
    int fill_slot = 0;
    auto fill = [&](int b) {  // buffer fill_slot is free: V_b in (or just released)
      uint64_t* bar = &vfull[fill_slot];
      unsigned char* buf = base + fill_slot * buf_bytes;
      if (A.V && A.ready != nullptr) {
        wait_ready(A.ready + b + A.ready_shift, A.epoch, A.status, A.slab0 + b);
        // the producer's generic-proxy stores, acquired above, before the
        // async-proxy (TMA) read of the same block
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
      }
      if (A.V) {
        mbar_arrive_expect_tx(bar, bytes);
        for (int r = 0; r < X.rows; r += X.box_rows)
          tma_load_2d(buf + r * 128, X.v, 0, b * X.rows + r, bar);
      } else {
        mbar_arrive(bar);
      }
      if (++fill_slot == nbuf) fill_slot = 0;
    };
    if (lane == 0)
      for (int b = 0; b < nbuf && b < A.count; ++b) fill(b);
    int slot = 0;
    unsigned phase = 0;
    for (int s = 0; s < A.count; ++s) {
      mbar_wait(&wfull[slot], phase);
      const unsigned char* buf = base + slot * buf_bytes;
      if (lane == 0) {
        for (int r = 0; r < X.rows; r += X.box_rows)
          tma_store_2d(X.w, 0, s * X.rows + r, buf + r * 128);
        bulk_commit();
      }
      __syncwarp();
      if (lane == 0 && s + nbuf < A.count) {
        bulk_wait_read();  // the store has read the buffer out
        fill(s + nbuf);
      }
      if (++slot == nbuf) {
        slot = 0;
        phase ^= 1u;
      }
    }
    if (lane == 0) bulk_wait_all();
    return;
  }

  double y[S::NC][S::SUB];
  load_field<S>(y, A.start, tid, M);
  if (A.W0 != nullptr) {  // W_0 = V_0
#pragma unroll
    for (int c = 0; c < S::NC; ++c)
#pragma unroll
      for (int j = 0; j < S::SUB; ++j)
        if (S::point(tid, c, j) < M) A.W0[S::point(tid, c, j)] = y[c][j];
  }
  const StepLane L = step_lane<S>(P, *sh, tid);
  // the table-form correction vector of the thread's points in registers
  // (coarse layouts of few points per thread; others read it from smem)
  constexpr bool kZreg = S::MPT <= 16 && S::WARPS <= 8;
  double zreg[kZreg ? S::NC : 1][S::SUB];
#pragma unroll
  for (int c = 0; c < (kZreg ? S::NC : 1); ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; ++j) zreg[c][j] = P.narrow || !kZreg ? 0.0 : s_zc[S::slot(tid, c, j)];
  int slot = 0;
  unsigned phase = 0;
  const uint32_t base_s = smem_u32(base), vfull_s = smem_u32(vfull), wfull_s = smem_u32(wfull);
  // the thread's swizzled row offsets in a slab buffer (loop invariant)
  uint32_t swz[S::NC][S::SUB / 2 > 0 ? S::SUB / 2 : 1];
#pragma unroll
  for (int c = 0; c < S::NC; ++c)
#pragma unroll
    for (int j = 0; j < S::SUB; j += 2) swz[c][j / 2] = (uint32_t)swz_off<S>(S::point(tid, c, j));
  // non-finite detection off the step chain: pz accumulates fma(w, 0, pz)
  // over every W value (0 while all are finite, NaN for good after an inf
  // or nan); it is tested one slab later, when its FMAs have long retired,
  // and the first failing block is reported
  double pz = 0.0;
  int bad = 0x7fffffff;
  for (int b = 0; b < A.count; ++b) {
    const int slab = A.slab0 + b;
#ifdef PIT_PHASE_TIMING
    const long long sw0 = clock64();
#endif
    if (kZreg && !P.narrow)
      run_slab<S, SRC, true, true>(y, P, L, *sh, s_zc, tid, slab, 0, P.steps, zreg);
    else
      run_slab<S, SRC, true, false>(y, P, L, *sh, s_zc, tid, slab, 0, P.steps, zreg);
#ifdef PIT_PHASE_TIMING
    const long long sw1 = clock64();
#endif
    const uint32_t buf = base_s + (uint32_t)(slot * buf_bytes);
    mbar_wait_s(vfull_s + 8u * slot, phase);  // V_b landed / buffer free
#pragma unroll
    for (int c = 0; c < S::NC; ++c)
#pragma unroll
      for (int j = 0; j < S::SUB; j += 2) {
        const int pnt = S::point(tid, c, j);
        if (pnt < M) {
          const uint32_t q = buf + swz[c][j / 2];
          if (A.V) {
            const double2 v = lds_v2(q);
            y[c][j] = y[c][j] + v.x;
            y[c][j + 1] = y[c][j + 1] + v.y;
          }
          sts_v2(q, y[c][j], y[c][j + 1]);
        }
      }
    fence_proxy_async_smem();
    mbar_arrive_s(wfull_s + 8u * slot);
    if (++slot == nbuf) {
      slot = 0;
      phase ^= 1u;
    }
    if (bad == 0x7fffffff && !isfinite(pz)) bad = slab - 1;  // blocks up to b-1
    {
      // w * 0 is 0 for a finite w and nan otherwise; summed as a tree (warps
      // issue in order: a 16-deep fma chain here stalled the next step).
      // Ghost points hold exact zeros.
      constexpr int NV = S::NC * S::SUB;
      double q[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) q[i] = y[i / S::SUB][i % S::SUB] * 0.0;
#pragma unroll
      for (int w = 1; w < NV; w *= 2)
#pragma unroll
        for (int i = 0; i + w < NV; i += 2 * w) q[i] = q[i] + q[i + w];
      pz = pz + q[0];
    }
#ifdef PIT_PHASE_TIMING
    if (P.timing && (tid & 31) == 0 && (tid >> 5) < 2) {
      P.timing[(tid >> 5) * 16 + 10] += sw1 - sw0;        // propagation
      P.timing[(tid >> 5) * 16 + 11] += clock64() - sw1;  // V add + W store
    }
#endif
  }
  if (bad == 0x7fffffff && !isfinite(pz)) bad = A.slab0 + A.count - 1;
  if (bad != 0x7fffffff) {
    atomicMin(A.status, bad);
    if (A.fail_info != nullptr) {  // direct solve: no Krylov iterations
      A.fail_info[0] = __longlong_as_double(0x7ff8000000000000LL);
      A.fail_info[1] = 0.0;
      A.fail_info[2] = kFailNonFinite;
    }
  }
}

// Pieces per slab for a batch of nblk slabs over `slots` resident CTAs.
// Measured on B200 (tools/pieces_grid.py): between one and two waves, two
// pieces let the queue refill the slots of the first CTAs to finish (c2:
// 2.12 -> 1.78 ms); beyond two waves, minimise ceil(waves*q)/q plus a
// per-piece cost (c4: q = 3, 3.73 -> 3.60 ms).
inline int choose_pieces(int nblk, int slots) {
  if (slots <= 0 || nblk <= slots) return 1;
  if (nblk < 2 * slots) return 2;
  int best = 1;
  double best_cost = 1e30;
  for (int q = 1; q <= 8; ++q) {
    const long long rounds = ((long long)nblk * q + slots - 1) / slots;
    const double cost = (double)rounds / q + 0.02 * q;
    if (cost < best_cost - 1e-12) {
      best_cost = cost;
      best = q;
    }
  }
  return best;
}

template <class S, bool SRC>
cudaError_t slab_launch(const StepParams& P, const SlabArgs& A0, int ctas, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)zc_smem_len<S>(P.narrow);
  auto k = slab_kernel<S, SRC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  SlabArgs A = A0;
  A.nblk = ctas;
  int grid = ctas;
  if (A.state != nullptr) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, S::T, smem);
    if (e != cudaSuccess) return e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
      return e;
    const int slots = per_sm * (sms - (A0.reserve_sms < sms ? A0.reserve_sms : 0));
    A.pieces = A0.pieces > 0 ? A0.pieces : choose_pieces(ctas, slots);
    if (A.pieces > kMaxPieces) A.pieces = kMaxPieces;
    if (A.pieces > P.steps) A.pieces = P.steps;
    static const bool verbose = std::getenv("PIT_PIECES_VERBOSE") != nullptr;
    if (verbose)
      std::fprintf(stderr, "[pit] slab_kernel<%d,%d,%d,%d,%d> ctas=%d per_sm=%d slots=%d pieces=%d\n",
                   S::MPT, S::NSUB, S::NSEG, S::WARPS, (int)SRC, ctas, per_sm, slots, A.pieces);
    if (A.pieces <= 1 || slots <= 0) {
      A.state = nullptr;  // one wave-sequence of plain CTAs
    } else {
      const long long units = (long long)A.pieces * ctas;
      grid = (int)(units < slots ? units : slots);
      const size_t nq = 2 + (size_t)(A.pieces - 1) * ctas;
      if ((e = cudaMemsetAsync(A.sched, 0, sizeof(int) * nq, st)) != cudaSuccess) return e;
    }
  }
  k<<<grid, S::T, smem, st>>>(P, A);
  return cudaGetLastError();
}

// Resident slab CTAs of one K1 wave (occupancy x SMs): the device's
// "worker count" for the executor's timing report (executor.cpp:156-171).
template <class S, bool SRC>
cudaError_t slab_slots_t(const StepParams& P, int* slots) {
  const size_t smem = sizeof(double) * (size_t)zc_smem_len<S>(P.narrow);
  auto k = slab_kernel<S, SRC>;
  cudaError_t e;
  if (smem > 48 * 1024 &&
      (e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
          cudaSuccess)
    return e;
  int per_sm = 0, dev = 0, sms = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, S::T, smem)) != cudaSuccess)
    return e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return e;
  *slots = per_sm * sms;
  return cudaSuccess;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency: the library still loads on GPU-less hosts)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// [rows][16] doubles, 128-byte swizzled boxes of box_rows rows
bool encode_rows(void* out, const double* base, long long rows, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {16, (cuuint64_t)rows};
  cuuint64_t strides[1] = {16 * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
             const_cast<double*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// smallest M that streams V/W through TMA (measured, tools/sweep_time.py;
// PIT_SWEEP_TMA_MIN overrides for A/B runs)
inline int tma_min_points() {
  static const int v = [] {
    const char* e = std::getenv("PIT_SWEEP_TMA_MIN");
    return e ? std::atoi(e) : 1024;
  }();
  return v;
}

template <class S, bool SRC>
cudaError_t sweep_launch(const StepParams& P, const SweepArgs& A, cudaStream_t st) {
  SweepTma X{};
  // measured (tools/sweep_time.py): the TMA path wins for M >= 4096 (c2
  // G^-1 2.87 -> 2.28 ms, c4 11.1 -> 8.9 ms) and loses for c3 (M = 2048,
  // two coarse steps per slab amortise the slot-layout I/O)
  bool tma = S::NSEG == 1 && S::MPT % 2 == 0 && S::SUB % 2 == 0 && P.M % 16 == 0 &&
             P.M >= tma_min_points() &&
             (reinterpret_cast<uintptr_t>(A.W) % 16) == 0 &&
             (!A.V || (reinterpret_cast<uintptr_t>(A.V) % 16) == 0) &&
             std::getenv("PIT_NO_TMA") == nullptr;
  if (tma) {
    X.rows = P.M / 16;
    X.box_rows = X.rows;
    while (X.box_rows > 256) X.box_rows /= 2;
    tma = X.rows % X.box_rows == 0 && (X.box_rows % 8) == 0 &&
          encode_rows(X.w, A.W, (long long)A.count * X.rows, X.box_rows) &&
          (!A.V || encode_rows(X.v, A.V, (long long)A.count * X.rows, X.box_rows));
  }
  const size_t buf_bytes =
      tma ? (size_t)P.M * sizeof(double) : (size_t)S::T * (S::MPT + 1) * sizeof(double);
  const size_t fixed = sizeof(double) * (size_t)zc_smem_len<S>(P.narrow) + 1024 +
                       8 * sizeof(uint64_t);
  const size_t budget = 227 * 1024 - sizeof(StepShared<S::NSEG, S::WARPS>);  // static part
  X.nbuf = 2;
  if (tma)
    for (int n = 4; n >= 3; --n)
      if (fixed + n * buf_bytes <= budget) {
        X.nbuf = n;
        break;
      }
  const size_t smem = fixed + (size_t)X.nbuf * buf_bytes;
  static const bool legacy = std::getenv("PIT_SWEEP_LEGACY") != nullptr;  // A/B knob
  if (A.ready != nullptr && (!tma || legacy)) return cudaErrorNotSupported;  // needs the I/O warp
  auto k = tma ? (legacy ? sweep_kernel<S, SRC, true> : sweep_io_kernel<S, SRC>)
               : sweep_kernel<S, SRC, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int threads = tma && !legacy ? S::T + 32 : S::T;
  k<<<1, threads, smem, st>>>(P, A, X);
  return cudaGetLastError();
}

}  // namespace

// Layouts (points per thread, sub-chunks, segments, warps per slab) compiled
// here; SUB = points / (sub-chunks * segments).  Keep in sync with kLayouts
// in coeffs.cpp.
#define PIT_LAYOUTS(X)                                                                       \
  X(4, 1, 1, 1) X(4, 1, 1, 2) X(4, 1, 1, 4) X(4, 1, 1, 8) X(4, 1, 1, 16) X(4, 1, 1, 32)        \
  X(8, 1, 1, 4) X(8, 1, 1, 8) X(8, 1, 1, 16) X(8, 1, 1, 32) X(16, 1, 1, 4) X(16, 1, 1, 8)    \
  X(16, 1, 1, 16) X(16, 1, 1, 32) X(32, 2, 1, 4) X(32, 2, 1, 8) X(32, 1, 2, 4) X(32, 2, 2, 4) \
  X(64, 2, 2, 1) X(64, 2, 2, 2) X(64, 2, 2, 4) X(64, 4, 1, 2) X(64, 1, 4, 2) X(64, 4, 1, 1)  \
  X(64, 4, 1, 4) X(64, 1, 2, 2) X(32, 2, 2, 8) X(64, 2, 2, 8) X(16, 2, 1, 16) X(16, 2, 2, 8)   \
  X(64, 4, 1, 8) X(16, 2, 1, 8) X(16, 4, 1, 8) X(32, 4, 1, 8) X(32, 2, 1, 8) X(32, 4, 1, 4)

#define PIT_SHAPE(MP, NU, NS, W) Shape<(MP) / ((NU) * (NS)), NU, NS, W>

// Fine layouts specialised on the scan stage count (PIT_SCAN_SPECIAL(X):
// layout, stages).  Measured: a run-time stage count costs c4 8% against
// the compile-time loop.
#define PIT_SCAN_SPECIAL(X)                                                                  \
  X(64, 4, 1, 1, 0) X(64, 4, 1, 1, 1) X(64, 4, 1, 1, 2) X(64, 4, 1, 1, 3)                   \
  X(64, 4, 1, 2, 0) X(64, 4, 1, 2, 1) X(64, 4, 1, 2, 2) X(64, 4, 1, 2, 3)                   \
  X(64, 4, 1, 4, 0) X(64, 4, 1, 4, 1) X(64, 4, 1, 4, 2) X(64, 4, 1, 4, 3)

}  // namespace pitb
