// pit_k2.cu — K2 launchers (the coarse sweeps) for every compiled layout; see
// pit_kernels_impl.cuh.
#include "pit_kernels_impl.cuh"

namespace pitb {

cudaError_t launch_sweep(int mpt, int nsub, int nseg, int warps, bool src, const StepParams& P,
                         const SweepArgs& A, cudaStream_t st) {
  if (A.count <= 0) return cudaSuccess;
  // the coarse auto layouts with the full 5-stage scans (slowly decaying
  // coarse factors) compiled without the run-time stage checks
  if (!src && P.scan_f == 5 && P.scan_b == 5) {
#define X(MP, NU, NS, W)                                   \
  if (mpt == MP && nsub == NU && nseg == NS && warps == W) \
    return sweep_launch<Shape<(MP) / ((NU) * (NS)), NU, NS, W, 5>, false>(P, A, st);
    X(8, 1, 1, 8) X(16, 1, 1, 8) X(16, 1, 1, 16) X(16, 2, 1, 8) X(16, 4, 1, 8) X(32, 4, 1, 8)
    X(32, 2, 1, 8) X(16, 2, 1, 16) X(32, 4, 1, 4)
#undef X
  }
#define X(MP, NU, NS, W)                                                        \
  if (mpt == MP && nsub == NU && nseg == NS && warps == W)                      \
    return src ? sweep_launch<PIT_SHAPE(MP, NU, NS, W), true>(P, A, st)         \
               : sweep_launch<PIT_SHAPE(MP, NU, NS, W), false>(P, A, st);
  PIT_LAYOUTS(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

}  // namespace pitb
