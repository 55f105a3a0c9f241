// pit_k1.cu — K1 launchers: every compiled fine layout (PIT_LAYOUTS) and the
// scan-stage specialisations; see pit_kernels_impl.cuh.
#include "pit_kernels_impl.cuh"

namespace pitb {

cudaError_t launch_slab(int mpt, int nsub, int nseg, int warps, bool src, const StepParams& P,
                        const SlabArgs& A, int ctas, cudaStream_t st) {
  if (ctas <= 0) return cudaSuccess;
  if (!src && P.scan_f == P.scan_b) {
#define X(MP, NU, NS, W, K)                                                                  \
  if (mpt == MP && nsub == NU && nseg == NS && warps == W && P.scan_f == K)                  \
    return slab_launch<Shape<(MP) / ((NU) * (NS)), NU, NS, W, K>, false>(P, A, ctas, st);
    PIT_SCAN_SPECIAL(X)
#undef X
  }
#define X(MP, NU, NS, W)                                                        \
  if (mpt == MP && nsub == NU && nseg == NS && warps == W)                      \
    return src ? slab_launch<PIT_SHAPE(MP, NU, NS, W), true>(P, A, ctas, st)    \
               : slab_launch<PIT_SHAPE(MP, NU, NS, W), false>(P, A, ctas, st);
  PIT_LAYOUTS(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

cudaError_t slab_slots(int mpt, int nsub, int nseg, int warps, bool src, const StepParams& P,
                       int* slots) {
#define X(MP, NU, NS, W)                                                   \
  if (mpt == MP && nsub == NU && nseg == NS && warps == W)                 \
    return src ? slab_slots_t<PIT_SHAPE(MP, NU, NS, W), true>(P, slots)    \
               : slab_slots_t<PIT_SHAPE(MP, NU, NS, W), false>(P, slots);
  PIT_LAYOUTS(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

}  // namespace pitb
