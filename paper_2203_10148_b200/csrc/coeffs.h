// coeffs.h — host-side recipe for the chunked constant-factor backward-Euler
// step and the BASELINE layout choice.  Pure host C++.
#pragma once
#include <vector>

#include "pit_b200.h"

namespace pitb {

// Threads-per-slab layout: mpt points per thread, warps per slab CTA.
struct Layout {
  int mpt = 0;
  int nsub = 0;
  int nseg = 0;
  int warps = 0;
};

// Layouts the CUDA kernels are instantiated for (pit_kernels.cu).
bool layout_supported(int mpt, int nsub, int nseg, int warps);
Layout auto_layout(int M, int role);

// Fills coefficients for one propagator role; zc receives the [M]
// correction vector, ppos/qpos the [32*warps] per-thread segment-carry
// weights nl^(t*sub), nu^((T-1-t)*sub).  Returns PIT_OK or PIT_ERR_INVALID_ARGUMENT.
int build_step_coeffs(int M, int mpt, int nsub, int nseg, int warps, int steps, double band_lo,
                      double band_diag, double band_up, double dt, pit_step_coeffs* out,
                      std::vector<double>* zc, std::vector<double>* ppos,
                      std::vector<double>* qpos, std::vector<double>* zt);

}  // namespace pitb
