// pit_kernels2d.cuh — 2D (config 5) kernels: K4 explicit-Euler fine slabs
// and K5 coarse backward-Euler sweep with a cluster-resident Jacobi-PCG.
// DESIGN.md §3b.  Blocks are m x m values, x fastest (flat index j*m + i,
// SpatialGrid::flat_index, include/pit/grid.hpp), Dirichlet 0 outside.
#pragma once

#include <cuda_runtime.h>

#include "pit_kernels.cuh"

namespace pitb {

// K4: one thread-block cluster per slab; explicit Euler
//   y' = fma(ac, y, an * ((yW + yE) + (yN + yS)))
// ac = 1 - dt*diag, an = -dt*off (5-point operator, band_lo = band_up = off).
struct Ex2Params {
  int m;       // points per axis
  int steps;   // explicit steps per slab
  double ac, an;
  int scaled, R;  // scaled form (pit_step_coeffs_2d)
  double kappa, anR, anLast;
  long long* timing;  // PIT_PHASE_TIMING builds: [warp][8] cycle totals of cluster 0, CTA 0
};

// K5: one persistent cluster; per slab one BE step (I + dt*A) x = b solved
// by Jacobi-PCG (src/sparse.cpp:60-114 control flow) with
//   (S p)_i = fma(D, p_i, O * ((pW + pE) + (pN + pS))),  D = 1 + dt*diag,
//   O = dt*off (ImplicitStepSolver, src/pde.cpp:103-110), minv = 1/D.
struct Cg2Params {
  int m;
  int steps;       // backward-Euler steps per slab
  int rows;        // rows per CTA (cluster size C = ceil(m / rows))
  int cluster;     // C
  double D, O, minv;
  double rel_tol;  // kInnerSolveRelTol analogue
  long long cap;   // iteration cap (10 n, pde.hpp:79)
  long long* timing;  // PIT_PHASE_TIMING builds: phase cycle totals (CTA 0, thread 0)
};

constexpr int kCgRowsMax = 16;

// K4 layouts: rows per thread tile, columns per thread tile, CTAs per
// cluster, warps per CTA.  Covers m <= 32*TC columns and CL*WARPS*TR rows.
#define PIT_LAYOUTS_2D(X) \
  X(8, 8, 4, 8)           \
  X(8, 8, 8, 4)           \
  X(4, 4, 4, 8)           \
  X(4, 2, 2, 8)           \
  X(2, 1, 2, 8)

struct Layout2D {
  int tr, tc, cl, warps;
};
// smallest compiled K4 layout covering m (tr == 0: none)
Layout2D auto_layout_2d(int m);
bool layout2d_supported(int tr, int tc, int cl, int warps);

cudaError_t launch_explicit2d(const Layout2D& L, const Ex2Params& P, const SlabArgs& A, int slabs,
                              cudaStream_t st);

// K6 (pit_kernels2d_be.cu): 2D backward Euler on the reference's general
// 5-point operator (assemble_spatial_operator with velocity, pde.cpp:66-100),
// each step solved by Jacobi-PCG (symmetric) or Jacobi-BiCGStab with the
// reference's control flow (sparse.cpp:60-206).
struct Be2Params {
  int m, M;              // columns (points per axis in 2D), unknowns m*my
  int my;                // rows: m for a 2D grid, 1 for a general 1D operator
  int steps;             // backward-Euler steps per slab
  const double* coef;    // [5][M] device: south, west, centre, east, north of I + dt*A (0 = absent)
  const double* minv;    // [M] device: Jacobi inverse diagonal (jacobi_inverse_diagonal)
  double rel_tol;        // kInnerSolveRelTol (pde.hpp:78)
  int cap;               // kInnerSolveCapFactor * n (pde.hpp:79)
  int symmetric;         // 1: solve_cg, 0: solve_bicgstab (ImplicitStepSolver::solve)
  long long* iters;      // sweeps: cumulative inner iterations (optional)
  const double* tab;     // general source fl(dt*f) [N*steps][M] (PIT_SOURCE_TABLE) or nullptr
};
constexpr int kBe2Threads = 512;
// points per thread: up to 5 (m <= 50) everything a thread owns sits in
// registers and the stencil rows in shared memory; larger grids (m <= 101)
// run the same code on rounded-up point counts (8, 12, 16, 20) whose
// vectors the compiler keeps in local memory, read the stencil rows from
// global memory, and share one operand buffer between x and s^
constexpr int kBe2MaxPPT = 20;
size_t be2d_smem_bytes(int m, int my);
bool be2d_supported(int m, int my);
// src: add the source table before every step (Propagator::propagate);
// otherwise the homogeneous map
cudaError_t launch_be2d_batch(const Be2Params& P, const SlabArgs& A, int slabs, cudaStream_t st,
                              bool src = false);
cudaError_t launch_be2d_sweep(const Be2Params& P, const SweepArgs& A, cudaStream_t st,
                              bool src = false);
cudaError_t launch_cg_sweep2d(const Cg2Params& P, const SweepArgs& A, long long* iters,
                              cudaStream_t st);

}  // namespace pitb
