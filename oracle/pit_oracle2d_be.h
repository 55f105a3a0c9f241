/*
 * pit_oracle2d_be.h — 2D backward-Euler propagators on the reference's
 * general 5-point operator, in the K6 kernel's operation order.
 * TEST INFRASTRUCTURE ONLY (see pit_oracle2d_be.c).
 */
#ifndef PIT_ORACLE2D_BE_H
#define PIT_ORACLE2D_BE_H

#include "pit_oracle.h"

#ifdef __cplusplus
extern "C" {
#endif

/* assemble_spatial_operator, 2D (src/pde.cpp:66-100): out[5][m*m] = south,
 * west, centre, east, north entries (0 when absent); rotation: u = (-y, x). */
void orc_be2_stencil(int m, double lo, double hi, double mu, double r, int rotation, double* out);

typedef struct orc_be2_role {
  int m, steps;
  int my;       /* rows: m for the 2D presets, 1 for a general 1D operator (m = M columns) */
  double rel_tol;
  long long cap;
  int symmetric;
  double* coef; /* [5][m*m] of I + dt*A */
  double* minv; /* [m*m] */
} orc_be2_role;

void orc_be2_role_init(orc_be2_role* R, int m, const double* stencil, double dt, int steps,
                       double rel_tol, long long cap, int symmetric);
void orc_be2_role_free(orc_be2_role* R);
/* Propagator::run without source: returns 1, or 0 on InnerSolveError */
int orc_be2_propagate(const orc_be2_role* R, const double* in, double* out, long long* iterations);

typedef struct orc_be2d orc_be2d;
/* A general 1D operator (pit::SpatialOperator over any tridiagonal CSR,
 * include/pit/pde.hpp:36-37) as a 1-row grid of M columns: stencil[5][M] with
 * zero south/north rows; inner-product weight h (dimension 1, grid.cpp:113-114). */
orc_be2d* orc_be2d_create_1d(int M, double lo, double hi, const double* stencil, int nonsymmetric,
                             int N, double total_time, int fine_steps, int coarse_steps,
                             double fine_tol, long long fine_cap, double coarse_tol,
                             long long coarse_cap, const double* y0, int mode);
int orc_be2d_set_source_tables(orc_be2d* o, const double* fine, const double* coarse);
orc_be2d* orc_be2d_create(int m, double lo, double hi, const double* stencil, int nonsymmetric,
                          int N, double total_time, int fine_steps, int coarse_steps,
                          double fine_tol, long long fine_cap, double coarse_tol,
                          long long coarse_cap, const double* y0, int mode);
void orc_be2d_destroy(orc_be2d* o);
const orc_problem* orc_be2d_problem(orc_be2d* o);
long long orc_be2d_coarse_iterations(orc_be2d* o);

#ifdef __cplusplus
}
#endif
#endif
