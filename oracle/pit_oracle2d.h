/*
 * pit_oracle2d.h — config-5 (2D heat) propagators for the oracle.
 * TEST INFRASTRUCTURE ONLY (see pit_oracle.h and pit_oracle2d.c).
 */
#ifndef PIT_ORACLE2D_H
#define PIT_ORACLE2D_H

#include "pit_oracle.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc2_coeffs {
  int m;              /* points per axis; blocks are m*m, x fastest */
  int fine_steps, coarse_steps;
  double ac, an;      /* explicit Euler: y' = fma(ac, y, an*((w+e)+(n+s))) */
  int scaled, R;      /* scaled form: z' = fma(kappa, z, (w+e)+(n+s)), z *= anR every R */
  double kappa, anR, anLast;
  double D, O, minv;  /* BE step matrix I + dt*A: centre, neighbour, 1/D */
  double rel_tol;     /* CG relative tolerance */
  long long cap;      /* CG iteration cap */
  int rows, cluster, threads; /* K5 decomposition (reduction order) */
} orc2_coeffs;

void orc2_coefficients(int m, double band_off, double band_diag, double total_time, int slabs,
                       int fine_steps, int coarse_steps, double rel_tol, long long cap,
                       orc2_coeffs* c);
void orc2_explicit_propagate(const orc2_coeffs* c, const double* in, double* out);
/* one BE step by Jacobi-PCG; returns 1 converged, 0 failed (InnerSolveError) */
int orc2_cg_solve(const orc2_coeffs* c, const double* b, double* x, long long* iterations);
int orc2_coarse_propagate(const orc2_coeffs* c, const double* in, double* out,
                          long long* iterations);

typedef struct orc_2d orc_2d;
orc_2d* orc_2d_create(int m, double band_off, double band_diag, int N, double total_time,
                      int fine_steps, int coarse_steps, double rel_tol, long long cap,
                      const double* y0, int mode);
void orc_2d_destroy(orc_2d* o);
const orc_problem* orc_2d_problem(orc_2d* o);
const orc2_coeffs* orc_2d_coeffs(orc_2d* o);
long long orc_2d_coarse_iterations(orc_2d* o);

#ifdef __cplusplus
}
#endif
#endif
