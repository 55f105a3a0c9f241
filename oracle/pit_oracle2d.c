/*
 * pit_oracle2d.c — CPU restatement of the config-5 (2D heat) propagators.
 *
 * TEST INFRASTRUCTURE ONLY (see pit_oracle.h).  Mirrors, operation for
 * operation, paper_2203_10148_b200/csrc/pit_kernels2d.cu:
 *
 *   orc2_explicit_propagate   K4: steps of explicit Euler
 *       y' = fma(ac, y, an*((yW + yE) + (yN + yS))),  0 outside the square,
 *       ac = 1 - dt*diag, an = -dt*off (5-point operator; the reference's
 *       2D assemble_spatial_operator with zero velocity, src/pde.cpp:66-100).
 *   orc2_cg_solve             K5: one backward-Euler step (I + dt*A) x = b by
 *       Jacobi-PCG with the control flow of the reference's solve_cg
 *       (src/sparse.cpp:60-114: x0 = 0, tol = rel_tol*||b||, exit on
 *       res <= tol, stall on <p,q> == 0 or non-finite, true-residual
 *       confirmation and restart, iteration cap) and the matrix entries of
 *       ImplicitStepSolver (src/pde.cpp:103-110: O = off*dt, D = diag*dt + 1,
 *       Jacobi 1/D, sparse.cpp:43-50).  Sums use the kernel's order: per
 *       thread (column t of CTA c's row strip) an fma chain down the strip,
 *       a 32-lane xor butterfly per warp, then per lane the warp slots
 *       l, l+32, ... in order and a last butterfly.
 */
#include "pit_oracle2d.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

void orc2_coefficients(int m, double band_off, double band_diag, double total_time, int slabs,
                       int fine_steps, int coarse_steps, double rel_tol, long long cap,
                       orc2_coeffs* c) {
  const double slab = total_time / slabs;
  const double dtf = slab / fine_steps; /* Propagator::internal_dt */
  const double dtc = slab / coarse_steps;
  c->m = m;
  c->fine_steps = fine_steps;
  c->coarse_steps = coarse_steps;
  c->an = (double)(-(long double)dtf * (long double)band_off);
  c->ac = (double)(1.0L - (long double)dtf * (long double)band_diag);
  /* scaled form: an = 2^-sh exactly, kappa = ac/an exact (pit_capi.cu
   * explicit_scaling) */
  c->scaled = 0;
  c->R = 1;
  c->kappa = 0.0;
  c->anR = c->anLast = 1.0;
  {
    int e = 0;
    const double mant = frexp(c->an, &e);
    if (c->an > 0.0 && mant == 0.5 && e - 1 < 0) {
      const double k = c->ac / c->an;
      const int sh = 1 - e;
      int r = 768 / sh;
      if (isfinite(k) && k * c->an == c->ac && r >= 1) {
        if (r > fine_steps) r = fine_steps;
        const int j = fine_steps - r * ((fine_steps - 1) / r);
        c->scaled = 1;
        c->R = r;
        c->kappa = k;
        c->anR = ldexp(1.0, -sh * r);
        c->anLast = ldexp(1.0, -sh * j);
      }
    }
  }
  c->O = band_off * dtc;          /* v *= dt           (pde.cpp:107) */
  c->D = band_diag * dtc + 1.0;   /* diagonal += 1.0   (pde.cpp:108) */
  c->minv = c->D != 0.0 ? 1.0 / c->D : 1.0;
  c->rel_tol = rel_tol;
  c->cap = cap;
  c->rows = 16;
  c->cluster = (m + c->rows - 1) / c->rows;
  c->rows = (m + c->cluster - 1) / c->cluster;
  c->threads = 32 * ((m + 31) / 32);
}

void orc2_explicit_propagate(const orc2_coeffs* c, const double* in, double* out) {
  const int m = c->m;
  const size_t n = (size_t)m * m;
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  memcpy(a, in, n * sizeof(double));
  for (int k = 0; k < c->fine_steps; ++k) {
    /* scaled form: z = y / an^j, folded back by anR before every step
     * k = R, 2R, ... and by anLast after the last step */
    if (c->scaled && k > 0 && k % c->R == 0)
      for (size_t i = 0; i < n; ++i) a[i] = a[i] * c->anR;
    for (int r = 0; r < m; ++r)
      for (int q = 0; q < m; ++q) {
        const double y = a[(size_t)r * m + q];
        const double w = q > 0 ? a[(size_t)r * m + q - 1] : 0.0;
        const double e = q < m - 1 ? a[(size_t)r * m + q + 1] : 0.0;
        const double no = r > 0 ? a[(size_t)(r - 1) * m + q] : 0.0;
        const double so = r < m - 1 ? a[(size_t)(r + 1) * m + q] : 0.0;
        b[(size_t)r * m + q] = c->scaled ? fma(c->kappa, y, (w + e) + (no + so))
                                         : fma(c->ac, y, c->an * ((w + e) + (no + so)));
      }
    double* t = a;
    a = b;
    b = t;
  }
  if (c->scaled)
    for (size_t i = 0; i < n; ++i) a[i] = a[i] * c->anLast;
  memcpy(out, a, n * sizeof(double));
  free(a);
  free(b);
}

/* ---- K5 mirror --------------------------------------------------------- */

static void butterfly32(double* v) {
  for (int off = 16; off >= 1; off >>= 1) {
    double nv[32];
    for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ off];
    memcpy(v, nv, sizeof(nv));
  }
}

/* cluster-wide sum of a_i*b_i in the kernel's order */
static double cl_dot(const orc2_coeffs* c, const double* a, const double* b) {
  const int m = c->m, R = c->rows, C = c->cluster, NT = c->threads, W = NT / 32;
  const int nslot = C * W;
  double slot[4096];
  for (int cc = 0; cc < C; ++cc)
    for (int w = 0; w < W; ++w) {
      double v[32];
      for (int l = 0; l < 32; ++l) {
        const int t = 32 * w + l;
        double s = 0.0;
        if (t < m)
          for (int k = 0; k < R; ++k) {
            const int r = cc * R + k;
            if (r >= m) break;
            s = fma(a[(size_t)r * m + t], b[(size_t)r * m + t], s);
          }
        v[l] = s;
      }
      butterfly32(v);
      slot[cc * W + w] = v[0];
    }
  double u[32];
  for (int l = 0; l < 32; ++l) {
    double s = 0.0;
    for (int i = l; i < nslot; i += 32) s = s + slot[i];
    u[l] = s;
  }
  butterfly32(u);
  return u[0];
}

static void apply_S(const orc2_coeffs* c, const double* f, double* out) {
  const int m = c->m;
  for (int r = 0; r < m; ++r)
    for (int q = 0; q < m; ++q) {
      const double w = q > 0 ? f[(size_t)r * m + q - 1] : 0.0;
      const double e = q < m - 1 ? f[(size_t)r * m + q + 1] : 0.0;
      const double no = r > 0 ? f[(size_t)(r - 1) * m + q] : 0.0;
      const double so = r < m - 1 ? f[(size_t)(r + 1) * m + q] : 0.0;
      out[(size_t)r * m + q] = fma(c->D, f[(size_t)r * m + q], c->O * ((w + e) + (no + so)));
    }
}

int orc2_cg_solve(const orc2_coeffs* c, const double* b, double* x, long long* iterations) {
  const int m = c->m;
  const size_t n = (size_t)m * m;
  const double minv = c->minv;
  double* r = (double*)malloc(n * sizeof(double));
  double* z = (double*)malloc(n * sizeof(double));
  double* p = (double*)malloc(n * sizeof(double));
  double* q = (double*)malloc(n * sizeof(double));
  int ok = 1;
  long long it = 0;
  for (size_t i = 0; i < n; ++i) x[i] = 0.0;
  const double nb = sqrt(cl_dot(c, b, b));
  if (nb != 0.0) {
    const double tol = c->rel_tol * nb;
    for (size_t i = 0; i < n; ++i) {
      r[i] = b[i];
      z[i] = minv * r[i];
      p[i] = z[i];
    }
    double rz = cl_dot(c, r, z);
    double res = sqrt(cl_dot(c, r, r));
    int stalled = 0;
    for (;;) {
      while (res > tol && it < c->cap && !stalled) {
        apply_S(c, p, q);
        const double pq = cl_dot(c, p, q);
        if (pq == 0.0 || !isfinite(pq)) {
          stalled = 1;
          break;
        }
        const double alpha = rz / pq;
        for (size_t i = 0; i < n; ++i) {
          x[i] = fma(alpha, p[i], x[i]);
          r[i] = fma(-alpha, q[i], r[i]);
          z[i] = minv * r[i];
        }
        ++it;
        const double rr = cl_dot(c, r, r);
        const double rzn = cl_dot(c, r, z);
        res = sqrt(rr);
        if (!isfinite(res) || res <= tol) break;
        const double beta = rzn / rz;
        for (size_t i = 0; i < n; ++i) p[i] = fma(beta, p[i], z[i]);
        rz = rzn;
      }
      apply_S(c, x, q);
      for (size_t i = 0; i < n; ++i) {
        r[i] = b[i] - q[i];
        z[i] = minv * r[i];
      }
      res = sqrt(cl_dot(c, r, r));
      rz = cl_dot(c, r, z);
      if (res <= tol) break;
      if (it >= c->cap || stalled || !isfinite(res)) {
        ok = 0;
        break;
      }
      memcpy(p, z, n * sizeof(double));
    }
  }
  for (size_t i = 0; i < n && ok; ++i)
    if (!isfinite(x[i])) ok = 0;
  if (iterations) *iterations = it;
  free(r);
  free(z);
  free(p);
  free(q);
  return ok;
}

int orc2_coarse_propagate(const orc2_coeffs* c, const double* in, double* out,
                          long long* iterations) {
  const size_t n = (size_t)c->m * c->m;
  double* b = (double*)malloc(n * sizeof(double));
  memcpy(b, in, n * sizeof(double));
  long long total = 0;
  int ok = 1;
  for (int s = 0; s < c->coarse_steps && ok; ++s) {
    long long it = 0;
    ok = orc2_cg_solve(c, b, out, &it);
    total += it;
    memcpy(b, out, n * sizeof(double));
  }
  if (iterations) *iterations = total;
  free(b);
  return ok;
}

/* ---- a 2D orc_problem ------------------------------------------------- */

struct orc_2d {
  orc2_coeffs c;
  orc_problem* prob;
  double* y0;
  long long coarse_iterations;
};

static int prop2d(void* user, int role, int with_source, const double* in, int slab, double* out) {
  (void)with_source;
  (void)slab;
  orc_2d* o = (orc_2d*)user;
  if (role == ORC_FINE) {
    orc2_explicit_propagate(&o->c, in, out);
    return 0;
  }
  long long it = 0;
  const int ok = orc2_coarse_propagate(&o->c, in, out, &it);
  o->coarse_iterations += it;
  return ok ? 0 : 1;
}

orc_2d* orc_2d_create(int m, double band_off, double band_diag, int N, double total_time,
                      int fine_steps, int coarse_steps, double rel_tol, long long cap,
                      const double* y0, int mode) {
  orc_2d* o = (orc_2d*)calloc(1, sizeof(orc_2d));
  orc2_coefficients(m, band_off, band_diag, total_time, N, fine_steps, coarse_steps, rel_tol, cap,
                    &o->c);
  const size_t n = (size_t)m * m;
  o->y0 = (double*)malloc(n * sizeof(double));
  memcpy(o->y0, y0, n * sizeof(double));
  const double h = 1.0 / (m + 1);
  o->prob = orc_problem_new((int)n, N, h * h, 0, mode, o->y0, prop2d, o);
  o->prob->parallel = 1;
  return o;
}

void orc_2d_destroy(orc_2d* o) {
  if (!o) return;
  orc_problem_delete(o->prob);
  free(o->y0);
  free(o);
}

const orc_problem* orc_2d_problem(orc_2d* o) { return o->prob; }
const orc2_coeffs* orc_2d_coeffs(orc_2d* o) { return &o->c; }
long long orc_2d_coarse_iterations(orc_2d* o) { return o->coarse_iterations; }
