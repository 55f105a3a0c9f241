/*
 * pit_oracle2d_be.c — CPU restatement of the reference's 2D backward-Euler
 * propagators on its general 5-point operator, in the operation order of
 * the K6 kernels (paper_2203_10148_b200/csrc/pit_kernels2d_be.cu).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ (and smoke()) as the checker of
 * the CUDA path, never by the product.
 *
 * Follows:
 *   orc_be2_stencil      assemble_spatial_operator, 2D branch with velocity
 *                        (src/pde.cpp:66-100): 5-point diffusion, reaction,
 *                        first-order upwind of u = (-y, x) (Rotation); an
 *                        entry is absent (0 here) at the walls or when zero.
 *   orc_be2_role_init    ImplicitStepSolver (src/pde.cpp:103-110): entries
 *                        times dt, diagonal + 1; jacobi_inverse_diagonal
 *                        (src/sparse.cpp:43-50).
 *   be2_cg / be2_bicgstab solve_cg (src/sparse.cpp:60-114) and
 *                        solve_bicgstab (116-206), branch for branch.
 *   orc_be2_propagate    Propagator::run without source (src/propagator.cpp:50-71).
 * Arithmetic follows the kernel: every multiply-add an fma; dot products as
 * per-thread fma chains over points t, t+512, ... (in that order), a 32-lane
 * xor butterfly, then the 16 warp totals summed in warp order; the stencil
 * row in CSR column order (south, west, centre, east, north) as fma's into 0.
 * Pinned against the reference's own Propagator (oracle/_ref) in
 * tests/test_oracle2d_be.py.
 */
#include "pit_oracle2d_be.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define BE2_T 512
#define BE2_NW (BE2_T / 32)

void orc_be2_stencil(int m, double lo, double hi, double mu, double r, int rotation, double* out) {
  const int n = m * m;
  const double h = (hi - lo) / (double)(m + 2 - 1); /* SpatialGrid spacing, grid.cpp:19 */
  const double mu_h2 = mu / (h * h);
  for (int j = 0; j < m; ++j) {
    const double y = lo + (j + 1) * h; /* interior_coord, grid.hpp:33 */
    for (int i = 0; i < m; ++i) {
      const double x = lo + (i + 1) * h;
      double ux = 0.0, uy = 0.0;
      if (rotation) {
        ux = -y;
        uy = x;
      }
      const double centre = 4.0 * mu_h2 + r + (fabs(ux) + fabs(uy)) / h;
      double west = -mu_h2, east = -mu_h2, south = -mu_h2, north = -mu_h2;
      if (ux > 0.0)
        west -= ux / h;
      else if (ux < 0.0)
        east += ux / h;
      if (uy > 0.0)
        south -= uy / h;
      else if (uy < 0.0)
        north += uy / h;
      const int row = j * m + i;
      out[row] = (south != 0.0 && j > 0) ? south : 0.0;
      out[n + row] = (west != 0.0 && i > 0) ? west : 0.0;
      out[2 * n + row] = centre;
      out[3 * n + row] = (east != 0.0 && i < m - 1) ? east : 0.0;
      out[4 * n + row] = (north != 0.0 && j < m - 1) ? north : 0.0;
    }
  }
}

static void role_init_rect(orc_be2_role* R, int m, int my, const double* stencil, double dt,
                           int steps, double rel_tol, long long cap, int symmetric);
void orc_be2_role_init(orc_be2_role* R, int m, const double* stencil, double dt, int steps,
                       double rel_tol, long long cap, int symmetric) {
  role_init_rect(R, m, m, stencil, dt, steps, rel_tol, cap, symmetric);
}
static void role_init_rect(orc_be2_role* R, int m, int my, const double* stencil, double dt,
                           int steps, double rel_tol, long long cap, int symmetric) {
  const int n = m * my;
  R->m = m;
  R->my = my;
  R->steps = steps;
  R->rel_tol = rel_tol > 0.0 ? rel_tol : 1e-12;
  R->cap = cap > 0 ? cap : 10LL * n;
  R->symmetric = symmetric;
  R->coef = (double*)malloc(sizeof(double) * 5 * (size_t)n);
  R->minv = (double*)malloc(sizeof(double) * (size_t)n);
  for (int k = 0; k < 5 * n; ++k) R->coef[k] = stencil[k] * dt;
  for (int i = 0; i < n; ++i) {
    R->coef[2 * n + i] = R->coef[2 * n + i] + 1.0;
    const double d = R->coef[2 * n + i];
    R->minv[i] = d != 0.0 ? 1.0 / d : 1.0;
  }
}

void orc_be2_role_free(orc_be2_role* R) {
  free(R->coef);
  free(R->minv);
  R->coef = R->minv = NULL;
}

/* block-wide sum of per-point terms f_i in the kernel's order */
static double be2_reduce(int n, const double* term) {
  double part[BE2_T];
  for (int t = 0; t < BE2_T; ++t) {
    double s = 0.0;
    for (int i = t; i < n; i += BE2_T) s = fma(term[2 * i], term[2 * i + 1], s);
    part[t] = s;
  }
  double tot = 0.0;
  for (int w = 0; w < BE2_NW; ++w) {
    double v[32];
    memcpy(v, part + 32 * w, sizeof(v));
    for (int off = 16; off >= 1; off >>= 1) {
      double nv[32];
      for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ off];
      memcpy(v, nv, sizeof(nv));
    }
    tot = w == 0 ? v[0] : tot + v[0];
  }
  return tot;
}

typedef struct be2_ws {
  int n;
  double* pair; /* [2n] scratch (a_i, b_i) */
} be2_ws;

static double be2_dot(be2_ws* w, const double* a, const double* b) {
  for (int i = 0; i < w->n; ++i) {
    w->pair[2 * i] = a[i];
    w->pair[2 * i + 1] = b[i];
  }
  return be2_reduce(w->n, w->pair);
}

/* (A x)_i, CSR column order south, west, centre, east, north */
static double be2_row(const orc_be2_role* R, const double* x, int i) {
  const int m = R->m, n = m * R->my, ix = i % m, iy = i / m;
  const double xs = iy > 0 ? x[i - m] : 0.0, xw = ix > 0 ? x[i - 1] : 0.0;
  const double xe = ix < m - 1 ? x[i + 1] : 0.0, xn = iy < R->my - 1 ? x[i + m] : 0.0;
  double s = 0.0;
  s = fma(R->coef[i], xs, s);
  s = fma(R->coef[n + i], xw, s);
  s = fma(R->coef[2 * n + i], x[i], s);
  s = fma(R->coef[3 * n + i], xe, s);
  s = fma(R->coef[4 * n + i], xn, s);
  return s;
}

static double be2_true_residual(const orc_be2_role* R, be2_ws* w, const double* b, const double* x,
                                double* r) {
  for (int i = 0; i < w->n; ++i) r[i] = b[i] - be2_row(R, x, i);
  return sqrt(be2_dot(w, r, r));
}

static int be2_cg(const orc_be2_role* R, be2_ws* w, const double* b, double* x, long long* iters) {
  const int n = w->n;
  double* r = (double*)malloc(sizeof(double) * n * 3);
  double *z = r + n, *p = r + 2 * n;
  double* q = (double*)malloc(sizeof(double) * n);
  int ok = 0;
  memset(x, 0, sizeof(double) * n);
  const double norm_b = sqrt(be2_dot(w, b, b));
  *iters = 0;
  if (norm_b == 0.0) {
    ok = 1;
    goto done;
  }
  const double tol = R->rel_tol * norm_b;
  for (int i = 0; i < n; ++i) {
    r[i] = b[i];
    z[i] = R->minv[i] * r[i];
    p[i] = z[i];
  }
  double rz = be2_dot(w, r, z), res = sqrt(be2_dot(w, r, r));
  long long it = 0;
  int stalled = 0;
  for (;;) {
    while (res > tol && it < R->cap && !stalled) {
      for (int i = 0; i < n; ++i) q[i] = be2_row(R, p, i);
      const double pq = be2_dot(w, p, q);
      if (pq == 0.0 || !isfinite(pq)) {
        stalled = 1;
        break;
      }
      const double alpha = rz / pq;
      for (int i = 0; i < n; ++i) {
        x[i] = fma(alpha, p[i], x[i]);
        r[i] = fma(-alpha, q[i], r[i]);
        z[i] = R->minv[i] * r[i];
      }
      ++it;
      res = sqrt(be2_dot(w, r, r));
      const double rzn = be2_dot(w, r, z);
      if (!isfinite(res) || res <= tol) break;
      const double beta = rzn / rz;
      for (int i = 0; i < n; ++i) p[i] = fma(beta, p[i], z[i]);
      rz = rzn;
    }
    res = be2_true_residual(R, w, b, x, r);
    *iters = it;
    if (res <= tol) {
      ok = 1;
      break;
    }
    if (it >= R->cap || stalled || !isfinite(res)) break;
    for (int i = 0; i < n; ++i) {
      z[i] = R->minv[i] * r[i];
      p[i] = z[i];
    }
    rz = be2_dot(w, r, z);
  }
done:
  free(r);
  free(q);
  return ok;
}

static int be2_bicgstab(const orc_be2_role* R, be2_ws* w, const double* b, double* x,
                        long long* iters) {
  const int n = w->n;
  double* buf = (double*)malloc(sizeof(double) * n * 8);
  double *r = buf, *rt = buf + n, *p = buf + 2 * n, *ph = buf + 3 * n, *v = buf + 4 * n,
         *s = buf + 5 * n, *sh = buf + 6 * n, *t = buf + 7 * n;
  int ok = 0;
  memset(x, 0, sizeof(double) * n);
  memset(v, 0, sizeof(double) * n);
  const double norm_b = sqrt(be2_dot(w, b, b));
  *iters = 0;
  if (norm_b == 0.0) {
    ok = 1;
    goto done;
  }
  const double tol = R->rel_tol * norm_b;
  double rho_prev = 1.0, alpha = 1.0, omega = 1.0, res = 0.0;
  long long it = 0;
  int restart = 1, first = 1;
  while (it < R->cap) {
    if (restart) {
      res = be2_true_residual(R, w, b, x, r);
      if (res <= tol) {
        ok = 1;
        goto out;
      }
      if (!isfinite(res)) goto out;
      memcpy(rt, r, sizeof(double) * n);
      first = 1;
      restart = 0;
      rho_prev = alpha = omega = 1.0;
    }
    const double rho = be2_dot(w, rt, r);
    if (rho == 0.0 || !isfinite(rho)) {
      restart = 1;
      ++it;
      continue;
    }
    if (first) {
      memcpy(p, r, sizeof(double) * n);
      first = 0;
    } else {
      const double beta = (rho / rho_prev) * (alpha / omega);
      for (int i = 0; i < n; ++i) p[i] = fma(beta, fma(-omega, v[i], p[i]), r[i]);
    }
    for (int i = 0; i < n; ++i) ph[i] = R->minv[i] * p[i];
    for (int i = 0; i < n; ++i) v[i] = be2_row(R, ph, i);
    const double rv = be2_dot(w, rt, v);
    if (rv == 0.0 || !isfinite(rv)) {
      restart = 1;
      ++it;
      continue;
    }
    alpha = rho / rv;
    for (int i = 0; i < n; ++i) s[i] = fma(-alpha, v[i], r[i]);
    if (sqrt(be2_dot(w, s, s)) <= tol) {
      for (int i = 0; i < n; ++i) x[i] = fma(alpha, ph[i], x[i]);
      ++it;
      res = be2_true_residual(R, w, b, x, r);
      if (res <= tol) {
        ok = 1;
        goto out;
      }
      if (!isfinite(res)) goto out;
      memcpy(rt, r, sizeof(double) * n);
      first = 1;
      rho_prev = alpha = omega = 1.0;
      continue;
    }
    for (int i = 0; i < n; ++i) sh[i] = R->minv[i] * s[i];
    for (int i = 0; i < n; ++i) t[i] = be2_row(R, sh, i);
    const double tt = be2_dot(w, t, t), ts = be2_dot(w, t, s);
    omega = tt == 0.0 ? 0.0 : ts / tt;
    for (int i = 0; i < n; ++i) {
      x[i] = fma(omega, sh[i], fma(alpha, ph[i], x[i]));
      r[i] = fma(-omega, t[i], s[i]);
    }
    ++it;
    res = sqrt(be2_dot(w, r, r));
    if (!isfinite(res)) {
      restart = 1;
      continue;
    }
    if (res <= tol) {
      res = be2_true_residual(R, w, b, x, r);
      if (res <= tol) {
        ok = 1;
        goto out;
      }
    }
    if (omega == 0.0) restart = 1;
    rho_prev = rho;
  }
  res = be2_true_residual(R, w, b, x, r);
  ok = res <= tol;
out:
  *iters = it;
done:
  free(buf);
  return ok;
}

static int propagate_tab(const orc_be2_role* R, const double* in, double* out,
                         long long* iterations, const double* tab);
int orc_be2_propagate(const orc_be2_role* R, const double* in, double* out, long long* iterations) {
  return propagate_tab(R, in, out, iterations, NULL);
}
/* tab: general source fl(dt*f) [steps][n] added before every step, or NULL */
static int propagate_tab(const orc_be2_role* R, const double* in, double* out,
                         long long* iterations, const double* tab) {
  const int n = R->m * R->my;
  be2_ws w;
  w.n = n;
  w.pair = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  double* b = (double*)malloc(sizeof(double) * n);
  double* x = (double*)malloc(sizeof(double) * n);
  memcpy(b, in, sizeof(double) * n);
  int ok = 1;
  for (int step = 0; step < R->steps && ok; ++step) {
    long long it = 0;
    if (tab)
      for (int i = 0; i < n; ++i) b[i] = b[i] + tab[(size_t)step * n + i];
    ok = R->symmetric ? be2_cg(R, &w, b, x, &it) : be2_bicgstab(R, &w, b, x, &it);
    if (iterations) *iterations += it;
    for (int i = 0; i < n && ok; ++i)
      if (!isfinite(x[i])) ok = 0;
    double* tmp = b;
    b = x;
    x = tmp;
  }
  memcpy(out, b, sizeof(double) * n);
  free(w.pair);
  free(b);
  free(x);
  return ok;
}

/* ---- orc_problem over the two roles ------------------------------------ */

struct orc_be2d {
  orc_be2_role role[2];
  orc_problem* prob;
  double* y0;
  long long coarse_iterations;
  double* tab[2]; /* general source fl(dt*f) [N][steps][n] per role, or NULL */
  double dt[2];
  int N;
};

static int prop_be2(void* user, int role, int with_source, const double* in, int slab,
                    double* out) {
  orc_be2d* o = (orc_be2d*)user;
  long long it = 0;
  const orc_be2_role* R = &o->role[role];
  const double* tab = NULL;
  if (with_source && o->tab[role])
    tab = o->tab[role] + (size_t)slab * R->steps * R->m * R->my;
  const int ok = propagate_tab(R, in, out, &it, tab);
  if (role == ORC_COARSE) o->coarse_iterations += it;
  return ok ? 0 : 1;
}

static orc_be2d* create_rect(int m, int my, double lo, double hi, const double* stencil,
                             int nonsymmetric, int N, double total_time, int fine_steps,
                             int coarse_steps, double fine_tol, long long fine_cap,
                             double coarse_tol, long long coarse_cap, const double* y0, int mode) {
  orc_be2d* o = (orc_be2d*)calloc(1, sizeof(orc_be2d));
  const double slab = total_time / N;
  role_init_rect(&o->role[ORC_FINE], m, my, stencil, slab / fine_steps, fine_steps, fine_tol,
                 fine_cap, !nonsymmetric);
  role_init_rect(&o->role[ORC_COARSE], m, my, stencil, slab / coarse_steps, coarse_steps,
                 coarse_tol, coarse_cap, !nonsymmetric);
  o->dt[ORC_FINE] = slab / fine_steps;
  o->dt[ORC_COARSE] = slab / coarse_steps;
  o->N = N;
  const size_t n = (size_t)m * my;
  o->y0 = (double*)malloc(n * sizeof(double));
  memcpy(o->y0, y0, n * sizeof(double));
  const double h = (hi - lo) / (double)(m + 1);
  /* inner_product weight h^d (grid.cpp:113-114) */
  o->prob = orc_problem_new((int)n, N, my == 1 ? h : h * h, 0, mode, o->y0, prop_be2, o);
  o->prob->parallel = 1;
  return o;
}

orc_be2d* orc_be2d_create(int m, double lo, double hi, const double* stencil, int nonsymmetric,
                          int N, double total_time, int fine_steps, int coarse_steps,
                          double fine_tol, long long fine_cap, double coarse_tol,
                          long long coarse_cap, const double* y0, int mode) {
  return create_rect(m, m, lo, hi, stencil, nonsymmetric, N, total_time, fine_steps, coarse_steps,
                     fine_tol, fine_cap, coarse_tol, coarse_cap, y0, mode);
}

orc_be2d* orc_be2d_create_1d(int M, double lo, double hi, const double* stencil, int nonsymmetric,
                             int N, double total_time, int fine_steps, int coarse_steps,
                             double fine_tol, long long fine_cap, double coarse_tol,
                             long long coarse_cap, const double* y0, int mode) {
  return create_rect(M, 1, lo, hi, stencil, nonsymmetric, N, total_time, fine_steps, coarse_steps,
                     fine_tol, fine_cap, coarse_tol, coarse_cap, y0, mode);
}

/* General source tables f(t_k, x_i) of both roles ([N][steps][n]); stored as
 * fl(dt*f) (PIT_SOURCE_TABLE). */
int orc_be2d_set_source_tables(orc_be2d* o, const double* fine, const double* coarse) {
  const double* f[2] = {fine, coarse};
  for (int r = 0; r < 2; ++r) {
    const orc_be2_role* R = &o->role[r];
    const size_t cnt = (size_t)o->N * R->steps * R->m * R->my;
    free(o->tab[r]);
    o->tab[r] = (double*)malloc(cnt * sizeof(double));
    if (!o->tab[r]) return -1;
    for (size_t i = 0; i < cnt; ++i) o->tab[r][i] = o->dt[r] * f[r][i];
  }
  o->prob->has_source = 1;
  return 0;
}

void orc_be2d_destroy(orc_be2d* o) {
  if (!o) return;
  free(o->tab[0]);
  free(o->tab[1]);
  orc_problem_delete(o->prob);
  orc_be2_role_free(&o->role[0]);
  orc_be2_role_free(&o->role[1]);
  free(o->y0);
  free(o);
}

const orc_problem* orc_be2d_problem(orc_be2d* o) { return o->prob; }
long long orc_be2d_coarse_iterations(orc_be2d* o) { return o->coarse_iterations; }
