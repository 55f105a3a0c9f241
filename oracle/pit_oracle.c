/*
 * pit_oracle.c — CPU restatement of the reference PiTSBiCG hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see pit_oracle.h).  Compiled with
 * -ffp-contract=off: every fused multiply-add below is an explicit fma(),
 * exactly where the CUDA kernels issue a DFMA, so results match bit for bit.
 */
#include "pit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Coefficient recipe of the chunked constant-factor step.    */
/* Written independently of paper_2203_10148_b200/csrc/coeffs.cpp; a test    */
/* checks both produce identical bits.                                       */
/* ------------------------------------------------------------------------ */

int orc_stepper_init(orc_stepper* s, int M, int m, int nsub, int nseg, int warps, int steps,
                     double band_lo, double band_diag, double band_up, double dt) {
  typedef long double ld;
  memset(s, 0, sizeof(*s));
  if (M < 1 || m < 1 || m > ORC_MAX_M || nsub < 1 || nsub > 8 || nseg < 1 || m % (nsub * nseg) ||
      m / (nsub * nseg) > 32 || warps < 1 || steps < 1)
    return -1;
  s->M = M;
  s->m = m;
  s->nsub = nsub;
  s->nseg = nseg;
  s->warps = warps;
  s->Mp = 32 * warps * m;
  if (s->Mp < M) return -1;
  s->steps = steps;
  /* ImplicitStepSolver: val *= dt, then diagonal += 1 (pde.cpp:103-110) */
  s->delta = band_diag * dt + 1.0;
  s->lam = band_lo * dt;
  s->mu = band_up * dt;
  const ld D = s->delta, L = s->lam, U = s->mu;
  const ld disc = D * D - 4.0L * L * U;
  if (!(disc > 0.0L)) return -2;
  const ld dst = (D + sqrtl(disc)) * 0.5L;
  s->nl = (double)(-L / dst);
  s->nu = (double)(-U / dst);
  const ld nl = s->nl, nu = s->nu;
  /* inv makes the row sum of the factored operator exact (smooth modes) */
  const ld inv = (1.0L - nl) * (1.0L - nu) / (D + L + U);
  s->inv = (double)inv;
  s->dstar = (double)(1.0L / (ld)s->inv);

  /* z' = U^-1 L^-1 e0 with unit bidiagonal factors */
  s->zc = (double*)calloc((size_t)M, sizeof(double));
  ld* z = (ld*)calloc((size_t)M, sizeof(ld));
  if (!s->zc || !z) {
    free(z);
    return -3;
  }
  z[0] = 1.0L;
  for (int i = 1; i < M; ++i) z[i] = nl * z[i - 1];
  for (int i = M - 2; i >= 0; --i) z[i] = z[i] + nu * z[i + 1];
  for (int i = 0; i < M; ++i) s->zc[i] = (double)z[i];
  {
    const ld invd = s->inv;
    const ld sigma = D - 1.0L / invd;
    const ld a = sigma * invd;
    s->gneg = (double)(-(a / (1.0L + a * z[0])));
    const ld thr = fabsl(z[0]) * 8.470329472543003e-22L; /* 2^-70 */
    int k0 = 1;
    for (int i = M - 1; i >= 1; --i) {
      if (fabsl(z[i]) > thr) {
        k0 = i + 1;
        break;
      }
    }
    s->K0 = k0;
  }
  const ld z0 = z[0];
  free(z);
  {
    /* sub-chunk = sub points; thread chunk = ch = nsub*sub (warp scan
     * multiplier nl^ch); segment = T*ch */
    const int sub = m / (nsub * nseg), ch = nsub * sub, T = 32 * warps;
    ld nlp[65], nup[65];
    nlp[0] = 1.0L;
    nup[0] = 1.0L;
    for (int k = 1; k <= 64; ++k) {
      nlp[k] = nlp[k - 1] * nl;
      nup[k] = nup[k - 1] * nu;
    }
    for (int j = 0; j < sub; ++j) s->nlpow[j] = (double)nlp[j];
    for (int u = 0; u < nsub; ++u) s->pw[u] = (double)nlp[u * sub];
    s->pS = (double)nlp[sub];
    s->qS = (double)nup[sub];
    ld pk = nlp[ch], qk = nup[ch];
    s->scan_f = s->scan_b = 5;
    for (int k = 0; k < 5; ++k) {
      if (s->scan_f == 5 && fabsl(pk) <= 8.470329472543003e-22L) s->scan_f = k;
      if (s->scan_b == 5 && fabsl(qk) <= 8.470329472543003e-22L) s->scan_b = k;
      s->pp[k] = (double)pk;
      s->qq[k] = (double)qk;
      pk = pk * pk;
      qk = qk * qk;
    }
    s->p32 = (double)pk;
    s->q32 = (double)qk;
    ld pl = 1.0L, ql = 1.0L;
    for (int l = 0; l < 32; ++l) {
      s->plane[l] = (double)pl;
      s->qlane[31 - l] = (double)ql;
      pl = pl * nlp[ch];
      ql = ql * nup[ch];
    }
    s->ppos = (double*)calloc((size_t)T, sizeof(double));
    s->qpos = (double*)calloc((size_t)T, sizeof(double));
    s->zt = (double*)calloc((size_t)T, sizeof(double));
    ld pt = 1.0L, qt = 1.0L;
    for (int t = 0; t < T; ++t) {
      s->ppos[t] = (double)pt;
      s->qpos[T - 1 - t] = (double)qt;
      s->zt[t] = (double)(z0 * pt);
      pt = pt * nlp[ch];
      qt = qt * nup[ch];
    }
    s->Pseg = (double)pt;
    s->Qseg = (double)qt;
    const ld decay = powl(fabsl(nl * nu), (ld)(M - s->K0));
    s->narrow = (s->K0 <= 32 * ch && decay < 7.7e-34L) ? 1 : 0;
  }
  {
    double lg = log2(s->dstar);
    int R = steps;
    if (lg > 0.0) {
      double r = floor(512.0 / lg);
      if (r < (double)steps) R = r < 1.0 ? 1 : (int)r;
    }
    s->R = R;
    const ld invd = s->inv;
    ld p = 1.0L;
    for (int k = 0; k < R; ++k) p = p * invd;
    s->invR = (double)p;
    const int last = steps % R;
    p = 1.0L;
    for (int k = 0; k < last; ++k) p = p * invd;
    s->invLast = (double)p;
  }
  return 0;
}

void orc_stepper_free(orc_stepper* s) {
  free(s->zc);
  free(s->ppos);
  free(s->qpos);
  free(s->zt);
  s->zc = s->ppos = s->qpos = s->zt = NULL;
}

/* One unscaled solve y <- U^-1 L^-1 b plus the corner correction, on the
 * padded array y[Mp], chunked exactly like the CUDA step (pit_step.cuh
 * be_solve).  The padded slab is nseg segments of lseg = T*ch points; thread
 * k owns chunk k (ch = nsub*sub contiguous points) of every segment, split
 * into nsub sub-chunks.  Per direction and segment: pass 1 sweeps each
 * sub-chunk with zero carry (end value only); the chunk end combines its
 * sub-chunks; warp Kogge-Stone scan + sequential cross-warp combine; segment
 * totals chained segment to segment; chunk carry = local carry + pos_k *
 * segment carry; sub-chunk carries; pass 2 reruns each sub-chunk's sweep. */
static void chunked_solve(const orc_stepper* s, double* y, double* scratch) {
  const int W = s->warps, T = 32 * W, M = s->M;
  const int nu_ = s->nsub, ns = s->nseg, sub = s->m / (nu_ * ns), ch = nu_ * sub, lseg = T * ch;
  double* Z = scratch;          /* [T] chunk end values / scan */
  double* C = scratch + T;      /* [T] local carries */
  double* tot = scratch + 2 * T;/* [W] */
  double* tmp = scratch + 2 * T + W; /* [32] */
  double E[8];

  /* ---- forward ---- */
  double S = 0.0; /* segment carry-in */
  for (int q = 0; q < ns; ++q) {
    double* seg = y + (size_t)q * lseg;
    for (int k = 0; k < T; ++k) { /* pass 1 */
      const double* c = seg + (size_t)k * ch;
      for (int u = 0; u < nu_; ++u) {
        const double* cu = c + u * sub;
        double z = cu[0];
        for (int j = 1; j < sub; ++j) z = fma(s->nl, z, cu[j]);
        E[u] = z;
      }
      double z = E[0];
      for (int u = 1; u < nu_; ++u) z = fma(s->pS, z, E[u]);
      Z[k] = z;
    }
    for (int w = 0; w < W; ++w) {
      double* I = Z + 32 * w;
      for (int st = 0; st < s->scan_f; ++st) {
        int off = 1 << st;
        for (int l = 0; l < 32; ++l) tmp[l] = (l >= off) ? fma(s->pp[st], I[l - off], I[l]) : I[l];
        memcpy(I, tmp, 32 * sizeof(double));
      }
      tot[w] = I[31];
    }
    for (int w = 0; w < W; ++w) {
      double Wc = 0.0;
      for (int v = 0; v < w; ++v) Wc = fma(s->p32, Wc, tot[v]);
      for (int l = 0; l < 32; ++l) {
        int k = 32 * w + l;
        C[k] = (l == 0) ? Wc : fma(s->plane[l], Wc, Z[k - 1]);
      }
    }
    double segtot = 0.0;
    for (int v = 0; v < W; ++v) segtot = fma(s->p32, segtot, tot[v]);
    for (int k = 0; k < T; ++k) { /* pass 2 from the true carries */
      double* c = seg + (size_t)k * ch;
      for (int u = 0; u < nu_; ++u) { /* sub-chunk end values with zero carry */
        const double* cu = c + u * sub;
        double z = cu[0];
        for (int j = 1; j < sub; ++j) z = fma(s->nl, z, cu[j]);
        E[u] = z;
      }
      double Ck = q > 0 ? fma(s->ppos[k], S, C[k]) : C[k];
      for (int u = 0; u < nu_; ++u) {
        double* cu = c + u * sub;
        const double Cu = Ck;
        if (u + 1 < nu_) Ck = fma(s->pS, Ck, E[u]);
        cu[0] = fma(s->nl, Cu, cu[0]);
        for (int j = 1; j < sub; ++j) cu[j] = fma(s->nl, cu[j - 1], cu[j]);
      }
    }
    S = fma(s->Pseg, S, segtot); /* carry into segment q+1 */
  }
  for (int i = M; i < ns * lseg; ++i) y[i] = 0.0; /* Dirichlet padding */
  /* ---- backward ---- */
  S = 0.0;
  for (int q = ns - 1; q >= 0; --q) {
    double* seg = y + (size_t)q * lseg;
    for (int k = 0; k < T; ++k) { /* pass 1 */
      const double* c = seg + (size_t)k * ch;
      for (int u = 0; u < nu_; ++u) {
        const double* cu = c + u * sub;
        double h = cu[sub - 1];
        for (int j = sub - 2; j >= 0; --j) h = fma(s->nu, h, cu[j]);
        E[u] = h;
      }
      double h = E[nu_ - 1];
      for (int u = nu_ - 2; u >= 0; --u) h = fma(s->qS, h, E[u]);
      Z[k] = h;
    }
    for (int w = 0; w < W; ++w) {
      double* J = Z + 32 * w;
      for (int st = 0; st < s->scan_b; ++st) {
        int off = 1 << st;
        for (int l = 0; l < 32; ++l)
          tmp[l] = (l < 32 - off) ? fma(s->qq[st], J[l + off], J[l]) : J[l];
        memcpy(J, tmp, 32 * sizeof(double));
      }
      tot[w] = J[0];
    }
    for (int w = 0; w < W; ++w) {
      double Vc = 0.0;
      for (int v = W - 1; v > w; --v) Vc = fma(s->q32, Vc, tot[v]);
      for (int l = 0; l < 32; ++l) {
        int k = 32 * w + l;
        C[k] = (l == 31) ? Vc : fma(s->qlane[l], Vc, Z[k + 1]);
      }
    }
    double segtot = 0.0;
    for (int v = W - 1; v >= 0; --v) segtot = fma(s->q32, segtot, tot[v]);
    for (int k = 0; k < T; ++k) { /* pass 2 */
      double* c = seg + (size_t)k * ch;
      for (int u = 0; u < nu_; ++u) {
        const double* cu = c + u * sub;
        double h = cu[sub - 1];
        for (int j = sub - 2; j >= 0; --j) h = fma(s->nu, h, cu[j]);
        E[u] = h;
      }
      double Rk = q < ns - 1 ? fma(s->qpos[k], S, C[k]) : C[k];
      for (int u = nu_ - 1; u >= 0; --u) {
        double* cu = c + u * sub;
        const double Ru = Rk;
        if (u > 0) Rk = fma(s->qS, Rk, E[u]);
        cu[sub - 1] = fma(s->nu, Ru, cu[sub - 1]);
        for (int j = sub - 2; j >= 0; --j) cu[j] = fma(s->nu, cu[j + 1], cu[j]);
      }
    }
    S = fma(s->Qseg, S, segtot);
  }
  /* corner rank-1 correction */
  {
    const double cc = s->gneg * y[0];
    if (s->narrow) {
      for (int k = 0; k < 32 && k * ch < s->K0; ++k) {
        const double a = cc * s->zt[k];
        for (int u = 0; u < nu_ && u * sub < s->K0; ++u) {
          const double au = a * s->pw[u];
          for (int j = 0; j < sub; ++j) {
            double* v = y + (size_t)k * ch + u * sub + j;
            *v = fma(au, s->nlpow[j], *v);
          }
        }
      }
    } else {
      for (int i = 0; i < s->K0; ++i) y[i] = fma(cc, s->zc[i], y[i]);
    }
  }
}

void orc_stepper_propagate(const orc_stepper* s, const double* in, const double* ds,
                           const double* g, double* out) {
  const int T = 32 * s->warps;
  double* y = (double*)calloc((size_t)s->Mp, sizeof(double));
  double* scratch = (double*)calloc((size_t)(2 * T + s->warps + 32), sizeof(double));
  memcpy(y, in, (size_t)s->M * sizeof(double));
  if (ds) {
    /* with source: unscaled state every step (R = 1) */
    for (int k = 0; k < s->steps; ++k) {
      for (int i = 0; i < s->M; ++i) y[i] = fma(ds[k], g[i], y[i]);
      chunked_solve(s, y, scratch);
      for (int i = 0; i < s->M; ++i) y[i] = y[i] * s->inv;
    }
  } else {
    for (int k = 1; k <= s->steps; ++k) {
      chunked_solve(s, y, scratch);
      if (k % s->R == 0) {
        for (int i = 0; i < s->M; ++i) y[i] = y[i] * s->invR;
      }
    }
    if (s->steps % s->R) {
      for (int i = 0; i < s->M; ++i) y[i] = y[i] * s->invLast;
    }
  }
  memcpy(out, y, (size_t)s->M * sizeof(double));
  free(y);
  free(scratch);
}

/* General source (PIT_SOURCE_TABLE): tab[k*M + i] = fl(dt * f(t_k, x_i)) is
 * added before step k, the reference's rhs.axpy(dt, sample_source(t))
 * (src/propagator.cpp:60-62); unscaled state every step, as with ds. */
void orc_stepper_propagate_table(const orc_stepper* s, const double* in, const double* tab,
                                 double* out) {
  const int T = 32 * s->warps;
  double* y = (double*)calloc((size_t)s->Mp, sizeof(double));
  double* scratch = (double*)calloc((size_t)(2 * T + s->warps + 32), sizeof(double));
  memcpy(y, in, (size_t)s->M * sizeof(double));
  for (int k = 0; k < s->steps; ++k) {
    const double* tk = tab + (size_t)k * s->M;
    for (int i = 0; i < s->M; ++i) y[i] = y[i] + tk[i];
    chunked_solve(s, y, scratch);
    for (int i = 0; i < s->M; ++i) y[i] = y[i] * s->inv;
  }
  memcpy(out, y, (size_t)s->M * sizeof(double));
  free(y);
  free(scratch);
}

void orc_thomas_propagate(int M, int steps, double band_lo, double band_diag, double band_up,
                          double dt, const double* in, const double* ds, const double* g,
                          double* out) {
  const double delta = band_diag * dt + 1.0, lam = band_lo * dt, mu = band_up * dt;
  double* cp = (double*)malloc((size_t)M * sizeof(double));
  double* iv = (double*)malloc((size_t)M * sizeof(double));
  double* y = (double*)malloc((size_t)M * sizeof(double));
  /* precomputed factors: d_i = delta - lam*c'_{i-1}; c'_i = mu/d_i */
  double dprev = delta;
  iv[0] = 1.0 / dprev;
  cp[0] = mu * iv[0];
  for (int i = 1; i < M; ++i) {
    double d = delta - lam * cp[i - 1];
    iv[i] = 1.0 / d;
    cp[i] = mu * iv[i];
  }
  memcpy(y, in, (size_t)M * sizeof(double));
  for (int k = 0; k < steps; ++k) {
    if (ds)
      for (int i = 0; i < M; ++i) y[i] = y[i] + ds[k] * g[i];
    else if (g) /* ds == NULL, g != NULL: g is a table [steps][M] of fl(dt*f) */
      for (int i = 0; i < M; ++i) y[i] = y[i] + g[(size_t)k * M + i];
    y[0] = y[0] * iv[0];
    for (int i = 1; i < M; ++i) y[i] = (y[i] - lam * y[i - 1]) * iv[i];
    for (int i = M - 2; i >= 0; --i) y[i] = y[i] - cp[i] * y[i + 1];
  }
  memcpy(out, y, (size_t)M * sizeof(double));
  free(cp);
  free(iv);
  free(y);
}

/* ------------------------------------------------------------------------ */
/* Block-vector algebra                                                      */
/* ------------------------------------------------------------------------ */

#define ORC_DOT_THREADS 256

/* inner_product of one block (grid.cpp:107-116) in the selected order */
double orc_block_partial(const orc_problem* p, const double* a, const double* b) {
  const int M = p->M;
  if (p->mode == ORC_MODE_REFERENCE) {
    double sum = 0.0;
    for (int i = 0; i < M; ++i) sum += a[i] * b[i];
    return p->weight * sum;
  }
  /* device order: pit_vec.cu block_dot — thread t accumulates i = t + 256j with
   * fma, warp butterfly over shfl_xor 16..1, warp totals summed in order. */
  double acc[ORC_DOT_THREADS];
  for (int t = 0; t < ORC_DOT_THREADS; ++t) {
    double v = 0.0;
    for (int i = t; i < M; i += ORC_DOT_THREADS) v = fma(a[i], b[i], v);
    acc[t] = v;
  }
  double wsum[ORC_DOT_THREADS / 32];
  for (int w = 0; w < ORC_DOT_THREADS / 32; ++w) {
    double v[32], nv[32];
    memcpy(v, acc + 32 * w, sizeof v);
    for (int off = 16; off >= 1; off >>= 1) {
      for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ off];
      memcpy(v, nv, sizeof v);
    }
    wsum[w] = v[0];
  }
  double s = wsum[0];
  for (int w = 1; w < ORC_DOT_THREADS / 32; ++w) s = s + wsum[w];
  return p->weight * s;
}

double orc_block_dot(const orc_problem* p, const double* a, const double* b) {
  double sum = 0.0;
  for (int n = 0; n < p->N; ++n)
    sum += orc_block_partial(p, a + (size_t)n * p->M, b + (size_t)n * p->M);
  return sum;
}

double orc_block_norm(const orc_problem* p, const double* a) {
  double worst = 0.0;
  for (int n = 0; n < p->N; ++n) {
    const double* x = a + (size_t)n * p->M;
    double v = sqrt(orc_block_partial(p, x, x));
    worst = worst > v ? worst : v; /* std::max(worst, v) */
  }
  return worst;
}

static size_t nm(const orc_problem* p) { return (size_t)p->N * (size_t)p->M; }

/* y += a*x */
static void vaxpy(const orc_problem* p, double* y, double a, const double* x) {
  size_t n = nm(p);
  if (p->mode == ORC_MODE_REFERENCE)
    for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
  else
    for (size_t i = 0; i < n; ++i) y[i] = fma(a, x[i], y[i]);
}

/* ------------------------------------------------------------------------ */
/* Block operators (block_system.cpp:115-195)                                */
/* ------------------------------------------------------------------------ */

int orc_apply_F(const orc_problem* p, const double* L, double* out, orc_history* h) {
  const int M = p->M, N = p->N;
  memcpy(out, L, (size_t)M * sizeof(double));
  int rc = 0, bad = N;
  /* slabs are independent (block_system.cpp:123-132); the lowest failing
   * slab's code wins, as SlabExecutor reports it (executor.cpp:142-152) */
#pragma omp parallel for schedule(dynamic, 1) if (p->parallel)
  for (int n = 1; n < N; ++n) {
    double* o = out + (size_t)n * M;
    int r = p->prop(p->user, ORC_FINE, 0, L + (size_t)(n - 1) * M, n - 1, o);
    if (r) {
#pragma omp critical(orc_slab_error)
      if (n < bad) {
        bad = n;
        rc = r;
      }
      continue;
    }
    const double* Ln = L + (size_t)n * M;
    for (int i = 0; i < M; ++i) o[i] = Ln[i] - o[i];
  }
  if (rc) return rc;
  if (h) h->fine_applications += N - 1;
  return 0;
}

int orc_assemble_rhs(const orc_problem* p, double* rhs, orc_history* h) {
  const int M = p->M, N = p->N;
  memset(rhs, 0, nm(p) * sizeof(double));
  memcpy(rhs, p->y0, (size_t)M * sizeof(double));
  if (!p->has_source) return 0;
  double* zero = (double*)calloc((size_t)M, sizeof(double));
  int rc = 0, bad = N;
#pragma omp parallel for schedule(dynamic, 1) if (p->parallel)
  for (int n = 1; n < N; ++n) {
    int r = p->prop(p->user, ORC_FINE, 1, zero, n - 1, rhs + (size_t)n * M);
    if (r) {
#pragma omp critical(orc_slab_error)
      if (n < bad) {
        bad = n;
        rc = r;
      }
    }
  }
  free(zero);
  if (rc) return rc;
  if (h) h->fine_applications += N - 1;
  return 0;
}

int orc_apply_G_inverse(const orc_problem* p, const double* V, double* out, orc_history* h) {
  const int M = p->M, N = p->N;
  memcpy(out, V, (size_t)M * sizeof(double));
  for (int n = 1; n < N; ++n) {
    double* o = out + (size_t)n * M;
    int rc = p->prop(p->user, ORC_COARSE, 0, out + (size_t)(n - 1) * M, n - 1, o);
    if (rc) return rc;
    const double* v = V + (size_t)n * M;
    for (int i = 0; i < M; ++i) o[i] += v[i];
  }
  if (h) h->coarse_applications += N - 1;
  return 0;
}

int orc_initial_guess(const orc_problem* p, int zero, double* out, orc_history* h) {
  const int M = p->M, N = p->N;
  memset(out, 0, nm(p) * sizeof(double));
  if (zero) return 0;
  memcpy(out, p->y0, (size_t)M * sizeof(double));
  for (int n = 1; n < N; ++n) {
    int rc = p->prop(p->user, ORC_COARSE, 1, out + (size_t)(n - 1) * M, n - 1,
                     out + (size_t)n * M);
    if (rc) return rc;
  }
  if (h) h->coarse_applications += N - 1;
  return 0;
}

int orc_sequential_fine(const orc_problem* p, double* out) {
  const int M = p->M, N = p->N;
  memset(out, 0, nm(p) * sizeof(double));
  memcpy(out, p->y0, (size_t)M * sizeof(double));
  for (int n = 1; n < N; ++n) {
    int rc = p->prop(p->user, ORC_FINE, 1, out + (size_t)(n - 1) * M, n - 1,
                     out + (size_t)n * M);
    if (rc) return rc;
  }
  return 0;
}

/* r = rhs; r -= apply_F(lambda); r = G^-1 r   (solvers.cpp:66-71) */
int orc_preconditioned_residual(const orc_problem* p, const double* lambda, const double* rhs,
                                double* out, orc_history* h) {
  size_t n = nm(p);
  double* f = (double*)malloc(n * sizeof(double));
  int rc = orc_apply_F(p, lambda, f, h);
  if (!rc) {
    for (size_t i = 0; i < n; ++i) f[i] = rhs[i] - f[i];
    rc = orc_apply_G_inverse(p, f, out, h);
  }
  free(f);
  return rc;
}

static void record(orc_history* h, int k, double res) {
  if (h->count < h->max_records) {
    orc_record* r = &h->records[h->count];
    r->k = k;
    r->residual = res;
    r->fine_applications = h->fine_applications;
    r->coarse_applications = h->coarse_applications;
  }
  h->count++;
}

/* pitsbicg_solve (solvers.cpp:116-220), op for op. */
int orc_pitsbicg(const orc_problem* p, double tol, double eps0, int max_iter, int zero_guess,
                 const double* lambda_init, double* lambda, double* first_residual,
                 orc_history* h) {
  if (!(tol > eps0) || !(eps0 > 0.0) || max_iter < 1) return -100; /* ConfigError */
  const size_t n = nm(p);
  const size_t bytes = n * sizeof(double);
  int rc = 0;
  h->count = 0;
  h->restarts = 0;
  h->converged = 0;
  h->fine_applications = h->coarse_applications = 0;
  h->min_restart_margin = INFINITY;
  if (lambda_init)
    memcpy(lambda, lambda_init, bytes);
  else if ((rc = orc_initial_guess(p, zero_guess, lambda, h)))
    return rc;
  double* rhs = (double*)malloc(bytes);
  double* r = (double*)malloc(bytes);
  double* rs = (double*)malloc(bytes);
  double* pv = (double*)malloc(bytes);
  double* d = (double*)malloc(bytes);
  double* s = (double*)malloc(bytes);
  double* t = (double*)malloc(bytes);
  double* f = (double*)malloc(bytes);
  if ((rc = orc_assemble_rhs(p, rhs, h))) goto done;
  if ((rc = orc_preconditioned_residual(p, lambda, rhs, r, h))) goto done;
  if (first_residual) memcpy(first_residual, r, bytes);
  double r_norm = orc_block_norm(p, r);
  record(h, 0, r_norm);
  if (r_norm <= tol) {
    h->converged = 1;
    goto done;
  }
  memcpy(rs, r, bytes);
  memcpy(pv, r, bytes);
  for (int k = 1; k <= max_iter; ++k) {
    const double rho = orc_block_dot(p, r, rs);
    if ((rc = orc_apply_F(p, pv, f, h))) goto done;
    if ((rc = orc_apply_G_inverse(p, f, d, h))) goto done;
    const double d_dot = orc_block_dot(p, d, rs);
    if (fabs(d_dot) < 1e-300) {
      memcpy(rs, r, bytes);
      memcpy(pv, r, bytes);
      h->restarts++;
      record(h, k, r_norm);
      continue;
    }
    const double alpha = rho / d_dot;
    memcpy(s, r, bytes);
    vaxpy(p, s, -alpha, d);
    const double s_norm = orc_block_norm(p, s);
    if (s_norm <= tol) {
      vaxpy(p, lambda, alpha, pv);
      memcpy(r, s, bytes);
      record(h, k, s_norm);
      h->converged = 1;
      goto done;
    }
    if ((rc = orc_apply_F(p, s, f, h))) goto done;
    if ((rc = orc_apply_G_inverse(p, f, t, h))) goto done;
    const double tt = orc_block_dot(p, t, t);
    if (tt < 1e-300) {
      memcpy(rs, r, bytes);
      memcpy(pv, r, bytes);
      h->restarts++;
      record(h, k, r_norm);
      continue;
    }
    const double omega = orc_block_dot(p, t, s) / tt;
    if (fabs(omega) < 1e-300) {
      memcpy(rs, r, bytes);
      memcpy(pv, r, bytes);
      h->restarts++;
      record(h, k, r_norm);
      continue;
    }
    vaxpy(p, lambda, alpha, pv);
    vaxpy(p, lambda, omega, s);
    vaxpy(p, s, -omega, t);
    memcpy(r, s, bytes);
    r_norm = orc_block_norm(p, r);
    record(h, k, r_norm);
    if (r_norm <= tol) {
      h->converged = 1;
      goto done;
    }
    const double r_dot = orc_block_dot(p, r, rs);
    {
      double margin = fabs(r_dot) / eps0;
      if (margin < h->min_restart_margin) h->min_restart_margin = margin;
    }
    if (fabs(r_dot) <= eps0) {
      memcpy(rs, r, bytes);
      memcpy(pv, r, bytes);
      h->restarts++;
    } else {
      const double beta = (alpha / omega) * (r_dot / rho);
      if (p->mode == ORC_MODE_REFERENCE) {
        vaxpy(p, pv, -omega, d);
        for (size_t i = 0; i < n; ++i) pv[i] *= beta;
        for (size_t i = 0; i < n; ++i) pv[i] += r[i];
      } else {
        for (size_t i = 0; i < n; ++i) pv[i] = fma(fma(-omega, d[i], pv[i]), beta, r[i]);
      }
    }
  }
done:
  free(rhs);
  free(r);
  free(rs);
  free(pv);
  free(d);
  free(s);
  free(t);
  free(f);
  return rc;
}

/* parareal_solve (solvers.cpp:73-114), op for op. */
int orc_parareal(const orc_problem* p, double tol, double eps0, int max_iter, int zero_guess,
                 const double* lambda_init, double* lambda, double* first_residual,
                 orc_history* h) {
  if (!(tol > eps0) || !(eps0 > 0.0) || max_iter < 1) return -100;
  const size_t n = nm(p);
  const size_t bytes = n * sizeof(double);
  int rc = 0;
  h->count = 0;
  h->restarts = 0;
  h->converged = 0;
  h->fine_applications = h->coarse_applications = 0;
  if (lambda_init)
    memcpy(lambda, lambda_init, bytes);
  else if ((rc = orc_initial_guess(p, zero_guess, lambda, h)))
    return rc;
  double* rhs = (double*)malloc(bytes);
  double* corr = (double*)malloc(bytes);
  if ((rc = orc_assemble_rhs(p, rhs, h))) goto done;
  for (int k = 0;; ++k) {
    long fine_before = h->fine_applications, coarse_before = h->coarse_applications;
    if ((rc = orc_preconditioned_residual(p, lambda, rhs, corr, h))) goto done;
    if (k == 0 && first_residual) memcpy(first_residual, corr, bytes);
    double res = orc_block_norm(p, corr);
    long fa = h->fine_applications, ca = h->coarse_applications;
    h->fine_applications = fine_before;
    h->coarse_applications = coarse_before;
    record(h, k, res);
    h->fine_applications = fa;
    h->coarse_applications = ca;
    if (res <= tol) {
      h->converged = 1;
      break;
    }
    if (k == max_iter) break;
    if (p->mode == ORC_MODE_REFERENCE)
      for (size_t i = 0; i < n; ++i) lambda[i] += corr[i];
    else
      for (size_t i = 0; i < n; ++i) lambda[i] = lambda[i] + corr[i];
  }
done:
  free(rhs);
  free(corr);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Convenience 1D problem                                                    */
/* ------------------------------------------------------------------------ */

struct orc_1d {
  orc_problem prob;
  orc_stepper st[2];
  int use_thomas;
  double band[3];
  double dt[2];
  int steps[2];
  int N;
  double* y0;
  double* shape;
  double* ds[2]; /* [N][steps] */
  double* tab[2]; /* general source: [N][steps][M] fl(dt*f), or NULL */
};

static int orc_1d_prop(void* user, int role, int with_source, const double* in, int slab,
                       double* out) {
  orc_1d* o = (orc_1d*)user;
  const double* ds = NULL;
  if (with_source && o->prob.has_source && o->tab[role]) {
    const double* tab = o->tab[role] + (size_t)slab * o->steps[role] * o->prob.M;
    if (o->use_thomas)
      orc_thomas_propagate(o->prob.M, o->steps[role], o->band[0], o->band[1], o->band[2],
                           o->dt[role], in, NULL, tab, out);
    else
      orc_stepper_propagate_table(&o->st[role], in, tab, out);
    for (int i = 0; i < o->prob.M; ++i)
      if (!isfinite(out[i])) return -200 - slab;
    return 0;
  }
  if (with_source && o->prob.has_source) ds = o->ds[role] + (size_t)slab * o->steps[role];
  if (o->use_thomas)
    orc_thomas_propagate(o->prob.M, o->steps[role], o->band[0], o->band[1], o->band[2],
                         o->dt[role], in, ds, o->shape, out);
  else
    orc_stepper_propagate(&o->st[role], in, ds, o->shape, out);
  for (int i = 0; i < o->prob.M; ++i)
    if (!isfinite(out[i])) return -200 - slab; /* InnerSolveError analogue */
  return 0;
}

orc_1d* orc_1d_create(int M, double h, double band_lo, double band_diag, double band_up, int N,
                      double total_time, int fine_steps, int coarse_steps, int fine_m,
                      int fine_nsub, int fine_nseg, int fine_warps, int coarse_m,
                      int coarse_nsub, int coarse_nseg, int coarse_warps, const double* y0,
                      int has_source, const double* src_shape, double src_amp,
                      double src_omega, double src_phase, int use_thomas, int mode) {
  orc_1d* o = (orc_1d*)calloc(1, sizeof(orc_1d));
  o->use_thomas = use_thomas;
  o->band[0] = band_lo;
  o->band[1] = band_diag;
  o->band[2] = band_up;
  o->N = N;
  o->steps[0] = fine_steps;
  o->steps[1] = coarse_steps;
  const double slab = total_time / N; /* TimeSlabPartition::slab_length */
  o->dt[0] = slab / fine_steps;       /* Propagator::internal_dt */
  o->dt[1] = slab / coarse_steps;
  if (orc_stepper_init(&o->st[0], M, fine_m, fine_nsub, fine_nseg, fine_warps, fine_steps,
                       band_lo, band_diag, band_up, o->dt[0]) ||
      orc_stepper_init(&o->st[1], M, coarse_m, coarse_nsub, coarse_nseg, coarse_warps,
                       coarse_steps, band_lo, band_diag, band_up, o->dt[1])) {
    orc_1d_destroy(o);
    return NULL;
  }
  o->y0 = (double*)malloc((size_t)M * sizeof(double));
  memcpy(o->y0, y0, (size_t)M * sizeof(double));
  if (has_source) {
    o->shape = (double*)malloc((size_t)M * sizeof(double));
    memcpy(o->shape, src_shape, (size_t)M * sizeof(double));
    for (int r = 0; r < 2; ++r) {
      o->ds[r] = (double*)malloc((size_t)N * o->steps[r] * sizeof(double));
      for (int n = 0; n < N; ++n) {
        const double t0 = n * slab; /* breakpoint(n) = n * (T/N) */
        for (int k = 1; k <= o->steps[r]; ++k) {
          const double t = t0 + k * o->dt[r];
          const double sv = src_amp * sin(src_omega * t + src_phase);
          o->ds[r][(size_t)n * o->steps[r] + (k - 1)] = o->dt[r] * sv;
        }
      }
    }
  }
  o->prob.M = M;
  o->prob.N = N;
  o->prob.weight = h;
  o->prob.has_source = has_source;
  o->prob.mode = mode;
  o->prob.y0 = o->y0;
  o->prob.prop = orc_1d_prop;
  o->prob.user = o;
  o->prob.parallel = 1;
  return o;
}

/* General source tables f(t_k, x_i) of both roles ([N][steps][M], the layout
 * of pit_problem_desc::source_table_*): stored as fl(dt*f). */
int orc_1d_set_source_tables(orc_1d* o, const double* fine, const double* coarse) {
  const double* f[2] = {fine, coarse};
  for (int r = 0; r < 2; ++r) {
    const size_t n = (size_t)o->N * o->steps[r] * o->prob.M;
    free(o->tab[r]);
    o->tab[r] = (double*)malloc(n * sizeof(double));
    if (!o->tab[r]) return -1;
    for (size_t i = 0; i < n; ++i) o->tab[r][i] = o->dt[r] * f[r][i];
  }
  o->prob.has_source = 1;
  return 0;
}

void orc_1d_destroy(orc_1d* o) {
  if (!o) return;
  free(o->tab[0]);
  free(o->tab[1]);
  orc_stepper_free(&o->st[0]);
  orc_stepper_free(&o->st[1]);
  free(o->y0);
  free(o->shape);
  free(o->ds[0]);
  free(o->ds[1]);
  free(o);
}

const orc_problem* orc_1d_problem(orc_1d* o) { return &o->prob; }
const orc_stepper* orc_1d_stepper(orc_1d* o, int role) { return &o->st[role]; }
const double* orc_1d_ds(orc_1d* o, int role, int slab) {
  return o->ds[role] ? o->ds[role] + (size_t)slab * o->steps[role] : NULL;
}

/* Heap-allocated problem for FFI callers (ctypes). */
orc_problem* orc_problem_new(int M, int N, double weight, int has_source, int mode,
                             const double* y0, orc_prop_fn prop, void* user) {
  orc_problem* p = (orc_problem*)calloc(1, sizeof(orc_problem));
  double* y = (double*)malloc((size_t)M * sizeof(double));
  memcpy(y, y0, (size_t)M * sizeof(double));
  p->M = M;
  p->N = N;
  p->weight = weight;
  p->has_source = has_source;
  p->mode = mode;
  p->y0 = y;
  p->prop = prop;
  p->user = user;
  return p;
}

void orc_problem_delete(orc_problem* p) {
  if (!p) return;
  free((void*)p->y0);
  free(p);
}

/* Elementwise BiCGStab phases in the device op order (pit_kernels.cu K3),
 * for drivers that split block vectors across ranks (tests only). */
void orc_vec_update_s(long n, double alpha, const double* r, const double* d, double* s) {
  const double na = -alpha;
  for (long i = 0; i < n; ++i) s[i] = fma(na, d[i], r[i]);
}
void orc_vec_update_lr(long n, double alpha, double omega, const double* p, const double* s,
                       const double* t, double* lam, double* r) {
  const double nw = -omega;
  for (long i = 0; i < n; ++i) {
    double l = fma(alpha, p[i], lam[i]);
    lam[i] = fma(omega, s[i], l);
    r[i] = fma(nw, t[i], s[i]);
  }
}
void orc_vec_update_p(long n, double omega, double beta, const double* d, const double* r,
                      double* p) {
  const double nw = -omega;
  for (long i = 0; i < n; ++i) p[i] = fma(fma(nw, d[i], p[i]), beta, r[i]);
}
void orc_vec_axpy(long n, double a, const double* x, double* y) {
  for (long i = 0; i < n; ++i) y[i] = fma(a, x[i], y[i]);
}

int orc_problem_propagate(const orc_problem* p, int role, int with_source, const double* in,
                          int slab, double* out) {
  return p->prop(p->user, role, with_source, in, slab, out);
}
