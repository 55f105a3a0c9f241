// coeffs.cpp — coefficient recipe of the chunked constant-factor BE step.
//
// The step matrix of the reference is I + dt*A, built exactly as
// ImplicitStepSolver does (src/pde.cpp:103-110: val *= dt, diagonal += 1).
// For constant tridiagonal bands (lam, delta, mu) it factors as
//     I + dt*A = Ttilde + sigma e0 e0^T,   Ttilde = (1/inv) (I - nl S)(I - nu S^T)
// with constant unit-bidiagonal factors (the converged LU of the Toeplitz
// matrix) and a rank-1 corner correction (Sherman-Morrison).  All derived
// quantities are evaluated in x87 long double from the double inputs and
// rounded once; inv is chosen so that the factored operator reproduces the
// row sum delta + lam + mu exactly, which pins the smooth modes that survive
// many steps.  Compiled with -ffp-contract=off.
#include "coeffs.h"

#include <cmath>
#include <cstring>

namespace pitb {

namespace {
struct L { int mpt, nsub, nseg, warps; };
// layouts compiled into pit_kernels.cu (keep in sync with PIT_LAYOUTS there)
const L kLayouts[] = {
    {4, 1, 1, 1},   {4, 1, 1, 2},   {4, 1, 1, 4},  {4, 1, 1, 8},  {4, 1, 1, 16}, {4, 1, 1, 32},
    {8, 1, 1, 4},   {8, 1, 1, 8},   {8, 1, 1, 16}, {8, 1, 1, 32}, {16, 1, 1, 4}, {16, 1, 1, 8},
    {16, 1, 1, 16}, {16, 1, 1, 32}, {32, 2, 1, 4}, {32, 2, 1, 8}, {32, 1, 2, 4}, {32, 2, 2, 4},
    {64, 2, 2, 1},  {64, 2, 2, 2},  {64, 2, 2, 4}, {64, 4, 1, 2}, {64, 1, 4, 2}, {64, 4, 1, 1},
    {64, 4, 1, 4},  {64, 1, 2, 2},  {32, 2, 2, 8}, {64, 2, 2, 8}, {16, 2, 1, 16}, {16, 2, 2, 8}, {64, 4, 1, 8},
    {16, 2, 1, 8},  {16, 4, 1, 8},  {32, 4, 1, 8}, {32, 2, 1, 8}, {32, 4, 1, 4}};
}  // namespace

bool layout_supported(int mpt, int nsub, int nseg, int warps) {
  for (const L& l : kLayouts)
    if (l.mpt == mpt && l.nsub == nsub && l.nseg == nseg && l.warps == warps) return true;
  return false;
}

Layout auto_layout(int M, int role) {
  // fine: 64 contiguous points per thread as 4 sub-chunks of 16 (four
  // interleaved chains, one warp scan per direction); coarse (one persistent
  // CTA, latency bound): 8 warps (16 at M = 8192), few points each.  Measured on B200,
  // profiles/README.md.
  static const L fine[] = {{4, 1, 1, 1},  {4, 1, 1, 2},  {4, 1, 1, 4},  {8, 1, 1, 4},
                           {64, 4, 1, 1}, {64, 4, 1, 2}, {64, 4, 1, 4}, {64, 4, 1, 8}};
  // (c2: 4 sub-chunks of 4 per thread, 1.84 -> 1.71 ms per G^-1; c4: 2 of
  // 8, 5.53 -> 5.35 ms; tools/coarse_layouts.py, profiles/r2k_coarse_layouts.txt)
  static const L coarse[] = {{4, 1, 1, 1},  {4, 1, 1, 2},   {4, 1, 1, 4},  {4, 1, 1, 8},
                             {8, 1, 1, 8},  {16, 4, 1, 8},  {16, 2, 1, 16}, {16, 1, 1, 32}};
  const L* list = role == PIT_FINE ? fine : coarse;
  for (int i = 0; i < 8; ++i)
    if (32 * list[i].warps * list[i].mpt >= M)
      return {list[i].mpt, list[i].nsub, list[i].nseg, list[i].warps};
  return {0, 0, 0, 0};
}

int build_step_coeffs(int M, int mpt, int nsub, int nseg, int warps, int steps, double band_lo,
                      double band_diag, double band_up, double dt, pit_step_coeffs* c,
                      std::vector<double>* zc, std::vector<double>* ppos,
                      std::vector<double>* qpos, std::vector<double>* zt) {
  typedef long double ld;
  std::memset(c, 0, sizeof(*c));
  if (M < 1 || mpt < 1 || mpt > 64 || nsub < 1 || nsub > 8 || nseg < 1 || mpt % (nsub * nseg) ||
      mpt / (nsub * nseg) > 32 || warps < 1 || steps < 1)
    return PIT_ERR_INVALID_ARGUMENT;
  if (32 * warps * mpt < M) return PIT_ERR_INVALID_ARGUMENT;
  if (!(dt > 0.0)) return PIT_ERR_INVALID_ARGUMENT;
  c->M = M;
  c->mpt = mpt;
  c->nsub = nsub;
  c->nseg = nseg;
  c->warps = warps;
  c->steps = steps;
  c->delta = band_diag * dt + 1.0;
  c->lam = band_lo * dt;
  c->mu = band_up * dt;
  const ld D = c->delta, Lm = c->lam, U = c->mu;
  const ld disc = D * D - 4.0L * Lm * U;
  if (!(disc > 0.0L)) return PIT_ERR_INVALID_ARGUMENT;  // not diagonally dominant enough
  const ld dst = (D + sqrtl(disc)) * 0.5L;
  c->nl = (double)(-Lm / dst);
  c->nu = (double)(-U / dst);
  const ld nl = c->nl, nu = c->nu;
  c->inv = (double)((1.0L - nl) * (1.0L - nu) / (D + Lm + U));
  c->dstar = (double)(1.0L / (ld)c->inv);

  std::vector<ld> z((size_t)M);
  z[0] = 1.0L;
  for (int i = 1; i < M; ++i) z[i] = nl * z[i - 1];
  for (int i = M - 2; i >= 0; --i) z[i] = z[i] + nu * z[i + 1];
  zc->assign((size_t)M, 0.0);
  for (int i = 0; i < M; ++i) (*zc)[(size_t)i] = (double)z[(size_t)i];
  {
    const ld invd = c->inv;
    const ld sigma = D - 1.0L / invd;
    const ld a = sigma * invd;
    c->gneg = (double)(-(a / (1.0L + a * z[0])));
    const ld thr = fabsl(z[0]) * 8.470329472543003e-22L;  // 2^-70
    int k0 = 1;
    for (int i = M - 1; i >= 1; --i) {
      if (fabsl(z[(size_t)i]) > thr) {
        k0 = i + 1;
        break;
      }
    }
    c->K0 = k0;
  }
  {
    // sub-chunk = sub points; thread chunk = ch = nsub*sub points (warp scan
    // multiplier nl^ch); segment = lseg = T*ch points.
    const int sub = mpt / (nsub * nseg), ch = nsub * sub, T = 32 * warps, lseg = T * ch;
    ld nlp[65], nup[65];
    nlp[0] = 1.0L;
    nup[0] = 1.0L;
    for (int k = 1; k <= 64; ++k) {
      nlp[k] = nlp[k - 1] * nl;
      nup[k] = nup[k - 1] * nu;
    }
    for (int j = 0; j < sub; ++j) c->nlpow[j] = (double)nlp[j];
    for (int u = 0; u < nsub; ++u) c->pw[u] = (double)nlp[u * sub];
    c->pS = (double)nlp[sub];
    c->qS = (double)nup[sub];
    ld pk = nlp[ch], qk = nup[ch];
    c->scan_f = 5;
    c->scan_b = 5;
    for (int k = 4; k >= 0; --k) {  // smallest s with (nl^ch)^(2^s) <= 2^-70
      ld a = nlp[ch], b = nup[ch];
      for (int r = 0; r < k; ++r) a = a * a, b = b * b;
      if (fabsl(a) <= 8.470329472543003e-22L) c->scan_f = k;
      if (fabsl(b) <= 8.470329472543003e-22L) c->scan_b = k;
    }
    for (int k = 0; k < 5; ++k) {
      c->pp[k] = (double)pk;
      c->qq[k] = (double)qk;
      pk = pk * pk;
      qk = qk * qk;
    }
    c->p32 = (double)pk;
    c->q32 = (double)qk;
    ld pl = 1.0L, ql = 1.0L;
    for (int l = 0; l < 32; ++l) {
      c->plane[l] = (double)pl;
      c->qlane[31 - l] = (double)ql;
      pl = pl * nlp[ch];
      ql = ql * nup[ch];
    }
    ppos->assign((size_t)T, 0.0);
    qpos->assign((size_t)T, 0.0);
    zt->assign((size_t)T, 0.0);
    ld pt = 1.0L, qt = 1.0L;
    for (int t = 0; t < T; ++t) {
      (*ppos)[(size_t)t] = (double)pt;
      (*qpos)[(size_t)(T - 1 - t)] = (double)qt;
      (*zt)[(size_t)t] = (double)(z[0] * pt);
      pt = pt * nlp[ch];
      qt = qt * nup[ch];
    }
    c->Pseg = (double)pt;  // nl^(T*ch) = nl^lseg
    c->Qseg = (double)qt;
    // narrow corner: every point below K0 in warp 0's chunks of segment 0,
    // and zc geometric there to double precision ((nl nu)^(M-K0) negligible)
    const ld decay = powl(fabsl(nl * nu), (ld)(M - c->K0));
    c->narrow = (c->K0 <= 32 * ch && decay < 7.7e-34L /* 2^-110 */) ? 1 : 0;
    (void)lseg;
  }
  {
    const double lg = std::log2(c->dstar);
    int R = steps;
    if (lg > 0.0) {
      const double r = std::floor(512.0 / lg);
      if (r < (double)steps) R = r < 1.0 ? 1 : (int)r;
    }
    c->R = R;
    const ld invd = c->inv;
    ld p = 1.0L;
    for (int k = 0; k < R; ++k) p = p * invd;
    c->invR = (double)p;
    const int last = steps % R;
    p = 1.0L;
    for (int k = 0; k < last; ++k) p = p * invd;
    c->invLast = (double)p;
  }
  return PIT_OK;
}

}  // namespace pitb
