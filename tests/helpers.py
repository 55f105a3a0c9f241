"""Shared test helpers: build CPU-oracle problems that mirror a product
Problem1D and its kernel layouts (TEST INFRASTRUCTURE)."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

import oracle_lib as O
from paper_2203_10148_b200 import api


class OracleProblem:
    """orc_1d / orc_2d wrapper: propagators mirror the CUDA kernels
    (use_thomas=False) or plain Thomas (True, 1D); block algebra in
    MODE_DEVICE or MODE_REFERENCE."""

    def __init__(self, p, mode=O.MODE_DEVICE, use_thomas=False, fine_layout=None,
                 coarse_layout=None):
        if isinstance(p, api.Problem2D):
            self._init_2d(p, mode)
            return
        if isinstance(p, api.Problem2DImplicit):
            self._init_be2d(p, mode)
            return
        if isinstance(p, api.Problem1DGeneral):
            self._init_be1d(p, mode)
            return
        self.dim = 1
        fc, _ = api.step_coefficients(p, 0, fine_layout, coarse_layout)
        cc, _ = api.step_coefficients(p, 1, fine_layout, coarse_layout)
        self.p = p
        self.lib = O.orc()
        src = p.source if isinstance(p.source, api.SeparableSource) else None
        self._keep = [np.ascontiguousarray(p.y0)]
        shape = None
        if src is not None:
            shape = np.ascontiguousarray(src.shape)
            self._keep.append(shape)
        self.o = self.lib.orc_1d_create(
            p.M, p.spacing, p.band_lo, p.band_diag, p.band_up, p.N, p.T, p.fine_steps,
            p.coarse_steps, fc.mpt, fc.nsub, fc.nseg, fc.warps, cc.mpt, cc.nsub, cc.nseg, cc.warps,
            O.ptr(self._keep[0]),
            1 if src else 0, O.ptr(shape) if src else None, src.amp if src else 0.0,
            src.omega if src else 0.0, src.phase if src else 0.0, 1 if use_thomas else 0, mode)
        assert self.o, "orc_1d_create failed"
        if isinstance(p.source, api.TableSource):
            tf = np.ascontiguousarray(p.source.fine, dtype=np.float64)
            tc = np.ascontiguousarray(p.source.coarse, dtype=np.float64)
            assert self.lib.orc_1d_set_source_tables(self.o, O.ptr(tf), O.ptr(tc)) == 0
        self.prob = self.lib.orc_1d_problem(self.o)

    def _init_2d(self, p, mode):
        self.dim = 2
        self.p = p
        self.lib = O.orc()
        self._keep = [np.ascontiguousarray(p.y0, dtype=np.float64).reshape(-1)]
        c = api.step_coefficients_2d(p)
        self.o = self.lib.orc_2d_create(p.m, p.band_off, p.band_diag, p.N, p.T, p.fine_steps,
                                        p.coarse_steps, c.rel_tol, c.cap, O.ptr(self._keep[0]),
                                        mode)
        assert self.o, "orc_2d_create failed"
        self.prob = self.lib.orc_2d_problem(self.o)
        self.coeffs = self.lib.orc_2d_coeffs(self.o).contents

    def _init_be2d(self, p, mode):
        self.dim = 3  # 2D backward Euler (K6 mirror)
        self.p = p
        self.lib = O.orc()
        st = np.ascontiguousarray(p.stencil, dtype=np.float64).reshape(-1)
        self._keep = [np.ascontiguousarray(p.y0, dtype=np.float64).reshape(-1), st]
        self.o = self.lib.orc_be2d_create(p.m, p.grid_lo, p.grid_hi, O.ptr(st),
                                          1 if p.nonsymmetric else 0, p.N, p.T, p.fine_steps,
                                          p.coarse_steps, p.fine_tolerance, p.fine_max_iterations,
                                          p.coarse_tolerance, p.coarse_max_iterations,
                                          O.ptr(self._keep[0]), mode)
        assert self.o, "orc_be2d_create failed"
        self._tables(p)
        self.prob = self.lib.orc_be2d_problem(self.o)

    def _tables(self, p):
        if isinstance(p.source, api.TableSource):
            tf = np.ascontiguousarray(p.source.fine, dtype=np.float64)
            tc = np.ascontiguousarray(p.source.coarse, dtype=np.float64)
            assert self.lib.orc_be2d_set_source_tables(self.o, O.ptr(tf), O.ptr(tc)) == 0

    def _init_be1d(self, p, mode):
        self.dim = 3  # the K6 mirror on a one-row grid
        self.p = p
        self.lib = O.orc()
        st3 = np.ascontiguousarray(p.stencil, dtype=np.float64).reshape(3, p.M)
        st = np.zeros((5, p.M))  # south, west, centre, east, north
        st[1, 1:], st[2], st[3, :-1] = st3[0, 1:], st3[1], st3[2, :-1]
        st = np.ascontiguousarray(st.reshape(-1))
        self._keep = [np.ascontiguousarray(p.y0, dtype=np.float64).reshape(-1), st]
        self.o = self.lib.orc_be2d_create_1d(p.M, p.grid_lo, p.grid_hi, O.ptr(st),
                                             1 if p.nonsymmetric else 0, p.N, p.T, p.fine_steps,
                                             p.coarse_steps, p.fine_tolerance,
                                             p.fine_max_iterations, p.coarse_tolerance,
                                             p.coarse_max_iterations, O.ptr(self._keep[0]), mode)
        assert self.o, "orc_be2d_create_1d failed"
        self._tables(p)
        self.prob = self.lib.orc_be2d_problem(self.o)

    def coarse_iterations(self):
        if self.dim == 3:
            return self.lib.orc_be2d_coarse_iterations(self.o)
        return self.lib.orc_2d_coarse_iterations(self.o) if self.dim == 2 else 0

    def close(self):
        if self.o:
            if self.dim == 3:
                self.lib.orc_be2d_destroy(self.o)
            elif self.dim == 2:
                self.lib.orc_2d_destroy(self.o)
            else:
                self.lib.orc_1d_destroy(self.o)
            self.o = None

    def __del__(self):
        self.close()

    def _z(self):
        return np.zeros((self.p.N, self.p.M))

    def apply_F(self, L):
        out = self._z()
        assert self.lib.orc_apply_F(self.prob, O.ptr(np.ascontiguousarray(L)), O.ptr(out), None) == 0
        return out

    def apply_G_inverse(self, V):
        out = self._z()
        assert self.lib.orc_apply_G_inverse(self.prob, O.ptr(np.ascontiguousarray(V)), O.ptr(out),
                                            None) == 0
        return out

    def assemble_rhs(self):
        out = self._z()
        assert self.lib.orc_assemble_rhs(self.prob, O.ptr(out), None) == 0
        return out

    def initial_guess(self, zero=False):
        out = self._z()
        assert self.lib.orc_initial_guess(self.prob, 1 if zero else 0, O.ptr(out), None) == 0
        return out

    def sequential_fine(self):
        out = self._z()
        assert self.lib.orc_sequential_fine(self.prob, O.ptr(out)) == 0
        return out

    def preconditioned_residual(self, lam, rhs):
        out = self._z()
        assert self.lib.orc_preconditioned_residual(
            self.prob, O.ptr(np.ascontiguousarray(lam)), O.ptr(np.ascontiguousarray(rhs)),
            O.ptr(out), None) == 0
        return out

    def propagate(self, role, x, slab, with_source=False):
        out = np.zeros(self.p.M)
        assert self.lib.orc_problem_propagate(self.prob, role, 1 if with_source else 0,
                                              O.ptr(np.ascontiguousarray(x)), slab, O.ptr(out)) == 0
        return out

    def block_dot(self, a, b):
        return self.lib.orc_block_dot(self.prob, O.ptr(np.ascontiguousarray(a)),
                                      O.ptr(np.ascontiguousarray(b)))

    def block_norm(self, a):
        return self.lib.orc_block_norm(self.prob, O.ptr(np.ascontiguousarray(a)))

    def solve(self, tol, which="pitsbicg", eps0=1e-12, max_iter=200, zero_guess=False, init=None):
        recs = (O.OrcRecord * (max_iter + 2))()
        h = O.OrcHistory()
        h.records, h.max_records = recs, max_iter + 2
        lam = self._z()
        first = self._z()
        fn = self.lib.orc_pitsbicg if which == "pitsbicg" else self.lib.orc_parareal
        rc = fn(self.prob, tol, eps0, max_iter, 1 if zero_guess else 0,
                O.ptr(np.ascontiguousarray(init)) if init is not None else None, O.ptr(lam),
                O.ptr(first), C.byref(h))
        assert rc == 0, rc
        rows = [(recs[i].k, recs[i].residual, recs[i].fine_applications,
                 recs[i].coarse_applications) for i in range(min(h.count, max_iter + 2))]
        return dict(lam=lam, first=first, rows=rows, restarts=h.restarts, converged=h.converged,
                    margin=h.min_restart_margin)


def rel_block(a, b):
    """worst per-block relative L2 difference."""
    worst = 0.0
    for n in range(b.shape[0]):
        nb = np.linalg.norm(b[n])
        worst = max(worst, np.linalg.norm(a[n] - b[n]) / (nb if nb > 0 else 1.0))
    return worst


def modal_heat_1d(p: api.Problem1D, coeffs: np.ndarray, slabs: int, reaction: float = 0.0):
    """Closed form of `slabs` fine slabs of BE steps on the sine modes
    sum_k coeffs[k] sin((k+1) pi x): the discrete sine modes are exact
    eigenvectors of the constant Dirichlet Laplacian."""
    h = p.spacing
    dt = (p.T / p.N) / p.fine_steps
    x = p.coords()
    out = np.zeros(p.M)
    for k, a in enumerate(coeffs):
        lam = 4.0 / h ** 2 * math.sin((k + 1) * math.pi * h / 2) ** 2 + reaction
        rho = 1.0 / (1.0 + dt * lam)
        out += a * rho ** (p.fine_steps * slabs) * np.sin((k + 1) * math.pi * x)
    return out
