"""Config 5 (2D heat) oracle on CPU: coefficients shared bit for bit with the
product, the explicit propagator against closed-form sine modes, the CG
coarse step against a direct solve and against the reference's own 2D
backward-Euler propagator (solve_cg at 1e-12, oracle/_ref), and the solver
loop on 2D propagators."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

import oracle_lib as O
from helpers import OracleProblem, rel_block
from paper_2203_10148_b200 import api, configs


def coeffs(p):
    c = O.Orc2Coeffs()
    pc = api.step_coefficients_2d(p)
    O.orc().orc2_coefficients(p.m, p.band_off, p.band_diag, p.T, p.N, p.fine_steps,
                              p.coarse_steps, pc.rel_tol, pc.cap, C.byref(c))
    return c, pc


@pytest.mark.parametrize("m,slabs", [(256, None), (32, 4), (100, 3), (17, 5)])
def test_2d_coefficients_match_product_bitwise(m, slabs):
    p = configs.make("c5", slabs=slabs, M=m)
    c, pc = coeffs(p)
    for f in ("ac", "an", "scaled", "R", "kappa", "anR", "anLast", "D", "O", "minv", "rel_tol",
              "cap", "rows", "cluster", "threads"):
        assert getattr(c, f) == getattr(pc, f), f
    if m == 256:
        # dt = h^2/8 exactly representable ratios at the BASELINE size
        assert (pc.ac, pc.an, pc.D, pc.O) == (0.5, 0.125, 2049.0, -512.0)
        assert (pc.scaled, pc.kappa, pc.R) == (1, 4.0, 256)
        assert pc.rel_tol == configs.C5_COARSE_TOL and pc.cap == 10 * 256 * 256
        assert (pc.cluster, pc.rows, pc.threads) == (16, 16, 256)


def mode(m, j, k):
    h = 1.0 / (m + 1)
    x = np.array([(i + 1) * h for i in range(m)])
    return np.outer(np.sin(k * math.pi * x), np.sin(j * math.pi * x)).reshape(-1)


@pytest.mark.parametrize("m", [16, 31])
def test_explicit_propagator_closed_form_modes(m):
    p = configs.make("c5", slabs=3, M=m)
    h = p.spacing
    p.fine_steps = 300
    p.T = p.N * p.fine_steps * (h * h / 8.0)  # keep dt = h^2/8
    c, _ = coeffs(p)
    y0 = np.zeros(m * m)
    amps = {(1, 1): 1.0, (2, 3): 0.5, (m, m - 1): 0.25}
    for (j, k), a in amps.items():
        y0 += a * mode(m, j, k)
    out = np.zeros_like(y0)
    O.orc().orc2_explicit_propagate(C.byref(c), O.ptr(y0), O.ptr(out))
    exact = np.zeros_like(y0)
    for (j, k), a in amps.items():
        rho = c.ac + c.an * (2 * math.cos(j * math.pi * h) + 2 * math.cos(k * math.pi * h))
        exact += a * rho ** p.fine_steps * mode(m, j, k)
    assert np.linalg.norm(out - exact) / np.linalg.norm(exact) < 1e-13


def stencil_S(c, m, x):
    X = x.reshape(m, m)
    P = np.pad(X, 1)
    nb = (P[1:-1, :-2] + P[1:-1, 2:]) + (P[:-2, 1:-1] + P[2:, 1:-1])
    return (c.D * X + c.O * nb).reshape(-1)


@pytest.mark.parametrize("m", [16, 33, 64])
def test_cg_step_solves_backward_euler(m):
    p = configs.make("c5", slabs=4, M=m)
    c, _ = coeffs(p)
    rng = np.random.default_rng(3)
    b = rng.normal(size=m * m)
    x = np.zeros_like(b)
    it = C.c_longlong()
    assert O.orc().orc2_cg_solve(C.byref(c), O.ptr(b), O.ptr(x), C.byref(it)) == 1
    res = np.linalg.norm(b - stencil_S(c, m, x)) / np.linalg.norm(b)
    assert res <= c.rel_tol
    # dense direct solve of the same matrix
    n = m * m
    S = np.zeros((n, n))
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        S[:, i] = stencil_S(c, m, e)
    xd = np.linalg.solve(S, b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-11
    assert 0 < it.value < 10 * n


def test_cg_zero_rhs_and_cap_failure():
    p = configs.make("c5", slabs=3, M=16)
    c, _ = coeffs(p)
    b = np.zeros(256)
    x = np.ones(256)
    it = C.c_longlong()
    assert O.orc().orc2_cg_solve(C.byref(c), O.ptr(b), O.ptr(x), C.byref(it)) == 1
    assert not x.any() and it.value == 0
    c.cap = 3  # InnerSolveError analogue: cap hit before the tolerance
    b = np.random.default_rng(0).normal(size=256)
    assert O.orc().orc2_cg_solve(C.byref(c), O.ptr(b), O.ptr(x), C.byref(it)) == 0


@pytest.mark.skipif(not O.ref_available(), reason="reference not built (no /root/reference)")
@pytest.mark.parametrize("m", [12, 20])
def test_cg_coarse_step_matches_reference_propagator(m):
    # the reference's own 2D backward-Euler propagator (SpatialGrid 2D,
    # assemble_spatial_operator, ImplicitStepSolver -> solve_cg at 1e-12)
    p = configs.make("c5", slabs=4, M=m)
    p.coarse_tolerance = 1e-12
    c, _ = coeffs(p)
    R = O.ref()
    y0 = np.ascontiguousarray(p.y0)
    h = R.pitref_create_2d(m, 0.0, 1.0, 1.0, 0.0, p.N, p.T, p.fine_steps, p.coarse_steps,
                           O.ptr(y0))
    assert h, R.pitref_last_error()
    try:
        assert abs(R.pitref_spacing(h) - p.spacing) == 0.0
        rng = np.random.default_rng(8)
        for slab in range(2):
            b = np.ascontiguousarray(rng.uniform(-1, 1, m * m))
            ref = np.zeros_like(b)
            assert R.pitref_propagate(h, 1, 0, O.ptr(b), slab, O.ptr(ref)) == 0
            mine = np.zeros_like(b)
            it = C.c_longlong()
            assert O.orc().orc2_coarse_propagate(C.byref(c), O.ptr(b), O.ptr(mine),
                                                 C.byref(it)) == 1
            assert np.linalg.norm(mine - ref) / np.linalg.norm(ref) < 5e-12
    finally:
        R.pitref_destroy(h)


def test_2d_pitsbicg_converges_to_sequential_fine():
    p = configs.make("c5", slabs=6, M=12)
    p.fine_steps = 64
    p.T = p.N * p.fine_steps * (p.spacing ** 2 / 8.0)
    o = OracleProblem(p)
    seq = o.sequential_fine()
    r = o.solve(1e-10)
    assert r["converged"] == 1
    assert rel_block(r["lam"], seq) < 1e-8
    assert o.coarse_iterations() > 0


def test_c5_cg_tolerance_floor():
    # Why c5 runs CG to 1e-12 rather than BASELINE's 1e-13: the true
    # residual of the correctly rounded exact solution is already above 1e-13.
    from scipy.fft import dstn, idstn
    p = configs.make("c5")
    c = api.step_coefficients_2d(p)
    m, h = p.m, p.spacing
    j = np.arange(1, m + 1)
    lam = c.D + 2 * c.O * (np.cos(j * np.pi * h)[:, None] + np.cos(j * np.pi * h)[None, :])
    b = p.y0.reshape(m, m)
    x = idstn(dstn(b, type=1) / lam, type=1)
    P = np.pad(x, 1)
    nb = (P[1:-1, :-2] + P[1:-1, 2:]) + (P[:-2, 1:-1] + P[2:, 1:-1])
    r = b - (c.D * x + c.O * nb)
    floor = np.linalg.norm(r) / np.linalg.norm(b)
    assert configs.C5_BASELINE_COARSE_TOL < floor < configs.C5_COARSE_TOL
