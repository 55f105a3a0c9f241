"""General 1D operators (any tridiagonal SpatialOperator, include/pit/pde.hpp:36-37;
variable coefficients): the oracle's restatement against the reference built
over the same CSR (CPU), and the device path (K6 on a one-row grid) against the
oracle bit for bit (GPU)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_lib as O
from helpers import OracleProblem
from paper_2203_10148_b200 import api


def variable_operator(M, advection=0.0, reaction=0.5):
    """-(mu(x) u')' + a(x) u' + r u, mu = 1 + 0.5 sin(2 pi x), a = advection (1 + x),
    conservative second differences + central first differences on (0, 1)."""
    h = 1.0 / (M + 1)
    x = np.array([(k + 1) * h for k in range(M)])
    mu_m = 1.0 + 0.5 * np.sin(2 * math.pi * (x - h / 2))
    mu_p = 1.0 + 0.5 * np.sin(2 * math.pi * (x + h / 2))
    a = advection * (1.0 + x)
    sub = -mu_m / (h * h) - a / (2 * h)
    sup = -mu_p / (h * h) + a / (2 * h)
    diag = (mu_m + mu_p) / (h * h) + reaction
    sub[0] = 0.0
    sup[-1] = 0.0
    return np.ascontiguousarray(np.stack([sub, diag, sup])), x


def make(M, N, nonsym, fine_steps=20):
    st, x = variable_operator(M, advection=30.0 if nonsym else 0.0)
    y0 = np.sin(math.pi * x) + 0.3 * np.sin(5 * math.pi * x)
    # step sizes that keep I + dt*A well inside what Jacobi-PCG reaches at
    # 1e-12 (the reference's inner solver stalls on stiffer steps, as on c2)
    h = 1.0 / (M + 1)
    T = min(0.05 * N / 8, N * fine_steps * 4.0 * h * h)
    return api.Problem1DGeneral(M=M, stencil=st, nonsymmetric=nonsym, N=N, T=T,
                                fine_steps=fine_steps, coarse_steps=1, y0=y0)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("nonsym", [False, True])
def test_general_operator_matches_reference(nonsym):
    R = O.ref()
    p = make(120, 8, nonsym)
    st = np.ascontiguousarray(p.stencil)
    y0 = np.ascontiguousarray(p.y0)
    hr = R.pitref_create_1d_csr(p.M, 0.0, 1.0, O.ptr(st[0]), O.ptr(st[1]), O.ptr(st[2]),
                                0 if nonsym else 1, p.N, p.T, p.fine_steps, p.coarse_steps,
                                O.ptr(y0), 0)
    assert hr, R.pitref_last_error()
    o = OracleProblem(p)
    # one fine slab and the coarse sweep: both sides iterate to 1e-12
    rng = np.random.default_rng(3)
    v = np.ascontiguousarray(rng.uniform(-1, 1, p.M))
    ref = np.zeros(p.M)
    assert R.pitref_propagate(hr, 0, 0, O.ptr(v), 2, O.ptr(ref)) == 0
    L = np.zeros((p.N, p.M))
    L[1] = v
    mine = L[2] - o.apply_F(L)[2]
    assert np.abs(mine - ref).max() <= 2e-10 * np.abs(ref).max()
    r = o.solve(1e-9)
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    ref_lam = np.zeros((p.N, p.M))
    assert R.pitref_pitsbicg(hr, 1e-9, 1e-12, 200, 0, 2, None, O.ptr(ref_lam), None, k, res, fa, ca,
                             cap, C.byref(nrec), C.byref(rs), C.byref(conv)) == 0
    R.pitref_destroy(hr)
    assert conv.value == 1 and r["rows"][-1][1] <= 1e-9
    assert abs(r["rows"][-1][0] - k[nrec.value - 1]) <= 1
    assert np.abs(r["lam"] - ref_lam).max() <= 1e-8 * np.abs(ref_lam).max()


@pytest.mark.gpu
@pytest.mark.parametrize("M", [7, 100, 333, 2500, 4096, 10240])
@pytest.mark.parametrize("nonsym", [False, True])
def test_general_operator_bitwise_vs_oracle(M, nonsym):
    p = make(M, 4, nonsym, fine_steps=3 if M > 1000 else 10)
    o = OracleProblem(p)
    rng = np.random.default_rng(M + nonsym)
    L = np.ascontiguousarray(rng.uniform(-1, 1, (p.N, p.M)))
    with api.BlockOperatorContext(p) as ctx:
        assert np.array_equal(api.apply_F(ctx, L), o.apply_F(L))
        assert np.array_equal(api.apply_G_inverse(ctx, L), o.apply_G_inverse(L))
        assert np.array_equal(api.sequential_fine_solve(ctx), o.sequential_fine())


@pytest.mark.gpu
def test_general_operator_pitsbicg_bitwise_vs_oracle():
    p = make(300, 8, True)
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-9))
    r = o.solve(1e-9)
    assert res.history.records[-1].residual_norm <= 1e-9
    assert [(x.k, x.residual_norm) for x in res.history.records] == [(a[0], a[1]) for a in r["rows"]]
    assert np.array_equal(res.solution, r["lam"])


@pytest.mark.gpu
def test_general_operator_limits():
    p = make(100, 4, False)
    p.M = 10241
    p.stencil = np.zeros((3, 10241))
    p.y0 = np.zeros(10241)
    with pytest.raises(ValueError):
        api.BlockOperatorContext(p)


def general_source(t, x):
    """oracle/ref_driver.cpp's non-separable test source."""
    return 2.0 * ((1.0 + t) * x * (1.0 - x) + math.sin(3.0 * t) * np.cos(2.0 * math.pi * x))


def with_source(p):
    p.source = api.TableSource.sample(general_source, p.M, p.N, p.T, p.fine_steps, p.coarse_steps,
                                      p.grid_lo, p.grid_hi)
    return p


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_general_operator_with_source_matches_reference():
    R = O.ref()
    p = with_source(make(120, 8, True))
    st = np.ascontiguousarray(p.stencil)
    y0 = np.ascontiguousarray(p.y0)
    hr = R.pitref_create_1d_csr(p.M, 0.0, 1.0, O.ptr(st[0]), O.ptr(st[1]), O.ptr(st[2]), 0, p.N, p.T,
                                p.fine_steps, p.coarse_steps, O.ptr(y0), 1)
    assert hr, R.pitref_last_error()
    o = OracleProblem(p)
    r = o.solve(1e-9)
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    ref_lam = np.zeros((p.N, p.M))
    assert R.pitref_pitsbicg(hr, 1e-9, 1e-12, 200, 0, 2, None, O.ptr(ref_lam), None, k, res, fa, ca,
                             cap, C.byref(nrec), C.byref(rs), C.byref(conv)) == 0
    R.pitref_destroy(hr)
    assert conv.value == 1 and r["rows"][-1][1] <= 1e-9
    assert np.abs(r["lam"] - ref_lam).max() <= 1e-8 * np.abs(ref_lam).max()
    homog = OracleProblem(make(120, 8, True)).solve(1e-9)["lam"]
    assert np.abs(homog - ref_lam).max() > 1e-4 * np.abs(ref_lam).max()  # the source matters


@pytest.mark.gpu
@pytest.mark.parametrize("M,nonsym", [(100, False), (333, True), (4096, True)])
def test_general_operator_with_source_bitwise_vs_oracle(M, nonsym):
    p = with_source(make(M, 4, nonsym, fine_steps=3 if M > 1000 else 10))
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        assert np.array_equal(api.assemble_rhs(ctx), o.assemble_rhs())
        assert np.array_equal(api.initial_guess(ctx, api.InitialGuessPolicy.CoarseSweep),
                              o.initial_guess())
        assert np.array_equal(api.sequential_fine_solve(ctx), o.sequential_fine())
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-9))
    r = o.solve(1e-9)
    assert [(x.k, x.residual_norm) for x in res.history.records] == [(a[0], a[1]) for a in r["rows"]]
    assert np.array_equal(res.solution, r["lam"])


@pytest.mark.gpu
def test_2d_preset_with_source_bitwise_vs_oracle():
    """The reference samples sources on 2D grids too (propagator.cpp:36-44);
    the presets have none, so a table over the desk rotation preset."""
    from paper_2203_10148_b200 import presets
    p = presets.build_problem(presets.make_preset("advection_diffusion_reaction", "desk"), 4)
    h = p.spacing
    xs = np.array([p.grid_lo + (k + 1) * h for k in range(p.m)])
    X, Y = np.meshgrid(xs, xs)  # flat index: x fastest

    def f(t, _):
        return ((1.0 + t) * np.exp(-8 * (X ** 2 + Y ** 2)) + np.sin(3 * t) * X * Y).reshape(-1)

    slab = p.T / p.N
    tabs = []
    for steps in (p.fine_steps, p.coarse_steps):
        tab = np.empty((p.N, steps, p.M))
        for n in range(p.N):
            for k in range(1, steps + 1):
                tab[n, k - 1] = f(n * slab + k * slab / steps, None)
        tabs.append(tab)
    p.source = api.TableSource(tabs[0], tabs[1])
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        assert np.array_equal(api.assemble_rhs(ctx), o.assemble_rhs())
        assert np.array_equal(api.sequential_fine_solve(ctx), o.sequential_fine())
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-8))
    r = o.solve(1e-8)
    assert np.array_equal(res.solution, r["lam"])


@pytest.mark.gpu
def test_pit_verify_on_a_general_operator():
    """run_oracle_checks (src/dense_oracle.cpp, `pit verify`) through the
    device operators of a variable-coefficient context, with the negative
    control."""
    from paper_2203_10148_b200 import verify
    p = make(40, 3, True)
    with api.BlockOperatorContext(p) as ctx:
        rep = verify.run_oracle_checks(ctx, trials=5, tolerance=1e-9)
        assert all(c.passed for c in rep.checks), [(c.name, c.worst_relative_error) for c in rep.checks]
        bad = verify.run_oracle_checks(ctx, trials=5, tolerance=1e-9, inject_fault=True)
        assert not all(c.passed for c in bad.checks)
