"""General sources (PIT_SOURCE_TABLE; pit::SourceFn, include/pit/pde.hpp:13):
the oracle's table path against its separable path and against the reference
built with a non-separable SourceFn (CPU), and the device path against the
oracle bit for bit (GPU)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_lib as O
from helpers import OracleProblem
from paper_2203_10148_b200 import api, configs


def general_source(t, x):
    """The non-separable test source of oracle/ref_driver.cpp (has_source == 2,
    amp 2, omega 3, phase 2 pi)."""
    return 2.0 * ((1.0 + t) * x * (1.0 - x) + math.sin(3.0 * t) * np.cos(2.0 * math.pi * x))


def with_table(p, f=general_source):
    src = api.TableSource.sample(f, p.M, p.N, p.T, p.fine_steps, p.coarse_steps, p.grid_lo, p.grid_hi)
    return api.Problem1D(M=p.M, band_lo=p.band_lo, band_diag=p.band_diag, band_up=p.band_up, N=p.N,
                         T=p.T, fine_steps=p.fine_steps, coarse_steps=p.coarse_steps, y0=p.y0,
                         grid_lo=p.grid_lo, grid_hi=p.grid_hi, source=src)


def test_table_of_a_separable_source_matches_the_separable_path():
    p = configs.make("c4", slabs=4, M=200)
    s = p.source
    q = with_table(p, lambda t, x: s.amp * math.sin(s.omega * t + s.phase) * np.asarray(s.shape))
    a, b = OracleProblem(p), OracleProblem(q)
    # fma(dt*s, g, y) against y + fl(dt*s*g): rounding-level agreement
    for u, v in ((a.assemble_rhs(), b.assemble_rhs()), (a.initial_guess(), b.initial_guess()),
                 (a.sequential_fine(), b.sequential_fine())):
        assert np.abs(u - v).max() <= 1e-13 * max(1.0, np.abs(u).max())


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_general_source_matches_reference_solve():
    """c1's operator and partition with the non-separable source, solved by
    the reference's own pitsbicg_solve and by the oracle on tables sampled
    from the reference's SourceFn."""
    R = O.ref()
    p = configs.make("c1")
    y0 = np.ascontiguousarray(p.y0)
    hr = R.pitref_create_1d(p.M, 0.0, 1.0, 1.0, 0.0, 0, 0.0, 0.0, 0.0, 1, p.N, p.T, p.fine_steps,
                            p.coarse_steps, O.ptr(y0), 2, None, 2.0, 3.0, 2.0 * math.pi)
    assert hr, R.pitref_last_error()
    slab = p.T / p.N
    tabs = []
    for steps in (p.fine_steps, p.coarse_steps):
        tab = np.zeros((p.N, steps, p.M))
        row = np.zeros(p.M)
        for n in range(p.N):
            for k in range(1, steps + 1):
                assert R.pitref_sample_source(hr, n * slab + k * (slab / steps), O.ptr(row)) == 0
                tab[n, k - 1] = row
        tabs.append(tab)
    # the Python sampler evaluates the same function at the same points
    mine = api.TableSource.sample(general_source, p.M, p.N, p.T, p.fine_steps, p.coarse_steps)
    assert np.abs(mine.fine - tabs[0]).max() < 1e-14 and np.abs(mine.coarse - tabs[1]).max() < 1e-14
    q = api.Problem1D(M=p.M, band_lo=p.band_lo, band_diag=p.band_diag, band_up=p.band_up, N=p.N,
                      T=p.T, fine_steps=p.fine_steps, coarse_steps=p.coarse_steps, y0=p.y0,
                      source=api.TableSource(tabs[0], tabs[1]))
    o = OracleProblem(q)
    r = o.solve(1e-10)
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    ref_lam = np.zeros((p.N, p.M))
    assert R.pitref_pitsbicg(hr, 1e-10, 1e-12, 200, 0, 2, None, O.ptr(ref_lam), None, k, res, fa,
                             ca, cap, C.byref(nrec), C.byref(rs), C.byref(conv)) == 0
    R.pitref_destroy(hr)
    assert conv.value == 1 and r["rows"][-1][1] <= 1e-10
    assert abs(r["rows"][-1][0] - k[nrec.value - 1]) <= 1  # iteration count +-1
    scale = np.abs(ref_lam).max()
    assert np.abs(r["lam"] - ref_lam).max() <= 1e-10 * scale
    # the source matters: the homogeneous solve differs at the 1e-2 level
    h = OracleProblem(p).solve(1e-10)["lam"]
    assert np.abs(h - ref_lam).max() > 1e-3 * scale


def same(a, b):
    return np.array_equal(a, b), float(np.abs(a - b).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name,slabs,M", [("c1", 16, 100), ("c2", 5, 4096), ("c4", 4, 8192),
                                          ("c3", 4, 333)])
def test_table_source_operators_bitwise_vs_oracle(name, slabs, M):
    base = configs.make(name, slabs=slabs, M=M)
    base.source = None
    if name != "c1":  # keep the tables small: fewer steps, the same per-step arithmetic
        base.fine_steps = 40
    p = with_table(base)
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        assert same(api.assemble_rhs(ctx), o.assemble_rhs())[0]
        assert same(api.initial_guess(ctx, api.InitialGuessPolicy.CoarseSweep), o.initial_guess())[0]
        assert same(api.sequential_fine_solve(ctx), o.sequential_fine())[0]
        lam = api.sequential_fine_solve(ctx)
        r = api.apply_F(ctx, lam) - api.assemble_rhs(ctx)
        assert np.abs(r).max() <= 1e-12 * max(1.0, np.abs(lam).max())  # the fixed point


@pytest.mark.gpu
def test_table_source_pitsbicg_bitwise_vs_oracle():
    p = with_table(configs.make("c1"))
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
    r = o.solve(1e-10)
    assert [(x.k, x.residual_norm) for x in res.history.records] == [(a[0], a[1]) for a in r["rows"]]
    assert np.array_equal(res.solution, r["lam"])


@pytest.mark.gpu
def test_table_source_needs_both_tables():
    p = with_table(configs.make("c1"))
    p.source.coarse = p.source.coarse[:, :, :-1]
    with pytest.raises(ValueError):
        api.BlockOperatorContext(p)
