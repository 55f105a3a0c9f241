"""CPU: the 2D backward-Euler oracle (K6 mirror, oracle/pit_oracle2d_be.c)
pinned to the reference's own desk/paper presets (oracle/_ref: build_context,
Propagator, pitsbicg_solve), and the preset builder (presets.py) pinned to
the reference's assembler and initial condition."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from helpers import OracleProblem
from paper_2203_10148_b200 import presets

CASES = list(enumerate(presets.CASES))


def _ref_solve(h, N, M, tol, which="pitsbicg"):
    R = O.ref()
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    lam = np.zeros((N, M))
    fn = R.pitref_pitsbicg if which == "pitsbicg" else R.pitref_parareal
    assert fn(h, tol, 1e-12, 200, 0, 4, None, O.ptr(lam), None, k, res, fa, ca, cap,
              C.byref(nrec), C.byref(rs), C.byref(conv)) == 0, R.pitref_last_error()
    rows = [(k[i], res[i], fa[i], ca[i]) for i in range(min(nrec.value, cap))]
    return dict(lam=lam, rows=rows, restarts=rs.value, converged=conv.value)


@pytest.mark.parametrize("scale", ["desk", "paper"])
@pytest.mark.parametrize("cid,case", CASES)
def test_stencil_matches_oracle_restatement(cid, case, scale):
    pr = presets.make_preset(case, scale)
    p = presets.build_problem(pr, 4)
    out = np.zeros(5 * p.M)
    O.orc().orc_be2_stencil(p.m, p.grid_lo, p.grid_hi, pr.mu, pr.r, 1 if pr.rotation else 0,
                            O.ptr(out))
    assert np.array_equal(out.reshape(5, -1), p.stencil)
    assert p.nonsymmetric == (case == "advection_diffusion_reaction")


def _ref_ctx(cid, scale, N):
    if not O.ref_available():
        pytest.skip("reference library not built (no /root/reference)")
    h = O.ref().pitref_create_preset(cid, 0 if scale == "desk" else 1, N)
    assert h, O.ref().pitref_last_error()
    return h


@pytest.mark.parametrize("cid,case", CASES)
def test_initial_value_and_fine_step_count_match_reference(cid, case):
    p = presets.build_problem(presets.make_preset(case), 16)
    h = _ref_ctx(cid, "desk", 16)
    y0 = np.zeros(p.M)
    O.ref().pitref_initial_value(h, O.ptr(y0))
    O.ref().pitref_destroy(h)
    assert np.array_equal(y0, p.y0)
    assert p.fine_steps == 100 and p.coarse_steps == 1


@pytest.mark.parametrize("cid,case", CASES)
def test_oracle_propagators_match_reference_propagator(cid, case):
    # one fine slab and one coarse step from y0: both sides solve every step
    # to a 1e-12 relative residual (different reduction orders), so they
    # agree to the inner-solve floor
    N = 16
    p = presets.build_problem(presets.make_preset(case), N)
    o = OracleProblem(p)
    h = _ref_ctx(cid, "desk", N)
    try:
        for role in (0, 1):
            ref = np.zeros(p.M)
            assert O.ref().pitref_propagate(h, role, 0, O.ptr(np.ascontiguousarray(p.y0)), 0,
                                            O.ptr(ref)) == 0
            got = o.propagate(role, p.y0, 0)
            rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert rel < 1e-10, (role, rel)
    finally:
        O.ref().pitref_destroy(h)


@pytest.mark.parametrize("cid,case", CASES)
def test_oracle_pitsbicg_matches_reference(cid, case):
    N = 8
    p = presets.build_problem(presets.make_preset(case), N)
    o = OracleProblem(p)
    r = o.solve(1e-8)
    h = _ref_ctx(cid, "desk", N)
    try:
        ref = _ref_solve(h, p.N, p.M, 1e-8)
    finally:
        O.ref().pitref_destroy(h)
    assert r["rows"][-1][0] == ref["rows"][-1][0]  # iteration count
    assert r["restarts"] == ref["restarts"]
    for a, b in zip(r["rows"], ref["rows"]):
        assert abs(a[1] - b[1]) <= 1e-6 * abs(b[1]) + 1e-13
    scale = np.max(np.abs(ref["lam"]))
    assert np.max(np.abs(r["lam"] - ref["lam"])) <= 1e-9 * scale


# ---- against the committed reference fixtures (tests/golden/make_golden_presets.py)

def _gold():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                "presets_desk_reference.npz"))


def _relmax(a, b):
    return np.max(np.linalg.norm(a - b, axis=1)) / np.max(np.linalg.norm(b, axis=1))


@pytest.mark.parametrize("case", presets.CASES)
def test_oracle_matches_reference_fixtures(case):
    g = _gold()
    p = presets.build_problem(presets.make_preset(case), 4)
    assert np.array_equal(p.y0, g[f"{case}_y0"])
    o = OracleProblem(p)
    assert _relmax(o.sequential_fine(), g[f"{case}_seq4"]) < 1e-10
    assert _relmax(o.apply_F(g[f"{case}_probe4"]), g[f"{case}_F4"]) < 1e-10
    assert _relmax(o.apply_G_inverse(g[f"{case}_probe4"]), g[f"{case}_G4"]) < 1e-10
    for n, key in ((4, "4"), (8, "8")):
        q = presets.build_problem(presets.make_preset(case), n)
        r = OracleProblem(q).solve(1e-8)
        rows = g[f"{case}_rows{key}"]
        assert [int(x[0]) for x in r["rows"]] == [int(x) for x in rows[:, 0]]
        assert [(x[2], x[3]) for x in r["rows"]] == [(int(a), int(b)) for a, b in rows[:, 2:4]]
        assert np.allclose([x[1] for x in r["rows"]], rows[:, 1], rtol=1e-6, atol=1e-13)
        assert r["restarts"] == int(g[f"{case}_restarts{key}"])
        if n == 4:
            assert _relmax(r["lam"], g[f"{case}_lam4"]) < 1e-9
