"""CPU tests: the oracle pinned against the reference (golden fixtures made by
tests/golden/make_golden.py from the unmodified reference, the loop pin,
closed-form known answers) and against the product's coefficient recipe.
No GPU needed."""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle_lib as O
from helpers import OracleProblem, modal_heat_1d, rel_block
from paper_2203_10148_b200 import api, configs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


# ---------------------------------------------------------------------------
# coefficient recipe: oracle (C, independent) == product (C++) bit for bit
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
@pytest.mark.parametrize("role", [0, 1])
def test_coefficients_bitwise_equal_product(name, role):
    p = configs.make(name, slabs=4)
    c, zc = api.step_coefficients(p, role)
    steps = p.fine_steps if role == 0 else p.coarse_steps
    dt = (p.T / p.N) / steps
    st = O.OrcStepper()
    assert O.orc().orc_stepper_init(C.byref(st), p.M, c.mpt, c.nsub, c.nseg, c.warps, steps,
                                    p.band_lo, p.band_diag, p.band_up, dt) == 0
    try:
        for f in ("delta", "lam", "mu", "dstar", "nl", "nu", "inv", "gneg", "invR", "invLast",
                  "p32", "q32", "pS", "qS", "Pseg", "Qseg"):
            assert getattr(st, f) == getattr(c, f), f
        for f in ("K0", "R", "narrow", "scan_f", "scan_b"):
            assert getattr(st, f) == getattr(c, f), f
        for f in ("pp", "qq", "plane", "qlane"):
            assert list(getattr(st, f)) == list(getattr(c, f)), f
        sub = c.mpt // (c.nsub * c.nseg)
        assert list(st.nlpow)[:sub] == list(c.nlpow)[:sub]
        assert list(st.pw)[: c.nsub] == list(c.pw)[: c.nsub]
        assert np.array_equal(np.ctypeslib.as_array(st.zc, (p.M,)), zc)
        pp, qp, zt = api.step_positions(p, role)
        T = 32 * c.warps
        assert np.array_equal(np.ctypeslib.as_array(st.ppos, (T,)), pp)
        assert np.array_equal(np.ctypeslib.as_array(st.qpos, (T,)), qp)
        assert np.array_equal(np.ctypeslib.as_array(st.zt, (T,)), zt)
    finally:
        O.orc().orc_stepper_free(C.byref(st))


# ---------------------------------------------------------------------------
# closed-form known answers (independent of any solver)
# ---------------------------------------------------------------------------

def test_closed_form_c1_one_slab():
    p = configs.make("c1")
    o = OracleProblem(p)
    seq = o.sequential_fine()
    for n in (1, 5, 15):
        exact = modal_heat_1d(p, [1.0], n)
        assert np.linalg.norm(seq[n] - exact) / np.linalg.norm(exact) < 1e-13 * n


def test_closed_form_c1_reference_value():
    # closed-form lambda_15[50] = 9.8671673279661e-05
    p = configs.make("c1")
    exact = modal_heat_1d(p, [1.0], 15)
    assert abs(exact[50] - 9.8671673279661e-05) < 1e-17
    g = gold("c1_reference.npz")
    assert abs(g["sequential_fine"][15][50] - exact[50]) / exact[50] < 1e-12


def test_closed_form_c2_modes_two_slabs():
    p = configs.make("c2", slabs=3)
    a = api.seeded_normal(configs.SEED, 8)
    o = OracleProblem(p)
    seq = o.sequential_fine()
    for n in (1, 2):
        exact = modal_heat_1d(p, a, n)
        err = np.linalg.norm(seq[n] - exact) / np.linalg.norm(exact)
        # exact-solver rounding grows linearly with the sequential step count
        assert err < 2e-15 * p.fine_steps * n, err
    th = OracleProblem(p, use_thomas=True).sequential_fine()
    assert rel_block(seq, th) < 1e-12


def test_closed_form_c4_source_mode():
    # c4 with a smooth initial value: the source lives on mode 1 only, so the
    # per-mode recurrence c <- (c + dt s(t_end)) / (1 + dt(mu_1 + r)) is exact.
    p = configs.make("c4", slabs=3, M=512)
    x = p.coords()
    p.y0 = np.ascontiguousarray(np.sin(math.pi * x) + 0.5 * np.sin(3 * math.pi * x))
    o = OracleProblem(p)
    seq = o.sequential_fine()
    h = p.spacing
    dt = (p.T / p.N) / p.fine_steps
    mu1 = 4.0 / h ** 2 * math.sin(math.pi * h / 2) ** 2 + 5.0
    mu3 = 4.0 / h ** 2 * math.sin(3 * math.pi * h / 2) ** 2 + 5.0
    c1, c3 = 1.0, 0.5
    for n in range(1, 3):
        for k in range(1, p.fine_steps + 1):
            t = (n - 1) * (p.T / p.N) + k * dt
            c1 = (c1 + dt * math.sin(2 * math.pi * t)) / (1 + dt * mu1)
            c3 = c3 / (1 + dt * mu3)
        exact = c1 * np.sin(math.pi * x) + c3 * np.sin(3 * math.pi * x)
        assert np.linalg.norm(seq[n] - exact) / np.linalg.norm(exact) < 1e-12


# ---------------------------------------------------------------------------
# the oracle against the reference itself (golden fixtures)
# ---------------------------------------------------------------------------

def test_c1_operators_match_reference():
    g = gold("c1_reference.npz")
    p = configs.make("c1")
    assert np.array_equal(p.y0, g["y0"])
    o = OracleProblem(p)
    probe = g["probe"]
    assert rel_block(o.apply_F(probe), g["apply_F"]) < 1e-10
    assert rel_block(o.apply_G_inverse(probe), g["apply_G_inverse"]) < 1e-10
    assert rel_block(o.initial_guess(), g["initial_guess"]) < 1e-10
    assert rel_block(o.sequential_fine(), g["sequential_fine"]) < 1e-10


@pytest.mark.parametrize("mode", [O.MODE_DEVICE, O.MODE_REFERENCE])
def test_c1_pitsbicg_matches_reference(mode):
    g = gold("c1_reference.npz")
    p = configs.make("c1")
    r = OracleProblem(p, mode=mode).solve(1e-10)
    hist = g["pitsbicg_hist"]
    assert [row[0] for row in r["rows"]] == [int(k) for k in hist[:, 0]]
    assert r["restarts"] == int(g["pitsbicg_restarts"]) == 1
    for row, ref in zip(r["rows"], hist):
        assert abs(row[1] - ref[1]) <= 1e-6 * ref[1]
        assert row[2] == ref[2] and row[3] == ref[3]  # (2k+1)(N-1) cost model
    assert rel_block(r["lam"], g["pitsbicg_lambda"]) < 1e-10
    assert rel_block(r["first"], g["pitsbicg_first"]) < 1e-10


def test_c1_parareal_matches_reference():
    g = gold("c1_reference.npz")
    r = OracleProblem(configs.make("c1")).solve(1e-10, which="parareal")
    assert [row[0] for row in r["rows"]] == [int(k) for k in g["parareal_hist"][:, 0]]
    assert [row[2] for row in r["rows"]] == [int(v) for v in g["parareal_hist"][:, 2]]
    assert rel_block(r["lam"], g["parareal_lambda"]) < 1e-10


def test_c3_n16_pitsbicg_matches_reference():
    g = gold("c3_n16_reference.npz")
    p = configs.make("c3", slabs=16)
    r = OracleProblem(p).solve(1e-10)
    assert [row[0] for row in r["rows"]] == [int(k) for k in g["pitsbicg_hist"][:, 0]]
    assert r["restarts"] == int(g["pitsbicg_restarts"])
    # Floor: the reference's own inner-solve inexactness (Jacobi-BiCGStab to
    # 1e-12 per step, ~2e-11 drift per slab) — a direct solve
    # cannot get closer; plain Thomas lands on the same 2.0e-10.
    assert rel_block(r["lam"], g["pitsbicg_lambda"]) < 5e-10
    th = OracleProblem(p, use_thomas=True).solve(1e-10)
    assert rel_block(r["lam"], th["lam"]) < 1e-12


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_c2_c4_fine_propagation_matches_reference(name):
    g = gold(f"{name}_n4_reference.npz")
    p = configs.make(name, slabs=4)
    o = OracleProblem(p)
    L = np.ascontiguousarray(np.tile(p.y0, (p.N, 1)))
    # per-slab floor of the reference's PCG inner solves
    assert rel_block(o.apply_F(L)[1:], g["apply_F"][1:]) < 2e-10
    rhs = o.assemble_rhs()
    assert rel_block(rhs, g["assemble_rhs"]) < 2e-10


def test_c2_reference_coarse_sweep_raises_inner_solve_error():
    # The reference cannot run c2 end to end: coarse CG hits its 10n cap.
    g = gold("c2_n4_reference.npz")
    assert int(g["g_inverse_rc"]) == 2  # InnerSolveError
    assert "did not converge" in str(g["g_inverse_error"])


# ---------------------------------------------------------------------------
# the loop pin: restated loop + reference propagators == pit::pitsbicg_solve
# ---------------------------------------------------------------------------

@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("which", ["pitsbicg", "parareal"])
def test_loop_pin_bitwise(which):
    R = O.ref()
    lib = O.orc()
    p = configs.make("c1")
    y0 = np.ascontiguousarray(p.y0)
    hr = R.pitref_create_1d(p.M, 0.0, 1.0, 1.0, 0.0, 0, 0.0, 0.0, 0.0, 1, p.N, p.T, p.fine_steps,
                            p.coarse_steps, O.ptr(y0), 0, None, 0.0, 0.0, 0.0)
    assert hr
    cb = C.cast(R.pitref_prop_callback, C.c_void_p)
    prob = lib.orc_problem_new(p.M, p.N, R.pitref_spacing(hr), 0, O.MODE_REFERENCE, O.ptr(y0), cb,
                               hr)
    recs = (O.OrcRecord * 64)()
    h = O.OrcHistory()
    h.records, h.max_records = recs, 64
    lam = np.zeros((p.N, p.M))
    fn = lib.orc_pitsbicg if which == "pitsbicg" else lib.orc_parareal
    assert fn(prob, 1e-10, 1e-12, 200, 0, None, O.ptr(lam), None, C.byref(h)) == 0
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    ref_lam = np.zeros((p.N, p.M))
    rfn = R.pitref_pitsbicg if which == "pitsbicg" else R.pitref_parareal
    assert rfn(hr, 1e-10, 1e-12, 200, 0, 2, None, O.ptr(ref_lam), None, k, res, fa, ca, cap,
               C.byref(nrec), C.byref(rs), C.byref(conv)) == 0
    assert h.count == nrec.value
    assert [recs[i].residual for i in range(h.count)] == [res[i] for i in range(nrec.value)]
    assert [recs[i].fine_applications for i in range(h.count)] == [fa[i] for i in range(nrec.value)]
    assert h.restarts == rs.value
    assert np.array_equal(lam, ref_lam)
    lib.orc_problem_delete(prob)
    R.pitref_destroy(hr)


# ---------------------------------------------------------------------------
# algorithm cross-checks
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("layout", [(8, 1, 1, 16), (16, 1, 1, 8), (4, 1, 1, 32), (32, 2, 1, 4),
                                    (64, 2, 2, 2), (64, 4, 1, 2), (64, 1, 4, 2), (64, 1, 2, 2),
                                    (32, 2, 2, 4), (16, 2, 2, 8)])
def test_chunked_stepper_layout_independent_to_rounding(layout):
    p = configs.make("c2", slabs=2)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, p.M)
    c, _ = api.step_coefficients(p, 0, fine_layout=layout)
    dt = (p.T / p.N) / p.fine_steps
    st = O.OrcStepper()
    lib = O.orc()
    assert lib.orc_stepper_init(C.byref(st), p.M, c.mpt, c.nsub, c.nseg, c.warps, 50, p.band_lo,
                                p.band_diag, p.band_up, dt) == 0
    out = np.zeros(p.M)
    lib.orc_stepper_propagate(C.byref(st), O.ptr(x), None, None, O.ptr(out))
    th = np.zeros(p.M)
    lib.orc_thomas_propagate(p.M, 50, p.band_lo, p.band_diag, p.band_up, dt, O.ptr(x), None, None,
                             O.ptr(th))
    assert np.linalg.norm(out - th) / np.linalg.norm(th) < 1e-13
    lib.orc_stepper_free(C.byref(st))


def test_device_mode_dot_is_fixed_tree():
    p = configs.make("c1")
    o = OracleProblem(p)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((p.N, p.M))
    b = rng.standard_normal((p.N, p.M))
    ref = float(np.sum(p.spacing * np.sum(a * b, axis=1)))
    assert abs(o.block_dot(a, b) - ref) < 1e-12 * abs(ref) + 1e-14
    assert o.block_norm(a) == pytest.approx(max(np.sqrt(p.spacing * np.sum(a * a, axis=1))),
                                            rel=1e-14)


def test_c3_full_size_pitsbicg_matches_reference():
    # the full BASELINE c3 (N = 512) against the reference binary's own solve
    # (tests/golden/c3_full_reference.npz, make_golden_c3_full.py): same k,
    # restarts and counters; lambda within the reference's inner-solve floor
    # (its BiCGStab steps stop at 1e-12; 6.7e-10 at full N)
    g = gold("c3_full_reference.npz")
    p = configs.make("c3")
    o = OracleProblem(p)
    r = o.solve(1e-10)
    lam_n = o.propagate(0, r["lam"][-1], p.N - 1, True)
    o.close()
    hist = g["pitsbicg_hist"]
    assert [row[0] for row in r["rows"]] == [int(k) for k in hist[:, 0]] == [0, 1, 2, 3]
    assert [(row[2], row[3]) for row in r["rows"]] == [(int(a), int(b)) for a, b in hist[:, 2:4]]
    assert r["restarts"] == int(g["pitsbicg_restarts"]) == 0
    assert abs(r["rows"][-1][1] - hist[-1, 1]) < 1e-4 * hist[-1, 1]
    assert rel_block(r["lam"][g["blocks"]], g["lambda_blocks"]) < 7e-10
    norms = np.linalg.norm(r["lam"], axis=1)
    assert np.max(np.abs(norms - g["lambda_block_norms"]) / g["lambda_block_norms"]) < 7e-10
    # lambda_N adds one more fine slab of the reference's drift (7.01e-10)
    assert np.linalg.norm(lam_n - g["lambda_N"]) / np.linalg.norm(g["lambda_N"]) < 7.5e-10
