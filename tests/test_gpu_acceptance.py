"""GPU: the reference's acceptance gate (proj/tests/acceptance.cpp, criteria
1-8) criterion for criterion on the device path — the desk presets through
K6, the device PiTSBiCG / parareal drivers, the runner and `pit verify`."""
from __future__ import annotations

import io
import os

import numpy as np
import pytest

from paper_2203_10148_b200 import api, presets, runner, verify

pytestmark = pytest.mark.gpu


def small_problem(dim, points, n):
    """acceptance.cpp small_context: mu = 1 on [-0.5, 0.5]^dim, T = 0.1 N,
    10 fine / 1 coarse BE steps per slab, Gaussian y0 (sigma 0.1)."""
    m, lo, hi = points - 2, -0.5, 0.5
    if dim == 2:
        return api.Problem2DImplicit(
            m=m, stencil=presets.stencil_2d(m, lo, hi, 1.0, 0.0, False), nonsymmetric=False, N=n,
            T=0.1 * n, fine_steps=10, coarse_steps=1, y0=presets.gaussian_2d(m, lo, hi, 0.1),
            grid_lo=lo, grid_hi=hi)
    h = (hi - lo) / (m + 1)
    b = api.diffusion_reaction_bands(1.0, 0.0, h)
    x = np.array([lo + (k + 1) * h for k in range(m)])
    return api.Problem1D(M=m, band_lo=b[0], band_diag=b[1], band_up=b[2], N=n, T=0.1 * n,
                         fine_steps=10, coarse_steps=1, y0=np.exp(-x * x / 0.02), grid_lo=lo,
                         grid_hi=hi)


def norm(ctx, a):
    return api.block_norm_n_inf(ctx, a)


def desk(case, n):
    return api.BlockOperatorContext(presets.build_problem(presets.make_preset(case, "desk"), n))


def test_criterion1_operators_match_dense_system():
    for dim, points, n in ((1, 7, 3), (2, 5, 2)):
        with api.BlockOperatorContext(small_problem(dim, points, n)) as ctx:
            rep = verify.run_oracle_checks(ctx, trials=20, tolerance=1e-12)
        assert rep.all_passed(), [(c.name, c.worst_relative_error) for c in rep.checks]


def test_criterion2_sequential_trajectory_solves_continuity_system():
    for case in presets.CASES:
        with desk(case, 8) as ctx:
            exact = api.sequential_fine_solve(ctx)
            res = api.apply_F(ctx, exact) - api.assemble_rhs(ctx)
            assert norm(ctx, res) <= 1e-10


def test_criterion3_parareal_settles_blocks_in_order():
    with desk("diffusion", 8) as ctx:
        ref = api.sequential_fine_solve(ctx)
        full = api.parareal_solve(ctx, api.SolverConfig())
        k_final = full.history.records[-1].k
        assert full.history.status == api.SolveStatus.Converged and k_final <= 7
        h = ctx.spacing
        for k in range(k_final + 1):
            # the iterate row k describes: the initial guess, or parareal
            # stopped at max_iterations = k (it breaks before the update)
            if k == 0:
                it = api.initial_guess(ctx, api.InitialGuessPolicy.CoarseSweep)
            else:
                it = api.parareal_solve(ctx, api.SolverConfig(max_iterations=k)).solution
            for b in range(min(k, 7) + 1):
                assert np.sqrt(h * h * np.sum((it[b] - ref[b]) ** 2)) <= 1e-10, (k, b)


def test_criterion4_and_5_pitsbicg_converges_and_counters_follow_cost_model():
    for case in presets.CASES:
        for n in (4, 8, 16):
            with desk(case, n) as ctx:
                ref = api.sequential_fine_solve(ctx)
                bi = api.pitsbicg_solve(ctx, api.SolverConfig())
                pr = api.parareal_solve(ctx, api.SolverConfig())
                assert bi.history.status == api.SolveStatus.Converged
                assert bi.history.records[-1].residual_norm <= 1e-8
                assert norm(ctx, bi.solution - ref) <= 1e-7
            for row in pr.history.records:
                assert row.fine_applications == row.k * (n - 1)
            rows = bi.history.records
            for i, row in enumerate(rows):
                full, half = (2 * row.k + 1) * (n - 1), 2 * row.k * (n - 1)
                assert row.fine_applications == full or (i == len(rows) - 1 and
                                                         row.fine_applications == half)


def test_criterion6_pitsbicg_beats_parareal_on_rotation_case():
    with desk("advection_diffusion_reaction", 16) as ctx:
        pr = api.parareal_solve(ctx, api.SolverConfig())
        bi = api.pitsbicg_solve(ctx, api.SolverConfig())

    def first_below(h):
        return next(r for r in h.records if r.residual_norm <= 1e-8)

    assert first_below(bi.history).fine_applications < first_below(pr.history).fine_applications


def test_criterion7_runner_csv_deterministic(tmp_path):
    # the reference runs the sweep with 1 and 4 workers; the device path is
    # deterministic by construction (fixed reduction trees), so two runs
    # must agree byte for byte apart from the timing column
    outs = []
    for d in ("a", "b"):
        preset = presets.make_preset("diffusion_reaction")
        preset.slab_counts = [4, 8, 16]
        path = runner.run_experiment(runner.RunSpec(preset=preset, out_dir=str(tmp_path / d)),
                                     io.StringIO())
        with open(path) as f:
            outs.append([line.rsplit(",", 1)[0] for line in f])
    assert outs[0] == outs[1]


def test_criterion8_solvers_start_from_identical_first_residual():
    with desk("diffusion", 8) as ctx:
        a, b = ctx.zero_vector(), ctx.zero_vector()
        api.parareal_solve(ctx, api.SolverConfig(), options=api.SolveOptions(first_residual_out=a))
        api.pitsbicg_solve(ctx, api.SolverConfig(), options=api.SolveOptions(first_residual_out=b))
    assert np.array_equal(a, b)


# ---- the reference's doctest cases that pin this path ----------------------

def _identity_problems(n):
    """dy/dt = 0 (A = 0): 1D bands 0 and the 2D 5-point K6 path with a zero
    stencil (test_block_system.cpp:82-103, test_solvers.cpp:167-197)."""
    rng = np.random.default_rng(11)
    p1 = api.Problem1D(M=40, band_lo=0.0, band_diag=0.0, band_up=0.0, N=n, T=1.0, fine_steps=4,
                       coarse_steps=2, y0=rng.uniform(-1, 1, 40))
    m = 5
    p2 = api.Problem2DImplicit(m=m, stencil=np.zeros((5, m * m)), nonsymmetric=False, N=n, T=1.0,
                               fine_steps=4, coarse_steps=2, y0=rng.uniform(-1, 1, m * m))
    return p1, p2


def test_identity_dynamics_F_telescopes_and_G_inverse_accumulates():
    for p in _identity_problems(4):
        x = np.random.default_rng(200).uniform(-1, 1, (p.N, p.M))
        with api.BlockOperatorContext(p) as ctx:
            fx, gx = api.apply_F(ctx, x), api.apply_G_inverse(ctx, x)
        assert np.array_equal(fx[0], x[0])
        for n in range(1, p.N):
            assert np.array_equal(fx[n], x[n] - x[n - 1])
        acc = x[0].copy()
        assert np.array_equal(gx[0], acc)
        for n in range(1, p.N):
            acc = acc + x[n]
            assert np.array_equal(gx[n], acc)


def test_half_step_exit_on_identity_dynamics():
    n = 6
    for p in _identity_problems(n):
        with api.BlockOperatorContext(p) as ctx:
            res = api.pitsbicg_solve(ctx, api.SolverConfig(
                initial_guess=api.InitialGuessPolicy.Zero))
        rows = res.history.records
        assert res.history.status == api.SolveStatus.Converged and len(rows) == 2
        assert (rows[0].k, rows[0].fine_applications, rows[0].coarse_applications) == (0, n - 1, n - 1)
        assert rows[1].k == 1 and rows[1].residual_norm == 0.0
        assert rows[1].fine_applications == rows[1].coarse_applications == 2 * (n - 1)
        for b in range(n):
            assert np.array_equal(res.solution[b], p.y0)


def test_restart_engages_on_desk_diffusion():
    with desk("diffusion", 8) as ctx:
        res = api.pitsbicg_solve(ctx, api.SolverConfig())
    assert res.history.status == api.SolveStatus.Converged
    assert res.history.restarts >= 1 and res.history.records[-1].residual_norm <= 1e-8
