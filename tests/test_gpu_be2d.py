"""GPU: K6 (2D backward Euler on the reference's general 5-point operator,
the desk/paper presets) bit for bit against its CPU mirror
(oracle/pit_oracle2d_be.c), which tests/test_oracle2d_be.py pins to the
reference's own Propagator and pitsbicg_solve."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from helpers import OracleProblem
from paper_2203_10148_b200 import api, presets

pytestmark = pytest.mark.gpu


def same(a, b):
    return np.array_equal(a, b)


@pytest.mark.parametrize("case", presets.CASES)
def test_desk_operators_bitwise_vs_oracle(case):
    p = presets.build_problem(presets.make_preset(case, "desk"), 8)
    o = OracleProblem(p)
    rng = np.random.default_rng(3)
    L = rng.uniform(-1, 1, (p.N, p.M))
    with api.BlockOperatorContext(p) as ctx:
        assert same(api.apply_F(ctx, L), o.apply_F(L))
        assert same(api.apply_G_inverse(ctx, L), o.apply_G_inverse(L))
        assert same(api.assemble_rhs(ctx), o.assemble_rhs())
        assert same(api.initial_guess(ctx, api.InitialGuessPolicy.CoarseSweep), o.initial_guess())
        assert same(api.sequential_fine_solve(ctx), o.sequential_fine())
        rhs = o.assemble_rhs()
        assert same(api.preconditioned_residual(ctx, L, rhs), o.preconditioned_residual(L, rhs))
        assert ctx.coarse_iterations() == o.coarse_iterations()


@pytest.mark.parametrize("which", ["pitsbicg", "parareal"])
@pytest.mark.parametrize("case", presets.CASES)
def test_desk_solvers_bitwise_vs_oracle(case, which):
    p = presets.build_problem(presets.make_preset(case, "desk"), 8)
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        fn = api.pitsbicg_solve if which == "pitsbicg" else api.parareal_solve
        res = fn(ctx, api.SolverConfig(tolerance=1e-8))
    r = o.solve(1e-8, which=which)
    assert [(x.k, x.residual_norm, x.fine_applications, x.coarse_applications)
            for x in res.history.records] == r["rows"]
    assert res.history.restarts == r["restarts"]
    assert np.array_equal(res.solution, r["lam"])


@pytest.mark.parametrize("case", ["diffusion", "advection_diffusion_reaction"])
def test_paper_scale_apply_F_bitwise(case):
    # m = 49: five points per thread, 208 KB of shared memory per CTA
    p = presets.build_problem(presets.make_preset(case, "paper"), 4)
    p = dataclasses.replace(p, fine_steps=40, T=p.T * 40 / p.fine_steps)  # keep dt, fewer steps
    o = OracleProblem(p)
    L = np.random.default_rng(5).uniform(-1, 1, (p.N, p.M))
    with api.BlockOperatorContext(p) as ctx:
        assert same(api.apply_F(ctx, L), o.apply_F(L))
        assert same(api.apply_G_inverse(ctx, L), o.apply_G_inverse(L))


def test_inner_solve_cap_raises_reference_errors():
    p = presets.build_problem(presets.make_preset("advection_diffusion_reaction", "desk"), 4)
    L = np.random.default_rng(1).uniform(-1, 1, (p.N, p.M))
    with api.BlockOperatorContext(dataclasses.replace(p, fine_max_iterations=1)) as ctx:
        with pytest.raises(api.SlabError) as e:
            api.apply_F(ctx, L)
        assert e.value.slab_index == 0
    with api.BlockOperatorContext(dataclasses.replace(p, coarse_max_iterations=1)) as ctx:
        with pytest.raises(api.InnerSolveError):
            api.apply_G_inverse(ctx, L)
        # the context survives (executor.cpp:142-152 analogue)
        assert np.isfinite(api.apply_F(ctx, L)).all()


def test_desk_all_slab_counts_converge():
    # the preset's slab counts {4, ..., 64} through the device solver
    for n in presets.make_preset("diffusion").slab_counts:
        p = presets.build_problem(presets.make_preset("diffusion"), n)
        with api.BlockOperatorContext(p) as ctx:
            res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-8))
            seq = api.sequential_fine_solve(ctx)
        assert res.history.status == api.SolveStatus.Converged
        assert np.max(np.abs(res.solution - seq)) < 1e-6 * np.max(np.abs(seq))


@pytest.mark.parametrize("case,dim", [("diffusion", 2), ("diffusion_reaction", 2),
                                      ("advection_diffusion_reaction", 2), ("diffusion", 1),
                                      ("diffusion_reaction", 1)])
def test_pit_verify_presets_through_device_operators(case, dim):
    # `pit verify` (cli.cpp:58-89: grid 5 points/axis, 3 slabs, 20 trials,
    # 1e-10) on the device operators, and its inject-fault negative control
    from paper_2203_10148_b200 import verify

    p = verify.preset_problem(case, dim, 5, 3)
    with api.BlockOperatorContext(p) as ctx:
        rep = verify.run_oracle_checks(ctx, trials=20, tolerance=1e-10)
        bad = verify.run_oracle_checks(ctx, trials=1, tolerance=1e-10, inject_fault=True)
    assert rep.all_passed(), [(c.name, c.worst_relative_error) for c in rep.checks]
    assert not any(c.passed for c in bad.checks)
    assert verify.main(["--case", case, "--dim", str(dim)]) == 0


def test_pit_verify_rejects_rotation_in_1d():
    from paper_2203_10148_b200 import verify

    assert verify.main(["--case", "advection_diffusion_reaction", "--dim", "1"]) == 2


@pytest.mark.parametrize("m", [1, 3, 22, 23, 39, 45, 50, 51, 64, 75, 88, 99, 101])
@pytest.mark.parametrize("nonsym", [False, True])
def test_k6_all_thread_layouts_bitwise(m, nonsym):
    # every points-per-thread instantiation (1..5; stencil rows in registers
    # up to 3, in shared memory beyond; 8, 12, 16, 20 for grids above 50
    # points per axis: stencil rows from global memory, vectors in local
    # memory, x and s^ sharing an operand buffer) on a random 5-point operator (the
    # rotation preset's structure: diagonally dominant, upwind-like
    # off-diagonals), fine batch and coarse sweep against the oracle
    rng = np.random.default_rng(m * 7 + nonsym)
    st = presets.stencil_2d(m, -0.5, 0.5, 0.2, 0.5, nonsym)
    if nonsym:  # symmetric operators keep CG's assumptions
        st[[0, 1, 3, 4]] *= rng.uniform(0.8, 1.2, (4, m * m))
    p = api.Problem2DImplicit(m=m, stencil=st, nonsymmetric=nonsym, N=3, T=0.03, fine_steps=3,
                              coarse_steps=1, y0=rng.uniform(-1, 1, m * m))
    o = OracleProblem(p)
    L = rng.uniform(-1, 1, (p.N, p.M))
    with api.BlockOperatorContext(p) as ctx:
        assert same(api.apply_F(ctx, L), o.apply_F(L))
        assert same(api.apply_G_inverse(ctx, L), o.apply_G_inverse(L))
        assert ctx.coarse_iterations() == o.coarse_iterations()


@pytest.mark.parametrize("case", presets.CASES)
def test_device_matches_reference_fixtures(case):
    # the reference's own outputs on its desk presets (committed fixtures, no
    # reference tree needed on the box): operators and PiTSBiCG
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "presets_desk_reference.npz"))

    def relmax(a, b):
        return np.max(np.linalg.norm(a - b, axis=1)) / np.max(np.linalg.norm(b, axis=1))

    p = presets.build_problem(presets.make_preset(case), 4)
    with api.BlockOperatorContext(p) as ctx:
        assert relmax(api.sequential_fine_solve(ctx), g[f"{case}_seq4"]) < 1e-10
        assert relmax(api.apply_F(ctx, g[f"{case}_probe4"]), g[f"{case}_F4"]) < 1e-10
        assert relmax(api.apply_G_inverse(ctx, g[f"{case}_probe4"]), g[f"{case}_G4"]) < 1e-10
        r4 = api.pitsbicg_solve(ctx, api.SolverConfig())
    assert relmax(r4.solution, g[f"{case}_lam4"]) < 1e-9
    q = presets.build_problem(presets.make_preset(case), 8)
    with api.BlockOperatorContext(q) as ctx:
        r8 = api.pitsbicg_solve(ctx, api.SolverConfig())
    for r, key in ((r4, "4"), (r8, "8")):
        rows = g[f"{case}_rows{key}"]
        assert [(x.k, x.fine_applications, x.coarse_applications) for x in r.history.records] == \
            [(int(a), int(b), int(c)) for a, b, c in rows[:, [0, 2, 3]]]
        assert np.allclose([x.residual_norm for x in r.history.records], rows[:, 1], rtol=1e-6,
                           atol=1e-13)
        assert r.history.restarts == int(g[f"{case}_restarts{key}"])


def test_grid_points_101_preset_runs_on_the_device():
    """The reference accepts any grid_points (presets.cpp:36, config.cpp:98-99);
    grid_points = 101 (m = 99) solves on the device and matches the oracle."""
    pre = presets.make_preset("advection_diffusion_reaction", "desk")
    pre.grid_points = 101
    p = presets.build_problem(pre, 4)
    o = OracleProblem(p)
    with api.BlockOperatorContext(p) as ctx:
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-8))
    r = o.solve(1e-8)
    assert res.history.records[-1].residual_norm <= 1e-8
    assert [(x.k, x.residual_norm) for x in res.history.records] == [(a[0], a[1]) for a in r["rows"]]
    assert np.array_equal(res.solution, r["lam"])
    with pytest.raises(ValueError):
        pre.grid_points = 104  # m = 102: beyond the compiled point counts
        api.BlockOperatorContext(presets.build_problem(pre, 4))
