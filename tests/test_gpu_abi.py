"""The C ABI's reference-facing extras on the GPU: the InnerSolveError
payload (include/pit/errors.hpp:15-21), SolveOptions::iterate_observer
(solvers.hpp:54), the executor's busy-time bookkeeping (RunStats::
fine_busy_ms, executor.cpp:124-128) and the device worker count."""
from __future__ import annotations

import math

import numpy as np
import pytest

from helpers import OracleProblem
from paper_2203_10148_b200 import _lib, api, configs, presets

pytestmark = pytest.mark.gpu


def test_inner_solve_error_payload_cap():
    # K5 (2D coarse CG) stopped by a 5-iteration cap: the reference's message
    # and payload ("did not converge (relative residual R after I iterations)")
    p = configs.make("c5", slabs=3, M=32)
    p.coarse_max_iterations = 5
    x = np.random.default_rng(0).normal(size=(p.N, p.M))
    with api.BlockOperatorContext(p) as ctx:
        with pytest.raises(api.InnerSolveError) as e:
            api.apply_G_inverse(ctx, x)
        assert e.value.iterations == 5
        assert e.value.achieved_relative_residual > 1e-12
        assert f"after 5 iterations" in str(e.value)
        assert "relative residual" in str(e.value)
        # the context survives and the next call is clean
        p.coarse_max_iterations = 0
    with api.BlockOperatorContext(p) as ctx:
        assert np.isfinite(api.apply_G_inverse(ctx, x)).all()


def test_inner_solve_error_payload_matches_reference_nan():
    # K6 (the reference's desk preset): a NaN right-hand side stops the
    # coarse CG at iteration 0 with a NaN residual, as pit::solve_cg does
    import oracle_lib as O

    q = presets.build_problem(presets.make_preset("diffusion"), 4)
    x = np.cos(0.1 * np.arange(q.N)[:, None] + 0.02 * np.arange(q.M)[None, :])
    x[1, 5] = np.nan
    with api.BlockOperatorContext(q) as ctx:
        with pytest.raises(api.InnerSolveError) as e:
            api.apply_G_inverse(ctx, x)
    assert e.value.iterations == 0 and math.isnan(e.value.achieved_relative_residual)
    assert "did not converge" in str(e.value)
    if O.ref_available():
        R = O.ref()
        h = R.pitref_create_preset(presets.CASES.index("diffusion"), 0, 4)
        out = np.zeros_like(x)
        assert R.pitref_apply_G_inverse(h, O.ptr(np.ascontiguousarray(x)), O.ptr(out)) != 0
        msg = R.pitref_last_error().decode()
        R.pitref_destroy(h)
        assert msg.replace("-nan", "nan") == str(e.value).replace("-nan", "nan")


def test_iterate_observer_rows_and_iterates():
    p = configs.make("c1")
    seen = []
    with api.BlockOperatorContext(p) as ctx:
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10),
                                 options=api.SolveOptions(
                                     iterate_observer=lambda r, lam: seen.append((r, lam))))
        guess = api.initial_guess(ctx, api.InitialGuessPolicy.CoarseSweep)
        # the observer is cleared after the solve
        api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
    assert len(seen) == len(res.history.records) == 6
    assert [r.k for r, _ in seen] == [r.k for r in res.history.records]
    assert np.array_equal(seen[0][1], guess)          # row 0 describes the initial guess
    assert np.array_equal(seen[-1][1], res.solution)  # the last row the solution
    o = OracleProblem(p)
    assert np.array_equal(res.solution, o.solve(1e-10)["lam"])


def test_run_stats_busy_time_and_worker_count():
    import ctypes as C

    p = configs.make("c2", slabs=200)
    L = np.tile(p.y0, (p.N, 1))
    with api.BlockOperatorContext(p) as ctx:
        st = api.RunStats()
        api.apply_F(ctx, L, stats=st)
        api.apply_F(ctx, L, stats=st)
        slots = C.c_int()
        api._check(_lib.lib().pit_context_slots(ctx.handle, C.byref(slots)))
    assert st.fine_applications == 2 * (p.N - 1)
    assert slots.value >= 148
    # busy time = the summed per-slab kernel times: below slots x wall time
    # (parallel_efficiency <= 1) and, per slab, the duration of one slab's
    # 1000 steps (~0.8 ms alone on an SM, a few ms when sharing one)
    assert 0.0 < st.fine_busy_ms <= slots.value * st.fine_parallel_ms
    assert 0.3 < st.fine_busy_ms / st.fine_applications < 5.0


def test_reference_rows_do_not_change_the_solve():
    # SolveOptions::reference adds error_vs_reference to every row; the
    # iterates and the history must be those of the plain solve
    for p in (configs.make("c1"), presets.build_problem(presets.make_preset("diffusion"), 8)):
        tol = 1e-10 if p.__class__.__name__ == "Problem1D" else 1e-8
        with api.BlockOperatorContext(p) as ctx:
            plain = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=tol))
            seq = api.sequential_fine_solve(ctx)
            withref = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=tol),
                                         options=api.SolveOptions(reference=seq))
        assert np.array_equal(plain.solution, withref.solution)
        assert [(r.k, r.residual_norm) for r in plain.history.records] == \
            [(r.k, r.residual_norm) for r in withref.history.records]
        assert all(r.error_vs_reference is not None for r in withref.history.records)


@pytest.mark.parametrize("env", [{"PIT_HOST_SCALARS": "1"},
                                 {"PIT_HOST_SCALARS": "0", "PIT_GF_OVERLAP": "1"},
                                 {"PIT_HOST_SCALARS": "1", "PIT_GF_OVERLAP": "1"},
                                 {"PIT_HOST_SCALARS": "0", "PIT_GF_OVERLAP": "0"}])
def test_solver_loop_variants_bitwise(env, tmp_path):
    # the host loop, the device-resident loop, each with and without K2
    # overlapped on K1: the oracle's bits every time (fresh processes: the
    # switches are read once per process)
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "lam.npz")
    code = ("import sys; sys.path.insert(0, '.'); import numpy as np; "
            "from paper_2203_10148_b200 import api, configs; r = {}\n"
            "for name, n in (('c2', 9), ('c4', 5), ('c1', 16)):\n"
            "    p = configs.make(name, slabs=n)\n"
            "    with api.BlockOperatorContext(p) as ctx:\n"
            "        s = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))\n"
            "    r[name] = s.solution; r[name + '_rows'] = np.array([(x.k, x.residual_norm, "
            "x.fine_applications, x.coarse_applications) for x in s.history.records])\n"
            f"np.savez({out!r}, **r)\n")
    res = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         timeout=300, env={**os.environ, **env})
    assert res.returncode == 0, res.stdout + res.stderr
    g = np.load(out)
    for name, n in (("c2", 9), ("c4", 5), ("c1", 16)):
        o = OracleProblem(configs.make(name, slabs=n)).solve(1e-10)
        assert np.array_equal(g[name], o["lam"]), (env, name)
        assert [tuple(r) for r in g[name + "_rows"].tolist()] == \
            [tuple(map(float, r)) for r in o["rows"]], (env, name)
