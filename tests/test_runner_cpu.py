"""CPU: the runner's output format (runner.cpp:17-55, 90-106) and argument
handling, without a device."""
from __future__ import annotations

import io

import pytest

from paper_2203_10148_b200 import api, presets, runner


def _hist():
    h = api.ConvergenceHistory()
    h.records = [api.IterationRecord(0, 0.5, 3, 6, 1.25, 0.125),
                 api.IterationRecord(1, 1.0 / 3.0, 9, 12, 2.5, None)]
    h.status = api.SolveStatus.Converged
    h.restarts = 1
    h.stats.fine_applications, h.stats.coarse_applications = 9, 12
    return h


def test_csv_rows_and_log_line():
    out = io.StringIO()
    runner.append_csv_rows(out, "diffusion", "pitsbicg", 4, _hist())
    assert out.getvalue().splitlines() == [
        "diffusion,pitsbicg,4,0,0.5,3,6,0.125,1.25",
        "diffusion,pitsbicg,4,1,0.33333333333333331,9,12,,2.5"]
    log = io.StringIO()
    runner.log_result(log, "diffusion", "pitsbicg", 4, _hist(), "B200")
    assert log.getvalue() == ("diffusion N=4 pitsbicg: converged at k=1, residual 0.333, fine 9, "
                              "coarse 12, restarts 1, 2.5 ms (B200)\n")
    assert runner.HEADER == ("case,solver,N,k,residual_N_inf,fine_applications,"
                             "coarse_applications,error_vs_reference,wall_ms\n")


def test_slab_list_and_presets():
    assert runner.parse_slab_list("4, 8,16") == [4, 8, 16]
    with pytest.raises(ValueError):
        runner.parse_slab_list("4,x")
    # the reference's parse_slab_list (config.cpp:50-66): getline on ',' and strtol
    assert runner.parse_slab_list("4,8,") == [4, 8]
    assert runner.parse_slab_list("+4") == [4]
    for bad in ("4,,8", ",4", "1_6", "4.0", "1", "", " "):
        with pytest.raises(runner.ConfigError):
            runner.parse_slab_list(bad)
    p = presets.make_preset("advection_diffusion_reaction", "paper")
    assert (p.grid_points, p.total_time, p.mu, p.r, p.rotation) == (51, 6.4, 0.1, 0.5, True)
    with pytest.raises(ValueError, match="unknown case"):
        presets.make_preset("nope")
    with pytest.raises(ValueError, match="not a multiple"):
        presets.fine_steps(1.6, 3, 1e-3)
    assert presets.fine_steps(1.6, 64, 1e-3) == 25


def test_config_overrides():
    # parse_config_text / apply_overrides (config.cpp:68-151)
    ov = runner.parse_config_text("""
        # comment
        case = advection_diffusion_reaction
        mu = 0.2          # trailing comment
        slabs = 4, 8
        epsilon = 1e-9
        max_iters = 50
        workers = 3
    """)
    p = presets.make_preset("diffusion", "paper")
    cfg = api.SolverConfig()
    runner.apply_overrides(ov, p, cfg)
    assert (p.case_name, p.rotation, p.mu, p.r, p.grid_points) == \
        ("advection_diffusion_reaction", True, 0.2, 0.5, 51)
    assert p.slab_counts == [4, 8] and cfg.tolerance == 1e-9 and cfg.max_iterations == 50
    for bad, msg in (("mu 1", "expected key = value"), ("nope = 1", "unknown key"),
                     ("grid_points = x", "expected an integer"), ("slabs = 1,4", ">= 2"),
                     ("velocity = swirl", "unknown velocity")):
        with pytest.raises(runner.ConfigError, match=msg):
            runner.parse_config_text(bad)
