"""GPU: `pit run` on the device (paper_2203_10148_b200/runner.py) — the
reference's runner CSV schema and counters, per-row error_vs_reference, and
agreement with the reference's own run_experiment (oracle/_ref) on the desk
presets."""
from __future__ import annotations

import csv
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib as O
from paper_2203_10148_b200 import api, presets, runner

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_rows(path):
    with open(path) as f:
        head = f.readline()
        rows = list(csv.reader(f))
    return head, rows


@pytest.mark.parametrize("case", ["diffusion", "advection_diffusion_reaction"])
def test_runner_csv_matches_device_solvers_and_reference(case, tmp_path):
    preset = presets.make_preset(case, "desk")
    preset.slab_counts = [4, 8]
    spec = runner.RunSpec(preset=preset, solver="both", out_dir=str(tmp_path / "gpu"))
    path = runner.run_experiment(spec, open(os.devnull, "w"))
    head, rows = read_rows(path)
    assert head == runner.HEADER
    # every row: the device solver's history, error column filled
    for n in preset.slab_counts:
        p = presets.build_problem(preset, n)
        with api.BlockOperatorContext(p) as ctx:
            seq = api.sequential_fine_solve(ctx)
            for solver, fn in (("parareal", api.parareal_solve), ("pitsbicg", api.pitsbicg_solve)):
                res = fn(ctx, api.SolverConfig())
                mine = [r for r in rows if r[1] == solver and int(r[2]) == n]
                assert [(int(r[3]), r[4], int(r[5]), int(r[6])) for r in mine] == \
                    [(x.k, runner.fmt(x.residual_norm), x.fine_applications, x.coarse_applications)
                     for x in res.history.records]
                assert all(r[7] != "" for r in mine)
                err = float(mine[-1][7])
                want = max(np.sqrt(p.spacing ** 2 * np.sum((res.solution - seq) ** 2, axis=1)))
                assert abs(err - want) <= 1e-10 * want + 1e-300
    if not O.ref_available():
        return
    out = str(tmp_path / "ref")
    slabs = (O.C.c_int * 2)(4, 8)
    cid = presets.CASES.index(case)
    assert O.ref().pitref_run_experiment(cid, 0, slabs, 2, 2, 1e-8, out.encode()) == 0
    rhead, rrows = read_rows(os.path.join(out, case + ".csv"))
    assert rhead == head
    assert len(rrows) == len(rows)
    for a, b in zip(rows, rrows):
        assert a[:4] == b[:4] and a[5:7] == b[5:7]           # case, solver, N, k, counters
        assert abs(float(a[4]) - float(b[4])) <= 1e-6 * float(b[4]) + 1e-13
        assert abs(float(a[7]) - float(b[7])) <= 1e-4 * float(b[7]) + 1e-11


def test_runner_cli(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2203_10148_b200.runner", "run", "--case",
                        "diffusion_reaction", "--solver", "pitsbicg", "--slabs", "4",
                        "--out", str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "diffusion_reaction N=4 pitsbicg: converged" in r.stdout
    assert os.path.exists(tmp_path / "diffusion_reaction.csv")
    bad = subprocess.run([sys.executable, "-m", "paper_2203_10148_b200.runner", "run", "--case",
                          "nope"], cwd=ROOT, capture_output=True, text=True)
    assert bad.returncode == 2 and "unknown case" in bad.stderr
