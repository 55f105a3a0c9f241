"""`pit run` on the device: the reference's experiment runner
(src/runner.cpp:86-147, src/cli.cpp:35-58) over the B200 operators.

For every slab count of the preset: build the context (build_context,
runner.cpp:75-88 -> presets.build_problem), the sequential fine trajectory as
the reference solution (runner.cpp:123), then parareal and/or PiTSBiCG with
`SolveOptions.reference` so every history row carries error_vs_reference;
rows go to <out>/<case>.csv with the reference's header and `%.17g` fields
(write_csv_header / append_csv_rows, runner.cpp:90-106) and one log line per
solve (log_result, runner.cpp:31-55; the executor's worker count and
fine-phase efficiency are replaced by the device name).

    python -m paper_2203_10148_b200.runner run --case diffusion --solver both \\
        --slabs 4,8 --scale desk --out out [--config overrides.txt]
"""
from __future__ import annotations

import argparse
import os
import sys
from dataclasses import dataclass, field
from typing import List, Optional, TextIO

from . import api, presets

HEADER = ("case,solver,N,k,residual_N_inf,fine_applications,coarse_applications,"
          "error_vs_reference,wall_ms\n")
SOLVERS = ("parareal", "pitsbicg", "both")


def fmt(v: float) -> str:
    """%.17g (runner.cpp:17-21)."""
    return "%.17g" % v


def fmt_short(v: float) -> str:
    return "%.3g" % v


@dataclass
class RunSpec:
    """pit::RunSpec (include/pit/runner.hpp:17-24)."""
    preset: presets.ExperimentPreset
    solver: str = "both"
    solver_config: api.SolverConfig = field(default_factory=api.SolverConfig)
    out_dir: str = "out"
    device: int = 0


def append_csv_rows(out: TextIO, case_label: str, solver_label: str, slab_count: int,
                    history: api.ConvergenceHistory) -> None:
    """append_csv_rows (runner.cpp:95-106)."""
    for r in history.records:
        err = fmt(r.error_vs_reference) if r.error_vs_reference is not None else ""
        out.write(f"{case_label},{solver_label},{slab_count},{r.k},{fmt(r.residual_norm)},"
                  f"{r.fine_applications},{r.coarse_applications},{err},{fmt(r.wall_ms)}\n")


def log_result(log: TextIO, case_label: str, solver_label: str, slab_count: int,
               hist: api.ConvergenceHistory, device: str) -> None:
    """log_result (runner.cpp:31-55)."""
    last = hist.records[-1]
    status = "converged" if hist.status == api.SolveStatus.Converged else "max-iterations"
    line = (f"{case_label} N={slab_count} {solver_label}: {status} at k={last.k}, residual "
            f"{fmt_short(last.residual_norm)}")
    if last.error_vs_reference is not None:
        line += f", error {fmt_short(last.error_vs_reference)}"
    line += f", fine {hist.stats.fine_applications}, coarse {hist.stats.coarse_applications}"
    if hist.restarts > 0:
        line += f", restarts {hist.restarts}"
    line += f", {fmt_short(last.wall_ms)} ms ({device})\n"
    log.write(line)


def run_experiment(spec: RunSpec, log: TextIO = sys.stdout) -> str:
    """run_experiment (runner.cpp:108-147); returns the CSV path."""
    spec.preset.validate()
    spec.solver_config.validate()
    if spec.solver not in SOLVERS:
        raise ValueError(f"unknown solver '{spec.solver}' (expected parareal, pitsbicg, or both)")
    os.makedirs(spec.out_dir, exist_ok=True)
    case_label = spec.preset.case_name
    path = os.path.join(spec.out_dir, case_label + ".csv")
    device = "B200" if api._lib.lib().pit_device_count() > 0 else "device"
    with open(path, "w") as csv:
        csv.write(HEADER)
        for n in spec.preset.slab_counts:
            p = presets.build_problem(spec.preset, n)
            with api.BlockOperatorContext(p, device=spec.device) as ctx:
                reference = api.sequential_fine_solve(ctx)
                opts = api.SolveOptions(reference=reference)
                if spec.solver in ("parareal", "both"):
                    res = api.parareal_solve(ctx, spec.solver_config, options=opts)
                    append_csv_rows(csv, case_label, "parareal", n, res.history)
                    log_result(log, case_label, "parareal", n, res.history, device)
                if spec.solver in ("pitsbicg", "both"):
                    res = api.pitsbicg_solve(ctx, spec.solver_config, options=opts)
                    append_csv_rows(csv, case_label, "pitsbicg", n, res.history)
                    log_result(log, case_label, "pitsbicg", n, res.history, device)
            csv.flush()
    return path


class ConfigError(ValueError):
    """pit::ConfigError (CLI exit code 2)."""


def parse_slab_list(text: str) -> List[int]:
    """parse_slab_list (config.cpp:50-66): comma-separated slab counts >= 2.
    Tokens are split like std::getline(',') (a trailing comma ends the list,
    an empty entry inside it is an error) and parsed like strtol: an optional
    sign and decimal digits, nothing else."""
    import re

    out = []
    parts = text.split(",")
    if parts and parts[-1] == "":
        parts = parts[:-1]  # getline yields no token after a trailing comma
    for item in parts:
        tok = item.strip()
        if not tok:
            raise ConfigError(f"empty entry in slab list '{text}'")
        if not re.fullmatch(r"[+-]?[0-9]+", tok) or int(tok) < 2:
            raise ConfigError(f"slab counts must be integers >= 2, got '{tok}'")
        out.append(int(tok))
    if not out:
        raise ConfigError(f"slab list '{text}' is empty")
    return out


_KEYS = {"case": str, "mu": float, "r": float, "velocity": str, "grid_points": int, "T": float,
         "dt_fine": float, "slabs": str, "epsilon": float, "epsilon0": float, "max_iters": int,
         "workers": int}


def parse_config_text(text: str) -> dict:
    """parse_config_text (config.cpp:68-118): `key = value` lines, `#`
    comments; unknown keys and malformed values are ConfigErrors."""
    out = {}
    for line_no, raw in enumerate(text.splitlines(), 1):
        entry = raw.split("#", 1)[0].strip()
        if not entry:
            continue
        if "=" not in entry:
            raise ConfigError(f"config line {line_no}: expected key = value")
        key, value = (x.strip() for x in entry.split("=", 1))
        if not key or not value:
            raise ConfigError(f"config line {line_no}: expected key = value")
        if key not in _KEYS:
            raise ConfigError(f"config line {line_no}: unknown key '{key}'")
        kind = _KEYS[key]
        if key == "case":
            if value not in presets.CASES:
                raise ConfigError(f"unknown case '{value}' (expected diffusion, "
                                  "diffusion_reaction, or advection_diffusion_reaction)")
            out[key] = value
        elif key == "velocity":
            if value not in ("zero", "rotation"):
                raise ConfigError(f"config line {line_no}: unknown velocity '{value}'")
            out[key] = value == "rotation"
        elif key == "slabs":
            out[key] = parse_slab_list(value)
        else:
            try:
                out[key] = kind(value)
            except ValueError:
                what = "an integer" if kind is int else "a number"
                raise ConfigError(f"config line {line_no}: expected {what}, got '{value}'") from None
    return out


def apply_overrides(ov: dict, preset: presets.ExperimentPreset, solver: api.SolverConfig) -> None:
    """apply_overrides (config.cpp:128-151); `workers` has no device meaning."""
    if "case" in ov:
        base = presets.make_preset(ov["case"], "desk")
        preset.case_name, preset.rotation, preset.mu, preset.r = (base.case_name, base.rotation,
                                                                  base.mu, base.r)
    if "mu" in ov:
        preset.mu = ov["mu"]
    if "r" in ov:
        preset.r = ov["r"]
    if "velocity" in ov:
        preset.rotation = ov["velocity"]
    if "grid_points" in ov:
        preset.grid_points = ov["grid_points"]
    if "T" in ov:
        preset.total_time = ov["T"]
    if "dt_fine" in ov:
        preset.dt_fine = ov["dt_fine"]
    if "slabs" in ov:
        preset.slab_counts = ov["slabs"]
    if "epsilon" in ov:
        solver.tolerance = ov["epsilon"]
    if "epsilon0" in ov:
        solver.restart_tolerance = ov["epsilon0"]
    if "max_iters" in ov:
        solver.max_iterations = ov["max_iters"]


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="pit", description="parallel-in-time benchmark: parareal "
                                 "and preconditioned BiCGStab over time slabs (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="run a benchmark case and write per-iteration CSV")
    run.add_argument("--case", default="diffusion",
                     help="diffusion | diffusion_reaction | advection_diffusion_reaction")
    run.add_argument("--solver", default="both", help="parareal | pitsbicg | both")
    run.add_argument("--slabs", default="", help="comma-separated slab counts (default preset sweep)")
    run.add_argument("--scale", default="desk", help="paper | desk")
    run.add_argument("--out", default="out", help="output directory")
    run.add_argument("--config", default="", help="key = value file overriding the flags")
    run.add_argument("--tolerance", type=float, default=None, help="solver tolerance")
    run.add_argument("--max-iterations", type=int, default=None)
    run.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    try:
        preset = presets.make_preset(args.case, args.scale)
        if args.slabs:
            preset.slab_counts = parse_slab_list(args.slabs)
        cfg = api.SolverConfig()
        if args.config:
            try:
                text = open(args.config).read()
            except OSError:
                raise ConfigError(f"cannot read config file '{args.config}'") from None
            apply_overrides(parse_config_text(text), preset, cfg)
        if args.tolerance is not None:
            cfg.tolerance = args.tolerance
        if args.max_iterations is not None:
            cfg.max_iterations = args.max_iterations
        spec = RunSpec(preset=preset, solver=args.solver, solver_config=cfg, out_dir=args.out,
                       device=args.device)
        path = run_experiment(spec, sys.stdout)
    except (ValueError, api.ConfigError) as e:  # ConfigError / invalid_argument -> 2 (cli.cpp:144-156)
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # other pit::Error -> 1
        print(f"error: {e}", file=sys.stderr)
        return 1
    print(f"wrote {path}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
