"""Dense verification of the device operators: the reference's
run_oracle_checks / `pit verify` (src/dense_oracle.cpp:110-237,
include/pit/dense_oracle.hpp; cli.cpp:59-96) driven through the B200 kernels.

The propagators are probed with unit fields through pit_propagate (the
slabs are uniform and time-independent, so one matrix per role suffices),
the flat block systems F and G are assembled densely, G is inverted, and the
matrix-free device apply_F / apply_G_inverse are compared with the dense
products on seeded random block vectors (std::mt19937_64(42), uniform(-1, 1),
the reference's draws).  `inject_fault` perturbs the dense matrices first:
a working checker then reports failures (negative control).

This is a verification tool over the GPU operators (like the reference's
own dense oracle), not a compute path: it refuses problems above
kDenseOracleLimit = 2000 flat unknowns.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

from .api import (BlockOperatorContext, ConfigError, apply_F, apply_G_inverse, coarse, fine,
                  seeded_uniform)

DENSE_ORACLE_LIMIT = 2000


@dataclass
class DenseBlockSystem:
    F: np.ndarray
    G: np.ndarray
    G_inverse: np.ndarray
    block_count: int
    nodes_per_block: int


@dataclass
class OracleCheck:
    name: str
    worst_relative_error: float = 0.0
    passed: bool = False


@dataclass
class OracleCheckReport:
    checks: List[OracleCheck] = field(default_factory=list)

    def all_passed(self) -> bool:
        return all(c.passed for c in self.checks)


def relative_difference(got: np.ndarray, want: np.ndarray) -> float:
    """||got - want|| / ||want|| (1 when want = 0), dense_oracle.cpp:19-28."""
    if got.shape != want.shape:
        raise ValueError("relative_difference: size mismatch")
    scale = float(np.sqrt(np.sum(want * want)))
    return float(np.sqrt(np.sum((got - want) ** 2))) / (scale if scale > 0.0 else 1.0)


def assemble_dense_system(ctx: BlockOperatorContext) -> DenseBlockSystem:
    nodes, count = ctx.M, ctx.N
    flat = nodes * count
    if flat > DENSE_ORACLE_LIMIT:
        raise ConfigError(f"dense oracle limited to {DENSE_ORACLE_LIMIT} unknowns; requested {flat} "
                          f"({count} blocks x {nodes} nodes)")
    p_fine = np.zeros((nodes, nodes))
    p_coarse = np.zeros((nodes, nodes))
    fp, cp = fine(ctx), coarse(ctx)
    for j in range(nodes):
        unit = np.zeros(nodes)
        unit[j] = 1.0
        p_fine[:, j] = fp.propagate_homogeneous(unit, 0)
        p_coarse[:, j] = cp.propagate_homogeneous(unit, 0)
    F = np.eye(flat)
    G = np.eye(flat)
    for n in range(1, count):
        F[n * nodes:(n + 1) * nodes, (n - 1) * nodes:n * nodes] = -p_fine
        G[n * nodes:(n + 1) * nodes, (n - 1) * nodes:n * nodes] = -p_coarse
    return DenseBlockSystem(F=F, G=G, G_inverse=np.linalg.inv(G), block_count=count,
                            nodes_per_block=nodes)


def run_oracle_checks(ctx: BlockOperatorContext, trials: int = 3, tolerance: float = 1e-10,
                      inject_fault: bool = False) -> OracleCheckReport:
    if trials < 1:
        raise ValueError("run_oracle_checks: trials must be >= 1")
    sys_ = assemble_dense_system(ctx)
    if inject_fault:
        i = sys_.nodes_per_block  # first row of the second block
        sys_.F[i, 0] += 0.5
        sys_.G[i, 0] += 0.5
        sys_.G_inverse[i, 0] += 0.5
    flat = sys_.block_count * sys_.nodes_per_block
    draws = seeded_uniform(42, trials * flat, -1.0, 1.0)
    f_check = OracleCheck("apply_F vs dense F")
    g_check = OracleCheck("apply_G_inverse vs dense inverse")
    for t in range(trials):
        x = draws[t * flat:(t + 1) * flat]
        bx = x.reshape(sys_.block_count, sys_.nodes_per_block)
        f_free = apply_F(ctx, bx).reshape(-1)
        f_check.worst_relative_error = max(f_check.worst_relative_error,
                                           relative_difference(f_free, sys_.F @ x))
        g_free = apply_G_inverse(ctx, bx).reshape(-1)
        g_check.worst_relative_error = max(g_check.worst_relative_error,
                                           relative_difference(g_free, sys_.G_inverse @ x))
    f_check.passed = f_check.worst_relative_error <= tolerance
    g_check.passed = g_check.worst_relative_error <= tolerance
    ident = OracleCheck("dense inverse times dense G vs identity")
    ident.worst_relative_error = float(np.max(np.abs(sys_.G_inverse @ sys_.G - np.eye(flat))))
    ident.passed = ident.worst_relative_error <= tolerance
    return OracleCheckReport([f_check, g_check, ident])


def preset_problem(case: str, dimension: int = 2, grid_points: int = 5, slabs: int = 3):
    """cli.cpp do_verify's context (cli.cpp:58-75): the case's coefficients on
    make_unit(dimension, grid_points), T = 0.1 over `slabs` slabs, fine dt =
    slab/8, one coarse step, the Gaussian initial value."""
    from . import api, presets

    pr = presets.make_preset(case, "desk")
    if dimension == 1 and pr.rotation:
        raise ValueError("the rotation velocity field needs a 2D grid; pick another case")
    m = grid_points - 2
    lo, hi = -0.5, 0.5
    T = 0.1
    if dimension == 2:
        return api.Problem2DImplicit(
            m=m, stencil=presets.stencil_2d(m, lo, hi, pr.mu, pr.r, pr.rotation),
            nonsymmetric=pr.rotation, N=slabs, T=T, fine_steps=8, coarse_steps=1,
            y0=presets.gaussian_2d(m, lo, hi, pr.gaussian_sigma), grid_lo=lo, grid_hi=hi)
    h = (hi - lo) / (m + 1)
    lo_b, di_b, up_b = api.diffusion_reaction_bands(pr.mu, pr.r, h)
    x = np.array([lo + (k + 1) * h for k in range(m)])
    y0 = np.exp(-(x * x) / (2.0 * pr.gaussian_sigma ** 2))
    return api.Problem1D(M=m, band_lo=lo_b, band_diag=di_b, band_up=up_b, N=slabs, T=T,
                         fine_steps=8, coarse_steps=1, y0=y0, grid_lo=lo, grid_hi=hi)


def main(argv=None) -> int:
    """`python -m paper_2203_10148_b200.verify [--case diffusion] [--dim 2]
    [--grid-points 5] [--slabs 3] [--trials 20] [--tolerance 1e-10]
    [--inject-fault]` — `pit verify` (cli.cpp:58-89) over the device
    operators; or `verify c1..c5 [--slabs N] [--grid-points M]` for the
    BASELINE configs reduced to the dense limit."""
    import argparse

    from . import configs

    ap = argparse.ArgumentParser(description="dense cross-check of the device operators")
    ap.add_argument("config", nargs="?", choices=sorted(configs.SHAPES), default=None)
    ap.add_argument("--case", default="diffusion")
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--slabs", type=int, default=None)
    ap.add_argument("--grid-points", type=int, default=None)
    ap.add_argument("--trials", type=int, default=None)
    ap.add_argument("--tolerance", type=float, default=1e-10)
    ap.add_argument("--inject-fault", action="store_true")
    a = ap.parse_args(argv)
    if a.config:
        slabs = a.slabs or 4
        trials = a.trials or 3
        m = a.grid_points or (12 if a.config == "c5" else max(2, DENSE_ORACLE_LIMIT // slabs))
        p = configs.make(a.config, slabs=slabs, M=m)
        label = f"{a.config}, {p.N} slabs x {p.M} nodes"
    else:
        trials = a.trials or 20
        try:
            p = preset_problem(a.case, a.dim, a.grid_points or 5, a.slabs or 3)
        except ValueError as e:
            print(f"error: {e}")
            return 2
        label = f"{a.case}, {a.dim}D, {a.grid_points or 5} points/axis, N={p.N}"
    with BlockOperatorContext(p) as ctx:
        rep = run_oracle_checks(ctx, trials, a.tolerance, a.inject_fault)
    print(f"oracle checks on {label}, {trials} trials, tolerance {a.tolerance}")
    for c in rep.checks:
        print(f"  [{'pass' if c.passed else 'FAIL'}] {c.name:40s} worst relative error "
              f"{c.worst_relative_error:.3e}")
    print("all checks passed" if rep.all_passed() else "CHECKS FAILED")
    return 0 if rep.all_passed() else 1


if __name__ == "__main__":
    raise SystemExit(main())
