"""The reference's experiment presets (src/presets.cpp) and context builder
(runner.cpp:75-88, build_context) as Problem2DImplicit instances.

Cases: diffusion (mu 1, r 0), diffusion_reaction (mu 1, r 1.5),
advection_diffusion_reaction (mu 0.1, r 0.5, rotation u = (-y, x)); scales:
desk (33 points per axis on [-0.5, 0.5], T 1.6) and paper (51 points, T 6.4);
dt_fine 1e-3, slab counts {4, 8, 16, 32, 64}; coarse propagator one
backward-Euler step per slab (make_coarse_propagator, propagator.cpp:100-103);
y0 the unit Gaussian at the origin with sigma 0.1
(gaussian_initial_condition, grid.cpp:120-141)."""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .api import Problem2DImplicit

CASES = ("diffusion", "diffusion_reaction", "advection_diffusion_reaction")
SCALES = ("desk", "paper")


@dataclass
class ExperimentPreset:
    """pit::ExperimentPreset (include/pit/presets.hpp:25-40)."""
    case_name: str = "diffusion"
    rotation: bool = False
    mu: float = 1.0
    r: float = 0.0
    grid_points: int = 33
    total_time: float = 1.6
    dt_fine: float = 1e-3
    slab_counts: List[int] = field(default_factory=lambda: [4, 8, 16, 32, 64])
    gaussian_sigma: float = 0.1

    def validate(self) -> None:
        """ExperimentPreset::validate (presets.cpp:35-46)."""
        if self.grid_points < 3:
            raise ValueError("grid_points must be >= 3")
        if not self.total_time > 0.0:
            raise ValueError("T must be positive")
        if not self.dt_fine > 0.0:
            raise ValueError("dt_fine must be positive")
        if self.mu < 0.0:
            raise ValueError("mu must be nonnegative")
        if not self.slab_counts:
            raise ValueError("at least one slab count is required")
        if any(n < 2 for n in self.slab_counts):
            raise ValueError("slab counts must be >= 2")
        if not self.gaussian_sigma > 0.0:
            raise ValueError("gaussian sigma must be positive")


def make_preset(case_name: str, scale: str = "desk") -> ExperimentPreset:
    """make_preset (presets.cpp:48-77)."""
    if case_name not in CASES:
        raise ValueError(f"unknown case '{case_name}' (expected diffusion, diffusion_reaction, "
                         "or advection_diffusion_reaction)")
    if scale not in SCALES:
        raise ValueError(f"unknown scale '{scale}' (expected paper or desk)")
    p = ExperimentPreset(case_name=case_name)
    if case_name == "diffusion":
        p.rotation, p.mu, p.r = False, 1.0, 0.0
    elif case_name == "diffusion_reaction":
        p.rotation, p.mu, p.r = False, 1.0, 1.5
    else:
        p.rotation, p.mu, p.r = True, 0.1, 0.5
    if scale == "paper":
        p.grid_points, p.total_time = 51, 6.4
    else:
        p.grid_points, p.total_time = 33, 1.6
    return p


def stencil_2d(m: int, lo: float, hi: float, mu: float, r: float, rotation: bool) -> np.ndarray:
    """assemble_spatial_operator, 2D branch (src/pde.cpp:66-100), op for op:
    [5, m*m] south, west, centre, east, north (0 where the CSR row has no
    entry: at the walls, or when the value is exactly zero)."""
    h = (hi - lo) / (m + 2 - 1)
    mu_h2 = mu / (h * h)
    n = m * m
    out = np.zeros((5, n))
    for j in range(m):
        y = lo + (j + 1) * h
        for i in range(m):
            x = lo + (i + 1) * h
            ux, uy = (-y, x) if rotation else (0.0, 0.0)
            centre = 4.0 * mu_h2 + r + (abs(ux) + abs(uy)) / h
            west = east = south = north = -mu_h2
            if ux > 0.0:
                west -= ux / h
            elif ux < 0.0:
                east += ux / h
            if uy > 0.0:
                south -= uy / h
            elif uy < 0.0:
                north += uy / h
            row = j * m + i
            out[0, row] = south if (south != 0.0 and j > 0) else 0.0
            out[1, row] = west if (west != 0.0 and i > 0) else 0.0
            out[2, row] = centre
            out[3, row] = east if (east != 0.0 and i < m - 1) else 0.0
            out[4, row] = north if (north != 0.0 and j < m - 1) else 0.0
    return out


def gaussian_2d(m: int, lo: float, hi: float, sigma: float) -> np.ndarray:
    """gaussian_initial_condition at the origin (grid.cpp:120-141)."""
    h = (hi - lo) / (m + 2 - 1)
    inv = 1.0 / (2.0 * sigma * sigma)
    out = np.empty(m * m)
    for j in range(m):
        dy = (lo + (j + 1) * h) - 0.0
        for i in range(m):
            dx = (lo + (i + 1) * h) - 0.0
            out[j * m + i] = math.exp(-(dx * dx + dy * dy) * inv)
    return out


def fine_steps(total_time: float, slab_count: int, dt_target: float) -> int:
    """make_fine_propagator's step count (propagator.cpp:88-98)."""
    ratio = (total_time / slab_count) / dt_target
    steps = max(1, int(math.floor(ratio + 0.5)))
    if abs(ratio - steps) > 1e-9 * steps:
        raise ValueError("make_fine_propagator: slab length is not a multiple of dt")
    return steps


def build_problem(preset: ExperimentPreset, slab_count: int) -> Problem2DImplicit:
    """build_context (runner.cpp:75-88) as a device problem description."""
    preset.validate()
    if slab_count < 2:
        raise ValueError("TimeSlabPartition: need at least 2 slabs")
    m = preset.grid_points - 2
    lo, hi = -0.5, 0.5  # SpatialGrid::make_unit (grid.cpp:26-28)
    return Problem2DImplicit(
        m=m, stencil=stencil_2d(m, lo, hi, preset.mu, preset.r, preset.rotation),
        nonsymmetric=preset.rotation, N=slab_count, T=preset.total_time,
        fine_steps=fine_steps(preset.total_time, slab_count, preset.dt_fine), coarse_steps=1,
        y0=gaussian_2d(m, lo, hi, preset.gaussian_sigma), grid_lo=lo, grid_hi=hi)
