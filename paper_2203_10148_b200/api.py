"""Python mirror of the reference's pit:: operator and solver API.

Same names, argument meaning and error behaviour as the C++ reference
(/root/reference/proj/include/pit/*.hpp), backed by the sm_100a kernels
through the C ABI in include/pit_b200.h.  Block vectors are numpy arrays of
shape (N, M) (block-major, x-fastest: the reference's flat convention,
src/dense_oracle.cpp:153-177).

Reference exception -> Python exception:
  std::invalid_argument  -> ValueError            (PIT_ERR_INVALID_ARGUMENT)
  pit::InnerSolveError   -> InnerSolveError       (PIT_ERR_INNER_SOLVE)
  pit::SlabError         -> SlabError(slab_index) (PIT_ERR_SLAB)
  pit::ConfigError       -> ConfigError           (PIT_ERR_CONFIG)
  (CUDA failure)         -> DeviceError           (PIT_ERR_CUDA)
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from ._lib import dptr


class PitError(RuntimeError):
    """pit::Error (include/pit/errors.hpp:9-12)."""


class InnerSolveError(PitError):
    """pit::InnerSolveError (errors.hpp:15-21): carries the inner solve's
    achieved relative residual and iteration count (thrown at
    src/pde.cpp:119-128; NaN and 0 for the 1D direct solve)."""

    def __init__(self, what: str, achieved_relative_residual: float = float("nan"),
                 iterations: int = 0):
        super().__init__(what)
        self.achieved_relative_residual = achieved_relative_residual
        self.iterations = iterations


class SlabError(PitError):
    """pit::SlabError (errors.hpp:24-29): carries the lowest failing slab."""

    def __init__(self, slab_index: int, what: str):
        super().__init__(what)
        self.slab_index = slab_index


class ConfigError(PitError):
    """pit::ConfigError (errors.hpp:32-34)."""


class DeviceError(PitError):
    """CUDA failure (no reference counterpart: the reference is CPU-only)."""


def _check(rc: int) -> None:
    if rc == _lib.PIT_OK:
        return
    L = _lib.lib()
    msg = (L.pit_last_error() or b"").decode()
    if rc == _lib.PIT_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == _lib.PIT_ERR_INNER_SOLVE:
        rel, its = C.c_double(float("nan")), C.c_int64(0)
        L.pit_last_error_detail(C.byref(rel), C.byref(its))
        raise InnerSolveError(msg, rel.value, its.value)
    if rc == _lib.PIT_ERR_SLAB:
        raise SlabError(L.pit_last_error_slab(), msg)
    if rc == _lib.PIT_ERR_CONFIG:
        raise ConfigError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------------------
# Problem description (SpatialGrid + SpatialOperator + partition + propagators)
# ---------------------------------------------------------------------------

@dataclass
class SeparableSource:
    """f(t, x_i) = amp * sin(omega*t + phase) * shape[i]  (a pit::SourceFn,
    include/pit/pde.hpp:13, restricted to the separable form the kernels
    evaluate from a host-built table)."""
    amp: float
    omega: float
    phase: float
    shape: np.ndarray


@dataclass
class TableSource:
    """A general pit::SourceFn f(t, x) (include/pit/pde.hpp:13) sampled where
    Propagator::run samples it (src/propagator.cpp:56-63, the end of every
    step): fine[n, k-1, i] = f(breakpoint(n) + k*dt_fine, x_i), k = 1 ..
    fine_steps, and coarse likewise with the coarse steps.  N*steps*M doubles
    per propagator: for moderate problems (SeparableSource needs no table)."""
    fine: np.ndarray
    coarse: np.ndarray

    @staticmethod
    def sample(f, M: int, N: int, T: float, fine_steps: int, coarse_steps: int,
               grid_lo: float = 0.0, grid_hi: float = 1.0) -> "TableSource":
        """Tables of the Python callable f(t, x) (x: array of the M interior
        coordinates; returns an array of M values)."""
        h = (grid_hi - grid_lo) / (M + 1)
        x = np.array([grid_lo + (k + 1) * h for k in range(M)])
        slab = T / N
        out = []
        for steps in (fine_steps, coarse_steps):
            dt = slab / steps
            tab = np.empty((N, steps, M))
            for n in range(N):
                t0 = n * slab
                for k in range(1, steps + 1):
                    tab[n, k - 1] = f(t0 + k * dt, x)
            out.append(tab)
        return TableSource(out[0], out[1])


def _attach_tables(d, keep, source, N, fine_steps, coarse_steps, M):
    """PIT_SOURCE_TABLE fields of a problem description."""
    if source is None:
        return
    if not isinstance(source, TableSource):
        raise ValueError("this problem class takes its source as a TableSource")
    tabs = []
    for tab, steps in ((source.fine, fine_steps), (source.coarse, coarse_steps)):
        t = np.ascontiguousarray(tab, dtype=np.float64)
        if t.shape != (N, steps, M):
            raise ValueError("TableSource: tables are [N, steps, M] per propagator")
        keep.append(t)
        tabs.append(t)
    d.source_kind = _lib.PIT_SOURCE_TABLE
    d.source_table_fine, d.source_table_coarse = dptr(tabs[0]), dptr(tabs[1])


@dataclass
class Problem1D:
    """Everything BlockOperatorContext needs for a 1D problem.

    bands (lo, diag, up) of A with dy/dt = -A y + f, as built by
    assemble_spatial_operator (src/pde.cpp:55-64) or any constant tridiagonal
    operator; grid [lo, hi] with M interior nodes (h = (hi-lo)/(M+1),
    src/grid.cpp:19); partition T, N (src/propagator.cpp:8-17)."""
    M: int
    band_lo: float
    band_diag: float
    band_up: float
    N: int
    T: float
    fine_steps: int
    coarse_steps: int
    y0: np.ndarray
    grid_lo: float = 0.0
    grid_hi: float = 1.0
    source: Optional[object] = None  # SeparableSource or TableSource

    @property
    def spacing(self) -> float:
        return (self.grid_hi - self.grid_lo) / (self.M + 2 - 1)

    def coords(self) -> np.ndarray:
        """SpatialGrid::interior_coord (include/pit/grid.hpp:31)."""
        h = self.spacing
        return np.array([self.grid_lo + (k + 1) * h for k in range(self.M)])

    def desc(self, device: int = 0, fine_layout=None, coarse_layout=None):
        d = _lib.ProblemDesc()
        d.dimension = 1
        d.interior = self.M
        d.grid_lo, d.grid_hi = self.grid_lo, self.grid_hi
        d.band_lo, d.band_diag, d.band_up = self.band_lo, self.band_diag, self.band_up
        d.slab_count = self.N
        d.total_time = self.T
        d.fine_steps, d.coarse_steps = self.fine_steps, self.coarse_steps
        keep = []
        y0 = np.ascontiguousarray(self.y0, dtype=np.float64)
        keep.append(y0)
        d.initial_value = dptr(y0)
        if isinstance(self.source, TableSource):
            tabs = []
            for tab, steps in ((self.source.fine, self.fine_steps),
                               (self.source.coarse, self.coarse_steps)):
                t = np.ascontiguousarray(tab, dtype=np.float64)
                if t.shape != (self.N, steps, self.M):
                    raise ValueError("TableSource: tables are [N, steps, M] per propagator")
                keep.append(t)
                tabs.append(t)
            d.source_kind = _lib.PIT_SOURCE_TABLE
            d.source_table_fine, d.source_table_coarse = dptr(tabs[0]), dptr(tabs[1])
        elif self.source is not None:
            sh = np.ascontiguousarray(self.source.shape, dtype=np.float64)
            keep.append(sh)
            d.source_kind = _lib.PIT_SOURCE_SEPARABLE
            d.source_amp, d.source_omega, d.source_phase = (self.source.amp, self.source.omega,
                                                            self.source.phase)
            d.source_shape = dptr(sh)
        d.device = device
        # layouts: (points/thread, warps/slab) or
        # (points/thread, sub-chunks/thread, segments/slab, warps/slab)
        if fine_layout:
            d.fine_mpt, d.fine_nsub, d.fine_nseg, d.fine_warps = _layout4(fine_layout)
        if coarse_layout:
            d.coarse_mpt, d.coarse_nsub, d.coarse_nseg, d.coarse_warps = _layout4(coarse_layout)
        return d, keep


@dataclass
class Problem2D:
    """A 2D problem (config 5): dy/dt = -A y on the square [lo, hi]^2 with m
    interior points per axis (h = (hi-lo)/(m+1)), A the isotropic 5-point
    operator (centre band_diag, each neighbour band_off) — the reference's
    2D assemble_spatial_operator with zero velocity (src/pde.cpp:66-100).
    Fine propagator: explicit Euler (fine_steps per slab); coarse: backward
    Euler (coarse_steps per slab) solved by Jacobi-PCG to coarse_tolerance
    (the reference's solve_cg control flow, src/sparse.cpp:60-114).  Blocks
    hold m*m values, x fastest (SpatialGrid::flat_index)."""
    m: int
    band_off: float
    band_diag: float
    N: int
    T: float
    fine_steps: int
    coarse_steps: int
    y0: np.ndarray
    grid_lo: float = 0.0
    grid_hi: float = 1.0
    coarse_tolerance: float = 1e-12
    coarse_max_iterations: int = 0
    source: Optional[SeparableSource] = None  # always None in 2D

    @property
    def M(self) -> int:
        return self.m * self.m

    @property
    def spacing(self) -> float:
        return (self.grid_hi - self.grid_lo) / (self.m + 2 - 1)

    def coords(self) -> np.ndarray:
        h = self.spacing
        return np.array([self.grid_lo + (k + 1) * h for k in range(self.m)])

    def desc(self, device: int = 0, fine_layout=None, coarse_layout=None):
        d = _lib.ProblemDesc()
        d.dimension = 2
        d.interior = self.m
        d.grid_lo, d.grid_hi = self.grid_lo, self.grid_hi
        d.band_lo, d.band_diag, d.band_up = self.band_off, self.band_diag, self.band_off
        d.slab_count = self.N
        d.total_time = self.T
        d.fine_steps, d.coarse_steps = self.fine_steps, self.coarse_steps
        y0 = np.ascontiguousarray(self.y0, dtype=np.float64).reshape(-1)
        keep = [y0]
        d.initial_value = dptr(y0)
        d.device = device
        d.fine_scheme = _lib.PIT_SCHEME_EXPLICIT_EULER
        d.coarse_tolerance = self.coarse_tolerance
        d.coarse_max_iterations = self.coarse_max_iterations
        if fine_layout:  # (tile rows, tile cols, CTAs per cluster, warps per CTA)
            d.tile_rows, d.tile_cols, d.tile_cluster, d.tile_warps = tuple(fine_layout)
        return d, keep


@dataclass
class Problem2DImplicit:
    """A 2D problem with backward-Euler fine and coarse propagators on the
    reference's general 5-point operator: the desk/paper presets
    (src/presets.cpp:47-77, assembled by runner.cpp:75-88; see presets.py).
    `stencil` is [5, m*m]: the south, west, centre, east, north entries of A
    per interior node exactly as assemble_spatial_operator emits them
    (src/pde.cpp:66-100), 0 where the row has no such entry.  Every step is
    solved by Jacobi-PCG (symmetric operator) or Jacobi-BiCGStab
    (`nonsymmetric`, e.g. the rotation velocity) to the reference's 1e-12
    within 10 n iterations (ImplicitStepSolver, src/pde.cpp:112-130).  m <= 101."""
    m: int
    stencil: np.ndarray
    nonsymmetric: bool
    N: int
    T: float
    fine_steps: int
    coarse_steps: int
    y0: np.ndarray
    grid_lo: float = -0.5
    grid_hi: float = 0.5
    fine_tolerance: float = 1e-12
    coarse_tolerance: float = 1e-12
    fine_max_iterations: int = 0
    coarse_max_iterations: int = 0
    source: Optional[object] = None  # a TableSource (the presets have f = 0)

    @property
    def M(self) -> int:
        return self.m * self.m

    @property
    def spacing(self) -> float:
        return (self.grid_hi - self.grid_lo) / (self.m + 2 - 1)

    def coords(self) -> np.ndarray:
        h = self.spacing
        return np.array([self.grid_lo + (k + 1) * h for k in range(self.m)])

    def desc(self, device: int = 0, fine_layout=None, coarse_layout=None):
        d = _lib.ProblemDesc()
        d.dimension = 2
        d.interior = self.m
        d.grid_lo, d.grid_hi = self.grid_lo, self.grid_hi
        st = np.ascontiguousarray(self.stencil, dtype=np.float64).reshape(-1)
        if st.size != 5 * self.M:
            raise ValueError("stencil must be [5, m*m]")
        d.band_lo, d.band_diag, d.band_up = 0.0, 0.0, 0.0
        d.slab_count = self.N
        d.total_time = self.T
        d.fine_steps, d.coarse_steps = self.fine_steps, self.coarse_steps
        y0 = np.ascontiguousarray(self.y0, dtype=np.float64).reshape(-1)
        keep = [y0, st]
        d.initial_value = dptr(y0)
        d.stencil = dptr(st)
        d.nonsymmetric = 1 if self.nonsymmetric else 0
        d.device = device
        d.fine_scheme = _lib.PIT_SCHEME_BACKWARD_EULER
        d.fine_tolerance, d.coarse_tolerance = self.fine_tolerance, self.coarse_tolerance
        d.fine_max_iterations = self.fine_max_iterations
        d.coarse_max_iterations = self.coarse_max_iterations
        _attach_tables(d, keep, self.source, self.N, self.fine_steps, self.coarse_steps, self.M)
        return d, keep


@dataclass
class Problem1DGeneral:
    """A 1D problem whose operator is any tridiagonal matrix — what the
    reference's propagators accept through the SpatialOperator CSR constructor
    (include/pit/pde.hpp:36-37), e.g. variable coefficients.  `stencil` is
    [3, M]: the sub-diagonal, diagonal and super-diagonal entry of A per
    interior node (0 where absent).  Every backward-Euler step is solved as
    the reference solves it (ImplicitStepSolver, src/pde.cpp:112-130):
    Jacobi-PCG, or Jacobi-BiCGStab when `nonsymmetric`, to 1e-12.  Constant
    bands should use Problem1D (the direct solve); M <= 10240; a source, if
    any, as a TableSource."""
    M: int
    stencil: np.ndarray
    nonsymmetric: bool
    N: int
    T: float
    fine_steps: int
    coarse_steps: int
    y0: np.ndarray
    grid_lo: float = 0.0
    grid_hi: float = 1.0
    fine_tolerance: float = 1e-12
    coarse_tolerance: float = 1e-12
    fine_max_iterations: int = 0
    coarse_max_iterations: int = 0
    source: Optional[object] = None  # a TableSource, or None

    @property
    def spacing(self) -> float:
        return (self.grid_hi - self.grid_lo) / (self.M + 2 - 1)

    def coords(self) -> np.ndarray:
        h = self.spacing
        return np.array([self.grid_lo + (k + 1) * h for k in range(self.M)])

    def desc(self, device: int = 0, fine_layout=None, coarse_layout=None):
        d = _lib.ProblemDesc()
        d.dimension = 1
        d.interior = self.M
        d.grid_lo, d.grid_hi = self.grid_lo, self.grid_hi
        st = np.ascontiguousarray(self.stencil, dtype=np.float64).reshape(-1)
        if st.size != 3 * self.M:
            raise ValueError("stencil must be [3, M]")
        d.slab_count = self.N
        d.total_time = self.T
        d.fine_steps, d.coarse_steps = self.fine_steps, self.coarse_steps
        y0 = np.ascontiguousarray(self.y0, dtype=np.float64).reshape(-1)
        keep = [y0, st]
        d.initial_value = dptr(y0)
        d.stencil = dptr(st)
        d.nonsymmetric = 1 if self.nonsymmetric else 0
        d.device = device
        d.fine_tolerance, d.coarse_tolerance = self.fine_tolerance, self.coarse_tolerance
        d.fine_max_iterations = self.fine_max_iterations
        d.coarse_max_iterations = self.coarse_max_iterations
        _attach_tables(d, keep, self.source, self.N, self.fine_steps, self.coarse_steps, self.M)
        return d, keep


def heat_2d_bands(diffusion: float, h: float):
    """(neighbour, centre) of the 2D 5-point -mu*Laplacian, as
    assemble_spatial_operator's 2D branch builds them (src/pde.cpp:66-100:
    centre 4*mu/h^2 + r, neighbours -mu/h^2; zero velocity, r = 0)."""
    mu_h2 = diffusion / (h * h)
    return -mu_h2, 4.0 * mu_h2


def step_coefficients_2d(problem: "Problem2D", fine_layout=None):
    """Host-side 2D coefficient struct (no GPU needed)."""
    d, keep = problem.desc(0, fine_layout)
    c = _lib.StepCoeffs2DC()
    _check(_lib.lib().pit_step_coefficients_2d(C.byref(d), C.byref(c)))
    return c


def _layout4(lay):
    lay = tuple(lay)
    if len(lay) == 2:
        return lay[0], 1, 1, lay[1]
    if len(lay) == 4:
        return lay
    raise ValueError("layout must be (mpt, warps) or (mpt, nsub, nseg, warps)")


def diffusion_reaction_bands(diffusion: float, reaction: float, h: float):
    """assemble_spatial_operator, 1D branch (src/pde.cpp:55-64), op for op."""
    mu_h2 = diffusion / (h * h)
    return -mu_h2, 2.0 * mu_h2 + reaction, -mu_h2


def advection_diffusion_bands(nu: float, a: float, h: float):
    """Central-difference -nu u_xx + a u_x (no reference assembler exists;
    the reference runs it through a hand-built CSR, pde.hpp:36-37)."""
    mu_h2 = nu / (h * h)
    adv = a / (2.0 * h)
    return -mu_h2 - adv, 2.0 * mu_h2, -mu_h2 + adv


def step_coefficients(problem: Problem1D, role: int = _lib.PIT_FINE, fine_layout=None,
                      coarse_layout=None):
    """Host-side coefficient struct of one propagator role (no GPU needed)."""
    d, keep = problem.desc(0, fine_layout, coarse_layout)
    c = _lib.StepCoeffsC()
    _check(_lib.lib().pit_step_coefficients(C.byref(d), role, C.byref(c)))
    zc = np.zeros(problem.M)
    _check(_lib.lib().pit_step_correction(C.byref(d), role, dptr(zc)))
    return c, zc


def step_positions(problem: Problem1D, role: int = _lib.PIT_FINE, fine_layout=None,
                   coarse_layout=None):
    """Per-thread weights (ppos, qpos, zt) of one role."""
    c, _ = step_coefficients(problem, role, fine_layout, coarse_layout)
    d, keep = problem.desc(0, fine_layout, coarse_layout)
    T = 32 * c.warps
    pp, qp, zt = np.zeros(T), np.zeros(T), np.zeros(T)
    _check(_lib.lib().pit_step_positions(C.byref(d), role, dptr(pp), dptr(qp), dptr(zt)))
    return pp, qp, zt


# ---------------------------------------------------------------------------
# RunStats / history / config (include/pit/executor.hpp, solvers.hpp)
# ---------------------------------------------------------------------------

@dataclass
class RunStats:
    fine_applications: int = 0
    coarse_applications: int = 0
    fine_parallel_ms: float = 0.0
    fine_busy_ms: float = 0.0
    coarse_sequential_ms: float = 0.0

    def _accumulate(self, s: "_lib.RunStatsC") -> None:
        self.fine_applications += s.fine_applications
        self.coarse_applications += s.coarse_applications
        self.fine_parallel_ms += s.fine_parallel_ms
        self.fine_busy_ms += s.fine_busy_ms
        self.coarse_sequential_ms += s.coarse_sequential_ms


class SolveStatus(enum.Enum):
    Converged = "converged"
    MaxIterations = "max-iterations"


class InitialGuessPolicy(enum.IntEnum):
    CoarseSweep = _lib.PIT_GUESS_COARSE_SWEEP
    Zero = _lib.PIT_GUESS_ZERO


@dataclass
class IterationRecord:
    k: int
    residual_norm: float
    fine_applications: int
    coarse_applications: int
    wall_ms: float = 0.0
    error_vs_reference: Optional[float] = None


@dataclass
class ConvergenceHistory:
    records: List[IterationRecord] = field(default_factory=list)
    status: SolveStatus = SolveStatus.MaxIterations
    restarts: int = 0
    stats: RunStats = field(default_factory=RunStats)
    min_restart_margin: float = float("inf")


@dataclass
class SolverConfig:
    tolerance: float = 1e-8
    restart_tolerance: float = 1e-12
    max_iterations: int = 200
    initial_guess: InitialGuessPolicy = InitialGuessPolicy.CoarseSweep

    def validate(self) -> None:
        """SolverConfig::validate (src/solvers.cpp:33-38)."""
        if not (self.tolerance > self.restart_tolerance) or not (self.restart_tolerance > 0.0):
            raise ConfigError("solver tolerances must satisfy tolerance > restart_tolerance > 0")
        if self.max_iterations < 1:
            raise ConfigError("max_iterations must be >= 1")

    def _c(self):
        c = _lib.SolverConfigC()
        c.tolerance = self.tolerance
        c.restart_tolerance = self.restart_tolerance
        c.max_iterations = self.max_iterations
        c.initial_guess = int(self.initial_guess)
        return c


@dataclass
class SolveOptions:
    initial_guess_override: Optional[np.ndarray] = None
    reference: Optional[np.ndarray] = None
    first_residual_out: Optional[np.ndarray] = None  # filled in place, shape (N, M)
    # called after every history row with (IterationRecord, lambda (N, M)),
    # as SolveOptions::iterate_observer (solvers.hpp:54); lambda is a copy
    iterate_observer: Optional[Callable] = None


@dataclass
class SolveResult:
    solution: np.ndarray
    history: ConvergenceHistory


# ---------------------------------------------------------------------------
# BlockOperatorContext
# ---------------------------------------------------------------------------

class BlockOperatorContext:
    """pit::BlockOperatorContext (include/pit/block_system.hpp:55-72): the
    partition, both propagators and the initial value, resident on one GPU."""

    def __init__(self, problem, device: int = 0, fine_layout=None,
                 coarse_layout=None):
        self.problem = problem
        d, keep = problem.desc(device, fine_layout, coarse_layout)
        h = C.c_void_p()
        _check(_lib.lib().pit_context_create(C.byref(d), C.byref(h)))
        self._h = h
        self.M = problem.M
        self.N = problem.N
        self.spacing = problem.spacing

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().pit_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def block_count(self) -> int:
        return self.N

    def coarse_iterations(self) -> int:
        """Cumulative inner CG iterations of the 2D coarse sweeps (0 in 1D)."""
        v = C.c_int64()
        _check(_lib.lib().pit_coarse_iterations(self._h, C.byref(v)))
        return v.value

    def zero_vector(self) -> np.ndarray:
        return np.zeros((self.N, self.M))

    def initial_value(self) -> np.ndarray:
        return np.asarray(self.problem.y0, dtype=np.float64)

    def _vec(self, v: np.ndarray, what: str) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.ndim != 2 or v.shape[0] != self.N:
            raise ValueError(f"{what}: block count does not match the partition")
        if v.shape[1] != self.M:
            raise ValueError("ScalarField: grid mismatch")
        return v


def _stats_out(stats: Optional[RunStats]):
    return _lib.RunStatsC() if stats is not None else None


def _stats_in(stats, sc):
    if stats is not None:
        stats._accumulate(sc)


def apply_F(ctx: BlockOperatorContext, L: np.ndarray, exec=None,
            stats: Optional[RunStats] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
    """(F L)_0 = L_0, (F L)_n = L_n - FineHom(L_{n-1})  (block_system.cpp:115-147).
    `exec` (a SlabExecutor) is accepted for signature compatibility; the
    slab fan-out is the kernel grid.  With page-locked `L` and `out` (e.g.
    torch pin_memory) the copies overlap the kernel (pit_apply_F)."""
    L = ctx._vec(L, "apply_F")
    if out is None:
        out = np.empty_like(L)
    elif out.shape != L.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("apply_F: out must be a C-contiguous float64 array of L's shape")
    sc = _stats_out(stats)
    _check(_lib.lib().pit_apply_F(ctx.handle, dptr(L), dptr(out), C.byref(sc) if sc else None))
    _stats_in(stats, sc)
    return out


def assemble_rhs(ctx: BlockOperatorContext, exec=None,
                 stats: Optional[RunStats] = None) -> np.ndarray:
    """B_0 = y0, B_n = fine.source_contribution(n-1)  (block_system.cpp:149-172)."""
    out = ctx.zero_vector()
    sc = _stats_out(stats)
    _check(_lib.lib().pit_assemble_rhs(ctx.handle, dptr(out), C.byref(sc) if sc else None))
    _stats_in(stats, sc)
    return out


def apply_G_inverse(ctx: BlockOperatorContext, V: np.ndarray,
                    stats: Optional[RunStats] = None) -> np.ndarray:
    """W_0 = V_0, W_n = CoarseHom(W_{n-1}) + V_n  (block_system.cpp:174-195)."""
    V = ctx._vec(V, "apply_G_inverse")
    out = np.empty_like(V)
    sc = _stats_out(stats)
    _check(_lib.lib().pit_apply_G_inverse(ctx.handle, dptr(V), dptr(out),
                                          C.byref(sc) if sc else None))
    _stats_in(stats, sc)
    return out


def initial_guess(ctx: BlockOperatorContext, policy: InitialGuessPolicy,
                  stats: Optional[RunStats] = None) -> np.ndarray:
    """solvers.cpp:49-64."""
    out = ctx.zero_vector()
    sc = _stats_out(stats)
    _check(_lib.lib().pit_initial_guess(ctx.handle, int(policy), dptr(out),
                                        C.byref(sc) if sc else None))
    _stats_in(stats, sc)
    return out


def preconditioned_residual(ctx: BlockOperatorContext, lam: np.ndarray, rhs: np.ndarray,
                            exec=None, stats: Optional[RunStats] = None) -> np.ndarray:
    """G^-1 (B - F lam)  (solvers.cpp:66-71)."""
    lam = ctx._vec(lam, "apply_F")
    rhs = ctx._vec(rhs, "apply_F")
    out = np.empty_like(lam)
    sc = _stats_out(stats)
    _check(_lib.lib().pit_preconditioned_residual(ctx.handle, dptr(lam), dptr(rhs), dptr(out),
                                                  C.byref(sc) if sc else None))
    _stats_in(stats, sc)
    return out


def sequential_fine_solve(ctx: BlockOperatorContext) -> np.ndarray:
    """solvers.cpp:40-47: lambda*_n = fine.propagate(lambda*_{n-1}, n-1)."""
    out = ctx.zero_vector()
    _check(_lib.lib().pit_sequential_fine_solve(ctx.handle, dptr(out)))
    return out


class _PropagatorView:
    def __init__(self, ctx: BlockOperatorContext, role: int):
        self.ctx, self.role = ctx, role

    def _run(self, lam, slab, with_source):
        ctx = self.ctx
        out = np.empty(ctx.M)
        if lam is not None:
            lam = np.ascontiguousarray(lam, dtype=np.float64)
            if lam.shape != (ctx.M,):
                raise ValueError("Propagator: field grid does not match operator grid")
        _check(_lib.lib().pit_propagate(ctx.handle, self.role, int(with_source), dptr(lam),
                                        int(slab), dptr(out)))
        return out

    def propagate(self, lam, slab_index: int):
        """Propagator::propagate (propagator.hpp:38)."""
        return self._run(lam, slab_index, True)

    def propagate_homogeneous(self, lam, slab_index: int):
        """Propagator::propagate_homogeneous (propagator.hpp:41)."""
        return self._run(lam, slab_index, False)

    def source_contribution(self, slab_index: int):
        """Propagator::source_contribution (propagator.hpp:44)."""
        return self._run(None, slab_index, True)


def fine(ctx: BlockOperatorContext) -> _PropagatorView:
    return _PropagatorView(ctx, _lib.PIT_FINE)


def coarse(ctx: BlockOperatorContext) -> _PropagatorView:
    return _PropagatorView(ctx, _lib.PIT_COARSE)


def block_inner_product(ctx: BlockOperatorContext, a: np.ndarray, b: np.ndarray) -> float:
    """block_system.cpp:76-81 (device reduction order)."""
    a = ctx._vec(a, "block_inner_product")
    b = ctx._vec(b, "block_inner_product")
    out = C.c_double()
    _check(_lib.lib().pit_block_inner_product(ctx.handle, dptr(a), dptr(b), C.byref(out)))
    return out.value


def block_norm_n_inf(ctx: BlockOperatorContext, a: np.ndarray) -> float:
    """block_system.cpp:83-87."""
    a = ctx._vec(a, "block_norm_n_inf")
    out = C.c_double()
    _check(_lib.lib().pit_block_norm_n_inf(ctx.handle, dptr(a), C.byref(out)))
    return out.value


def _solve(which: int, ctx: BlockOperatorContext, config: SolverConfig,
           options: Optional[SolveOptions]) -> SolveResult:
    config.validate()
    options = options or SolveOptions()
    init = None
    if options.initial_guess_override is not None:
        init = ctx._vec(options.initial_guess_override, "initial guess")
    lam = ctx.zero_vector()
    first = None
    if options.first_residual_out is not None:
        first = ctx.zero_vector()
    cap = config.max_iterations + 2
    recs = (_lib.RecordC * cap)()
    info = _lib.SolveInfoC()
    cfg = config._c()
    fn = _lib.lib().pit_pitsbicg_solve if which == 0 else _lib.lib().pit_parareal_solve
    ref = None
    if options.reference is not None:
        ref = ctx._vec(options.reference, "reference")
        _check(_lib.lib().pit_set_reference(ctx.handle, dptr(ref)))
    cb = None
    if options.iterate_observer is not None:
        user_fn = options.iterate_observer

        def _observe(row, lam_p, n, m, _user):
            r = row.contents
            rec = IterationRecord(r.k, r.residual_norm, r.fine_applications, r.coarse_applications,
                                  r.wall_ms, r.error_vs_reference if r.has_error else None)
            user_fn(rec, np.ctypeslib.as_array(lam_p, shape=(n, m)).copy())

        cb = _lib.ITERATE_OBSERVER(_observe)
        _check(_lib.lib().pit_set_iterate_observer(ctx.handle, cb, None))
    try:
        _check(fn(ctx.handle, C.byref(cfg), dptr(init), dptr(lam), dptr(first), recs, cap,
                  C.byref(info)))
    finally:
        if ref is not None:
            _lib.lib().pit_set_reference(ctx.handle, None)
        if cb is not None:
            _lib.lib().pit_set_iterate_observer(ctx.handle, _lib.ITERATE_OBSERVER(), None)
    hist = ConvergenceHistory()
    for i in range(info.record_count):
        r = recs[i]
        hist.records.append(IterationRecord(r.k, r.residual_norm, r.fine_applications,
                                            r.coarse_applications, r.wall_ms,
                                            r.error_vs_reference if r.has_error else None))
    hist.status = SolveStatus.Converged if info.status == _lib.PIT_CONVERGED \
        else SolveStatus.MaxIterations
    hist.restarts = info.restarts
    hist.stats._accumulate(info.stats)
    hist.min_restart_margin = info.min_restart_margin
    if first is not None:
        options.first_residual_out[...] = first
    return SolveResult(lam, hist)


def pitsbicg_solve(ctx: BlockOperatorContext, config: SolverConfig = SolverConfig(), exec=None,
                   options: Optional[SolveOptions] = None) -> SolveResult:
    """Left-preconditioned BiCGStab on G^-1 F L = G^-1 B  (solvers.cpp:116-220)."""
    return _solve(0, ctx, config, options)


def parareal_solve(ctx: BlockOperatorContext, config: SolverConfig = SolverConfig(), exec=None,
                   options: Optional[SolveOptions] = None) -> SolveResult:
    """Fixed-point L <- L + G^-1 (B - F L)  (solvers.cpp:73-114)."""
    return _solve(1, ctx, config, options)


def seeded_uniform(seed: int, n: int, a: float = -1.0, b: float = 1.0) -> np.ndarray:
    out = np.empty(n)
    _lib.lib().pit_seeded_uniform(seed, n, a, b, dptr(out))
    return out


def seeded_normal(seed: int, n: int, mean: float = 0.0, stddev: float = 1.0) -> np.ndarray:
    out = np.empty(n)
    _lib.lib().pit_seeded_normal(seed, n, mean, stddev, dptr(out))
    return out
