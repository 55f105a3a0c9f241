#!/usr/bin/env python
"""bench.py — PiT matvec throughput (fine-propagation gridpoint-steps/s).

Workload: BASELINE config c2 (1D heat, M=4096, N=1024 slabs, 1000 backward
Euler steps per slab) — the configuration BASELINE.json's metric is quoted on
(configs[1]).  One "step" = one apply_F over all slabs of the shard:
M * 1000 * (slabs propagated) gridpoint-steps, inputs resident in HBM.  c4
(the largest single-GPU 1D config) is measured the same way in `c4`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 re-launches itself under torch.distributed.run (one rank per
GPU, NCCL) unless it already runs under it: every rank owns a c2-size shard
(1024 slabs) of a 1024*N-slab problem and exchanges one boundary block per
apply (weak scaling).

The reference arm (--impl reference) times the reference's own CPU apply_F
(oracle/_ref/libpitref.so, compiled from the unmodified /root/reference
sources by oracle/Makefile) on the box's host cores, on rank 0 only, each
step a bounded sample of the same workload.  It does not import this
package (inputs come from the reference driver's own seeded generators).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-propagation gridpoint-steps/s (PiT matvec apply_F)"
UNIT = "gridpoint-steps/s"
HEADLINE = "c2"
FLOPS_PER_GP_STEP = 5  # 1D BE step with precomputed LU factors
SEED = 1234

# Workload shapes (BASELINE.json configs; the same numbers as
# paper_2203_10148_b200/configs.py, restated here so that the reference arm
# never imports the product package).
WORKLOADS = {
    "c1": dict(M=100, N=16, fine=100, coarse=1,
               desc="1D heat u_t=u_xx, M=100, N=16, T=1, fine 100 BE/slab, coarse 1, "
                    "y0=sin(pi x)"),
    "c2": dict(M=4096, N=1024, fine=1000, coarse=1,
               desc="1D heat, M=4096, N=1024, fine 1000 BE/slab, coarse 1, "
                    "y0=sum_8 N(0,1) sine modes"),
    "c4": dict(M=8192, N=2048, fine=500, coarse=1,
               desc="1D react-diff r=5 + sin(2pi t)sin(pi x), M=8192, N=2048, fine 500 BE/slab, "
                    "coarse 1"),
}

# Issue ceiling of any chunked (parallel) tridiagonal solve: every point is
# swept twice per direction, >= 4 DFMA = 8 pipe flops per
# point-step against the 5 credited flops; K1 issues 4.69 DFMA per point-step
# (ncu, profiles/r1b_ncu_slab_kernel_c2.txt).
ISSUE_CEILING = {"any_chunked_solve": 5.0 / 8.0, "this_kernel": 5.0 / (2 * 4.69),
                 "source": "DESIGN.md §6; DFMA count from profiles/r1b_ncu_slab_kernel_c2.txt"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the per-config apply_F and time-to-tolerance lines")
    ap.add_argument("--cpu-ttt-all", action="store_true",
                    help="also time the reference's c3 solve and the oracle's c4 solve on the host "
                         "(minutes)")
    return ap.parse_args()


def workload_config(name, world):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    w = WORKLOADS[name]
    total = w["N"] * world
    return {"workload": f"{name}: {w['desc']}", "M": w["M"], "slabs_per_gpu": w["N"],
            "slabs_total": total, "fine_steps": w["fine"],
            "gp_steps_per_apply_total": w["M"] * w["fine"] * (total - 1),
            "l2": "flushed between timed iterations (256 MB write)",
            "parallelism": f"slab-sharded x{world}" if world > 1 else "single GPU"}


# ---------------------------------------------------------------------------
# clocks during the timed region (pynvml sampling thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# the reference on the host cores (no product import on this path)
# ---------------------------------------------------------------------------
def _ref():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O

    if not os.path.exists(O.REF_SO):
        return None, O
    return O.ref(), O


def ref_inputs(R, O, name, M):
    """BASELINE inputs from the reference driver's seeded
    generators: x_i = (i+1)h, seed 1234."""
    h = 1.0 / (M + 1)
    x = np.array([(k + 1) * h for k in range(M)])
    if name == "c1":
        return np.ascontiguousarray(np.sin(math.pi * x))
    if name == "c2":
        a = np.zeros(8)
        R.pitref_seeded_normal(SEED, 8, 0.0, 1.0, O.ptr(a))
        y0 = np.zeros(M)
        for k in range(8):
            y0 += a[k] * np.sin((k + 1) * math.pi * x)
        return np.ascontiguousarray(y0)
    raise KeyError(name)


class RefSample:
    """The reference's pit::apply_F with SlabExecutor(cores) on a bounded
    sample of the workload: 4*cores + 1 blocks (4*cores fine propagations at
    the config's own dt and steps per slab), so every pool round is full."""

    def __init__(self, name="c2"):
        self.R, self.O = _ref()
        if self.R is None:
            raise RuntimeError("oracle/_ref/libpitref.so not built")
        w = WORKLOADS[name]
        self.cores = os.cpu_count() or 1
        self.slabs = 4 * self.cores + 1
        M, fs = w["M"], w["fine"]
        T = 1.0 * self.slabs / w["N"]  # the full config's slab length
        y0 = ref_inputs(self.R, self.O, name, M)
        self.h = self.R.pitref_create_1d(M, 0.0, 1.0, 1.0, 0.0, 0, 0.0, 0.0, 0.0, 1, self.slabs, T,
                                         fs, w["coarse"], self.O.ptr(y0), 0, None, 0.0, 0.0, 0.0)
        assert self.h, self.R.pitref_last_error()
        self.L = np.ascontiguousarray(np.tile(y0, (self.slabs, 1)))
        self.out = np.zeros_like(self.L)
        self.gp = M * fs * (self.slabs - 1)
        self.sample = (f"pit::apply_F on {self.slabs} blocks ({self.slabs - 1} fine propagations "
                       f"of 1000 BE steps at the {name} dt) per step, SlabExecutor({self.cores})")

    def step(self):
        t0 = time.perf_counter()
        rc = self.R.pitref_apply_F(self.h, self.O.ptr(self.L), self.O.ptr(self.out), self.cores)
        dt = time.perf_counter() - t0
        if rc:
            raise RuntimeError(self.R.pitref_last_error())
        return dt

    def close(self):
        self.R.pitref_destroy(self.h)


def ref_time_to_tolerance_c1(R, O):
    """The reference's pitsbicg_solve on full c1 (SurveY §8(d) metric 2),
    SlabExecutor(cores): wall time, k, restarts."""
    w = WORKLOADS["c1"]
    cores = os.cpu_count() or 1
    y0 = ref_inputs(R, O, "c1", w["M"])
    h = R.pitref_create_1d(w["M"], 0.0, 1.0, 1.0, 0.0, 0, 0.0, 0.0, 0.0, 1, w["N"], 1.0, w["fine"],
                           w["coarse"], O.ptr(y0), 0, None, 0.0, 0.0, 0.0)
    return _ref_solve(R, O, h, w["N"], w["M"], cores, "full c1")


def _ref_solve(R, O, h, N, M, cores, what, tol=1e-10, reps=3):
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    lam = np.zeros((N, M))
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        rc = R.pitref_pitsbicg(h, tol, 1e-12, 200, 0, cores, None, O.ptr(lam), None, k, res, fa, ca,
                               cap, C.byref(nrec), C.byref(rs), C.byref(conv))
        dt = (time.perf_counter() - t0) * 1e3
        if rc:
            R.pitref_destroy(h)
            return {"error": R.pitref_last_error().decode()}
        best = dt if best is None else min(best, dt)
    n = min(nrec.value, cap)
    R.pitref_destroy(h)
    return {"ms": best, "cores": cores, "k": k[n - 1], "restarts": rs.value,
            "residual": res[n - 1], "kind": "reference", "sample": f"{what}, best of {reps}"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return  # rank 0 alone times the host CPU path
    S = RefSample(HEADLINE)
    for _ in range(args.warmup):
        S.step()
    times = [S.step() for _ in range(args.steps)]
    total = float(np.sum(times))
    v = S.gp * args.steps / total
    cpu = {"value": v, "unit": UNIT, "cores": S.cores, "kind": "reference", "sample": S.sample}
    ttt = ref_time_to_tolerance_c1(S.R, S.O)
    S.close()
    cpu["time_to_tolerance"] = {"c1": ttt}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {HEADLINE} inputs, seed {SEED})",
        "config": workload_config(HEADLINE, world),
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def device_apply_rate(name, reps=3, slabs=None):
    """Best-of-reps device apply_F (inputs resident, dedicated stream) of a
    full BASELINE config (or the same per-slab work on `slabs` slabs):
    (gp-steps/s, ms, gp-steps)."""
    import torch

    from paper_2203_10148_b200 import _lib, api, configs

    L = _lib.lib()
    p = configs.make(name, slabs=slabs)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream), api.BlockOperatorContext(p) as ctx:
        x = torch.tensor(np.tile(p.y0, (p.N, 1)), device="cuda")
        out = torch.empty_like(x)
        f = lambda: api._check(L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(),
                                                    0, p.N, stream.cuda_stream))
        f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            f()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        api._check(L.pit_sync_status(ctx.handle, stream.cuda_stream))
    gp = configs.gp_steps_per_apply(p)
    ms = min(ts)
    return gp / (ms * 1e-3), ms, gp


def measure_single(name, steps, warmup, peak, flush):
    """One config on one GPU: device-resident apply_F over `steps` timed
    launches (L2 flushed between them, CUDA events on the launching stream),
    the roofline of K1, and the e2e rate of the public host-buffer call."""
    import torch

    from paper_2203_10148_b200 import _lib, api, configs

    L = _lib.lib()
    p = configs.make(name)
    gp = configs.gp_steps_per_apply(p)
    stream = torch.cuda.Stream()
    rng = np.random.default_rng(SEED)
    Lh = np.ascontiguousarray(np.tile(p.y0, (p.N, 1)) * (1.0 + 0.01 * rng.standard_normal((p.N, 1))))
    out_line = {}
    with torch.cuda.stream(stream), api.BlockOperatorContext(p) as ctx:
        Ld = torch.tensor(Lh, device="cuda")
        out = torch.empty_like(Ld)
        st = stream.cuda_stream

        def kernel():
            rc = L.pit_apply_F_device(ctx.handle, Ld.data_ptr(), None, out.data_ptr(), 0, p.N, st)
            if rc:
                api._check(rc)

        for _ in range(warmup):
            kernel()
            flush.zero_()
        torch.cuda.synchronize()
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        for i in range(steps):
            flush.zero_()
            e0[i].record(stream)
            kernel()
            e1[i].record(stream)
        torch.cuda.synchronize()
        api._check(L.pit_sync_status(ctx.handle, st))
        ms = [e0[i].elapsed_time(e1[i]) for i in range(steps)]
        kms = float(np.mean(ms))
        # e2e: the public host call on pinned buffers, copies inside
        Lpin = torch.from_numpy(Lh).pin_memory()
        Opin = torch.empty_like(Lpin).pin_memory()
        Ln, On = Lpin.numpy(), Opin.numpy()
        api.apply_F(ctx, Ln, out=On)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            r = L.pit_apply_F(ctx.handle, _lib.dptr(Ln), _lib.dptr(On), None)
            if r:
                api._check(r)
        e2e_s = time.perf_counter() - t0
    achieved = FLOPS_PER_GP_STEP * gp / (kms * 1e-3) / 1e12
    out_line = {
        "value": gp / (kms * 1e-3), "unit": UNIT, "ms_per_step": kms, "steps": steps,
        "config": workload_config(name, 1),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "algorithmic": f"{FLOPS_PER_GP_STEP} flop per gridpoint-step x {gp} "
                                    "gp-steps per launch",
                     "kernel_ms": kms},
        "e2e": {"value": gp * steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(Ln.nbytes), "d2h_bytes_per_step": int(On.nbytes),
                "api": "pit_apply_F (host buffers, pinned)"},
        "gpu_launches": steps,
    }
    return out_line


def device_time_to_tolerance(name):
    """PiTSBiCG (SURVEY §8(d) metric 2) through pit_pitsbicg_solve_device:
    wall time from solver entry (inputs resident) to ||R|| <= tol, including
    initial_guess, assemble_rhs and every iteration."""
    import torch

    from paper_2203_10148_b200 import _lib, api, configs

    L = _lib.lib()
    p = configs.make(name)
    tol = configs.tolerance(name)
    with api.BlockOperatorContext(p) as ctx:
        lam = torch.empty((p.N, p.M), dtype=torch.float64, device="cuda")
        cfg = _lib.SolverConfigC(tol, 1e-12, 200, _lib.PIT_GUESS_COARSE_SWEEP)
        recs = (_lib.RecordC * 202)()
        info = _lib.SolveInfoC()
        # first solve allocates the context's work vectors; time the best of
        # the next ones
        api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(),
                                               recs, 202, C.byref(info), None))
        its0 = ctx.coarse_iterations()
        walls = []
        reps = 1 if name == "c5" else 3
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(),
                                                   recs, 202, C.byref(info), None))
            walls.append(time.perf_counter() - t0)
        n = min(info.record_count, 202)
        its = (ctx.coarse_iterations() - its0) // reps
    last = recs[n - 1] if n else None
    out = {"ms": min(walls) * 1e3, "k": last.k if last else None,
           "residual": last.residual_norm if last else None, "restarts": info.restarts,
           "converged": info.status == _lib.PIT_CONVERGED, "tolerance": tol,
           "fine_applications": int(info.stats.fine_applications),
           "coarse_applications": int(info.stats.coarse_applications)}
    if its:
        out["coarse_cg_iterations"] = int(its)
    if name == "c5":
        out["coarse_cg_tolerance"] = configs.C5_COARSE_TOL
        out["coarse_cg_tolerance_note"] = (
            f"BASELINE asks {configs.C5_BASELINE_COARSE_TOL:g}, below this system's FP64 "
            "true-residual floor (6.4e-13); the reference's own kInnerSolveRelTol is used "
            "(DESIGN.md §3.6)")
    return out


PRESET_LINES = (("diffusion", "desk", 16), ("advection_diffusion_reaction", "desk", 16),
                ("advection_diffusion_reaction", "paper", 64))


def preset_time_to_tolerance(case, scale, n, with_reference=False):
    """The reference's own experiments (presets.cpp; K6):
    device PiTSBiCG to the runner's default 1e-8 (warm solve, inputs
    resident), beside the reference's pitsbicg_solve on the host cores
    (oracle/_ref, SlabExecutor(nproc)) when that library is present."""
    import torch

    from paper_2203_10148_b200 import _lib, api, presets

    L = _lib.lib()
    p = presets.build_problem(presets.make_preset(case, scale), n)
    with api.BlockOperatorContext(p) as ctx:
        lam = torch.empty((p.N, p.M), dtype=torch.float64, device="cuda")
        cfg = _lib.SolverConfigC(1e-8, 1e-12, 200, _lib.PIT_GUESS_COARSE_SWEEP)
        recs = (_lib.RecordC * 202)()
        info = _lib.SolveInfoC()
        for _ in range(2):  # time the second (work vectors allocated by the first)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None,
                                                   lam.data_ptr(), recs, 202, C.byref(info), None))
            wall = time.perf_counter() - t0
    n_rec = min(info.record_count, 202)
    out = {"N": n, "m": p.m, "ms": wall * 1e3, "k": recs[n_rec - 1].k,
           "restarts": info.restarts, "converged": info.status == _lib.PIT_CONVERGED}
    R, O = _ref()
    if with_reference and R is not None:
        h = R.pitref_create_preset(presets.CASES.index(case), 0 if scale == "desk" else 1, n)
        out["reference_cpu"] = _ref_solve(R, O, h, p.N, p.M, os.cpu_count() or 1,
                                          f"{scale}/{case} N={n}", tol=1e-8, reps=1)
    return out


def secondary(include_c5_solve=True):
    out = {"apply_F": {}, "time_to_tolerance": {}, "presets_time_to_tolerance": {}}
    for case, scale, n in PRESET_LINES:
        try:
            out["presets_time_to_tolerance"][f"{scale}/{case}"] = preset_time_to_tolerance(
                case, scale, n)
        except Exception as e:  # pragma: no cover
            out["presets_time_to_tolerance"][f"{scale}/{case}"] = {"error": str(e)}
    for name in ("c1", "c3", "c5"):
        try:
            rate, ms, gp = device_apply_rate(name)
            out["apply_F"][name] = {"gp_steps_per_s": rate, "ms": ms, "gp_steps": gp}
        except Exception as e:  # pragma: no cover
            out["apply_F"][name] = {"error": str(e)}
    # the same K1 on ten waves of c2 slabs (8881 blocks): the rate the kernel
    # sustains when finished CTAs are replaced at once; c2's 1023 slabs are
    # 1.15 waves of 888 resident CTAs
    try:
        rate, ms, gp = device_apply_rate("c2", slabs=8881)
        out["apply_F"]["c2_ten_waves"] = {"gp_steps_per_s": rate, "ms": ms, "gp_steps": gp,
                                          "slabs": 8880}
    except Exception as e:  # pragma: no cover
        out["apply_F"]["c2_ten_waves"] = {"error": str(e)}
    for name in ("c1", "c2", "c3", "c4") + (("c5",) if include_c5_solve else ()):
        try:
            out["time_to_tolerance"][name] = device_time_to_tolerance(name)
        except Exception as e:  # pragma: no cover
            out["time_to_tolerance"][name] = {"error": str(e)}
    return out


def oracle_time_to_tolerance(name):
    """The restated oracle (CPU, OpenMP over slabs, all host cores) where the
    reference cannot run the config (c2/c4: its coarse CG hits the 10n cap;
    SURVEY §8(c)); labelled kind "port"."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import OracleProblem

    from paper_2203_10148_b200 import configs

    p = configs.make(name)
    o = OracleProblem(p)
    t0 = time.perf_counter()
    r = o.solve(configs.tolerance(name))
    ms = (time.perf_counter() - t0) * 1e3
    o.close()
    return {"ms": ms, "cores": os.cpu_count() or 1, "k": r["rows"][-1][0],
            "restarts": r["restarts"], "residual": r["rows"][-1][1], "kind": "port",
            "sample": f"full {name}: the restated oracle (oracle/pit_oracle.c, OpenMP over slabs); "
                      "the reference itself stops with InnerSolveError on this config"}


def cpu_baseline(args, include_ttt):
    S = RefSample(HEADLINE)
    times = [S.step() for _ in range(3)]
    v = S.gp / min(times)
    out = {"value": v, "unit": UNIT, "cores": S.cores, "kind": "reference",
           "sample": S.sample + ", best of 3"}
    if include_ttt:
        ttt = {"c1": ref_time_to_tolerance_c1(S.R, S.O), "c2": oracle_time_to_tolerance("c2")}
        if args.cpu_ttt_all:
            from paper_2203_10148_b200 import configs

            p = configs.make("c3")
            y0 = np.ascontiguousarray(p.y0)
            h = S.R.pitref_create_1d(p.M, 0.0, 1.0, 0.0, 0.0, 1, p.band_lo, p.band_diag, p.band_up,
                                     0, p.N, p.T, p.fine_steps, p.coarse_steps, S.O.ptr(y0), 0,
                                     None, 0.0, 0.0, 0.0)
            ttt["c3"] = _ref_solve(S.R, S.O, h, p.N, p.M, S.cores, "full c3", reps=1)
            ttt["c4"] = oracle_time_to_tolerance("c4")
        out["time_to_tolerance"] = ttt
        pre = {}
        for case, scale, n in PRESET_LINES:
            r = preset_time_to_tolerance(case, scale, n, with_reference=True)
            pre[f"{scale}/{case}"] = r.get("reference_cpu")
        out["presets_time_to_tolerance"] = pre
    S.close()
    return out


def run_ours(args, rank, world):
    import torch

    from paper_2203_10148_b200 import _lib, api, configs
    from paper_2203_10148_b200.distributed import Communicator, ShardedContext

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    L = _lib.lib()
    base = configs.make(HEADLINE)
    n_global = base.N * world  # weak scaling: one c2-size shard per rank
    p = configs.make(HEADLINE, slabs=n_global) if world > 1 else base
    ctx = api.BlockOperatorContext(p, device=dev)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream
    dist = None
    sc = comm = None
    if world > 1:
        import torch.distributed as dist

        # the library's own NCCL communicator (rank 0's id over the process
        # group): halo exchange overlapped with the interior slabs inside
        # pit_sharded_apply_F_device
        comm = Communicator.from_process_group(dev, transport="nccl")
        sc = ShardedContext(ctx, comm)
        first, count = sc.first, sc.count
    else:
        first, count = 0, p.N
    gp_local = p.M * p.fine_steps * (count - 1 if first == 0 else count)

    # inputs resident in HBM: the seeded trajectory-like block vector
    rng = np.random.default_rng(SEED + rank)
    Lh = np.ascontiguousarray(np.tile(p.y0, (count, 1)) * (1.0 + 0.01 * rng.standard_normal((count, 1))))
    Ld = torch.tensor(Lh, device="cuda")
    out = torch.empty_like(Ld)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2

    def kernel():
        if world > 1:
            rc = L.pit_sharded_apply_F_device(ctx.handle, Ld.data_ptr(), out.data_ptr(), st)
        else:
            rc = L.pit_apply_F_device(ctx.handle, Ld.data_ptr(), None, out.data_ptr(), 0, count, st)
        if rc:
            api._check(rc)

    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for _ in range(args.warmup):
        kernel()
        flush.zero_()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev)
    with sampler:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            e0[i].record(stream)
            kernel()
            e1[i].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    api._check(L.pit_sharded_sync_status(ctx.handle, st))
    step_ms = [e0[i].elapsed_time(e1[i]) for i in range(args.steps)]
    kern_ms = step_ms
    total_ms = float(np.sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    gpt = torch.tensor([float(gp_local)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(gpt, op=dist.ReduceOp.SUM)
    total_ms = float(t.item())
    gp_total = float(gpt.item())
    value = gp_total * args.steps / (total_ms * 1e-3)

    # ---- e2e: public API with pinned host buffers, H2D + D2H inside ------
    Lpin = torch.from_numpy(Lh).pin_memory()
    Opin = torch.empty_like(Lpin).pin_memory()
    if world == 1:
        Ln, On = Lpin.numpy(), Opin.numpy()
        api.apply_F(ctx, Ln, out=On)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = L.pit_apply_F(ctx.handle, _lib.dptr(Ln), _lib.dptr(On), None)
            if r:
                api._check(r)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": gp_local * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(Ln.nbytes), "d2h_bytes_per_step": int(On.nbytes),
               "api": "api.apply_F / pit_apply_F (host buffers)"}
    else:
        # sharded public API: host shard in, halo over NCCL, host shard out
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dL = Lpin.to("cuda", non_blocking=True)
            o = sc.apply_F(dL, stream)
            Opin.copy_(o, non_blocking=True)
            torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": gp_total * args.steps / float(tt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(Lh.nbytes), "d2h_bytes_per_step": int(Lh.nbytes),
               "api": "distributed.ShardedContext.apply_F (pit_sharded_apply_F_device, "
                      "host shards)"}

    # ---- roofline: FP64 pipe (measured in-run) ---------------------------
    peak = C.c_double()
    api._check(L.pit_measure_fp64_peak(dev, C.byref(peak)))
    kms = float(np.mean(kern_ms))
    achieved = FLOPS_PER_GP_STEP * gp_local / (kms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(HEADLINE)
        except Exception:
            traffic = None

    if rank != 0:
        if sc is not None:
            sc.detach()
            comm.close()
        ctx.close()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {HEADLINE} inputs: seeded 8-mode sine initial value, "
                f"seed {SEED})",
        "config": workload_config(HEADLINE, world),
        "kernel_layout": {"points_per_thread": api.step_coefficients(p)[0].mpt,
                          "warps_per_slab": api.step_coefficients(p)[0].warps},
        "e2e": e2e,
        # one slab_kernel launch per apply_F (two when sharded: the
        # interior slabs and, after the halo, the boundary slab)
        "gpu_launches": args.steps * (2 if world > 1 and rank > 0 else 1),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value,
                     "unit": "TFLOP/s", "frac": achieved / peak.value, "traffic": traffic,
                     "algorithmic": f"{FLOPS_PER_GP_STEP} flop per gridpoint-step x "
                                    f"{gp_local} gp-steps per launch",
                     "peak_source": "measured in-run: FP64 DFMA probe (MEASURED_PEAKS.json "
                                    "has no FP64 figure)",
                     "kernel_ms": kms, "issue_ceiling": ISSUE_CEILING},
        "clocks": sampler.summary(),
    }
    if world == 1:
        line["c4"] = measure_single("c4", args.steps, args.warmup, peak.value, flush)
    if world == 1 and not args.no_secondary:
        line["secondary"] = secondary()
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args, include_ttt=not args.no_secondary)
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    if sc is not None:
        sc.detach()
        comm.close()
    ctx.close()


def relaunch(args):
    """--gpus N without a torchrun environment: run N ranks of this script
    under torch.distributed.run (one process per GPU) and return its code."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus < 1:
        sys.exit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    from paper_2203_10148_b200.distributed import init_from_env

    rank, world = init_from_env("nccl")
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
