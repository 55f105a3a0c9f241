#!/usr/bin/env python
"""bench.py — PiT matvec throughput (fine-propagation gridpoint-steps/s).

Workload: BASELINE config c2 (1D heat, M=4096, N=1024 slabs, 1000 backward
Euler steps per slab) — the configuration BASELINE.json's metric is quoted on
(configs[1]).  One "step" = one apply_F over all slabs of the shard:
M * 1000 * (slabs propagated) gridpoint-steps, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL): every rank owns a c2-size
shard (1024 slabs) of a 1024*N-slab problem and exchanges one boundary block
per apply (weak scaling).  The reference arm times the reference's own CPU
apply_F (oracle/_ref/libpitref.so, built from /root/reference sources) on the
box's host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-propagation gridpoint-steps/s (PiT matvec apply_F)"
UNIT = "gridpoint-steps/s"
CONFIG_NAME = "c2"
FLOPS_PER_GP_STEP = 5  # 1D BE step with precomputed LU factors


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the per-config apply_F and time-to-tolerance lines")
    return ap.parse_args()


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
# CPU baselines (reference library; oracle port as fallback)
# ---------------------------------------------------------------------------
def cpu_reference_rate(p, target_s=12.0, max_passes=3):
    """Reference apply_F (unmodified pit::apply_F with SlabExecutor(ncores)) on
    a slab subset of the workload, same dt and steps/slab.  Returns
    (gp-steps/s, cores, kind, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O

    from paper_2203_10148_b200 import configs

    cores = os.cpu_count() or 1
    if os.path.exists(O.REF_SO):
        R = O.ref()
        slabs = 2 * cores + 1
        q = configs.make(CONFIG_NAME, slabs=slabs + 1)
        y0 = np.ascontiguousarray(q.y0)
        h = R.pitref_create_1d(q.M, q.grid_lo, q.grid_hi, 1.0, 0.0, 0, 0.0, 0.0, 0.0, 1, q.N, q.T,
                               q.fine_steps, q.coarse_steps, O.ptr(y0), 0, None, 0.0, 0.0, 0.0)
        L = np.ascontiguousarray(np.tile(q.y0, (q.N, 1)))
        out = np.zeros_like(L)
        times = []
        t_all = time.perf_counter()
        for _ in range(max_passes):
            t0 = time.perf_counter()
            rc = R.pitref_apply_F(h, O.ptr(L), O.ptr(out), cores)
            times.append(time.perf_counter() - t0)
            if rc or time.perf_counter() - t_all > target_s:
                break
        R.pitref_destroy(h)
        gp = q.M * q.fine_steps * (q.N - 1)
        return gp / min(times), cores, "reference", \
            f"pit::apply_F on {q.N - 1} of 1023 c2 slabs (same dt, 1000 BE steps/slab), " \
            f"SlabExecutor({cores}), best of {len(times)}"
    # fallback: the oracle port (single thread)
    from helpers import OracleProblem  # noqa

    q = configs.make(CONFIG_NAME, slabs=3)
    o = OracleProblem(q)
    L = np.ascontiguousarray(np.tile(q.y0, (q.N, 1)))
    t0 = time.perf_counter()
    o.apply_F(L)
    dt = time.perf_counter() - t0
    return q.M * q.fine_steps * (q.N - 1) / dt, 1, "port", "oracle port apply_F on 2 c2 slabs, 1 thread"


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2203_10148_b200 import configs

    p = configs.make(CONFIG_NAME)
    rates = []
    for i in range(args.warmup + args.steps):
        r, cores, kind, sample = cpu_reference_rate(p, target_s=1e9, max_passes=1)
        if i >= args.warmup:
            rates.append(r)
    v = float(np.median(rates))
    gp_full = configs.gp_steps_per_apply(p)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        # one full c2 apply_F at the sampled rate (the sample covers 2*cores+1 slabs)
        "ms_per_step": gp_full / v * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE c2 inputs, seed 1234)",
        "config": {"workload": f"{CONFIG_NAME}: {configs.DESCRIPTIONS[CONFIG_NAME]}",
                   "sample": sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def device_apply_rate(name, reps=3):
    """Best-of-reps device apply_F (inputs resident, dedicated stream) of a
    full BASELINE config: (gp-steps/s, ms, kernel name)."""
    import torch

    from paper_2203_10148_b200 import _lib, api, configs

    L = _lib.lib()
    p = configs.make(name)
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
        # first solve allocates the context's work vectors; time the second
        api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(),
                                               recs, 202, C.byref(info), None))
        its0 = ctx.coarse_iterations()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(),
                                               recs, 202, C.byref(info), None))
        wall = time.perf_counter() - t0
        n = min(info.record_count, 202)
        its = ctx.coarse_iterations() - its0
    last = recs[n - 1] if n else None
    return {"ms": wall * 1e3, "k": last.k if last else None,
            "residual": last.residual_norm if last else None, "restarts": info.restarts,
            "converged": info.status == _lib.PIT_CONVERGED, "tolerance": tol,
            "fine_applications": int(info.stats.fine_applications),
            "coarse_applications": int(info.stats.coarse_applications),
            **({"coarse_cg_iterations": int(its)} if its else {})}


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
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libpitref.so")
    if with_reference and os.path.exists(ref_so):
        R = C.CDLL(ref_so)
        R.pitref_create_preset.restype = C.c_void_p
        R.pitref_create_preset.argtypes = [C.c_int, C.c_int, C.c_int]
        R.pitref_destroy.argtypes = [C.c_void_p]
        h = R.pitref_create_preset(presets.CASES.index(case), 0 if scale == "desk" else 1, n)
        cap = 64
        k = (C.c_int * cap)()
        res = (C.c_double * cap)()
        fa = (C.c_long * cap)()
        ca = (C.c_long * cap)()
        nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
        lam_h = np.zeros((p.N, p.M))
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        R.pitref_pitsbicg(C.c_void_p(h), C.c_double(1e-8), C.c_double(1e-12), 200, 0, cores, None,
                          lam_h.ctypes.data_as(C.POINTER(C.c_double)), None, k, res, fa, ca, cap,
                          C.byref(nrec), C.byref(rs), C.byref(conv))
        out["reference_cpu"] = {"ms": (time.perf_counter() - t0) * 1e3, "cores": cores,
                                "k": k[max(0, min(nrec.value, cap) - 1)]}
        R.pitref_destroy(C.c_void_p(h))
    return out


def secondary(include_c5_solve=True):
    out = {"apply_F": {}, "time_to_tolerance": {}, "presets_time_to_tolerance": {}}
    for case, scale, n in PRESET_LINES:
        try:
            out["presets_time_to_tolerance"][f"{scale}/{case}"] = preset_time_to_tolerance(
                case, scale, n)
        except Exception as e:  # pragma: no cover
            out["presets_time_to_tolerance"][f"{scale}/{case}"] = {"error": str(e)}
    for name in ("c1", "c3", "c4", "c5"):
        try:
            rate, ms, gp = device_apply_rate(name)
            out["apply_F"][name] = {"gp_steps_per_s": rate, "ms": ms, "gp_steps": gp}
        except Exception as e:  # pragma: no cover
            out["apply_F"][name] = {"error": str(e)}
    for name in ("c1", "c2", "c3", "c4") + (("c5",) if include_c5_solve else ()):
        try:
            out["time_to_tolerance"][name] = device_time_to_tolerance(name)
        except Exception as e:  # pragma: no cover
            out["time_to_tolerance"][name] = {"error": str(e)}
    return out


def run_ours(args, rank, world):
    import torch

    from paper_2203_10148_b200 import _lib, api, configs
    from paper_2203_10148_b200.distributed import DeviceBackend, ShardedOperators

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    L = _lib.lib()
    base = configs.make(CONFIG_NAME)
    n_global = (base.N) * world  # weak scaling: one c2-size shard per rank
    p = configs.make(CONFIG_NAME, slabs=n_global) if world > 1 else base
    ctx = api.BlockOperatorContext(p, device=dev)
    coeff, _ = api.step_coefficients(p)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream
    first = rank * base.N
    count = base.N
    gp_local = p.M * p.fine_steps * (count - 1 if first == 0 else count)

    # inputs resident in HBM: the seeded trajectory-like block vector
    rng = np.random.default_rng(1234 + rank)
    Lh = np.ascontiguousarray(np.tile(p.y0, (count, 1)) * (1.0 + 0.01 * rng.standard_normal((count, 1))))
    Ld = torch.tensor(Lh, device="cuda")
    out = torch.empty_like(Ld)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2
    halo = torch.empty(p.M, dtype=torch.float64, device="cuda") if rank > 0 else None
    dist = None
    if world > 1:
        import torch.distributed as dist
    backend = DeviceBackend(ctx, first, count, stream)

    def exchange():
        if world == 1:
            return
        last = Ld[-1].contiguous()
        if rank % 2 == 0:
            if rank + 1 < world:
                dist.send(last, rank + 1)
            if rank > 0:
                dist.recv(halo, rank - 1)
        else:
            dist.recv(halo, rank - 1)
            if rank + 1 < world:
                dist.send(last, rank + 1)

    def kernel():
        rc = L.pit_apply_F_device(ctx.handle, Ld.data_ptr(), halo.data_ptr() if halo is not None else None,
                                  out.data_ptr(), first, count, st)
        if rc:
            api._check(rc)

    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for _ in range(args.warmup):
        exchange()
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
            exchange()
            k0[i].record(stream)
            kernel()
            e1[i].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    api._check(L.pit_sync_status(ctx.handle, st))
    step_ms = [e0[i].elapsed_time(e1[i]) for i in range(args.steps)]
    kern_ms = [k0[i].elapsed_time(e1[i]) for i in range(args.steps)]
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
    if world == 1:
        Lpin = torch.from_numpy(Lh).pin_memory()
        Opin = torch.empty_like(Lpin).pin_memory()
        Ln, On = Lpin.numpy(), Opin.numpy()
        api.apply_F(ctx, Ln)  # warm
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
        ops = ShardedOperators(backend, n_global)
        assert ops.shard.first == first and ops.shard.count == count
        Lpin = torch.from_numpy(Lh).pin_memory()
        Opin = torch.empty_like(Lpin).pin_memory()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dL = Lpin.to("cuda", non_blocking=True)
            o = ops.apply_F(dL)
            Opin.copy_(o, non_blocking=True)
            torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": gp_total * args.steps / float(tt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(Lh.nbytes), "d2h_bytes_per_step": int(Lh.nbytes),
               "api": "distributed.ShardedOperators.apply_F (host shards)"}

    # ---- roofline: FP64 pipe (measured in-run) ---------------------------
    peak = C.c_double()
    api._check(L.pit_measure_fp64_peak(dev, C.byref(peak)))
    kms = float(np.mean(kern_ms))
    achieved = FLOPS_PER_GP_STEP * gp_local / (kms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(CONFIG_NAME)
        except Exception:
            traffic = None

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE c2 inputs: seeded 8-mode sine initial value, seed 1234)",
        "config": {"workload": f"{CONFIG_NAME}: {configs.DESCRIPTIONS[CONFIG_NAME]}",
                   "slabs_per_gpu": count, "M": p.M, "fine_steps": p.fine_steps,
                   "gp_steps_per_apply_total": gp_total,
                   "layout": {"points_per_thread": coeff.mpt, "segments": coeff.nseg,
                              "warps_per_slab": coeff.warps},
                   "l2": "flushed between timed iterations (256 MB write)",
                   "parallelism": f"slab-sharded x{world}" if world > 1 else "single GPU"},
        "e2e": e2e,
        "gpu_launches": args.steps,  # one slab_kernel launch per apply_F
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value,
                     "unit": "TFLOP/s", "frac": achieved / peak.value, "traffic": traffic,
                     "algorithmic": f"{FLOPS_PER_GP_STEP} flop per gridpoint-step x "
                                    f"{gp_local} gp-steps per launch",
                     "peak_source": "measured in-run: FP64 DFMA probe (MEASURED_PEAKS.json "
                                    "has no FP64 figure)",
                     "kernel_ms": kms},
        "clocks": sampler.summary(),
    }
    if world == 1 and not args.no_secondary:
        line["secondary"] = secondary()
    if world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, kind, sample = cpu_reference_rate(p)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                    "sample": sample}
            if not args.no_secondary:
                # the reference's own pitsbicg_solve on the presets of
                # secondary.presets_time_to_tolerance, same host cores
                pre = {}
                for case, scale, n in PRESET_LINES:
                    r = preset_time_to_tolerance(case, scale, n, with_reference=True)
                    pre[f"{scale}/{case}"] = r.get("reference_cpu")
                line["cpu_baseline"]["presets_time_to_tolerance"] = pre
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    ctx.close()


def main():
    args = parse()
    from paper_2203_10148_b200.distributed import init_from_env

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, rank, world)
        return
    rank, world = init_from_env("nccl")
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
