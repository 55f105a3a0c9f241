"""Desk/paper preset timings: device apply_F and PiTSBiCG time-to-tolerance
(K6) next to the reference's own pitsbicg_solve on the host cores
(oracle/_ref, SlabExecutor(nproc))."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2203_10148_b200 import api, presets  # noqa: E402

import oracle_lib as O  # noqa: E402

scale = sys.argv[1] if len(sys.argv) > 1 else "desk"
slabs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "16,64").split(",")]
with_ref = O.ref_available() and os.environ.get("NO_REF") is None
nproc = os.cpu_count()
for cid, case in enumerate(presets.CASES):
    for n in slabs:
        p = presets.build_problem(presets.make_preset(case, scale), n)
        with api.BlockOperatorContext(p) as ctx:
            x = np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))
            api.apply_F(ctx, x)
            t = time.perf_counter()
            for _ in range(3):
                api.apply_F(ctx, x)
            fms = (time.perf_counter() - t) / 3 * 1e3
            api.pitsbicg_solve(ctx, api.SolverConfig())
            t = time.perf_counter()
            res = api.pitsbicg_solve(ctx, api.SolverConfig())
            sms = (time.perf_counter() - t) * 1e3
        line = (f"{scale} {case} N={n}: device apply_F {fms:.2f} ms, pitsbicg {sms:.1f} ms "
                f"k={res.history.records[-1].k}")
        if with_ref and n <= 64:
            h = O.ref().pitref_create_preset(cid, 0 if scale == "desk" else 1, n)
            cap = 64
            k = (C.c_int * cap)(); r = (C.c_double * cap)(); fa = (C.c_long * cap)(); ca = (C.c_long * cap)()
            nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
            lam = np.zeros((p.N, p.M))
            t = time.perf_counter()
            O.ref().pitref_pitsbicg(h, 1e-8, 1e-12, 200, 0, nproc, None, O.ptr(lam), None, k, r, fa,
                                    ca, cap, C.byref(nrec), C.byref(rs), C.byref(conv))
            rms = (time.perf_counter() - t) * 1e3
            O.ref().pitref_destroy(h)
            line += f" | reference CPU ({nproc} threads) pitsbicg {rms:.0f} ms k={k[nrec.value - 1]}"
        print(line, flush=True)
