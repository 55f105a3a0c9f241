"""apply_GF (G^-1 F x) time through the solver's code path: serial (K1 then
K2) vs overlapped (K2 concurrent with K1, PIT_GF_OVERLAP), and the full
PiTSBiCG time-to-tolerance, per config."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    import torch
    from paper_2203_10148_b200 import _lib, api, configs
    L = _lib.lib()
    for name in sys.argv[2:]:
        p = configs.make(name)
        with api.BlockOperatorContext(p) as ctx:
            lam = torch.empty((p.N, p.M), dtype=torch.float64, device="cuda")
            cfg = _lib.SolverConfigC(configs.tolerance(name), 1e-12, 200, 0)
            recs = (_lib.RecordC * 202)()
            info = _lib.SolveInfoC()
            ts = []
            for _ in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None,
                                                       lam.data_ptr(), recs, 202, C.byref(info),
                                                       None))
                ts.append(time.perf_counter() - t0)
            s = info.stats
            print(f"{name} overlap={os.environ.get('PIT_GF_OVERLAP', '1')}: TTT {min(ts[1:])*1e3:.2f} ms "
                  f"k={recs[info.record_count-1].k} res={recs[info.record_count-1].residual_norm:.6e} "
                  f"fine {s.fine_parallel_ms:.2f} ms coarse {s.coarse_sequential_ms:.2f} ms", flush=True)
    sys.exit(0)
names = sys.argv[1:] or ["c2", "c3", "c4"]
for ov in ("0", "1"):
    subprocess.run([sys.executable, __file__, "child"] + names, env={**os.environ, "PIT_GF_OVERLAP": ov})
