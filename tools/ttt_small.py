"""PiTSBiCG time-to-tolerance of the launch-bound cases (c1, the desk
presets) with the device-resident loop and with the host loop
(PIT_HOST_SCALARS=1)."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_2203_10148_b200 import _lib, api, configs, presets
    L = _lib.lib()
    cases = [("c1", configs.make("c1"), 1e-10)]
    for case, scale, n in (("diffusion", "desk", 16), ("advection_diffusion_reaction", "desk", 16),
                           ("advection_diffusion_reaction", "paper", 64)):
        cases.append((f"{scale}/{case}", presets.build_problem(presets.make_preset(case, scale), n), 1e-8))
    for name, p, tol in cases:
        with api.BlockOperatorContext(p) as ctx:
            lam = torch.empty((p.N, p.M), dtype=torch.float64, device="cuda")
            cfg = _lib.SolverConfigC(tol, 1e-12, 200, 0)
            recs = (_lib.RecordC * 202)()
            info = _lib.SolveInfoC()
            ts = []
            for _ in range(6):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(),
                                                       recs, 202, C.byref(info), None))
                ts.append(time.perf_counter() - t0)
            print(f"{name} host_scalars={os.environ.get('PIT_HOST_SCALARS', '0')}: "
                  f"{min(ts[1:])*1e3:.3f} ms k={recs[info.record_count-1].k} restarts={info.restarts} "
                  f"res={recs[info.record_count-1].residual_norm:.6e}", flush=True)
    sys.exit(0)
for hs in ("1", "0"):
    subprocess.run([sys.executable, __file__, "child"], env={**os.environ, "PIT_HOST_SCALARS": hs})
