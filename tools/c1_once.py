"""One c1 PiTSBiCG solve through the device entry point (launch list for ncu)."""
import ctypes as C
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

L = _lib.lib()
p = configs.make("c1")
with api.BlockOperatorContext(p) as ctx:
    lam = torch.empty((p.N, p.M), dtype=torch.float64, device="cuda")
    cfg = _lib.SolverConfigC(1e-10, 1e-12, 200, 0)
    recs = (_lib.RecordC * 202)()
    info = _lib.SolveInfoC()
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(), recs,
                                               202, C.byref(info), None))
        print(f"solve {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms", flush=True)
