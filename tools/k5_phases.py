"""K5 per-iteration phase breakdown (instrumented build): CTA 0, thread 0."""
import ctypes as C
import os
import sys
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_timing.so")
import numpy as np
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

L = _lib.lib()
L.pit_debug_phase_timing.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_longlong)]
p = configs.make("c5", slabs=6)
with api.BlockOperatorContext(p) as ctx:
    x = np.tile(p.y0, (p.N, 1))
    api.apply_G_inverse(ctx, x)
    its = ctx.coarse_iterations()
    out = (C.c_longlong * 64)()
    assert L.pit_debug_phase_timing(ctx.handle, 1, out) == 0
names = ["", "SpMV+dot", "reduce pq", "x,r update", "reduce rr,rz", "p update+put", "publish(sync)"]
print(f"cg iterations {its}")
print(" | ".join(f"{names[i]} {out[i] / its:6.0f}" for i in range(1, 7)), "cycles/iteration")
