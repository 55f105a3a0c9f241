"""K4 per-step phase breakdown (instrumented build): cluster 0, CTA 0, each warp."""
import ctypes as C
import os
import sys
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_timing.so")
import numpy as np
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 34
L = _lib.lib()
L.pit_debug_phase_timing.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_longlong)]
p = configs.make("c5", slabs=slabs)
with api.BlockOperatorContext(p) as ctx:
    x = np.tile(p.y0, (p.N, 1))
    api.apply_F(ctx, x)
    out = (C.c_longlong * 64)()
    assert L.pit_debug_phase_timing(ctx.handle, 0, out) == 0
names = ["shfl", "wait", "boundary", "publish", "interior"]
for w in range(8):
    v = [out[w * 8 + i] / p.fine_steps for i in range(5)]
    print(f"slabs={slabs} warp{w}: total {sum(v):6.0f} cyc/step | " +
          " | ".join(f"{n} {c:5.0f}" for n, c in zip(names, v)))
