"""Per-phase cycle breakdown of the K2 coarse sweep (instrumented build,
libpit_b200_timing.so): cycles per coarse step for warps 0 and 1."""
import ctypes as C
import os
import sys
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_timing.so")
import numpy as np
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

L = _lib.lib()
L.pit_debug_phase_timing.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_longlong)]
names = ["fwd pass1", "fwd scan", "fwd xwarp", "fwd carry+pass2", "bwd pass1", "bwd scan",
         "bwd xwarp", "bwd carry+pass2", "corner", "rescale/loop", "propagate", "V add+W store"]
for name in sys.argv[1:] or ["c2"]:
    p = configs.make(name)
    ctx = api.BlockOperatorContext(p)
    x = np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))
    api.apply_G_inverse(ctx, x)
    out = (C.c_longlong * 64)()
    assert L.pit_debug_phase_timing(ctx.handle, 1, out) == 0
    n = (p.N - 1) * p.coarse_steps
    print(f"{name} I/O: wait W {out[12]/n:.0f} | store W {out[13]/n:.0f} | load V {out[14]/n:.0f}")
    for w in (0, 1):
        v = [out[w * 16 + k] / n for k in range(12)]
        print(f"{name} coarse warp{w}: " + " | ".join(f"{nm} {c:.0f}" for nm, c in zip(names, v)), flush=True)
    ctx.close()
