"""Per-phase cycle breakdown of one step (instrumented build, CTA 0)."""
import ctypes as C
import os
import sys
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_timing.so")
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
lay = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else None
L = _lib.lib()
L.pit_debug_phase_timing.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_longlong)]
names = ["fwd pass1", "fwd scan", "fwd xwarp", "fwd carry+pass2", "bwd pass1", "bwd scan",
         "bwd xwarp", "bwd carry+pass2", "corner", "rescale/loop"]
for slabs in (2, 889, 1024):
    p = configs.make(name, slabs=slabs)
    ctx = api.BlockOperatorContext(p, fine_layout=lay)
    x = np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))
    api.apply_F(ctx, x)
    out = (C.c_longlong * 32)()
    assert L.pit_debug_phase_timing(ctx.handle, 0, out) == 0
    steps = p.fine_steps
    for w in (0, 1):
        v = [out[w * 16 + k] / steps for k in range(10)]
        print(f"{name} {lay} slabs={slabs} warp{w}: total {sum(v):7.0f} cyc/step | " +
              " | ".join(f"{n} {c:5.0f}" for n, c in zip(names, v)), flush=True)
    if slabs == 1024:
        api.apply_G_inverse(ctx, x)
        out = (C.c_longlong * 32)()
        assert L.pit_debug_phase_timing(ctx.handle, 1, out) == 0
        n = (p.N - 1) * p.coarse_steps
        print(f"{name} coarse sweep I/O warp: wait W {out[12]/n:.0f} | store W {out[13]/n:.0f} | "
              f"load V {out[14]/n:.0f} cyc per slab", flush=True)
        for w in (0, 1):
            v = [out[w * 16 + k] / n for k in range(12)]
            print(f"{name} coarse sweep warp{w}: per coarse step | " +
                  " | ".join(f"{nm} {c:5.0f}" for nm, c in zip(names + ["propagate", "V add+W store"], v)),
                  flush=True)
    ctx.close()
