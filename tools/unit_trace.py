"""K1 schedule: per-unit {SM, start, end} from the trace build; summarises SM
occupancy over time and unit durations."""
import ctypes as C
import os
import sys
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_trace.so")
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1]
slabs = int(sys.argv[2])
pieces = sys.argv[3] if len(sys.argv) > 3 else "0"
os.environ["PIT_PIECES"] = pieces
L = _lib.lib()
L.pit_debug_trace.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]
p = configs.make(name, slabs=slabs)
ctx = api.BlockOperatorContext(p)
x = np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))
api.apply_F(ctx, x)
api.apply_F(ctx, x)
n = 64 * p.N
buf = (C.c_longlong * (8 * n))()
assert L.pit_debug_trace(ctx.handle, buf, n) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(n, 8)
t = t[t[:, 3] > 0]
t0 = t[:, 2].min()
st, en = (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3
dur = en - st
print(f"{name} slabs={slabs} pieces={pieces} units={len(t)} makespan={en.max():.1f}us "
      f"dur min/med/max={dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f}us")
ld = (t[:, 4] - t[:, 2]) / 1e3
cp = (t[:, 5] - t[:, 4]) / 1e3
sv = (t[:, 3] - t[:, 5]) / 1e3
print(f"phase medians: pop+load {np.median(ld):.2f}us compute {np.median(cp):.1f}us store+push {np.median(sv):.2f}us"
      f" | means {ld.mean():.2f} {cp.mean():.1f} {sv.mean():.2f}")
gaps = []
for sm in np.unique(t[:, 0]):
    pass
sms = np.unique(t[:, 0])
per_sm = np.bincount(t[:, 0].astype(int), minlength=148)
print("units per SM: min", per_sm.min(), "max", per_sm.max(), "SMs used", len(sms))
print("start times quantiles (us):", np.round(np.quantile(st, [0, .1, .5, .8, .9, .95, 1]), 1))
print("end times quantiles (us):  ", np.round(np.quantile(en, [0, .1, .5, .8, .9, .95, 1]), 1))
for T in np.linspace(0, en.max(), 11)[:-1]:
    act = (st <= T) & (en > T)
    occ = np.bincount(t[act, 0].astype(int), minlength=148)
    print(f"t={T:7.1f}us active={act.sum():4d} per-SM min/max={occ.min()}/{occ.max()}")
ctx.close()
