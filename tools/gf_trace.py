"""K1 block-ready times inside the overlapped G^-1 F (last application of a
PiTSBiCG solve) from the trace build, and the bound they put on the coarse
chain: K2 cannot pass block b before ready_b, then needs (N-b) more steps.
usage: python tools/gf_trace.py [config] [us per coarse step]"""
import ctypes as C
import os
import sys
import time
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_trace.so")
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
step_us = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
L = _lib.lib()
L.pit_debug_trace.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]
p = configs.make(name)
ctx = api.BlockOperatorContext(p)
lam = torch.empty((p.N, p.M), dtype=torch.float64, device="cuda")
cfg = _lib.SolverConfigC(configs.tolerance(name), 1e-12, 200, 0)
recs = (_lib.RecordC * 202)()
info = _lib.SolveInfoC()
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    api._check(L.pit_pitsbicg_solve_device(ctx.handle, C.byref(cfg), None, lam.data_ptr(), recs, 202,
                                           C.byref(info), None))
    ttt = (time.perf_counter() - t0) * 1e3
n = p.N
buf = (C.c_longlong * (8 * n))()
assert L.pit_debug_trace(ctx.handle, buf, n) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(n, 8)
idx = np.nonzero(t[:, 3] > 0)[0]
t = t[idx]
base = t[:, 2].min()
st, end = (t[:, 2] - base) / 1e3, (t[:, 3] - base) / 1e3
print(f"{name}: TTT {ttt:.2f} ms, {info.stats.fine_applications} fine propagations; last K1 batch: "
      f"{len(t)} units, makespan {end.max():.0f} us")
for lo in range(0, len(t), max(1, len(t) // 8)):
    m = (idx >= lo) & (idx < lo + max(1, len(t) // 8))
    print(f" blocks {lo:5d}+: start {st[m].min():6.0f}..{st[m].max():6.0f}  ready "
          f"{np.round(np.quantile(end[m], [0, .5, 1]), 0)}")
nb = len(t)
chain = 0.0
stall = 0.0
for b in np.argsort(idx):
    if end[b] > chain:
        stall += end[b] - chain
        chain = end[b]
    chain += step_us
print(f" coarse chain at {step_us} us/step: ends >= {chain:.0f} us, of which {stall:.0f} us waiting for K1 "
      f"(first block ready at {end[np.argsort(idx)[0]]:.0f})")
ctx.close()
