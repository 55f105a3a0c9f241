"""Timeline of the pipelined pit_apply_F (pinned host buffers) on c2 from the
trace build (make -C paper_2203_10148_b200/csrc trace): when each unit got its
input, how long it computed, when it ended; per-SM occupancy over time.
usage: python tools/e2e_trace.py [pieces] [chunks]"""
import ctypes as C
import os
import sys
import time
os.environ["PIT_LIB"] = os.path.abspath("paper_2203_10148_b200/libpit_b200_trace.so")
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

pieces = sys.argv[1] if len(sys.argv) > 1 else "0"
os.environ["PIT_PIECES"] = pieces
os.environ["PIT_E2E_CHUNKS"] = sys.argv[2] if len(sys.argv) > 2 else "16"
L = _lib.lib()
L.pit_debug_trace.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]
p = configs.make("c2")
ctx = api.BlockOperatorContext(p)
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))).pin_memory().numpy()
o = torch.zeros((p.N, p.M), dtype=torch.float64).pin_memory().numpy()
for _ in range(3):
    t0 = time.perf_counter()
    api._check(L.pit_apply_F(ctx.handle, _lib.dptr(x), _lib.dptr(o), None))
    wall = (time.perf_counter() - t0) * 1e3
n = 64 * p.N
buf = (C.c_longlong * (8 * n))()
assert L.pit_debug_trace(ctx.handle, buf, n) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(n, 8)
idx = np.nonzero(t[:, 3] > 0)[0]
t = t[idx]
base = t[:, 2].min()
pop, got, done, end = [(t[:, k] - base) / 1e3 for k in (2, 4, 5, 3)]
print(f"pieces={pieces} wall={wall:.3f} ms units={len(t)} makespan={end.max():.1f} us")
nb = p.N - 1
q = idx // nb
for k in range(int(q.max()) + 1):
    m = q == k
    print(f" piece {k}: pop {np.round(np.quantile(pop[m], [0, .25, .5, .75, 1]), 0)}"
          f" input {np.round(np.quantile(got[m], [0, .25, .5, .75, 1]), 0)}"
          f" wait med {np.median((got - pop)[m]):.0f} compute med {np.median((done - got)[m]):.0f}"
          f" end {np.round(np.quantile(end[m], [0, .25, .5, .75, 1]), 0)}")
order = np.argsort(idx)
b = idx % nb
for lo in range(0, nb, 128):
    m = (b >= lo) & (b < lo + 128)
    print(f" slabs {lo:4d}+: input {got[m & (q == 0)].min():7.0f}..{got[m & (q == 0)].max():7.0f}"
          f"  compute {np.median((done - got)[m]):6.0f}  last end {end[m].max():7.0f}")
for T in np.linspace(0, end.max(), 13)[:-1]:
    act = (got <= T) & (done > T)
    occ = np.bincount(t[act, 0].astype(int), minlength=148)
    wt = ((pop <= T) & (got > T)).sum()
    print(f" t={T:7.1f} us computing={act.sum():4d} waiting={wt:4d} per-SM min/mean/max="
          f"{occ.min()}/{occ.mean():.2f}/{occ.max()}")
if int(pieces) != 1 and len(sys.argv) > 3:
    first = {int(u): (int(r[1]), int(r[0])) for u, r in zip(idx, t) if u < 48}
    print(" unit -> (blockIdx, SM):", [first[u] for u in sorted(first)])
ctx.close()
