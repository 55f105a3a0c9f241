"""Host<->device copy bandwidth and pit_apply_F (pinned, pipelined) timing
on the c2 workload: where the e2e time goes."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_10148_b200 import api, configs, _lib

n = 1024 * 4096
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
ms = t(lambda: d.copy_(h, non_blocking=True)); print(f"H2D {n*8/ms/1e6:.1f} GB/s {ms:.3f} ms")
ms = t(lambda: h.copy_(d, non_blocking=True)); print(f"D2H {n*8/ms/1e6:.1f} GB/s {ms:.3f} ms")
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
ms = t(both); print(f"H2D||D2H {2*n*8/ms/1e6:.1f} GB/s {ms:.3f} ms")
p = configs.make("c2")
L = np.random.default_rng(1).uniform(-1, 1, (p.N, p.M))
Lp = torch.from_numpy(L).pin_memory().numpy(); Op = torch.empty(p.N * p.M, dtype=torch.float64).pin_memory().numpy()
ctx = api.BlockOperatorContext(p)
lib = _lib.lib()
os.environ["PIT_E2E_DIRECT"] = "0"  # output through the D2H copy stream
for chunks in (os.environ.get("CHUNKS", "16").split(",")):
    os.environ["PIT_E2E_CHUNKS"] = chunks
    ctx.close(); ctx = api.BlockOperatorContext(p)
    f = lambda: lib.pit_apply_F(ctx.handle, _lib.dptr(Lp), _lib.dptr(Op), None)
    ms = t(f); print(f"pit_apply_F pinned direct=0 chunks={chunks}: {ms:.3f} ms  {p.M*p.fine_steps*(p.N-1)/ms/1e9:.3e} gp-steps/s")
ref = Op.copy()
for direct in ("1",):
    os.environ["PIT_E2E_DIRECT"] = direct
    for chunks in (os.environ.get("CHUNKS", "16").split(",")):
        os.environ["PIT_E2E_CHUNKS"] = chunks
        ctx.close(); ctx = api.BlockOperatorContext(p)
        Op[:] = 0
        f = lambda: lib.pit_apply_F(ctx.handle, _lib.dptr(Lp), _lib.dptr(Op), None)
        ms = t(f)
        print(f"pit_apply_F direct={direct} chunks={chunks}: {ms:.3f} ms  {p.M*p.fine_steps*(p.N-1)/ms/1e9:.3e} gp-steps/s  same={np.array_equal(Op, ref)}")

