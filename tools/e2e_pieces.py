"""pit_apply_F (pinned, pipelined) on c2 for PIT_PIECES x PIT_E2E_CHUNKS, and
the resident apply_F time beside it."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_10148_b200 import api, configs, _lib

def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
p = configs.make("c2")
L = np.random.default_rng(1).uniform(-1, 1, (p.N, p.M))
Lp = torch.from_numpy(L).pin_memory().numpy(); Op = torch.empty(p.N * p.M, dtype=torch.float64).pin_memory().numpy()
lib = _lib.lib()
ref = None
for pieces in sys.argv[1].split(","):
    os.environ["PIT_PIECES"] = pieces
    for chunks in sys.argv[2].split(","):
        os.environ["PIT_E2E_CHUNKS"] = chunks
        ctx = api.BlockOperatorContext(p)
        f = lambda: lib.pit_apply_F(ctx.handle, _lib.dptr(Lp), _lib.dptr(Op), None)
        ms = t(f)
        if ref is None: ref = Op.copy()
        print(f"pieces={pieces} chunks={chunks}: {ms:.3f} ms  {p.M*p.fine_steps*(p.N-1)/ms/1e9:.3e}e12 gp-steps/s same={np.array_equal(Op, ref)}", flush=True)
        ctx.close()
