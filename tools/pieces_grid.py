"""apply_F ms for (slab count, forced piece count) pairs: per-piece overhead."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1]
counts = [int(v) for v in sys.argv[2].split(",")]
pieces = [int(v) for v in sys.argv[3].split(",")]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
for n in counts:
    p = configs.make(name, slabs=n)
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    row = []
    for q in pieces:
        os.environ["PIT_PIECES"] = str(q)
        ctx = api.BlockOperatorContext(p)
        f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
        f(); f(); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); f(); e1.record(stream); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row.append(f"q{q}={min(ts):.3f}")
        ctx.close()
    print(name, n, " ".join(row), flush=True)
