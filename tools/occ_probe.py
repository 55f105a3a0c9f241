"""apply_F time for several slab counts (same per-slab work), with K1's piece decision."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["PIT_PIECES_VERBOSE"] = "1"
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1]
counts = [int(v) for v in sys.argv[2].split(",")]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
for n in counts:
    p = configs.make(name, slabs=n)
    ctx = api.BlockOperatorContext(p)
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
    f(); f(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); f(); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{name} slabs={n} ms={ms:.3f} us/slab-step-per-SM={ms*1e3*148/((n-1)*p.fine_steps)*1e3:.1f}ns", flush=True)
    ctx.close()
