"""apply_F time vs slab count (exposes per-step latency vs throughput)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
lay = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else None
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
for slabs in (2, 149, 297, 445, 593, 741, 889, 1024):
    p = configs.make(name, slabs=slabs)
    ctx = api.BlockOperatorContext(p, fine_layout=lay)
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); f(); e1.record(stream); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name} {lay} slabs={slabs:5d} ms={ms:.3f} cycles/step={ms*1e-3*1.95e9/p.fine_steps:.0f}", flush=True)
    ctx.close()
