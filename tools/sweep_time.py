"""Coarse sweep (K2) time per slab for each config (G^-1, V added)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
for name in (sys.argv[1:] or ["c2", "c3", "c4"]):
    p = configs.make(name)
    with api.BlockOperatorContext(p) as ctx:
        x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
        out = torch.empty_like(x)
        for addv in (1, 0):
            f = lambda: L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, 0, addv, st)
            f(); torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream); f(); b.record(stream); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = min(ts)
            print(f"{name} sweep add_v={addv}: {ms:.3f} ms = {ms/(p.N-1)*1e3:.2f} us/slab "
                  f"({ms/(p.N-1)*1.965e6/p.coarse_steps:.0f} cyc per coarse step)", flush=True)
