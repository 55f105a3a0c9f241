"""G^-1 (K2) device time per coarse layout: name mpt,nsub,nseg,warps ..."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

L = _lib.lib()
name = sys.argv[1]
for lay in sys.argv[2:] or ["auto"]:
    cl = None if lay == "auto" else tuple(int(v) for v in lay.split(","))
    p = configs.make(name)
    ctx = api.BlockOperatorContext(p, coarse_layout=cl)
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    s = torch.cuda.Stream(); torch.cuda.set_stream(s); st = s.cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f = lambda: L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, 0, 1, st)
    assert f() == 0
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"{name} coarse {lay}: {sorted(ts)[2]:.3f} ms", flush=True)
    ctx.close()
