"""apply_F device timing only (for A/B builds selected with PIT_LIB)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

L = _lib.lib()
for arg in sys.argv[1:] or ["c2"]:
    name, _, lay = arg.partition(":")
    p = configs.make(name)
    ctx = api.BlockOperatorContext(p, fine_layout=tuple(int(v) for v in lay.split(",")) if lay else None)
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
    assert f() == 0
    ts = []
    for _ in range(7):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    gp = configs.gp_steps_per_apply(p)
    ms = sorted(ts)[3]
    print(f"{_lib.LIB_PATH.split('/')[-1]} {arg}: median {ms:.3f} ms  {gp/ms/1e9:.3f}e12 gp/s  frac {5*gp/ms/1e9/36.7:.3f}", flush=True)
    ctx.close()
