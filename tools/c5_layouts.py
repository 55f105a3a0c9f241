"""c5 apply_F timing per K4 tiling (tile rows, tile cols, CTAs per cluster,
warps per CTA); the explicit step is pointwise, so every tiling returns the
same bits (checked against the default)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 297
L = _lib.lib()
p = configs.make("c5", slabs=slabs)
x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
ref = None
for lay in [(8, 8, 4, 8)] + [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]]:
    ctx = api.BlockOperatorContext(p, fine_layout=lay)
    out = torch.empty_like(x)
    f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
    assert f() == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    o = out.cpu().numpy()
    if ref is None:
        ref = o
    gp = (p.N - 1) * p.M * p.fine_steps
    ms = sorted(ts)[1]
    print(f"c5 slabs={slabs} layout {lay}: {ms:.2f} ms  {gp/ms/1e9:.3f}e12 gp/s  "
          f"frac {6*gp/ms/1e9/36.8:.3f}  same bits: {np.array_equal(o, ref)}", flush=True)
    ctx.close()
