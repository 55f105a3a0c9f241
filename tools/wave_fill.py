import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs
L = _lib.lib()
for slabs in (149, 297, 445, 593, 741, 889, 1024):
    p = configs.make("c2", slabs=slabs)
    ctx = api.BlockOperatorContext(p)
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    s = torch.cuda.Stream(); torch.cuda.set_stream(s); st = s.cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]; gp = configs.gp_steps_per_apply(p)
    print(f"slabs={slabs-1}: {ms:.3f} ms  {gp/ms/1e9:.3f}e12 gp/s  frac {5*gp/ms/1e9/36.9:.3f}  per-slab-per-SM-slot {ms/((slabs-1)/888):.3f}", flush=True)
    ctx.close()
