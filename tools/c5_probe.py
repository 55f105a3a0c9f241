"""c5 timing probe: apply_F (K4) and one G^-1 sweep (K5) at full size."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tol = float(sys.argv[2]) if len(sys.argv) > 2 else None
lay = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
p = configs.make("c5", slabs=slabs)
if tol:
    p.coarse_tolerance = tol
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
ctx = api.BlockOperatorContext(p, fine_layout=lay)
x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
out = torch.empty_like(x)
f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
assert f() == 0
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); f(); e1.record(stream); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
gp = p.M * p.fine_steps * (p.N - 1)
ms = min(ts)
print(f"c5 slabs={slabs} layout={lay} apply_F ms={ms:.3f} gp-steps/s={gp/ms*1e3:.3e} "
      f"TF(6 flop)={gp*6/ms*1e3/1e12:.2f}", flush=True)
# one coarse sweep from the seq-like input
y = torch.tensor(np.tile(p.y0, (p.N, 1)), device="cuda")
w = torch.empty_like(y)
it0 = ctx.coarse_iterations()
t0 = time.time()
rc = L.pit_coarse_sweep_device(ctx.handle, y.data_ptr(), None, w.data_ptr(), 0, p.N, 0, 1, st)
r2 = L.pit_sync_status(ctx.handle, st)
dt = time.time() - t0
its = ctx.coarse_iterations() - it0
print(f"G^-1 rc={rc},{r2} {_lib.lib().pit_last_error().decode()} wall={dt*1e3:.1f} ms "
      f"cg_iters={its} per_slab={its/max(1,p.N-1):.1f} us/iter={dt*1e6/max(1,its):.2f}", flush=True)
