"""Launch each hot kernel a few times (for ncu): apply_F and G^-1 on a config."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = configs.make(name)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
st = stream.cuda_stream
L = _lib.lib()
lay = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
ctx = api.BlockOperatorContext(p, fine_layout=lay)
x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
out = torch.empty_like(x)
for _ in range(reps):
    assert L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st) == 0
    assert L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, 0, 1, st) == 0
torch.cuda.synchronize()
print("ok")
