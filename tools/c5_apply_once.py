"""One c5 apply_F (for ncu captures of K4)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 34
lay = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else None
p = configs.make("c5", slabs=slabs)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
ctx = api.BlockOperatorContext(p, fine_layout=lay)
x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
out = torch.empty_like(x)
L = _lib.lib()
for _ in range(2):
    assert L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st) == 0
torch.cuda.synchronize()
print("ok")
