"""One c5 apply_F and one c5 coarse sweep over a few slabs (for ncu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 34
p = configs.make("c5", slabs=slabs)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
with api.BlockOperatorContext(p) as ctx:
    x = torch.tensor(np.tile(p.y0, (p.N, 1)), device="cuda")
    out = torch.empty_like(x)
    assert L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st) == 0
    assert L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, min(p.N, 4),
                                     0, 1, st) == 0
    torch.cuda.synchronize()
print("ok")
