"""One warm-up and one measured G^-1 (K2 coarse sweep) of a BASELINE config
through the device entry point — the launch `ncu -k regex:sweep -s 1 -c 1`
captures."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
L = _lib.lib()
p = configs.make(name)
with api.BlockOperatorContext(p) as ctx:
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
    out = torch.empty_like(x)
    for _ in range(2):
        api._check(L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0,
                                             p.N, 0, 1, None))
    api._check(L.pit_sync_status(ctx.handle, None))
print("ok", name)
