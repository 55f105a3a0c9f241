"""apply_F time vs K1 piece count (PIT_PIECES; 0 = launcher's choice)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
lay = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] else None
pieces = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 0, 2, 3, 4, 5, 6, 8]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); st = stream.cuda_stream
L = _lib.lib()
p = configs.make(name)
x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for q in pieces:
    os.environ["PIT_PIECES"] = str(q)
    ctx = api.BlockOperatorContext(p, fine_layout=lay)
    out = torch.empty_like(x)
    f = lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)
    f(); torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    same = bool(torch.equal(out, ref))
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); f(); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name} {lay} pieces={q} ms={np.median(ts):.3f} min={min(ts):.3f} bitwise_same={same}", flush=True)
    ctx.close()
