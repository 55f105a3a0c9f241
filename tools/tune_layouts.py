"""Time apply_F / G^-1 over kernel layouts (development tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402

FINE = [(16, 1, 1, 8), (64, 2, 2, 2), (64, 4, 1, 2), (64, 1, 4, 2), (64, 1, 2, 2), (32, 2, 2, 4), (32, 2, 1, 4), (32, 1, 2, 4), (16, 2, 2, 8), (64, 2, 2, 1), (64, 4, 1, 1), (64, 2, 2, 4), (64, 4, 1, 4), (32, 2, 2, 8), (64, 2, 2, 8)]
COARSE = [(4, 1, 1, 16), (4, 1, 1, 32), (8, 1, 1, 8), (8, 1, 1, 16), (8, 1, 1, 32), (16, 1, 1, 8), (16, 1, 1, 16), (16, 1, 1, 32), (32, 2, 1, 4), (32, 2, 1, 8), (16, 2, 1, 16), (64, 2, 2, 2), (32, 2, 2, 4), (32, 2, 2, 8)]


def timeit(fn, reps=3):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    assert fn() == 0, _lib.lib().pit_last_error()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main(names):
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream
    L = _lib.lib()
    for name in names:
        p = configs.make(name)
        gp = configs.gp_steps_per_apply(p)
        x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device="cuda")
        out = torch.empty_like(x)
        for lay in FINE:
            if 32 * lay[0] * lay[-1] < p.M or 32 * lay[0] * lay[-1] >= 2 * p.M:
                continue
            ctx = api.BlockOperatorContext(p, fine_layout=lay, coarse_layout=None)
            ms = timeit(lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st))
            print(f"{name} fine {lay}: {ms:.3f} ms  {gp / ms / 1e9:.3e} gp-steps/s  {5 * gp / ms / 1e9 / 1e12 * 1e3:.2f} TF", flush=True)
            ctx.close()
        for lay in COARSE:
            if 32 * lay[0] * lay[-1] < p.M or 32 * lay[0] * lay[-1] >= 2 * p.M:
                continue
            ctx = api.BlockOperatorContext(p, coarse_layout=lay)
            ms = timeit(lambda: L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, 0, 1, st))
            print(f"{name} coarse {lay}: {ms:.3f} ms  {ms / (p.N - 1) * 1e3:.2f} us/slab", flush=True)
            ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
