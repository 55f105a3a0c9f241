"""Quick device timing of the PiT operators (development tool)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10148_b200 import _lib, api, configs  # noqa: E402


def main(name="c2", reps=5, layout=None):
    reps = int(reps)
    p = configs.make(name)
    fl = tuple(int(v) for v in layout.split(",")) if layout else None
    ctx = api.BlockOperatorContext(p, fine_layout=fl)
    L = _lib.lib()
    dev = torch.device("cuda:0")
    x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, (p.N, p.M)), device=dev)
    out = torch.empty_like(x)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gp = configs.gp_steps_per_apply(p)
    for label, fn in (
        ("apply_F", lambda: L.pit_apply_F_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, st)),
        ("G_inv", lambda: L.pit_coarse_sweep_device(ctx.handle, x.data_ptr(), None, out.data_ptr(), 0, p.N, 0, 1, st)),
    ):
        assert fn() == 0, L.pit_last_error()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0.record()
            assert fn() == 0
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        extra = f" {gp / (ms * 1e-3):.3e} gp-steps/s  {5 * gp / (ms * 1e-3) / 1e12:.2f} TF(5flop)" if label == "apply_F" else ""
        print(f"{name} {label}: best {ms:.3f} ms median {sorted(ts)[len(ts)//2]:.3f} ms{extra}", flush=True)
    t = time.time()
    res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=configs.tolerance(name)))
    dt = time.time() - t
    r = res.history.records
    print(f"{name} pitsbicg: k={r[-1].k} restarts={res.history.restarts} res={r[-1].residual_norm:.3e} "
          f"wall {dt*1e3:.1f} ms (incl. H2D/D2H) stats fine {res.history.stats.fine_parallel_ms:.1f} ms "
          f"coarse {res.history.stats.coarse_sequential_ms:.1f} ms", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
