"""K6 on grids above the presets' (m up to 101): apply_F and PiTSBiCG time of
the rotation case at N slabs."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_2203_10148_b200 import api, presets  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for gp in (33, 51, 66, 101):
    pre = presets.make_preset("advection_diffusion_reaction", "desk")
    pre.grid_points = gp
    p = presets.build_problem(pre, N)
    x = np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))
    with api.BlockOperatorContext(p) as ctx:
        api.apply_F(ctx, x)
        t0 = time.perf_counter(); api.apply_F(ctx, x); t1 = time.perf_counter()
        res = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-8))
        t2 = time.perf_counter()
    print(f"grid_points {gp} (m = {gp - 2}): apply_F {1e3 * (t1 - t0):.1f} ms, PiTSBiCG to 1e-8 "
          f"{1e3 * (t2 - t1):.1f} ms, k = {res.history.records[-1].k}", flush=True)
