"""Small cases of every kernel family with hand-rolled synchronisation, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck, one tool per
run): K1 piece scheduling (ld.acquire queue), K2's I/O warp (TMA ring,
mbarrier hand-offs), apply_GF with K2 overlapped on K1 (epoch flags), K3, K4
clusters (DSMEM st.async + mbarriers), K5 cluster CG, K6 (2D presets)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2203_10148_b200 import api, configs, presets  # noqa: E402

rng = np.random.default_rng(0)
os.environ.setdefault("PIT_PIECES", "3")
p = configs.make("c2", slabs=9)
with api.BlockOperatorContext(p) as ctx:
    L = rng.uniform(-1, 1, (p.N, p.M))
    api.apply_F(ctx, L)                        # K1, pieces (queue)
    api.apply_G_inverse(ctx, L)                # K2 I/O warp, TMA ring
    r = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))  # K1+K2+K3
    print("c2/9", r.history.records[-1].k, flush=True)
os.environ["PIT_GF_OVERLAP"] = "1"             # K2 waiting on K1's epoch flags
p = configs.make("c2", slabs=9)
with api.BlockOperatorContext(p) as ctx:
    r = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
    print("c2/9 overlapped", r.history.records[-1].k, flush=True)
q = configs.make("c4", slabs=4)
with api.BlockOperatorContext(q) as ctx:
    r = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))  # source paths
    print("c4/4", r.history.records[-1].k, flush=True)
c = configs.make("c5", slabs=3, M=32)
c.fine_steps = 64
c.T = c.N * c.fine_steps * (c.spacing ** 2 / 8.0)
with api.BlockOperatorContext(c) as ctx:
    X = rng.uniform(-1, 1, (c.N, c.M))
    api.apply_F(ctx, X)                        # K4 clusters
    api.apply_G_inverse(ctx, X)                # K5 cluster CG
    print("c5 small ok", flush=True)
d = presets.build_problem(presets.make_preset("advection_diffusion_reaction"), 4)
with api.BlockOperatorContext(d) as ctx:
    X = rng.uniform(-1, 1, (d.N, d.M))
    api.apply_F(ctx, X)                        # K6 batch (BiCGStab)
    api.apply_G_inverse(ctx, X)                # K6 sweep
    print("desk rotation ok", flush=True)
print("SANITIZE CASES DONE")
