"""One device PiTSBiCG solve of a config (for ncu captures of the K3 vector kernels)."""
import sys
sys.path.insert(0, ".")
from paper_2203_10148_b200 import api, configs  # noqa: E402

p = configs.make(sys.argv[1] if len(sys.argv) > 1 else "c2")
with api.BlockOperatorContext(p) as ctx:
    r = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=configs.tolerance("c2")))
print("k", r.history.records[-1].k)
