"""One K6 coarse sweep (apply_G_inverse) on a preset (for ncu captures): case scale N."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2203_10148_b200 import api, presets  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "advection_diffusion_reaction"
scale = sys.argv[2] if len(sys.argv) > 2 else "paper"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 16
p = presets.build_problem(presets.make_preset(case, scale), N)
x = np.random.default_rng(0).uniform(-1, 1, (p.N, p.M))
with api.BlockOperatorContext(p) as ctx:
    api.apply_G_inverse(ctx, x)
    api.apply_G_inverse(ctx, x)
print("ok")
