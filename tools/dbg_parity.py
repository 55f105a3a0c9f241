import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from helpers import OracleProblem
from paper_2203_10148_b200 import api, configs
p = configs.make('c2', slabs=8); o = OracleProblem(p)
L = np.ascontiguousarray(np.random.default_rng(11).uniform(-1,1,(p.N,p.M)))
with api.BlockOperatorContext(p) as ctx:
    for nm, a, b in (('F', api.apply_F(ctx, L), o.apply_F(L)), ('G', api.apply_G_inverse(ctx, L), o.apply_G_inverse(L)),
                     ('rhs', api.assemble_rhs(ctx), o.assemble_rhs()), ('ig', api.initial_guess(ctx, 0), o.initial_guess())):
        d = np.abs(a-b); print(nm, np.array_equal(a,b), d.max(), np.argwhere(d > 0)[:5].tolist(), np.abs(b).max())
