"""Problem factory shared by the multi-rank GPU test and its workers: the
BASELINE configs by name, plus the widened boundary's cases
  c1t   c1 with a non-separable source (PIT_SOURCE_TABLE)
  gen   a variable-coefficient 1D operator (K6 on a one-row grid) with a source."""
import math

import numpy as np

from paper_2203_10148_b200 import api, configs


def general_source(t, x):
    return 2.0 * ((1.0 + t) * x * (1.0 - x) + math.sin(3.0 * t) * np.cos(2.0 * math.pi * x))


def make_case(case, slabs):
    if case == "c1t":
        p = configs.make("c1", slabs=slabs)
        p.source = api.TableSource.sample(general_source, p.M, p.N, p.T, p.fine_steps,
                                          p.coarse_steps)
        return p
    if case == "gen":
        M = 150
        h = 1.0 / (M + 1)
        x = np.array([(k + 1) * h for k in range(M)])
        mu_m = 1.0 + 0.5 * np.sin(2 * math.pi * (x - h / 2))
        mu_p = 1.0 + 0.5 * np.sin(2 * math.pi * (x + h / 2))
        a = 20.0 * (1.0 + x)
        st = np.stack([-mu_m / (h * h) - a / (2 * h), (mu_m + mu_p) / (h * h) + 0.5,
                       -mu_p / (h * h) + a / (2 * h)])
        st[0, 0] = 0.0
        st[2, -1] = 0.0
        p = api.Problem1DGeneral(M=M, stencil=st, nonsymmetric=True, N=slabs, T=0.05 * slabs / 8,
                                 fine_steps=10, coarse_steps=1, y0=np.sin(math.pi * x))
        p.source = api.TableSource.sample(general_source, p.M, p.N, p.T, p.fine_steps,
                                          p.coarse_steps)
        return p
    return configs.make(case, slabs=slabs, M=32 if case == "c5" else None)
