"""Generate tests/golden/c3_full_reference.npz: the UNMODIFIED reference's
pit::pitsbicg_solve on the full BASELINE c3 (1D advection-diffusion,
central differences, M=2048, N=512, 2000/2 BE steps per slab, tol 1e-10),
driven through its public C++ API (oracle/ref_driver.cpp, oracle/_ref).

Run here (where /root/reference exists; ~3 min on 8 cores):
    python tests/golden/make_golden_c3_full.py
The fixture keeps the full history, the restart count, lambda_N (the
reference's own fine propagation of lambda_{N-1} across the last slab),
every block's norm and a subset of whole blocks (the first four, every 32nd,
the last two), so it stays small enough to commit.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402
from make_golden import O, configs  # noqa: E402

BLOCKS = sorted(set([0, 1, 2, 3] + list(range(0, 512, 32)) + [510, 511]))


def main():
    R = O.ref()
    p = configs.make("c3")
    N, M = p.N, p.M
    t0 = time.time()
    h = G.ref_ctx(p, use_bands=True, symmetric=False)
    s = G.solve(h, N, M, 1e-10)
    assert s["rc"] == 0, s
    lam = s["lam"]
    lamN = np.zeros(M)
    assert R.pitref_propagate(h, 0, 1, O.ptr(np.ascontiguousarray(lam[-1])), N - 1,
                              O.ptr(lamN)) == 0
    R.pitref_destroy(h)
    np.savez_compressed(os.path.join(HERE, "c3_full_reference.npz"),
                        blocks=np.array(BLOCKS), lambda_blocks=lam[BLOCKS],
                        lambda_block_norms=np.linalg.norm(lam, axis=1), lambda_N=lamN,
                        pitsbicg_hist=s["hist"], pitsbicg_restarts=s["restarts"],
                        workers=G.WORKERS, seconds=time.time() - t0)
    print("c3 full done", s["hist"][:, :2].tolist(), s["restarts"], time.time() - t0, flush=True)


if __name__ == "__main__":
    main()
