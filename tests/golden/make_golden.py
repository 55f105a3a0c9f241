"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libpitref.so (oracle/Makefile) and drives it through
the reference's public C++ API (oracle/ref_driver.cpp).  The fixtures are
committed so the GPU box (which has no /root/reference) can check against
them.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402
from paper_2203_10148_b200 import configs  # noqa: E402

WORKERS = os.cpu_count() or 4


def ref_ctx(p, use_bands=True, symmetric=True):
    R = O.ref()
    src = p.source
    shape = np.ascontiguousarray(src.shape) if src else None
    y0 = np.ascontiguousarray(p.y0)
    h = R.pitref_create_1d(p.M, p.grid_lo, p.grid_hi, 0.0, 0.0, 1 if use_bands else 0,
                           p.band_lo, p.band_diag, p.band_up, 1 if symmetric else 0, p.N, p.T,
                           p.fine_steps, p.coarse_steps, O.ptr(y0), 1 if src else 0,
                           O.ptr(shape) if src else None, src.amp if src else 0.0,
                           src.omega if src else 0.0, src.phase if src else 0.0)
    assert h, R.pitref_last_error()
    return h


def ref_create_coeffs(p, diffusion, reaction):
    """c1/c2/c4: the operator from the reference's own assembler."""
    R = O.ref()
    src = p.source
    shape = np.ascontiguousarray(src.shape) if src else None
    y0 = np.ascontiguousarray(p.y0)
    h = R.pitref_create_1d(p.M, p.grid_lo, p.grid_hi, diffusion, reaction, 0, 0.0, 0.0, 0.0, 1,
                           p.N, p.T, p.fine_steps, p.coarse_steps, O.ptr(y0), 1 if src else 0,
                           O.ptr(shape) if src else None, src.amp if src else 0.0,
                           src.omega if src else 0.0, src.phase if src else 0.0)
    assert h, R.pitref_last_error()
    return h


def solve(h, N, M, tol, which="pitsbicg", max_iter=200):
    R = O.ref()
    lam = np.zeros((N, M))
    first = np.zeros((N, M))
    cap = max_iter + 2
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, restarts, conv = C.c_int(), C.c_int(), C.c_int()
    fn = R.pitref_pitsbicg if which == "pitsbicg" else R.pitref_parareal
    rc = fn(h, tol, 1e-12, max_iter, 0, WORKERS, None, O.ptr(lam), O.ptr(first), k, res, fa, ca,
            cap, C.byref(nrec), C.byref(restarts), C.byref(conv))
    if rc:
        return dict(rc=rc, error=R.pitref_last_error().decode())
    n = nrec.value
    hist = np.array([[k[i], res[i], fa[i], ca[i]] for i in range(n)])
    return dict(rc=0, lam=lam, first=first, hist=hist, restarts=restarts.value,
                converged=conv.value)


def main():
    R = O.ref()
    out = {}
    t0 = time.time()
    # ---- c1: full size -------------------------------------------------------
    p = configs.make("c1")
    N, M = p.N, p.M
    h = ref_create_coeffs(p, 1.0, 0.0)
    rng = np.random.default_rng(7)
    probe = np.ascontiguousarray(rng.uniform(-1, 1, (N, M)))
    fL = np.zeros((N, M)); assert R.pitref_apply_F(h, O.ptr(probe), O.ptr(fL), WORKERS) == 0
    gV = np.zeros((N, M)); assert R.pitref_apply_G_inverse(h, O.ptr(probe), O.ptr(gV)) == 0
    ig = np.zeros((N, M)); assert R.pitref_initial_guess(h, O.ptr(ig)) == 0
    sq = np.zeros((N, M)); assert R.pitref_sequential_fine(h, O.ptr(sq)) == 0
    lamN = np.zeros(M); assert R.pitref_propagate(h, 0, 1, O.ptr(np.ascontiguousarray(sq[-1])), N - 1, O.ptr(lamN)) == 0
    s = solve(h, N, M, 1e-10)
    lamN_solve = np.zeros(M)
    assert R.pitref_propagate(h, 0, 1, O.ptr(np.ascontiguousarray(s["lam"][-1])), N - 1, O.ptr(lamN_solve)) == 0
    pr = solve(h, N, M, 1e-10, "parareal")
    np.savez_compressed(os.path.join(HERE, "c1_reference.npz"), y0=p.y0, probe=probe, apply_F=fL,
                        apply_G_inverse=gV, initial_guess=ig, sequential_fine=sq,
                        lambda_N_exact=lamN, pitsbicg_lambda=s["lam"], pitsbicg_first=s["first"],
                        pitsbicg_hist=s["hist"], pitsbicg_restarts=s["restarts"],
                        pitsbicg_lambda_N=lamN_solve, parareal_lambda=pr["lam"],
                        parareal_hist=pr["hist"])
    R.pitref_destroy(h)
    print("c1 done", s["hist"][:, :2].tolist(), s["restarts"], time.time() - t0, flush=True)

    # ---- c3: 16-slab truncation (same dt and steps/slab) ------------------
    p = configs.make("c3", slabs=16)
    N, M = p.N, p.M
    h = ref_ctx(p, use_bands=True, symmetric=False)
    sq = np.zeros((N, M)); assert R.pitref_sequential_fine(h, O.ptr(sq)) == 0
    s = solve(h, N, M, 1e-10)
    np.savez_compressed(os.path.join(HERE, "c3_n16_reference.npz"), sequential_fine=sq,
                        pitsbicg_lambda=s["lam"], pitsbicg_hist=s["hist"],
                        pitsbicg_restarts=s["restarts"])
    R.pitref_destroy(h)
    print("c3 done", s["hist"][:, :2].tolist(), s["restarts"], time.time() - t0, flush=True)

    # ---- c2 / c4: fine propagation of a few slabs; G^-1 fails in the ref ----
    for name, diff, reac in (("c2", 1.0, 0.0), ("c4", 1.0, 5.0)):
        p = configs.make(name, slabs=4)
        N, M = p.N, p.M
        h = ref_create_coeffs(p, diff, reac)
        L = np.ascontiguousarray(np.tile(p.y0, (N, 1)))
        fL = np.zeros((N, M)); assert R.pitref_apply_F(h, O.ptr(L), O.ptr(fL), WORKERS) == 0
        rhs = np.zeros((N, M)); assert R.pitref_assemble_rhs(h, O.ptr(rhs), WORKERS) == 0
        gV = np.zeros((N, M))
        rc = R.pitref_apply_G_inverse(h, O.ptr(L), O.ptr(gV))
        err = R.pitref_last_error().decode() if rc else ""
        np.savez_compressed(os.path.join(HERE, f"{name}_n4_reference.npz"), apply_F=fL,
                            assemble_rhs=rhs, g_inverse_rc=rc, g_inverse_error=err)
        R.pitref_destroy(h)
        print(name, "done rc(G^-1) =", rc, err[:80], time.time() - t0, flush=True)


if __name__ == "__main__":
    main()
