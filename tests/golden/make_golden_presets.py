"""Generate tests/golden/presets_desk_reference.npz from the UNMODIFIED
reference library (oracle/_ref, built from /root/reference by oracle/Makefile)
through its own build_context(make_preset(case, Desk), N) contexts:

  <case>_y0          initial value (gaussian_initial_condition)
  <case>_seq4        sequential_fine_solve, N = 4
  <case>_probe4 / <case>_F4 / <case>_G4
                     a seeded probe block vector and apply_F / apply_G_inverse of it, N = 4
  <case>_lam4, <case>_rows4, <case>_restarts4
                     pitsbicg_solve (SolverConfig defaults, tol 1e-8), N = 4
  <case>_rows8, <case>_restarts8
                     pitsbicg_solve history, N = 8

Run here:  python tests/golden/make_golden_presets.py
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402
from paper_2203_10148_b200 import presets  # noqa: E402


def solve(h, N, M):
    R = O.ref()
    cap = 64
    k = (C.c_int * cap)()
    res = (C.c_double * cap)()
    fa = (C.c_long * cap)()
    ca = (C.c_long * cap)()
    nrec, rs, conv = C.c_int(), C.c_int(), C.c_int()
    lam = np.zeros((N, M))
    assert R.pitref_pitsbicg(h, 1e-8, 1e-12, 200, 0, 4, None, O.ptr(lam), None, k, res, fa, ca,
                             cap, C.byref(nrec), C.byref(rs), C.byref(conv)) == 0
    rows = np.array([(k[i], res[i], fa[i], ca[i]) for i in range(nrec.value)], dtype=np.float64)
    return lam, rows, rs.value


def main():
    R = O.ref()
    out = {}
    for cid, case in enumerate(presets.CASES):
        h = R.pitref_create_preset(cid, 0, 4)
        M = 31 * 31
        y0 = np.zeros(M)
        R.pitref_initial_value(h, O.ptr(y0))
        seq = np.zeros((4, M))
        assert R.pitref_sequential_fine(h, O.ptr(seq)) == 0
        probe = np.random.default_rng(100 + cid).uniform(-1, 1, (4, M))
        F = np.zeros((4, M))
        G = np.zeros((4, M))
        assert R.pitref_apply_F(h, O.ptr(probe), O.ptr(F), 4) == 0
        assert R.pitref_apply_G_inverse(h, O.ptr(probe), O.ptr(G)) == 0
        lam, rows, rs = solve(h, 4, M)
        R.pitref_destroy(h)
        h8 = R.pitref_create_preset(cid, 0, 8)
        _, rows8, rs8 = solve(h8, 8, M)
        R.pitref_destroy(h8)
        out.update({f"{case}_y0": y0, f"{case}_seq4": seq, f"{case}_probe4": probe,
                    f"{case}_F4": F, f"{case}_G4": G, f"{case}_lam4": lam,
                    f"{case}_rows4": rows, f"{case}_restarts4": np.array(rs),
                    f"{case}_rows8": rows8, f"{case}_restarts8": np.array(rs8)})
        print(case, "k4", int(rows[-1, 0]), "k8", int(rows8[-1, 0]), "restarts", rs, rs8)
    np.savez_compressed(os.path.join(HERE, "presets_desk_reference.npz"), **out)


if __name__ == "__main__":
    main()
