"""Repetition stress of the hand-rolled synchronisation (compute-sanitizer is
closed on this GPU pool, so races are hunted by determinism instead): every
protocol is run many times on the same inputs and must return the same bits
each time, and the oracle's.

  * K1 piece scheduling: ld.acquire / st.release unit queue (PIT_PIECES)
  * K1 pipelined host copies: in-kernel chunk flags + stream memory ops
  * K2 I/O warp: TMA ring handed off through mbarriers
  * apply_GF with K2 waiting on K1's per-block epoch flags
  * K4 clusters: DSMEM st.async + per-warp mbarriers; K5 cluster CG
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import OracleProblem
from paper_2203_10148_b200 import api, configs

pytestmark = pytest.mark.gpu


def test_k1_pieces_and_k2_ring_repeatable(monkeypatch):
    monkeypatch.setenv("PIT_PIECES", "3")
    p = configs.make("c2", slabs=300)
    p.fine_steps = 100
    L = np.random.default_rng(1).uniform(-1, 1, (p.N, p.M))
    o = OracleProblem(p)
    fo, go = o.apply_F(L), o.apply_G_inverse(L)
    with api.BlockOperatorContext(p) as ctx:
        for _ in range(20):
            assert np.array_equal(api.apply_F(ctx, L), fo)
            assert np.array_equal(api.apply_G_inverse(ctx, L), go)


def test_pipelined_host_copies_repeatable():
    import torch

    p = configs.make("c2", slabs=64)
    p.fine_steps = 50
    L = np.random.default_rng(2).uniform(-1, 1, (p.N, p.M))
    Lp = torch.from_numpy(L).pin_memory().numpy()
    Op = torch.zeros((p.N, p.M), dtype=torch.float64).pin_memory().numpy()
    ref = OracleProblem(p).apply_F(L)
    with api.BlockOperatorContext(p) as ctx:
        for _ in range(30):
            Op[...] = np.nan
            api.apply_F(ctx, Lp, out=Op)
            assert np.array_equal(Op, ref)


def test_overlapped_apply_GF_repeatable(monkeypatch):
    # the overlap engages for batches of more than one wave; forced here on a
    # small one (PIT_GF_OVERLAP=1 is read per context)
    monkeypatch.setenv("PIT_GF_OVERLAP", "1")
    p = configs.make("c2", slabs=40)
    p.fine_steps = 60
    o = OracleProblem(p)
    r = o.solve(1e-10)
    L = np.random.default_rng(8).uniform(-1, 1, (p.N, p.M))
    rhs = o.assemble_rhs()
    pr = o.preconditioned_residual(L, rhs)
    with api.BlockOperatorContext(p) as ctx:
        for _ in range(8):
            s = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
            assert np.array_equal(s.solution, r["lam"])
            # G^-1 (rhs - F lam) takes the same overlapped path, in place
            assert np.array_equal(api.preconditioned_residual(ctx, L, rhs), pr)


@pytest.mark.parametrize("m,slabs,fs", [(48, 12, 128), (256, 6, 64)])
def test_overlapped_apply_GF_2d_bitwise_and_repeatable(m, slabs, fs, monkeypatch):
    # config 5: K5's cluster follows K4's clusters block by block through the
    # ready flags (engages by itself from two waves of clusters; forced here)
    monkeypatch.setenv("PIT_GF_OVERLAP", "1")
    p = configs.make("c5", slabs=slabs, M=m)
    p.fine_steps = fs
    p.T = p.N * fs * (p.spacing ** 2 / 8.0)
    o = OracleProblem(p)
    r = o.solve(1e-10)
    L = np.random.default_rng(9).uniform(-1, 1, (p.N, p.M))
    rhs = o.assemble_rhs()
    pr = o.preconditioned_residual(L, rhs)
    with api.BlockOperatorContext(p) as ctx:
        for _ in range(4):
            s = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
            assert [(x.k, x.residual_norm) for x in s.history.records] == \
                [(a[0], a[1]) for a in r["rows"]]
            assert np.array_equal(s.solution, r["lam"])
            assert np.array_equal(api.preconditioned_residual(ctx, L, rhs), pr)


def test_cluster_kernels_repeatable():
    p = configs.make("c5", slabs=4, M=48)
    p.fine_steps = 128
    p.T = p.N * p.fine_steps * (p.spacing ** 2 / 8.0)
    X = np.random.default_rng(3).uniform(-1, 1, (p.N, p.M))
    o = OracleProblem(p)
    fo, go = o.apply_F(X), o.apply_G_inverse(X)
    with api.BlockOperatorContext(p) as ctx:
        for _ in range(10):
            assert np.array_equal(api.apply_F(ctx, X), fo)
            assert np.array_equal(api.apply_G_inverse(ctx, X), go)
