"""The slab-sharded C-ABI path (pit_comm_*, pit_sharded_*) on
the GPU: bit-identical to the one-GPU operators and solvers.

* NCCL at world 1 (the only world size one GPU allows; NCCL refuses two
  ranks on one device): the whole sharded code path, every collective a
  no-op exchange.
* The host transport at world 2 and 3: one process per rank, all on cuda:0,
  exchanging through torch.distributed (gloo) — the same halo / chain /
  all-gather logic the NCCL transport runs, with real peers.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from cases import make_case
from paper_2203_10148_b200 import api, configs

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def rows_of(hist):
    return [(r.k, r.residual_norm, r.fine_applications, r.coarse_applications)
            for r in hist.records]


@pytest.mark.parametrize("case,slabs", [("c2", 9), ("c4", 6)])
def test_nccl_world1_sharded_bitwise(case, slabs):
    import torch

    from paper_2203_10148_b200.distributed import Communicator, ShardedContext

    p = configs.make(case, slabs=slabs)
    comm = Communicator.nccl(0, 1, 0, Communicator.nccl_unique_id())
    rng = np.random.default_rng(3)
    L = rng.uniform(-1, 1, (p.N, p.M))
    with api.BlockOperatorContext(p) as ctx:
        ref = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
        fref = api.apply_F(ctx, L)
        sc = ShardedContext(ctx, comm)
        assert (sc.first, sc.count) == (0, p.N)
        fx = sc.apply_F(torch.tensor(L, device="cuda"))
        lam, hist = sc.solve(api.SolverConfig(tolerance=1e-10))
        sc.detach()
    comm.close()
    assert np.array_equal(fx.cpu().numpy(), fref)
    assert np.array_equal(lam.cpu().numpy(), ref.solution)
    assert rows_of(hist) == rows_of(ref.history)
    assert hist.restarts == ref.history.restarts


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("case,slabs,world", [("c2", 9, 2), ("c4", 7, 3), ("c5", 5, 2),
                                              ("c1t", 7, 3), ("gen", 6, 2)])
def test_host_transport_multi_rank_bitwise(case, slabs, world, tmp_path):
    out = str(tmp_path / "res.npz")
    port = _port()
    worker = os.path.join(HERE, "workers", "sharded_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), str(port), case,
                               str(slabs), out], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              text=True) for r in range(world)]
    logs = []
    for pr in procs:
        try:
            logs.append(pr.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:  # pragma: no cover
            for q in procs:
                q.kill()
            raise
    assert all(pr.returncode == 0 for pr in procs), "\n".join(logs)
    g = np.load(out)
    p = make_case(case, slabs)
    with api.BlockOperatorContext(p) as ctx:
        fref = api.apply_F(ctx, g["L"])
        ref = api.pitsbicg_solve(ctx, api.SolverConfig(tolerance=1e-10))
        pref = api.parareal_solve(ctx, api.SolverConfig(tolerance=1e-10))
    assert np.array_equal(g["apply_F"], fref)
    assert np.array_equal(g["lam"], ref.solution)
    assert [tuple(r) for r in g["rows"].tolist()] == [tuple(map(float, r)) for r in rows_of(ref.history)]
    assert int(g["restarts"]) == ref.history.restarts
    assert np.array_equal(g["parareal"], pref.solution)
    assert [tuple(r) for r in g["prows"].tolist()] == [tuple(map(float, r)) for r in rows_of(pref.history)]
    # every rank raised the same SlabError (the lowest failing slab, owned by
    # the last rank)
    assert set(g["errors"].tolist()) == {f"SlabError {p.N - 2}"}
