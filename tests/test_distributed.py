"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the slab-sharded
operators and the sharded PiTSBiCG driver (paper_2203_10148_b200.distributed)
over an oracle-backed local backend must reproduce the single-process
oracle bit for bit — halo exchange, coarse-sweep chain across ranks,
reductions summed in global slab order."""
from __future__ import annotations

import ctypes as C
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest

import oracle_lib as O
from helpers import OracleProblem
from paper_2203_10148_b200 import configs
from paper_2203_10148_b200.distributed import ShardedOperators, shard_range


class OracleBackend:
    """Per-rank compute with the CPU oracle (device op order)."""

    def __init__(self, p, first, count):
        self.p = p
        self.o = OracleProblem(p)
        self.lib = O.orc()
        self.M = p.M
        self.first, self.count = first, count
        self.has_source = p.source is not None
        self.shape = np.ascontiguousarray(p.source.shape) if self.has_source else None
        self.st = [self.lib.orc_1d_stepper(self.o.o, r) for r in (0, 1)]

    def _prop(self, role, with_source, x, slab):
        out = np.zeros(self.M)
        ds = self.lib.orc_1d_ds(self.o.o, role, slab) if (with_source and self.has_source) else None
        self.lib.orc_stepper_propagate(self.st[role], O.ptr(np.ascontiguousarray(x)), ds,
                                       O.ptr(self.shape) if ds is not None else None, O.ptr(out))
        return out

    # vectors
    def y0(self):
        return np.ascontiguousarray(self.p.y0, dtype=np.float64)

    def zeros(self):
        return np.zeros((self.count, self.M))

    def block(self, x, i):
        import torch
        return torch.from_numpy(np.ascontiguousarray(x[i]))

    def set_block(self, x, i, v):
        x[i] = v

    def empty_block(self):
        import torch
        return torch.zeros(self.M, dtype=torch.float64)

    def copy(self, x):
        return x.copy()

    def to_host(self, x):
        return np.asarray(x)

    # operators
    def apply_F(self, L, halo, first, count):
        out = np.zeros_like(L)
        for b in range(count):
            n = first + b
            if n == 0:
                out[b] = L[b]
                continue
            prev = L[b - 1] if b > 0 else halo.numpy()
            out[b] = L[b] - self._prop(0, False, prev, n - 1)
        return out

    def residual(self, lam, halo, rhs, first, count):
        out = np.zeros_like(lam)
        for b in range(count):
            n = first + b
            if n == 0:
                out[b] = rhs[b] - lam[b]
                continue
            prev = lam[b - 1] if b > 0 else halo.numpy()
            a = lam[b] - self._prop(0, False, prev, n - 1)
            out[b] = rhs[b] - a
        return out

    def coarse_sweep(self, V, W_prev, first, count, with_source, add_v, out=None):
        W = out if out is not None else np.zeros((count, self.M))
        b0 = 0
        if first == 0:
            if add_v:
                W[0] = V[0]
            prev = W[0].copy()
            b0 = 1
        else:
            prev = W_prev.numpy()
        for b in range(b0, count):
            y = self._prop(1, with_source, prev, first + b - 1)
            if add_v:
                y = y + V[b]
            W[b] = y
            prev = y
        return W

    def fine_source(self, first, count):
        B = np.zeros((count, self.M))
        if not self.has_source:
            return B
        for b in range(count):
            n = first + b
            if n > 0:
                B[b] = self._prop(0, True, np.zeros(self.M), n - 1)
        return B

    # reductions / phases (device op order)
    def _part(self, a, b):
        p = self.o.prob
        return np.array([self.lib.orc_block_partial(p, O.ptr(np.ascontiguousarray(a[i])),
                                                    O.ptr(np.ascontiguousarray(b[i])))
                         for i in range(a.shape[0])])

    def partials(self, a, b):
        return self._part(a, b)

    def partials2(self, a0, b0, a1, b1):
        return np.stack([self._part(a0, b0), self._part(a1, b1)], axis=1).reshape(-1)

    def update_s(self, alpha, r, d):
        s = np.empty_like(r)
        self.lib.orc_vec_update_s(r.size, alpha, O.ptr(r), O.ptr(d), O.ptr(s))
        return s, self._part(s, s)

    def update_lr(self, alpha, omega, p, s, t, rs, lam):
        r = np.empty_like(s)
        self.lib.orc_vec_update_lr(s.size, alpha, omega, O.ptr(p), O.ptr(s), O.ptr(t), O.ptr(lam),
                                   O.ptr(r))
        return r, np.stack([self._part(r, r), self._part(r, rs)], axis=1).reshape(-1)

    def update_p(self, omega, beta, d, r, p):
        self.lib.orc_vec_update_p(p.size, omega, beta, O.ptr(d), O.ptr(r), O.ptr(p))

    def axpy(self, a, x, y):
        self.lib.orc_vec_axpy(y.size, a, O.ptr(x), O.ptr(y))


class OracleBackend2D(OracleBackend):
    """2D (config 5) propagators: K4 explicit / K5 CG mirrors."""

    def __init__(self, p, first, count):
        self.p = p
        self.o = OracleProblem(p)
        self.lib = O.orc()
        self.M = p.M
        self.first, self.count = first, count
        self.has_source = False
        self.shape = None
        self.c = self.o.coeffs

    def _prop(self, role, with_source, x, slab):
        out = np.zeros(self.M)
        xin = np.ascontiguousarray(x)
        if role == 0:
            self.lib.orc2_explicit_propagate(C.byref(self.c), O.ptr(xin), O.ptr(out))
        else:
            it = C.c_longlong()
            assert self.lib.orc2_coarse_propagate(C.byref(self.c), O.ptr(xin), O.ptr(out),
                                                  C.byref(it)) == 1
        return out


class OracleBackendBE2D(OracleBackend):
    """2D backward-Euler presets (K6 mirror)."""

    def __init__(self, p, first, count):
        self.p = p
        self.o = OracleProblem(p)
        self.lib = O.orc()
        self.M = p.M
        self.first, self.count = first, count
        self.has_source = False
        self.shape = None

    def _prop(self, role, with_source, x, slab):
        return self.o.propagate(role, x, slab)


def _problem(name, slabs, M, fine_steps):
    if name.startswith("preset:"):
        import dataclasses

        from paper_2203_10148_b200 import presets
        p = presets.build_problem(presets.make_preset(name.split(":")[1]), slabs)
        return dataclasses.replace(p, fine_steps=fine_steps, T=p.T * fine_steps / p.fine_steps)
    p = configs.make(name, slabs=slabs, M=M)
    p.fine_steps = fine_steps
    if name == "c5":
        p.T = p.N * fine_steps * (p.spacing ** 2 / 8.0)  # keep dt = h^2/8
    return p


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_path):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    name, slabs, M, fine_steps = case
    p = _problem(name, slabs, M, fine_steps)
    first, count = shard_range(p.N, world, rank)
    be = (OracleBackendBE2D if name.startswith("preset:") else
          OracleBackend2D if name == "c5" else OracleBackend)(p, first, count)
    ops = ShardedOperators(be, p.N)
    rng = np.random.default_rng(5)
    Lg = rng.uniform(-1, 1, (p.N, p.M))
    L = np.ascontiguousarray(Lg[first:first + count])
    fL = ops.apply_F(L)
    gV = ops.apply_G_inverse(L.copy())
    dot = ops.block_inner_product(L, fL)
    nrm = ops.block_norm_n_inf(gV)
    lam, rows, restarts, conv = ops.pitsbicg_solve(tolerance=1e-10)
    res = dict(rank=rank, first=first, fL=fL, gV=gV, dot=dot, nrm=nrm, lam=lam, rows=rows,
               restarts=restarts, conv=conv)
    with open(f"{out_path}.{rank}", "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


CASES = [("c2", 7, 300, 40), ("c4", 6, 256, 30), ("c3", 5, 200, 50), ("c5", 5, 12, 48),
         ("preset:advection_diffusion_reaction", 5, None, 10)]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES)
def test_sharded_operators_and_solver_bitwise(world, case):
    import torch.multiprocessing as mp

    name, slabs, M, fine_steps = case
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res")
        mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world,
                           join=True, start_method="spawn")
        parts = []
        for r in range(world):
            with open(f"{out}.{r}", "rb") as f:
                parts.append(pickle.load(f))
    parts.sort(key=lambda x: x["first"])
    p = _problem(name, slabs, M, fine_steps)
    o = OracleProblem(p)
    rng = np.random.default_rng(5)
    Lg = rng.uniform(-1, 1, (p.N, p.M))
    assert np.array_equal(np.concatenate([x["fL"] for x in parts]), o.apply_F(Lg))
    assert np.array_equal(np.concatenate([x["gV"] for x in parts]), o.apply_G_inverse(Lg))
    ref_dot = o.block_dot(Lg, o.apply_F(Lg))
    ref_nrm = o.block_norm(o.apply_G_inverse(Lg))
    for x in parts:
        assert x["dot"] == ref_dot and x["nrm"] == ref_nrm
    r = o.solve(1e-10)
    assert np.array_equal(np.concatenate([x["lam"] for x in parts]), r["lam"])
    for x in parts:
        assert [tuple(row) for row in x["rows"]] == [tuple(row) for row in r["rows"]]
        assert x["restarts"] == r["restarts"] and x["conv"] == bool(r["converged"])


def test_shard_ranges_cover_blocks():
    for n in (2, 7, 1024, 2048):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, w, r) for r in range(w)]
            assert got[0][0] == 0 and sum(c for _, c in got) == n
            for (f0, c0), (f1, _) in zip(got, got[1:]):
                assert f0 + c0 == f1
