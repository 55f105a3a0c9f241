"""Slab-sharded multi-GPU PiT operators (one process per GPU).

SURVEY.md §8(e): time slabs shard naturally — rank g owns the contiguous
global blocks [first, first+count).  apply_F needs one boundary block from
rank g-1 (L_{first-1}, the halo); the coarse sweep G^-1 is a chain: rank g
starts from W_{first-1} received from rank g-1 and sends W_{last} to g+1.
Block inner products are per-block partials all-gathered and summed in
global slab order on every rank, so the result is bit-identical to the
single-GPU reduction (block_system.cpp:76-81 structure).

The transport is torch.distributed (NCCL on GPUs; gloo in the CPU tests).
Device work goes through the C ABI (`pit_apply_F_device`,
`pit_coarse_sweep_device`, `pit_block_partials_device`).  A `LocalBackend`
object supplies the per-rank compute so the exchange logic can be tested on
CPU with an oracle backend (tests/test_distributed.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


def shard_range(n_blocks: int, world: int, rank: int):
    """Contiguous block range of `rank` (first, count): the first n % world
    ranks get one extra block."""
    base, extra = divmod(n_blocks, world)
    first = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return first, count


@dataclass
class Shard:
    first: int
    count: int
    rank: int
    world: int

    @property
    def last(self) -> int:
        return self.first + self.count - 1


class ShardedOperators:
    """Exchange logic of the sharded PiT operators over a local backend.

    backend must provide (all arrays are the backend's own array type):
      apply_F(L_local, halo, first, count) -> out_local
      coarse_sweep(V_local, W_prev, first, count) -> W_local
      block_partials(a_local, b_local) -> per-block partials (count,)
      to_host(x) / empty_block()
    and torch.distributed must be initialised.
    """

    def __init__(self, backend, n_blocks: int, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        first, count = shard_range(n_blocks, self.world, self.rank)
        self.shard = Shard(first, count, self.rank, self.world)
        self.backend = backend
        self.n_blocks = n_blocks

    # -- point-to-point halo of the last owned block -----------------------
    def _send_last(self, x_local):
        if self.rank + 1 < self.world:
            self.dist.send(self.backend.block(x_local, self.shard.count - 1), self.rank + 1,
                           group=self.group)

    def _recv_prev(self):
        if self.rank == 0:
            return None
        buf = self.backend.empty_block()
        self.dist.recv(buf, self.rank - 1, group=self.group)
        return buf

    def apply_F(self, L_local):
        """(F L)_n = L_n - FineHom(L_{n-1}) on the owned blocks; one halo block
        crosses each rank boundary (sent before the local batch starts)."""
        # even ranks send first, odd ranks receive first: no deadlock with
        # blocking send/recv
        if self.rank % 2 == 0:
            self._send_last(L_local)
            halo = self._recv_prev()
        else:
            halo = self._recv_prev()
            self._send_last(L_local)
        return self.backend.apply_F(L_local, halo, self.shard.first, self.shard.count)

    def apply_G_inverse(self, V_local):
        """W_n = G(W_{n-1}) + V_n: the sequential chain crosses ranks in order."""
        W_prev = self._recv_prev()
        W = self.backend.coarse_sweep(V_local, W_prev, self.shard.first, self.shard.count)
        self._send_last(W)
        return W

    def block_inner_product(self, a_local, b_local) -> float:
        """Sum over all blocks in global slab order (bit-identical to 1 GPU)."""
        import torch

        part = torch.as_tensor(self.backend.to_host(self.backend.block_partials(a_local, b_local)),
                               dtype=torch.float64)
        counts = [shard_range(self.n_blocks, self.world, r)[1] for r in range(self.world)]
        gathered = [torch.zeros(c, dtype=torch.float64, device=part.device) for c in counts]
        self.dist.all_gather(gathered, part.to(self._coll_device()), group=self.group)
        s = 0.0
        for g in gathered:
            for v in g.cpu().numpy():
                s += float(v)
        return s

    def block_norm_n_inf(self, a_local) -> float:
        import torch

        part = np.sqrt(self.backend.to_host(self.backend.block_partials(a_local, a_local)))
        m = torch.tensor([float(np.max(part)) if part.size else 0.0], dtype=torch.float64,
                         device=self._coll_device())
        self.dist.all_reduce(m, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(m.item())

    def _coll_device(self):
        import torch

        return torch.device("cuda", torch.cuda.current_device()) \
            if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu")


class DeviceBackend:
    """Per-rank compute on the local GPU through the C ABI.  Arrays are torch
    CUDA tensors of shape (count, M)."""

    def __init__(self, ctx, stream=None):
        import torch

        from . import _lib

        self.ctx = ctx
        self.M = ctx.M
        self.L = _lib.lib()
        self.torch = torch
        self.stream = stream or torch.cuda.current_stream()

    def _check(self, rc):
        from .api import _check

        _check(rc)

    def block(self, x, i):
        return x[i].contiguous()

    def empty_block(self):
        return self.torch.empty(self.M, dtype=self.torch.float64, device="cuda")

    def to_host(self, x):
        return x.detach().cpu().numpy()

    def apply_F(self, L_local, halo, first, count):
        out = self.torch.empty_like(L_local)
        self._check(self.L.pit_apply_F_device(
            self.ctx.handle, L_local.data_ptr(), halo.data_ptr() if halo is not None else None,
            out.data_ptr(), first, count, self.stream.cuda_stream))
        self._check(self.L.pit_sync_status(self.ctx.handle, self.stream.cuda_stream))
        return out

    def coarse_sweep(self, V_local, W_prev, first, count):
        W = self.torch.empty_like(V_local)
        self._check(self.L.pit_coarse_sweep_device(
            self.ctx.handle, V_local.data_ptr(), W_prev.data_ptr() if W_prev is not None else None,
            W.data_ptr(), first, count, 0, 1, self.stream.cuda_stream))
        self._check(self.L.pit_sync_status(self.ctx.handle, self.stream.cuda_stream))
        return W

    def block_partials(self, a, b):
        p = self.torch.empty(a.shape[0], dtype=self.torch.float64, device="cuda")
        self._check(self.L.pit_block_partials_device(self.ctx.handle, a.data_ptr(), b.data_ptr(),
                                                     p.data_ptr(), a.shape[0],
                                                     self.stream.cuda_stream))
        return p


def init_from_env(backend: str = "nccl"):
    """torch.distributed init from RANK/WORLD_SIZE/MASTER_* (torchrun)."""
    import os

    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend=backend)
        return dist.get_rank(), world
    return 0, 1
