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
    """Exchange logic of the sharded PiT operators and solver over a local
    backend (one rank per GPU; torch.distributed must be initialised).

    backend provides, on the rank's blocks (arrays of the backend's type):
      apply_F(L, halo, first, count) -> out           K1, (F L)_n
      residual(lam, halo, rhs, first, count) -> out   K1, rhs_n - (F lam)_n
      coarse_sweep(V, W_prev, first, count, with_source, add_v, out=None) -> W   K2
      fine_source(first, count) -> B                  K1 with source, zero input
      partials(a, b) / partials2(a0, b0, a1, b1)      K3 per-block h<.,.>
      update_s / update_lr / update_p / axpy / add / copy   K3 (device op order)
      y0(), zeros(), block(x, i), empty_block(), set_block(x, i, v), to_host(x)
    """

    def __init__(self, backend, n_blocks: int, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > n_blocks:
            raise ValueError(f"ShardedOperators: {self.world} ranks for {n_blocks} blocks "
                             "(every rank must own at least one block)")
        first, count = shard_range(n_blocks, self.world, self.rank)
        self.shard = Shard(first, count, self.rank, self.world)
        self.backend = backend
        self.n_blocks = n_blocks
        self.counts = [shard_range(n_blocks, self.world, r)[1] for r in range(self.world)]

    # -- point-to-point of the last owned block ------------------------------
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

    def _halo(self, x_local):
        # even ranks send first, odd ranks receive first: blocking send/recv
        # cannot deadlock
        if self.rank % 2 == 0:
            self._send_last(x_local)
            return self._recv_prev()
        halo = self._recv_prev()
        self._send_last(x_local)
        return halo

    # -- operators (block_system.cpp:115-195) ---------------------------------
    def apply_F(self, L_local):
        """(F L)_n = L_n - FineHom(L_{n-1}); one halo block per rank boundary."""
        halo = self._halo(L_local)
        return self.backend.apply_F(L_local, halo, self.shard.first, self.shard.count)

    def apply_G_inverse(self, V_local, out=None):
        """W_n = G(W_{n-1}) + V_n: the sequential chain crosses ranks in order."""
        W_prev = self._recv_prev()
        W = self.backend.coarse_sweep(V_local, W_prev, self.shard.first, self.shard.count,
                                      False, True, out)
        self._send_last(W)
        return W

    def initial_guess(self, zero: bool = False):
        """CoarseSweep (solvers.cpp:49-64): lambda_0 = y0, lambda_n = G(lambda_{n-1})."""
        be = self.backend
        lam = be.zeros()
        if zero:
            return lam
        if self.rank == 0:
            be.set_block(lam, 0, be.y0())
        W_prev = self._recv_prev()
        lam = be.coarse_sweep(None, W_prev, self.shard.first, self.shard.count, True, False, lam)
        self._send_last(lam)
        return lam

    def assemble_rhs(self):
        """B_0 = y0, B_n = fine.source_contribution(n-1) (block_system.cpp:149-172)."""
        be = self.backend
        rhs = be.fine_source(self.shard.first, self.shard.count)
        if self.rank == 0:
            be.set_block(rhs, 0, be.y0())
        return rhs

    def preconditioned_residual(self, lam, rhs):
        """G^-1 (rhs - F lam) (solvers.cpp:66-71)."""
        halo = self._halo(lam)
        f = self.backend.residual(lam, halo, rhs, self.shard.first, self.shard.count)
        return self.apply_G_inverse(f, out=f)

    # -- reductions: per-block partials, summed in global slab order ---------
    def _gather(self, part, np_):
        import torch

        part = torch.as_tensor(self.backend.to_host(part), dtype=torch.float64).reshape(-1)
        dev = self._coll_device()
        cmax = max(self.counts)
        padded = torch.zeros(cmax * np_, dtype=torch.float64, device=dev)  # equal sizes
        padded[: part.numel()] = part.to(dev)
        gathered = [torch.zeros(cmax * np_, dtype=torch.float64, device=dev) for _ in self.counts]
        self.dist.all_gather(gathered, padded, group=self.group)
        return np.concatenate([g[: c * np_].cpu().numpy() for g, c in zip(gathered, self.counts)]
                              ).reshape(-1, np_)

    @staticmethod
    def _sum(p):
        s = 0.0
        for v in p:
            s += float(v)
        return s

    @staticmethod
    def _max_sqrt(p):
        w = 0.0
        for v in p:
            w = max(w, float(np.sqrt(v)))
        return w

    def block_inner_product(self, a_local, b_local) -> float:
        return self._sum(self._gather(self.backend.partials(a_local, b_local), 1)[:, 0])

    def block_norm_n_inf(self, a_local) -> float:
        return self._max_sqrt(self._gather(self.backend.partials(a_local, a_local), 1)[:, 0])

    def _coll_device(self):
        import torch

        return torch.device("cuda", torch.cuda.current_device()) \
            if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu")

    # -- pitsbicg_solve (solvers.cpp:116-220), op for op ----------------------
    def pitsbicg_solve(self, tolerance=1e-8, restart_tolerance=1e-12, max_iterations=200,
                       zero_guess=False, lambda_init=None):
        """Returns (lambda_local, rows, restarts, converged); rows are
        (k, residual, fine_applications, coarse_applications).  Same branches,
        restart rules and reduction order as the single-GPU device driver
        (pit_capi.cu pitsbicg_dev), so the history is bit-identical."""
        if not (tolerance > restart_tolerance) or not (restart_tolerance > 0.0):
            raise ValueError("solver tolerances must satisfy tolerance > restart_tolerance > 0")
        be = self.backend
        Nm1 = self.n_blocks - 1
        fine = coarse = 0
        rows = []
        lam = lambda_init if lambda_init is not None else self.initial_guess(zero_guess)
        if lambda_init is None and not zero_guess:
            coarse += Nm1
        rhs = self.assemble_rhs()
        if be.has_source:
            fine += Nm1
        r = self.preconditioned_residual(lam, rhs)
        fine += Nm1
        coarse += Nm1
        part = self._gather(be.partials(r, r), 1)[:, 0]
        r_norm = self._max_sqrt(part)
        rr_shadow = self._sum(part)
        rows.append((0, r_norm, fine, coarse))
        if r_norm <= tolerance:
            return lam, rows, 0, True
        rs = be.copy(r)
        p = be.copy(r)
        restarts = 0
        for k in range(1, max_iterations + 1):
            rho = rr_shadow
            d = self.apply_G_inverse(self.apply_F(p))
            fine += Nm1
            coarse += Nm1
            d_dot = self._sum(self._gather(be.partials(d, rs), 1)[:, 0])
            if abs(d_dot) < 1e-300:
                rs, p = be.copy(r), be.copy(r)
                restarts += 1
                rows.append((k, r_norm, fine, coarse))
                rr_shadow = self._sum(self._gather(be.partials(r, r), 1)[:, 0])
                continue
            alpha = rho / d_dot
            s, ps = be.update_s(alpha, r, d)
            s_norm = self._max_sqrt(self._gather(ps, 1)[:, 0])
            if s_norm <= tolerance:
                be.axpy(alpha, p, lam)
                rows.append((k, s_norm, fine, coarse))
                return lam, rows, restarts, True
            t = self.apply_G_inverse(self.apply_F(s))
            fine += Nm1
            coarse += Nm1
            g2 = self._gather(be.partials2(t, t, t, s), 2)
            tt = self._sum(g2[:, 0])
            if tt < 1e-300:
                rs, p = be.copy(r), be.copy(r)
                restarts += 1
                rows.append((k, r_norm, fine, coarse))
                rr_shadow = self._sum(self._gather(be.partials(r, r), 1)[:, 0])
                continue
            omega = self._sum(g2[:, 1]) / tt
            if abs(omega) < 1e-300:
                rs, p = be.copy(r), be.copy(r)
                restarts += 1
                rows.append((k, r_norm, fine, coarse))
                rr_shadow = self._sum(self._gather(be.partials(r, r), 1)[:, 0])
                continue
            r, plr = be.update_lr(alpha, omega, p, s, t, rs, lam)
            g2 = self._gather(plr, 2)
            r_norm = self._max_sqrt(g2[:, 0])
            rr = self._sum(g2[:, 0])
            r_dot = self._sum(g2[:, 1])
            rows.append((k, r_norm, fine, coarse))
            if r_norm <= tolerance:
                return lam, rows, restarts, True
            if abs(r_dot) <= restart_tolerance:
                rs, p = be.copy(r), be.copy(r)
                restarts += 1
                rr_shadow = rr
            else:
                beta = (alpha / omega) * (r_dot / rho)
                be.update_p(omega, beta, d, r, p)
                rr_shadow = r_dot
        return lam, rows, restarts, False


class DeviceBackend:
    """Per-rank compute on the local GPU through the C ABI.  Arrays are torch
    CUDA tensors of shape (count, M) holding the rank's blocks."""

    def __init__(self, ctx, first: int, count: int, stream=None):
        import torch

        from . import _lib

        self.ctx = ctx
        self.M = ctx.M
        self.first, self.count = first, count
        self.L = _lib.lib()
        self.torch = torch
        self.stream = stream or torch.cuda.current_stream()
        self.has_source = ctx.problem.source is not None
        self._y0 = torch.tensor(np.ascontiguousarray(ctx.problem.y0), dtype=torch.float64,
                                device="cuda")

    def _check(self, rc):
        from .api import _check

        _check(rc)

    def _st(self):
        return self.stream.cuda_stream

    def _sync(self):
        self._check(self.L.pit_sync_status(self.ctx.handle, self._st()))

    def y0(self):
        return self._y0

    def zeros(self):
        return self.torch.zeros((self.count, self.M), dtype=self.torch.float64, device="cuda")

    def block(self, x, i):
        return x[i].contiguous()

    def set_block(self, x, i, v):
        x[i].copy_(v)

    def empty_block(self):
        return self.torch.empty(self.M, dtype=self.torch.float64, device="cuda")

    def copy(self, x):
        return x.clone()

    def to_host(self, x):
        return x.detach().cpu().numpy()

    def apply_F(self, L_local, halo, first, count):
        out = self.torch.empty_like(L_local)
        self._check(self.L.pit_apply_F_device(
            self.ctx.handle, L_local.data_ptr(), halo.data_ptr() if halo is not None else None,
            out.data_ptr(), first, count, self._st()))
        self._sync()
        return out

    def residual(self, lam, halo, rhs, first, count):
        out = self.torch.empty_like(lam)
        self._check(self.L.pit_residual_device(
            self.ctx.handle, lam.data_ptr(), halo.data_ptr() if halo is not None else None,
            rhs.data_ptr(), out.data_ptr(), first, count, self._st()))
        self._sync()
        return out

    def coarse_sweep(self, V, W_prev, first, count, with_source, add_v, out=None):
        W = out if out is not None else self.torch.empty((count, self.M), dtype=self.torch.float64,
                                                         device="cuda")
        self._check(self.L.pit_coarse_sweep_device(
            self.ctx.handle, V.data_ptr() if V is not None else None,
            W_prev.data_ptr() if W_prev is not None else None, W.data_ptr(), first, count,
            int(with_source), int(add_v), self._st()))
        self._sync()
        return W

    def fine_source(self, first, count):
        out = self.torch.empty((count, self.M), dtype=self.torch.float64, device="cuda")
        self._check(self.L.pit_fine_source_device(self.ctx.handle, out.data_ptr(), first, count,
                                                  self._st()))
        self._sync()
        return out

    def partials(self, a, b):
        p = self.torch.empty(a.shape[0], dtype=self.torch.float64, device="cuda")
        self._check(self.L.pit_block_partials_device(self.ctx.handle, a.data_ptr(), b.data_ptr(),
                                                     p.data_ptr(), a.shape[0], self._st()))
        return p

    def partials2(self, a0, b0, a1, b1):
        p = self.torch.empty(2 * a0.shape[0], dtype=self.torch.float64, device="cuda")
        self._check(self.L.pit_block_partials2_device(self.ctx.handle, a0.data_ptr(),
                                                      b0.data_ptr(), a1.data_ptr(), b1.data_ptr(),
                                                      p.data_ptr(), a0.shape[0], self._st()))
        return p

    def update_s(self, alpha, r, d):
        s = self.torch.empty_like(r)
        p = self.torch.empty(r.shape[0], dtype=self.torch.float64, device="cuda")
        self._check(self.L.pit_update_s_device(self.ctx.handle, alpha, r.data_ptr(), d.data_ptr(),
                                               s.data_ptr(), p.data_ptr(), r.shape[0], self._st()))
        return s, p

    def update_lr(self, alpha, omega, p, s, t, rs, lam):
        r = self.torch.empty_like(s)
        part = self.torch.empty(2 * s.shape[0], dtype=self.torch.float64, device="cuda")
        self._check(self.L.pit_update_lr_device(self.ctx.handle, alpha, omega, p.data_ptr(),
                                                s.data_ptr(), t.data_ptr(), rs.data_ptr(),
                                                lam.data_ptr(), r.data_ptr(), part.data_ptr(),
                                                s.shape[0], self._st()))
        return r, part

    def update_p(self, omega, beta, d, r, p):
        self._check(self.L.pit_update_p_device(self.ctx.handle, omega, beta, d.data_ptr(),
                                               r.data_ptr(), p.data_ptr(), p.shape[0], self._st()))

    def axpy(self, a, x, y):
        self._check(self.L.pit_axpy_device(self.ctx.handle, a, x.data_ptr(), y.data_ptr(),
                                           y.shape[0], self._st()))

    def add(self, x, y):
        self._check(self.L.pit_add_device(self.ctx.handle, x.data_ptr(), y.data_ptr(), y.shape[0],
                                          self._st()))


# ---------------------------------------------------------------------------
# The native sharded path: the C ABI's communicator and sharded solver
# (pit_comm_*, pit_sharded_*; csrc/pit_comm.cpp).  The whole
# exchange (halo overlapped with the interior slabs, the coarse chain, the
# partials all-gather) runs inside the library; Python only sets it up.
# ---------------------------------------------------------------------------

class Communicator:
    """pit_comm: NCCL (one rank per GPU) or host callbacks over a
    torch.distributed process group (any backend; the CPU-exchange tests use
    gloo with several processes on one GPU)."""

    def __init__(self, handle, rank: int, world: int, keep=None):
        self.handle, self.rank, self.world = handle, rank, world
        self._keep = keep

    @staticmethod
    def nccl_unique_id() -> bytes:
        import ctypes as C

        from . import _lib
        from .api import _check

        buf = C.create_string_buffer(128)
        _check(_lib.lib().pit_comm_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, rank: int, world: int, device: int, unique_id: bytes) -> "Communicator":
        import ctypes as C

        from . import _lib
        from .api import _check

        h = C.c_void_p()
        _check(_lib.lib().pit_comm_create_nccl(C.create_string_buffer(unique_id, 128), rank, world,
                                               device, C.byref(h)))
        return cls(h, rank, world)

    @classmethod
    def from_process_group(cls, device: int = 0, group=None, transport: str = "nccl"):
        """Every rank of `group` calls this: transport "nccl" shares rank 0's
        NCCL id over the group; "host" routes the exchange through the
        group's own send/recv/all_gather."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if transport == "host":
            return cls.host(rank, world, group)
        obj = [cls.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.nccl(rank, world, device, obj[0])

    @classmethod
    def host(cls, rank: int, world: int, group=None) -> "Communicator":
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib
        from .api import _check

        def view(buf, n):
            return torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))

        def send(buf, n, peer, _user):
            try:
                dist.send(view(buf, n), peer, group=group)
                return 0
            except Exception:  # pragma: no cover
                return 1

        def recv(buf, n, peer, _user):
            try:
                dist.recv(view(buf, n), peer, group=group)
                return 0
            except Exception:  # pragma: no cover
                return 1

        def allgather(buf, n, out, _user):
            try:
                parts = [torch.empty(n, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, view(buf, n).clone(), group=group)
                o = view(out, n * world)
                for r, t in enumerate(parts):
                    o[r * n:(r + 1) * n] = t
                return 0
            except Exception:  # pragma: no cover
                return 1

        cbs = (_lib.COMM_SEND(send), _lib.COMM_RECV(recv), _lib.COMM_ALLGATHER(allgather))
        ops = _lib.CommOpsC(cbs[0], cbs[1], cbs[2], None)
        h = C.c_void_p()
        _check(_lib.lib().pit_comm_create_host(C.byref(ops), rank, world, C.byref(h)))
        return cls(h, rank, world, keep=(cbs, ops))

    def close(self):
        from . import _lib

        if self.handle:
            _lib.lib().pit_comm_destroy(self.handle)
            self.handle = None


class ShardedContext:
    """A BlockOperatorContext (the whole problem, on this rank's GPU) with a
    Communicator attached: the rank owns the contiguous global blocks
    [first, first+count) and the operators and solvers run sharded through
    the C ABI (pit_sharded_*)."""

    def __init__(self, ctx, comm: Communicator):
        import ctypes as C

        from . import _lib
        from .api import _check

        self.ctx, self.comm = ctx, comm
        self.L = _lib.lib()
        _check(self.L.pit_context_attach_comm(ctx.handle, comm.handle))
        f, c = C.c_int(), C.c_int()
        _check(self.L.pit_context_shard(ctx.handle, C.byref(f), C.byref(c)))
        self.first, self.count = f.value, c.value

    def detach(self):
        self.L.pit_context_attach_comm(self.ctx.handle, None)

    def apply_F(self, L_local, stream=None):
        """(F L)_n of the rank's blocks; L_local / result: torch CUDA (count, M)."""
        import torch

        from .api import _check

        out = torch.empty_like(L_local)
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(self.L.pit_sharded_apply_F_device(self.ctx.handle, L_local.data_ptr(),
                                                 out.data_ptr(), st))
        _check(self.L.pit_sharded_sync_status(self.ctx.handle, st))
        return out

    def solve(self, config=None, which: str = "pitsbicg", init_local=None):
        """Sharded pitsbicg_solve / parareal_solve: (lambda of the rank's
        blocks as a torch CUDA tensor, ConvergenceHistory) — the history is the
        same on every rank and bit-identical to the one-GPU solve."""
        import ctypes as C

        import torch

        from . import _lib
        from .api import (ConvergenceHistory, IterationRecord, SolverConfig, SolveStatus, _check)

        config = config or SolverConfig()
        config.validate()
        lam = torch.empty((self.count, self.ctx.M), dtype=torch.float64, device="cuda")
        cap = config.max_iterations + 2
        recs = (_lib.RecordC * cap)()
        info = _lib.SolveInfoC()
        cfg = config._c()
        fn = (self.L.pit_sharded_pitsbicg_solve_device if which == "pitsbicg"
              else self.L.pit_sharded_parareal_solve_device)
        _check(fn(self.ctx.handle, C.byref(cfg),
                  init_local.data_ptr() if init_local is not None else None, lam.data_ptr(), recs,
                  cap, C.byref(info), torch.cuda.current_stream().cuda_stream))
        hist = ConvergenceHistory()
        for i in range(info.record_count):
            r = recs[i]
            hist.records.append(IterationRecord(r.k, r.residual_norm, r.fine_applications,
                                                r.coarse_applications, r.wall_ms,
                                                r.error_vs_reference if r.has_error else None))
        hist.status = (SolveStatus.Converged if info.status == _lib.PIT_CONVERGED
                       else SolveStatus.MaxIterations)
        hist.restarts = info.restarts
        hist.stats._accumulate(info.stats)
        return lam, hist


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
