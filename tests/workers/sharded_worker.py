"""One rank of the sharded C-ABI solver over the host transport (gloo),
used by tests/test_gpu_sharded.py: every rank runs on cuda:0 (the kernels of
different ranks never wait on one another: every exchange is a blocking host
call), solves, and rank 0 writes the gathered solution and history.

  python tests/workers/sharded_worker.py <rank> <world> <port> <case> <slabs> <out.npz>
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from cases import make_case  # noqa: E402
from paper_2203_10148_b200 import api  # noqa: E402
from paper_2203_10148_b200.distributed import Communicator, ShardedContext  # noqa: E402


def main():
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    case, slabs, out = sys.argv[4], int(sys.argv[5]), sys.argv[6]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    p = make_case(case, slabs)
    comm = Communicator.host(rank, world)
    with api.BlockOperatorContext(p) as ctx:
        sc = ShardedContext(ctx, comm)
        rng = np.random.default_rng(3)
        L = rng.uniform(-1, 1, (p.N, p.M))
        fx = sc.apply_F(torch.tensor(L[sc.first:sc.first + sc.count], device="cuda"))
        lam, hist = sc.solve(api.SolverConfig(tolerance=1e-10))
        par, phist = sc.solve(api.SolverConfig(tolerance=1e-10), which="parareal")
        # the error path: a NaN in one rank's input is reported identically
        # on every rank (lowest failing slab)
        bad = L.copy()
        bad[p.N - 2, 3] = np.nan  # propagated by slab N-2 (the last slab)
        err = ""
        try:
            sc.apply_F(torch.tensor(bad[sc.first:sc.first + sc.count], device="cuda"))
        except api.SlabError as e:
            err = f"SlabError {e.slab_index}"
        sc.detach()
    parts = [None] * world
    dist.all_gather_object(parts, (sc.first, fx.cpu().numpy(), lam.cpu().numpy(),
                                   par.cpu().numpy(), err))
    if rank == 0:
        parts.sort(key=lambda t: t[0])
        rows = np.array([(r.k, r.residual_norm, r.fine_applications, r.coarse_applications)
                         for r in hist.records])
        prow = np.array([(r.k, r.residual_norm, r.fine_applications, r.coarse_applications)
                         for r in phist.records])
        np.savez(out, apply_F=np.concatenate([t[1] for t in parts]),
                 lam=np.concatenate([t[2] for t in parts]),
                 parareal=np.concatenate([t[3] for t in parts]), rows=rows, prows=prow,
                 restarts=hist.restarts, errors=np.array([t[4] for t in parts]), L=L)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
