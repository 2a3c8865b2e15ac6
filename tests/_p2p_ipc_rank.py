"""One rank of the cross-PROCESS peer-memory transport test
(tests/test_gpu_p2p_ipc.py): launched by torch.distributed.run with the gloo
backend, every rank on cuda:0 (one GPU here), SEM_COMM=p2p -- the windows are
shared through CUDA IPC handles exchanged by the setup all-gather (the path
one-process-per-GPU runs use), the flags with release / acquire at system
scope.  Rank 0 writes a JSON verdict to the path in argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
from paper_1403_0968_b200 import meshgen, sem  # noqa: E402
from tests.test_gpu_multirank import partition, rank_ordered_dssum  # noqa: E402


def main():
    out_path = sys.argv[1]
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    N, elems = 4, (2, 4, 4)
    full, ranks, pos = partition(N, elems, P)
    n3 = (N + 1) ** 3
    G, J = oracle.geom(N, full.xyz)
    vfull = meshgen.random_field(full.nlocal, 5).reshape(full.nelem, n3)
    vs = [vfull[p].reshape(-1) for p in pos]
    e1 = rank_ordered_dssum(ranks, vs)
    e2 = rank_ordered_dssum(ranks, e1)
    _, f = meshgen.manufactured(full)
    b = oracle.mass_rhs(N, full.glo, full.dirichlet, J, f).reshape(full.nelem, n3)
    xr, its_r, _, _ = oracle.cg(N, full.glo, full.dirichlet, G, b.reshape(-1), tol=1e-8, maxit=2000)
    xr = xr.reshape(full.nelem, n3)
    ctx = sem.Context(ranks[rank], N, device=0, group=dist.group.WORLD)
    u = torch.from_numpy(vs[rank]).cuda()
    bb = torch.from_numpy(b[pos[rank]].reshape(-1)).cuda()
    d1, d2, x = torch.empty_like(u), torch.empty_like(u), torch.zeros_like(u)
    torch.cuda.synchronize()
    dist.barrier()
    d1.copy_(u)
    ctx.dssum(d1)
    d2.copy_(d1)
    ctx.dssum(d2)
    x, its, rel, ok = ctx.cg(bb, x, tol=1e-8, maxit=2000)
    ctx.status()
    res = {
        "rank": rank,
        "dssum1": bool(np.array_equal(d1.cpu().numpy(), e1[rank])),
        "dssum2": bool(np.array_equal(d2.cpu().numpy(), e2[rank])),
        "its": its, "its_oracle": its_r, "ok": bool(ok),
        "x_relerr": float(np.linalg.norm(x.cpu().numpy() - xr[pos[rank]].reshape(-1))
                          / np.linalg.norm(xr[pos[rank]].reshape(-1))),
    }
    gathered = [None] * P
    dist.all_gather_object(gathered, res)
    ctx.free()
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(gathered, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
