"""Cases of the peer-memory transport (SEM_COMM=p2p) on one GPU, run in a
fresh process by tests/test_gpu_p2p.py (CUDA_MODULE_LOADING=EAGER and
CUDA_DEVICE_MAX_CONNECTIONS=32 must be in the environment before CUDA
starts).  Each rank warms up (allocations) and meets the others at a host
barrier before its first device-side collective (include/sem.h: several
ranks on one device).  Prints one JSON line per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1403_0968_b200 import dist as sdist  # noqa: E402
from paper_1403_0968_b200 import meshgen, sem  # noqa: E402
from tests.test_gpu_multirank import partition, rank_ordered_dssum  # noqa: E402


def relerr(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def case(N, elems, P, method):
    full, ranks, pos = partition(N, elems, P)
    n3 = (N + 1) ** 3
    G, J = oracle.geom(N, full.xyz)
    vfull = meshgen.random_field(full.nlocal, 5).reshape(full.nelem, n3)
    vs = [vfull[p].reshape(-1) for p in pos]
    e1 = rank_ordered_dssum(ranks, vs)
    e2 = rank_ordered_dssum(ranks, e1)
    _, f = meshgen.manufactured(full)
    b = oracle.mass_rhs(N, full.glo, full.dirichlet, J, f).reshape(full.nelem, n3)
    if method == "sr":
        xr, its_r, _, _ = oracle.cg_single_reduction(N, full.glo, full.dirichlet, G, b.reshape(-1),
                                                     tol=1e-8, maxit=3000)
    else:
        xr, its_r, _, _ = oracle.cg(N, full.glo, full.dirichlet, G, b.reshape(-1), tol=1e-8,
                                    maxit=3000, precond="jacobi" if method == "jacobi" else "none")
    xr = xr.reshape(full.nelem, n3)
    kw = {"precond": "jacobi"} if method == "jacobi" else (
        {"variant": "single_reduction"} if method == "sr" else {})

    def body(lr):
        r = lr.rank
        ctx = sem.Context(ranks[r], N, device=0, loopback=lr)
        try:
            u = torch.from_numpy(vs[r]).cuda()
            bb = torch.from_numpy(b[pos[r]].reshape(-1)).cuda()
            d1, d2, x = torch.empty_like(u), torch.empty_like(u), torch.zeros_like(u)
            x2 = torch.zeros_like(u)
            torch.cuda.synchronize()
            lr.barrier()                         # warm, then the device-side collectives
            d1.copy_(u)
            ctx.dssum(d1)
            d2.copy_(d1)
            ctx.dssum(d2)
            x, its, rel, ok = ctx.cg(bb, x, tol=1e-8, maxit=3000, **kw)
            x2, its2, _, _ = ctx.cg(bb, x2, tol=1e-8, maxit=3000, **kw)   # graph replay
            ctx.status()
            return (d1.cpu().numpy(), d2.cpu().numpy(), x.cpu().numpy(), its, ok,
                    bool(torch.equal(x, x2)), its2)
        finally:
            ctx.free()

    out = sdist.LoopbackGroup(P, device=0).run(body)
    res = {"N": N, "P": P, "method": method, "its_oracle": its_r, "ok": True, "why": []}
    for r, (d1, d2, x, its, ok, same, its2) in enumerate(out):
        checks = {
            "dssum1 bit-identical": np.array_equal(d1, e1[r]),
            "dssum2 bit-identical": np.array_equal(d2, e2[r]),
            "converged": ok,
            "count": its == its_r and its2 == its,
            "x": relerr(x, xr[pos[r]].reshape(-1)) <= 1e-10,
            "repeat identical": same,
        }
        for k, v in checks.items():
            if not v:
                res["ok"] = False
                res["why"].append(f"rank {r}: {k} (its {its} vs {its_r})")
    return res


def main():
    cases = [(3, (4, 4, 4), 2, "cg"), (4, (4, 4, 4), 4, "cg"), (7, (4, 4, 4), 8, "cg"),
             (4, (2, 4, 4), 2, "jacobi"), (7, (2, 2, 4), 2, "sr"), (11, (2, 2, 4), 2, "cg"),
             (3, (4, 4, 4), 8, "sr")]
    for c in cases:
        print(json.dumps(case(*c)), flush=True)


if __name__ == "__main__":
    main()
