"""Small invocations of every libsem kernel family, for compute-sanitizer
(tools/sanitizer_sweep.sh): Ax (element-staged TMA, N=7 DMMA with 2 and 4
warps per element, high-order slice-streamed, tensor-core high-order, simple),
K1/K2 CG iterations, the resident CG kernel (SEM_CG_RESIDENT=1), the split
high-order K1 (x/p update + tensor-core operator), Jacobi PCG, single-reduction CG,
the gather-scatter, the boundary/interior K1 split, the multi-rank loopback
path (pack/combine/rank folds) and the FD stencil (both arithmetic forms).
Tiny meshes, few iterations: the sanitizers slow kernels down 10-100x.
Each case checks its result against the oracle so a silent miscompute under
the tool is caught too.  Usage: python tools/sanitize_driver.py [N ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1403_0968_b200 import dist as sdist  # noqa: E402
from paper_1403_0968_b200 import fd, meshgen, sem  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def case(N, elems, kernel, extra=None):
    env = {"SEM_AX_KERNEL": kernel or ""}
    env.update(extra or {})
    old = {k: os.environ.get(k) for k in env}
    for k, v in env.items():
        if v:
            os.environ[k] = v
        else:
            os.environ.pop(k, None)
    try:
        xi, _ = oracle.gll(N)
        m = meshgen.box_mesh(N, xi, elems=elems, eps=0.05)
        G, J = oracle.geom(N, m.xyz)
        ctx = sem.Context(m, N, device=0)
        dev = torch.device("cuda", 0)
        u = meshgen.random_field(m.nlocal, 1)
        w = ctx.ax(torch.from_numpy(u).to(dev))
        wr = oracle.ax(N, G, u)
        assert rel(w.cpu().numpy(), wr) <= 1e-12
        ctx.dssum(w)
        assert rel(w.cpu().numpy(), oracle.dssum(m.glo, wr)) <= 1e-12
        _, f = meshgen.manufactured(m)
        b = torch.from_numpy(oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)).to(dev)
        for kw in ({}, {"precond": "jacobi"}, {"variant": "single_reduction"}):
            if kw.get("variant") and kernel == "simple":
                continue
            x, its, _, _ = ctx.cg(b, tol=0.0, maxit=6, **kw)
            assert its == 6
        torch.cuda.synchronize()
        ctx.free()
        print(f"ok N={N} elems={elems} kernel={kernel or 'default'} {extra or ''}", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def multirank(N, elems, P):
    xi, _ = oracle.gll(N)
    parts = meshgen.default_parts(P)
    ranks = [meshgen.box_mesh(N, xi, elems=elems, eps=0.05, parts=parts, rank=r,
                              boundary_first=True) for r in range(P)]

    def body(lr):
        m = ranks[lr.rank]
        ctx = sem.Context(m, N, device=0, loopback=lr)
        try:
            u = torch.from_numpy(meshgen.random_field(m.nlocal, 2)).cuda()
            ctx.dssum(u)
            _, f = meshgen.manufactured(m)
            b = ctx.rhs(torch.from_numpy(f).cuda())
            for kw in ({}, {"precond": "jacobi"}, {"variant": "single_reduction"}):
                ctx.cg(b, tol=0.0, maxit=4, **kw)
        finally:
            ctx.free()

    sdist.LoopbackGroup(P, device=0).run(body)
    print(f"ok multirank N={N} P={P}", flush=True)


def fd_case():
    h, w = 40, 96
    rng = np.random.default_rng(3)
    for r in (1, 4, 7):
        u1, u2 = rng.uniform(-1, 1, (h, w)), rng.uniform(-1, 1, (h, w))
        om = fd.weights(r, 2.0 / w)
        g1, g2 = torch.from_numpy(u1).cuda(), torch.from_numpy(u2).cuda()
        g3 = torch.empty_like(g1)
        fd.step(g1, g2, g3, om, 0.01)
        assert np.array_equal(g3.cpu().numpy(), oracle.fd_step(u1, u2, om, 0.01))
        fd.run(g1, g2, g3, om, 0.01, 3, regrouped=True)
    torch.cuda.synchronize()
    print("ok fd", flush=True)


def main():
    Ns = [int(a) for a in sys.argv[1:]] or [3, 4, 7, 10, 15]
    for N in Ns:
        elems = (2, 2, 1) if N >= 10 else (2, 2, 2)
        case(N, elems, None)
        case(N, elems, "simple")
        if N <= 10:
            case(N, elems, "tma")
        if N >= 6:
            case(N, elems, "hi")
        if N == 7:
            case(N, elems, None, {"SEM_DMMA_W": "2"})
            case(N, elems, None, {"SEM_K1_SPLIT": "0.5"})
            case(N, elems, None, {"SEM_CG_RESIDENT": "1"})      # the resident CG kernel
            case(N, (3, 2, 1), None, {"SEM_CG_RESIDENT": "1"})
            case(N, elems, None, {"SEM_L2_PERSIST": "1"})
        if N >= 10:
            case(N, elems, None, {"SEM_DMMAG": "0"})
            case(N, elems, None, {"SEM_K1_AX": "fused" if N >= 11 else "split"})
    multirank(4, (2, 2, 2), 2)
    multirank(7, (2, 2, 2), 8)
    fd_case()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
