"""What the multi-rank code path costs, measured on ONE GPU: config c3 (4096
elements, N = 7, CG to 1e-8) split over P in-process ranks (the c5 block
partition of the 16^3 element grid), every rank on the same device with its
own stream, joined by the host-rendezvous loopback transport or the
peer-memory transport (SEM_COMM=p2p, CUDA graphs on).  The P ranks share the
GPU, so this is NOT a scaling measurement: it shows the per-iteration cost of
the exchange, the rank folds, the all-gathers and the K1 split against the
one-rank solve of the same mesh.

  SEM_COMM=p2p CUDA_MODULE_LOADING=EAGER CUDA_DEVICE_MAX_CONNECTIONS=32 \\
      python tools/loopback_bench.py --ranks 1 2 4 8
"""
import argparse
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_0968_b200 import dist as sdist  # noqa: E402
from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--N", type=int, default=7)
ap.add_argument("--elems", type=int, default=16)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

N, e = args.N, args.elems
xi, _ = sem.gll(N)
rows = []
for P in args.ranks:
    parts = meshgen.default_parts(P)
    meshes = [meshgen.box_mesh(N, xi, elems=(e, e, e), eps=0.05, parts=parts, rank=r,
                               boundary_first=P > 1) for r in range(P)]
    times = [None] * P
    iters = [None] * P

    def body(lr):
        r = lr.rank
        ctx = sem.Context(meshes[r], N, device=0, loopback=lr)
        try:
            _, f = meshgen.manufactured(meshes[r])
            fd = torch.from_numpy(f).cuda()
            b = torch.empty_like(fd)
            x = torch.zeros_like(fd)
            torch.cuda.synchronize()
            lr.barrier()
            b.copy_(ctx.rhs(fd))
            ctx.cg(b, x, tol=1e-8, maxit=5000)         # warm-up (graphs, caches)
            torch.cuda.synchronize()
            lr.barrier()
            t0 = time.perf_counter()
            for _ in range(args.reps):
                x.zero_()
                _, its, _, _ = ctx.cg(b, x, tol=1e-8, maxit=5000)
            torch.cuda.synchronize()
            lr.barrier()
            times[r] = (time.perf_counter() - t0) / args.reps
            iters[r] = its
            ctx.status()
        finally:
            ctx.free()

    sdist.LoopbackGroup(P, device=0).run(body)
    t = max(times)
    row = {"P": P, "transport": os.environ.get("SEM_COMM", "host") if P > 1 else "-",
           "iters": iters[0], "ms_per_solve": 1e3 * t, "us_per_iteration": 1e6 * t / iters[0]}
    rows.append(row)
    print(json.dumps(row), flush=True)
