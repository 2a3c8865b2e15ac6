"""Resident-CG phase clock at c3 (or --elems): per-iteration time of the whole
solve (CUDA events) and CTA 0's split into update+operator / barrier 1 /
DSSUM+r update / barrier 2 (sem_cg_phases), next to the two-kernel schedule.
Usage: python tools/rcg_phases.py [--elems 16 16 16] [--reps 3]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1403_0968_b200 import meshgen, sem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, nargs=3, default=(16, 16, 16))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tol", type=float, default=1e-8)
    args = ap.parse_args()
    os.environ["SEM_CG_RESIDENT"] = "1"      # the context gets the resident tables
    N = 7
    xi, _ = sem.gll(N)
    m = meshgen.box_mesh(N, xi, elems=tuple(args.elems), eps=0.05)
    _, f = meshgen.manufactured(m)
    ctx = sem.Context(m, N, device=0)
    b = ctx.mass(torch.from_numpy(f).cuda())
    out = {"elems": list(args.elems)}
    for mode in ("1", "0"):
        os.environ["SEM_CG_RESIDENT"] = mode
        ctx.cg(b, tol=args.tol, maxit=5000)
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            x, its, rel, ok = ctx.cg(b, tol=args.tol, maxit=5000)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        rec = {"its": its, "ms": min(ts), "us_per_it": 1e3 * min(ts) / max(its, 1)}
        if mode == "1":
            rec["phases_us"] = ctx.cg_phases()
        out["resident" if mode == "1" else "two_kernel"] = rec
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
