#!/usr/bin/env python
"""Config c2 (BASELINE.json configs[1]): 512 elements (8x8x8), N=7, Ax + DSSUM
throughput on one B200.  As SURVEY.md §8(d) prescribes, the applies run as one
CUDA graph of `reps` back-to-back (Ax, DSSUM) pairs (sem_kernel_replay
which=3) to amortise launch latency; the 16.8 MB working set is L2-resident,
so this is labelled "L2-resident", not a roofline claim.  Also Ax alone.
Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1403_0968_b200 import meshgen, sem
    N, elems, reps = 7, (8, 8, 8), 100
    xi, _ = sem.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=0.05)
    ctx = sem.Context(m, N, device=0)
    L = ctx.nlocal
    u = torch.from_numpy(meshgen.random_field(L, 0)).cuda()
    w = ctx.ax(u)
    ctx.cg(ctx.rhs(u), tol=0.0, maxit=2)          # fills the internal work vectors
    stream = torch.cuda.current_stream()
    out = {"config": "c2: 512 hex elements (8x8x8), N=7, eps=0.05, one B200",
           "local_dof": L, "unique_dof": ctx.nglobal, "reps_per_graph": reps,
           "note": "L2-resident (16.8 MB working set); CUDA events around one graph of reps applies"}
    for name in ("ax", "ax+dssum"):
        ctx.kernel_replay(name, reps)             # warm-up (and graph build)
        torch.cuda.synchronize()
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.kernel_replay(name, reps)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            best = ms if best is None else min(best, ms)
        out[name] = {"us_per_apply": 1e3 * best, "gdof_s": L / (best * 1e-3) / 1e9,
                     "model_gbs_ax": 64.0 * L / (best * 1e-3) / 1e9}
    print(json.dumps(out))
    ctx.free()


if __name__ == "__main__":
    main()
