"""c3 CG solve time (CUDA events, best of --reps) for the current environment;
prints one JSON line (us per iteration, GDOF/s, L2 attributes)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=7)
ap.add_argument("--elems", type=int, nargs=3, default=(16, 16, 16))
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--precond", default="none")
ap.add_argument("--variant", default="standard")
a = ap.parse_args()
xi, _ = sem.gll(a.N)
m = meshgen.box_mesh(a.N, xi, elems=tuple(a.elems), eps=0.05)
_, f = meshgen.manufactured(m)
ctx = sem.Context(m, a.N, device=0)
b = ctx.mass(torch.from_numpy(f).cuda())
ctx.cg(b, tol=1e-8, maxit=5000, precond=a.precond, variant=a.variant)
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    x, its, rel, ok = ctx.cg(b, tol=1e-8, maxit=5000, precond=a.precond, variant=a.variant)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
p = torch.cuda.get_device_properties(0)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SEM_")}, "N": a.N,
                  "its": its, "ms": min(ts), "us_per_it": 1e3 * min(ts) / its,
                  "gdof_s": m.nlocal * its / (min(ts) * 1e-3) / 1e9,
                  "l2_bytes": getattr(p, "L2_cache_size", None),
                  "persisting_max": getattr(p, "persisting_l2_cache_max_size", None)}))
