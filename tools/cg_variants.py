"""Time the c3 CG solve under the current SEM_* environment; print one line.
Usage: SEM_PDL=0 SEM_CG_GRAPH=1 python tools/cg_variants.py [N ex ey ez]"""
import os, sys, json
import torch
sys.path.insert(0, '.')
from paper_1403_0968_b200 import meshgen, sem
N = int(sys.argv[1]) if len(sys.argv) > 1 else 7
el = tuple(int(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (16, 16, 16)
xi, _ = sem.gll(N)
m = meshgen.box_mesh(N, xi, elems=el, eps=0.05)
ctx = sem.Context(m, N, device=0)
_, f = meshgen.manufactured(m)
b = ctx.rhs(torch.from_numpy(f).cuda())
x = torch.zeros_like(b)
for _ in range(3):
    x.zero_(); ctx.cg(b, x, tol=1e-8, maxit=5000)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 10
e0.record()
for _ in range(K):
    x.zero_(); _, its, rel, ok = ctx.cg(b, x, tol=1e-8, maxit=5000)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
ctx.profile(True)
for _ in range(2):
    x.zero_(); ctx.cg(b, x, tol=1e-8, maxit=5000)
pr = ctx.profile_read(); ctx.profile(False)
avg = {k: round(1e3 * v[0] / v[1], 2) for k, v in pr.items() if v[1]}
env = {k: v for k, v in os.environ.items() if k.startswith('SEM_')}
print(json.dumps({"env": env, "N": N, "elems": el, "ms_per_solve": round(ms, 3), "its": its,
                  "us_per_it": round(1e3 * ms / its, 2), "kernel_avg_us": avg}))
