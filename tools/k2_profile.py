"""Warm-cache profile target: the c3 CG solve (4096 el, N=7) run a few times,
for `ncu --replay-mode application` (every metric pass re-runs this script,
so the profiled kernel sees the L2 state of a real solve, unlike kernel
replay with its save/restore).  Usage under ncu:
  ncu --replay-mode application --cache-control none -k regex:k2 -s 40 -c 1 \
      --section SpeedOfLight ... python tools/k2_profile.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

N = int(os.environ.get("K2P_N", "7"))
e = int(os.environ.get("K2P_E", "16"))
xi, _ = sem.gll(N)
m = meshgen.box_mesh(N, xi, elems=(e, e, e), eps=0.05)
ctx = sem.Context(m, N, device=0)
_, f = meshgen.manufactured(m)
b = ctx.rhs(torch.from_numpy(f).cuda())
x = torch.zeros_like(b)
for _ in range(int(os.environ.get("K2P_SOLVES", "2"))):
    x.zero_()
    ctx.cg(b, x, tol=1e-8, maxit=5000)
torch.cuda.synchronize()
print("done")
