"""A few plain Ax applies at c4 size for one order N (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

N = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n3 = (N + 1) ** 3
E = max(1, round(16.8e6 / n3))
ex = round(E ** (1 / 3))
elems = (ex, ex, max(1, E // (ex * ex)))
xi, _ = sem.gll(N)
m = meshgen.box_mesh(N, xi, elems=elems, eps=0.05)
ctx = sem.Context(m, N, device=0)
u = torch.randn(m.nlocal, dtype=torch.float64, device="cuda")
for _ in range(reps):
    w = ctx.ax(u)
torch.cuda.synchronize()
print("N", N, "elems", elems)
