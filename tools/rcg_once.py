"""One resident CG solve at c3 with a fixed iteration count (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

os.environ.setdefault("SEM_CG_RESIDENT", "1")
its = int(sys.argv[1]) if len(sys.argv) > 1 else 30
N = 7
xi, _ = sem.gll(N)
m = meshgen.box_mesh(N, xi, elems=(16, 16, 16), eps=0.05)
_, f = meshgen.manufactured(m)
ctx = sem.Context(m, N, device=0)
b = ctx.mass(torch.from_numpy(f).cuda())
x, k, rel, ok = ctx.cg(b, tol=0.0, maxit=its)
torch.cuda.synchronize()
print("its", k, "phases", ctx.cg_phases())
