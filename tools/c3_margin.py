"""Residual history of the c3 CG solve near the 1e-8 crossing (GPU) and,
optionally, the oracle's iteration count on the same inputs."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1403_0968_b200 import meshgen, sem
import oracle
N = 7
xi, _ = oracle.gll(N)
m = meshgen.box_mesh(N, xi, elems=(16, 16, 16), eps=0.05)
G, J = oracle.geom(N, m.xyz)
_, f = meshgen.manufactured(m)
b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
ctx = sem.Context(m, N, device=0)
bd = torch.from_numpy(b).cuda()
for mi in range(668, 680):
    x, its, rel, ok = ctx.cg(bd, tol=0.0, maxit=mi)
    print('gpu maxit', mi, 'rel_res %.15e' % rel, flush=True)
x, its, rel, ok = ctx.cg(bd, tol=1e-8, maxit=5000)
print('gpu tol1e-8 its', its, rel)
if '--oracle' in sys.argv:
    t = time.time()
    xr, itr, relr, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=5000)
    print('oracle its', itr, 'rel %.15e' % relr, 'time', time.time() - t)
    print('x rel-L2', np.linalg.norm(x.cpu().numpy() - xr) / np.linalg.norm(xr))
    for mi in (itr - 1, itr, itr + 1):
        xr2, it2, rel2, _ = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=mi)
        print('oracle maxit', mi, 'rel_res %.15e' % rel2, flush=True)
