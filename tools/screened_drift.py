"""Drift of the GPU CG iterate from the oracle's at fixed iteration counts
(tol = 0) on a screened-Coulomb problem without Dirichlet nodes."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch, oracle
from paper_1403_0968_b200 import meshgen, sem
N, el = 3, (3, 3, 3)
for d in (False, True):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=el, eps=0.05, dirichlet_faces=d)
    kap, alp = meshgen.coefficients(m)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0, kappa=kap, alpha=alp)
    _, f = meshgen.manufactured(m)
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f + 1.0)
    bt = torch.from_numpy(b).cuda()
    for k in (1, 2, 5, 10, 20, 50, 100, 150, 173):
        x, its, rel, ok = ctx.cg(bt, tol=0.0, maxit=k)
        xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=k, J=J, kappa=kap, alpha=alp)
        xe = np.linalg.norm(x.cpu().numpy() - xr) / np.linalg.norm(xr)
        print("dirichlet" if d else "natural", k, "x rel %.2e" % xe, "res gpu %.6e oracle %.6e" % (rel, rel_r), flush=True)
