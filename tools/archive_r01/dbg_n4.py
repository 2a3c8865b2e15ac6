import sys, torch
sys.path.insert(0, '.')
from paper_1403_0968_b200 import meshgen, sem
N = int(sys.argv[1]); el = tuple(int(v) for v in sys.argv[2:5])
xi, _ = sem.gll(N)
m = meshgen.box_mesh(N, xi, elems=el, eps=0.05)
ctx = sem.Context(m, N, device=0)
u = torch.from_numpy(meshgen.random_field(m.nlocal, 0)).cuda()
w = ctx.ax(u)
torch.cuda.synchronize()
print("ok", N, el, m.nlocal, float(w.abs().max()))
