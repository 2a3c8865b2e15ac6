"""Back-to-back timing of single entry points on the c3 mesh (events around
200 launches) -- kernel time + launch gap, no profiler."""
import sys, json
import torch
sys.path.insert(0, '.')
from paper_1403_0968_b200 import meshgen, sem
N = int(sys.argv[1]) if len(sys.argv) > 1 else 7
el = tuple(int(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (16, 16, 16)
xi, _ = sem.gll(N)
m = meshgen.box_mesh(N, xi, elems=el, eps=0.05)
ctx = sem.Context(m, N, device=0)
u = torch.from_numpy(meshgen.random_field(m.nlocal, 0)).cuda()
w = torch.empty_like(u)
def t(fn, R=200):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(R): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / R * 1e3
res = {"ax_us": t(lambda: ctx.ax(u, w)), "dssum_us": t(lambda: ctx.dssum(w)), "mask_us": t(lambda: ctx.mask(w)),
       "mass_us": t(lambda: ctx.mass(u, w)), "copy_us": t(lambda: w.copy_(u))}
L = m.nlocal
res["ax_GBs"] = 64 * L / res["ax_us"] / 1e3
res["copy_GBs"] = 16 * L / res["copy_us"] / 1e3
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
