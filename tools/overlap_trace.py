"""Timeline evidence for the overlap of the interface exchange with the
interior-element K1 ("boundary-element Ax first, then the
exchange on a second stream concurrently with the interior-element Ax"; the
nsys trace SURVEY.md §8(d) asks for -- nsys is not in this image, CUPTI via
torch.profiler is).  Config: c3 split over P = 2 in-process ranks on one GPU
(1x1x2 blocks, boundary elements first), peer-memory transport with CUDA
graphs (SEM_COMM=p2p) or the host-rendezvous one.  Writes a JSON summary
(per iteration and rank: boundary K1, exchange kernels, interior K1 start /
end, and whether the exchange ran inside the interior K1's interval) and a
chrome trace of a few iterations.

  SEM_COMM=p2p CUDA_MODULE_LOADING=EAGER CUDA_DEVICE_MAX_CONNECTIONS=32 \\
      python tools/overlap_trace.py --out gpurun_out/overlap
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import kernel_trace  # noqa: E402
from paper_1403_0968_b200 import dist as sdist  # noqa: E402
from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/overlap")
ap.add_argument("--its", type=int, default=16)
args = ap.parse_args()
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)

N, P = 7, 2
xi, _ = sem.gll(N)
parts = meshgen.default_parts(P)
meshes = [meshgen.box_mesh(N, xi, elems=(16, 16, 16), eps=0.05, parts=parts, rank=r,
                           boundary_first=True) for r in range(P)]
ctxs = [None] * P
bufs = [None] * P
go = __import__("threading").Barrier(P + 1)
done = __import__("threading").Barrier(P + 1)


def body(lr):
    r = lr.rank
    ctx = sem.Context(meshes[r], N, device=0, loopback=lr)
    _, f = meshgen.manufactured(meshes[r])
    b = ctx.rhs(torch.from_numpy(f).cuda())
    x = torch.zeros_like(b)
    ctx.cg(b, x, tol=0.0, maxit=args.its)             # warm (graphs, caches)
    torch.cuda.synchronize()
    lr.barrier()
    go.wait()                                          # the profiler is on
    x.zero_()
    ctx.cg(b, x, tol=0.0, maxit=args.its)
    torch.cuda.synchronize()
    done.wait()
    ctx.free()


import threading  # noqa: E402
grp = sdist.LoopbackGroup(P, device=0)
runner = threading.Thread(target=lambda: grp.run(body))
runner.start()
events = []


def traced():
    go.wait()
    done.wait()


events = kernel_trace.trace(traced, export=args.out + ".trace.json")
runner.join()
# classify, then per rank and iteration: the exchange kernels (pack / sync /
# combine, on the rank's side branch) against that rank's interior K1.  With
# CUDA graphs (p2p) CUPTI reports the boundary K1 and the side branch on the
# rank's stream and the interior K1 on a graph-branch stream; a rank's
# interior K1 is the first K1 off the main streams that starts when its
# boundary K1 has ended.
rows = []
for name, t0, d, sid in events:
    c = kernel_trace.classify(name)
    kind = ("k1" if c == "k1" else
            "ex" if any(k in name for k in ("pack_kernel", "p2p_sync", "combine_kernel")) else "o")
    rows.append({"kind": kind, "name": name.split("(")[0].replace("sem::", "")[-30:], "t0": t0,
                 "t1": t0 + d, "s": sid})
rows.sort(key=lambda r: r["t0"])
k1s = [r for r in rows if r["kind"] == "k1"]
cnt = {}
mains = {}
for r in k1s:
    mains[r["s"]] = mains.get(r["s"], 0) + 1
main_ids = sorted(mains, key=lambda s: -mains[s])[:P]
n_ex, t_ex, t_in = {}, {}, {}
for b in [r for r in k1s if r["s"] not in main_ids] or k1s[1::2]:
    bnd = [r for r in k1s if r["s"] in main_ids and r["t1"] <= b["t0"] + 1.0 and r is not b]
    if not bnd:
        continue
    a = bnd[-1]
    nxt = [r for r in k1s if r["s"] == a["s"] and r["t0"] > a["t0"] and r is not b]
    tend = nxt[0]["t0"] if nxt else 1e18
    for r in rows:
        if r["kind"] != "ex" or not (a["t1"] - 0.5 <= r["t0"] < tend):
            continue
        if r["s"] in main_ids and r["s"] != a["s"]:
            continue
        nm = r["name"]
        n_ex[nm] = n_ex.get(nm, 0) + 1
        t_ex[nm] = t_ex.get(nm, 0.0) + r["t1"] - r["t0"]
        t_in[nm] = t_in.get(nm, 0.0) + max(0.0, min(r["t1"], b["t1"]) - max(r["t0"], b["t0"]))
out = {"config": f"c3 over P={P} loopback ranks on one GPU, transport "
                 f"{os.environ.get('SEM_COMM', 'host')}",
       "exchange_kernels": {k: {"launches": n_ex[k], "mean_us": t_ex[k] / n_ex[k],
                                "fraction_inside_interior_k1": t_in[k] / t_ex[k]} for k in n_ex}}
json.dump(out, open(args.out + ".json", "w"), indent=1)
print(json.dumps(out))
