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
# classify; each exchange kernel (pack / sync / combine) of an iteration is
# paired with the interior K1 it was forked beside: the latest LONG K1 launch
# (the interior range, >= 60% of the longest K1) that started before the
# rank's pack.  CUPTI's stream ids of graph nodes are not stable enough to
# tell the ranks apart, but the ranks' iterations alternate on the shared
# GPU, so "latest interior K1 before this pack" is the same rank's.
rows = []
for name, t0, d, sid in events:
    c = kernel_trace.classify(name)
    nm = name.split("(")[0].replace("sem::", "")
    kind = ("k1" if c == "k1" else
            "pack" if "pack_kernel" in nm else "sync" if "p2p_sync" in nm else
            "combine" if "combine_kernel" in nm else "o")
    rows.append({"kind": kind, "t0": t0, "t1": t0 + d})
rows.sort(key=lambda r: r["t0"])
k1s = [r for r in rows if r["kind"] == "k1"]
longest = max(r["t1"] - r["t0"] for r in k1s)
interior = [r for r in k1s if r["t1"] - r["t0"] >= 0.6 * longest]
stats = {k: [0, 0.0, 0.0] for k in ("pack", "sync", "combine")}
for i, r in enumerate(rows):
    if r["kind"] != "pack":
        continue
    cands = [b for b in interior if b["t0"] <= r["t0"] + 0.5]
    if not cands:
        continue
    b = cands[-1]
    # this pack and the sync / combine that follow it on the same side branch
    grp = [r] + [q for q in rows[i + 1:i + 12] if q["kind"] in ("sync", "combine")][:2]
    for q in grp:
        st = stats[q["kind"]]
        st[0] += 1
        st[1] += q["t1"] - q["t0"]
        st[2] += max(0.0, min(q["t1"], b["t1"]) - max(q["t0"], b["t0"]))
out = {"config": f"c3 over P={P} loopback ranks on one GPU, transport "
                 f"{os.environ.get('SEM_COMM', 'host')}",
       "interior_k1_mean_us": sum(b["t1"] - b["t0"] for b in interior) / max(len(interior), 1),
       "exchange_kernels": {k: {"launches": v[0], "mean_us": v[1] / max(v[0], 1),
                                "fraction_inside_interior_k1": v[2] / v[1] if v[1] else None}
                            for k, v in stats.items()}}
json.dump(out, open(args.out + ".json", "w"), indent=1)
print(json.dumps(out))
