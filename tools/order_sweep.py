"""Config c4 (BASELINE.json): order sweep N=3..15 at ~16M local DOF
(e = round(256/n) elements per side), Ax kernel HBM roofline
fraction.  Times sem_ax (u -> w, 64 B/node algorithmic) with CUDA events around
back-to-back launches on the library stream; inputs (~1.1 GB per apply) are
far larger than L2.  Also times one CG iteration block (tol = 0, 20 its).

    python tools/order_sweep.py [--orders 3 4 ... 15] [--out gpurun_out/order_sweep.json]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_0968_b200 import meshgen, sem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--orders", type=int, nargs="*", default=list(range(3, 16)))
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default="gpurun_out/order_sweep.json")
args = ap.parse_args()

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
rows = []
for N in args.orders:
    n = N + 1
    e = round(256 / n)
    t0 = time.time()
    xi, _ = sem.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(e, e, e), eps=0.05)
    ctx = sem.Context(m, N, device=0)
    L = ctx.nlocal
    u = torch.from_numpy(meshgen.random_field(L, 0)).cuda()
    w = torch.empty_like(u)
    for _ in range(3):
        ctx.ax(u, w)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        ctx.ax(u, w)
    b.record()
    torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / args.reps
    gbs = 64.0 * L / (us * 1e-6) / 1e9
    flops = (12 * n ** 4 + 15 * n ** 3) * (L // n ** 3)
    # CG: 20 iterations at tol = 0 (fixed work), per-iteration time
    _, f = meshgen.manufactured(m)
    bb = ctx.rhs(torch.from_numpy(f).cuda())
    x = torch.zeros_like(bb)
    ctx.cg(bb, x, tol=0.0, maxit=20)
    torch.cuda.synchronize()
    a.record()
    x.zero_()
    ctx.cg(bb, x, tol=0.0, maxit=200)
    b.record()
    torch.cuda.synchronize()
    cg_us = 1e3 * a.elapsed_time(b) / 200
    row = {"N": N, "elems": e ** 3, "local_dof": L, "unique_dof": ctx.nglobal,
           "ax_us": us, "ax_gdof_s": L / (us * 1e-6) / 1e9, "ax_gbs": gbs, "ax_frac": gbs / peak,
           "ax_tflops": flops / (us * 1e-6) / 1e12,
           "kernel": os.environ.get("SEM_AX_KERNEL") or (
               "ax_dmma_kernel" if N == 7 else "ax_dmmag_kernel" if N >= 10 else
               "ax_tma_kernel" if N <= 10 else "ax_hi_kernel"),
           "cg_us_per_it": cg_us, "cg_gdof_s": L / (cg_us * 1e-6) / 1e9,
           "setup_s": time.time() - t0}
    rows.append(row)
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}),
          flush=True)
    ctx.free()
    del u, w, bb, x, ctx
    torch.cuda.empty_cache()
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
json.dump({"peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs", "rows": rows},
          open(args.out, "w"), indent=1)
