#!/usr/bin/env python
"""Benchmark of the SEM Poisson hot path (arXiv 1403.0968) on B200.

One STEP = one full CG solve (Ax + DSSUM + mask + fused CG vector updates and
dot products) to rel. tol 1e-8 from x0 = 0 on config c3:
4096 hexahedra (16^3) of order N=7 per GPU, eps=0.05 deformed box, manufactured
sin right-hand side.  N GPUs = weak scaling (c5): each rank owns a 16^3-element
unit cube of the global box, ranks exchange interface partial sums over NCCL.

value = CG GDOF/s = (local DOF on all ranks) x (CG iterations) / time / 1e9,
with local DOF = E (N+1)^3 (SURVEY.md reading G13).  The line also carries CG
iterations/s, the Ax-only GDOF/s, the roofline of the dominant kernel, an
end-to-end number through the public API with host buffers, the plain-C oracle
timed on a bounded sample of the same workload, and SM clocks under load.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Ax GDOF/s and % of HBM roofline; CG iterations/s at 1/2/4/8 B200"
L2_BYTES = 126 * 2 ** 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["sem", "reference"], default="sem")
    ap.add_argument("--N", type=int, default=7)
    ap.add_argument("--elems", type=int, nargs=3, default=[16, 16, 16], help="elements per rank")
    ap.add_argument("--eps", type=float, default=0.05)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--maxit", type=int, default=5000)
    ap.add_argument("--ax-reps", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--operator", choices=["poisson", "screened"], default="poisson",
                    help="screened: -div(kappa grad u) + alpha u (NEXT-1) with meshgen.coefficients")
    ap.add_argument("--precond", choices=["none", "jacobi"], default="none",
                    help="jacobi: Jacobi-preconditioned CG (NEXT-2, sem_pcg)")
    ap.add_argument("--cg-variant", choices=["standard", "single_reduction"], default="standard",
                    help="single_reduction: Chronopoulos-Gear CG (NEXT-3, sem_cg_sr)")
    ap.add_argument("--workload", choices=["sem", "fd"], default="sem",
                    help="fd: the finite-difference wave step of lst:fdCode (NEXT-4), "
                         "MNodes/s over stencil sizes 3..15")
    ap.add_argument("--fd-size", type=int, default=8192, help="fd grid is size x size")
    ap.add_argument("--fd-radii", type=int, nargs="+", default=[1, 2, 3, 4, 5, 6, 7])
    ap.add_argument("--cpu-its", type=int, default=100,
                    help="oracle CG iterations timed for cpu_baseline (bounded sample)")
    ap.add_argument("--share-device", action="store_true",
                    help="HARNESS CHECK, not a measurement: every rank of --gpus N on cuda:0 "
                         "(gloo process group, the peer-memory transport over CUDA IPC, "
                         "SEM_COMM=p2p) -- runs the N > 1 code path of this script on a "
                         "one-GPU box")
    ap.add_argument("--ref-its", type=int, default=10,
                    help="oracle CG iterations per --impl reference step")
    ap.add_argument("--cpu-threads", type=int, default=0,
                    help="oracle threads for the all-core baseline (0 = the affinity count)")
    ap.add_argument("--cpu-c4", action="store_true",
                    help="cpu_baseline also times one oracle Ax per N = 3..15 at ~16M DOF (c4; slow)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernels=("ax_tma_kernel<7, true, false>", "ax_tma_kernel<7, 1>")):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of
    the dominant kernel from the newest committed ncu --set full summary
    (profiles/ncu_summary_*.json) that captured THAT kernel, or None."""
    d = os.path.join(ROOT, "profiles")
    if not os.path.isdir(d):
        return None
    files = sorted(f for f in os.listdir(d) if f.startswith("ncu_summary") and f.endswith(".json"))
    for f in reversed(files):   # newest tag that captured the dominant kernel
        try:
            s = json.load(open(os.path.join(d, f)))
        except Exception:
            continue
        dom = s.get("dominant") or {}
        if any(k in dom.get("kernel", "") for k in kernels):
            return dom.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def rank_mesh(args, rank, world, r1d):
    from paper_1403_0968_b200 import meshgen
    parts = meshgen.default_parts(world)
    elems = tuple(e * p for e, p in zip(args.elems, parts))
    lengths = tuple(float(p) for p in parts)
    return meshgen.box_mesh(args.N, r1d, elems=elems, lengths=lengths, eps=args.eps,
                            parts=parts, rank=rank, boundary_first=world > 1), parts


def workload_name(args, world):
    E = args.elems[0] * args.elems[1] * args.elems[2]
    op = ("" if args.operator == "poisson" else
          ", screened Coulomb -div(kappa grad u) + alpha u (meshgen.coefficients)")
    cg = "CG" if args.precond == "none" else "Jacobi PCG"
    if args.cg_variant != "standard":
        cg = "single-reduction (Chronopoulos-Gear) CG"
    return (f"c3/c5: {E} hex elements ({'x'.join(map(str, args.elems))}) of order N={args.N} "
            f"per GPU, eps={args.eps} deformed box, full {cg} to {args.tol:g} from x0=0{op}")


def coefficients(args, m):
    from paper_1403_0968_b200 import meshgen
    return meshgen.coefficients(m) if args.operator == "screened" else (None, None)


def host_cores():
    """Cores this process may run on (sched_getaffinity), and the oracle
    thread count for the all-core baseline."""
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    return n


def oracle_sample(args, its_per_call, calls):
    """Time the plain-C oracle's CG (tol = 0, fixed iterations) on rank 0's c3
    mesh.  Returns (seconds per call list, L); each entry is the time of a
    maxit = its_per_call solve minus that of a maxit = 0 solve (the oracle's
    own setup inside the call: sorting the global ids, the initial residual),
    so it covers exactly its_per_call iterations."""
    import oracle
    from paper_1403_0968_b200 import meshgen
    xi, _ = oracle.gll(args.N)
    m, _ = rank_mesh(args, 0, 1, xi)
    G, J = oracle.geom(args.N, m.xyz)
    _, f = meshgen.manufactured(m)
    b = oracle.mass_rhs(args.N, m.glo, m.dirichlet, J, f)
    kappa, alpha = coefficients(args, m)
    co = {} if kappa is None else {"J": J, "kappa": kappa, "alpha": alpha}
    def solve(its):
        t0 = time.perf_counter()
        if args.cg_variant == "single_reduction":
            oracle.cg_single_reduction(args.N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=its)
        else:
            oracle.cg(args.N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=its,
                      precond=args.precond, **co)
        return time.perf_counter() - t0

    t_setup = min(solve(0) for _ in range(2))
    times = [max(solve(its_per_call) - t_setup, 1e-9) for _ in range(calls)]
    return times, m.nlocal


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    steps, warm = args.steps, args.warmup
    cores = args.cpu_threads or host_cores()
    oracle.set_threads(cores)
    times, L = oracle_sample(args, args.ref_its, steps + warm)
    oracle.set_threads(1)
    t = sum(times[warm:])
    value = L * args.ref_its * steps / t / 1e9
    sample = (f"oracle (plain C, operator element loop on {cores} OpenMP threads, sequential "
              f"dot products / DSSUM) CG, {args.ref_its} iterations (tol=0) per step on the "
              f"c3 mesh of rank 0 ({L} local DOF); the oracle's setup (maxit = 0 call) "
              "subtracted")
    out = {"metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": steps,
           "warmup": warm, "ms_per_step": 1e3 * t / steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": workload_name(args, world), "N": args.N,
                      "elements_per_gpu": args.elems[0] * args.elems[1] * args.elems[2]},
           "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": cores, "kind": "oracle",
                            "sample": sample, "cpu": cpu_info(),
                            "affinity_cores": host_cores()},
           "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(args):
    """The plain-C oracle on this host (rank 0, N = 1): c3 CG throughput on 1
    core and on all cores (OpenMP over the operator's elements; dot products,
    DSSUM and the recurrence sequential -- bit-identical results), plus the
    other BASELINE.md §3 configs: c1 in full (setup + Ax + DSSUM + 20 CG
    iterations), c2 Ax + DSSUM x 10, and with --cpu-c4 one Ax per N at ~16M DOF.
    Bounded: ~10-30 s in total by default."""
    import oracle
    from paper_1403_0968_b200 import meshgen
    pc = "CG" if args.precond == "none" else "Jacobi PCG"
    cores = args.cpu_threads or host_cores()
    oracle.set_threads(1)
    t1, Lc = oracle_sample(args, args.cpu_its, 1)
    oracle.set_threads(cores)
    tn, _ = oracle_sample(args, args.cpu_its, 1)
    one = Lc * args.cpu_its / t1[0] / 1e9
    allc = Lc * args.cpu_its / tn[0] / 1e9
    out = {"value": allc, "unit": "GDOF/s", "cores": cores, "kind": "oracle", "cpu": cpu_info(),
           "affinity_cores": host_cores(), "omp_threads": cores,
           "sample": f"plain-C oracle {pc}, {args.cpu_its} iterations (tol=0) on the same c3 mesh "
                     f"({Lc} local DOF), operator element loop on {cores} OpenMP threads "
                     f"(sequential dot products / DSSUM / recurrence), {tn[0]:.1f} s; the oracle's "
                     "setup (maxit = 0 call) subtracted",
           "one_core": {"value": one, "unit": "GDOF/s", "cores": 1, "seconds": t1[0]}}
    cfg = {}
    # c1: 8 hex (2x2x2), N = 4: setup + 1 Ax + DSSUM + 20 CG iterations
    t0 = time.perf_counter()
    xi, _ = oracle.gll(4)
    m1 = meshgen.box_mesh(4, xi, elems=(2, 2, 2), eps=0.05)
    G1, J1 = oracle.geom(4, m1.xyz)
    u1 = meshgen.random_field(m1.nlocal, 0)
    oracle.dssum(m1.glo, oracle.ax(4, G1, u1))
    _, f1 = meshgen.manufactured(m1)
    b1 = oracle.mass_rhs(4, m1.glo, m1.dirichlet, J1, f1)
    oracle.cg(4, m1.glo, m1.dirichlet, G1, b1, tol=0.0, maxit=20)
    cfg["c1_full_ms"] = 1e3 * (time.perf_counter() - t0)
    # c2: 512 elements, N = 7: Ax + DSSUM, 10 repetitions (setup untimed)
    xi7, _ = oracle.gll(7)
    m2 = meshgen.box_mesh(7, xi7, elems=(8, 8, 8), eps=0.05)
    G2, _ = oracle.geom(7, m2.xyz)
    u2 = meshgen.random_field(m2.nlocal, 0)
    t0 = time.perf_counter()
    for _ in range(10):
        oracle.dssum(m2.glo, oracle.ax(7, G2, u2))
    dt = (time.perf_counter() - t0) / 10
    cfg["c2_ax_dssum"] = {"ms": 1e3 * dt, "gdof_s": m2.nlocal / dt / 1e9, "cores": cores}
    if args.cpu_c4:
        sweep = {}
        for N in range(3, 16):
            xiN, _ = oracle.gll(N)
            e = round(256 / (N + 1))
            mN = meshgen.box_mesh(N, xiN, elems=(e, e, e), eps=0.05)
            GN, _ = oracle.geom(N, mN.xyz)
            uN = meshgen.random_field(mN.nlocal, 0)
            t0 = time.perf_counter()
            oracle.ax(N, GN, uN)
            d = time.perf_counter() - t0
            sweep[str(N)] = {"gdof_s": mN.nlocal / d / 1e9, "s": d}
            del mN, GN, uN
        cfg["c4_ax"] = {"cores": cores, "per_N": sweep}
    oracle.set_threads(1)
    out["configs"] = cfg
    return out


FD_METRIC = "FD wave step MNodes/s vs stencil size (lst:fdCode), % of HBM roofline"


def run_fd(args, rank, world):
    """NEXT-4: fd2d_run over `steps` time steps of a size x size periodic grid
    per GPU (weak scaling: independent replicas, the stencil does not shard
    across this API), each stencil radius in --fd-radii; CUDA events on the
    launching stream, L2 flushed by the working set (3 x 512 MiB > L2)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1403_0968_b200 import fd

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.fd_size
    rng = np.random.default_rng(1 + rank)
    u1 = torch.from_numpy(rng.uniform(-1, 1, (n, n))).to(dev)
    u2 = torch.from_numpy(rng.uniform(-1, 1, (n, n))).to(dev)
    u3 = torch.empty_like(u1)
    stream = torch.cuda.current_stream()
    peak, peak_src = peaks()
    sweep = {}
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    def timed(r, regrouped):
        om = fd.weights(r, 2.0 / n)
        dt = 0.2 * 2.0 / n
        fd.run(u1, u2, u3, om, dt, max(args.warmup, 3), regrouped=regrouped)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fd.run(u1, u2, u3, om, dt, args.steps, regrouped=regrouped)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        nodes = float(n) * n * args.steps * world
        # input data was rotated: refresh so every run starts from finite values
        u1.uniform_(-1, 1)
        u2.uniform_(-1, 1)
        return {"mnodes_s": nodes / (ms * 1e-3) / 1e6, "us_per_step": 1e3 * ms / args.steps,
                "achieved_gbs": 24.0 * n * n / (ms / args.steps * 1e-3) / 1e9}

    # default (the listing's operation order, bit-exact with the oracle) and
    # the opt-in pair-regrouped FMA form (fd2d_run_ex FD_REGROUPED, reading R6c)
    regrouped = {}
    for r in args.fd_radii:
        sweep[2 * r + 1] = timed(r, False)
        regrouped[2 * r + 1] = timed(r, True)
    clocks = sampler.stop()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        m = 2048
        a, b = rng.uniform(-1, 1, (m, m)), rng.uniform(-1, 1, (m, m))
        r = args.fd_radii[-1]
        om = oracle.fd_weights(r, 2.0 / m)
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            oracle.fd_step(a, b, om, 0.1 / m)
        tc = (time.perf_counter() - t0) / reps
        cpu = {"value": m * m / tc / 1e6, "unit": "MNodes/s", "cores": 1, "kind": "oracle",
               "cpu": cpu_info(),
               "sample": f"plain-C oracle ora_fd_step, {m}x{m} grid, stencil size {2 * r + 1}, "
                         f"{reps} steps, 1 thread, {tc * reps:.1f} s"}
    if rank == 0:
        rmax = 2 * args.fd_radii[-1] + 1
        head = sweep[rmax]
        out = {"metric": FD_METRIC, "value": head["mnodes_s"], "unit": "MNodes/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": head["us_per_step"] / 1e3, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded U(-1,1) fields)",
               "config": {"workload": f"fd2d (lst:fdCode) {n}x{n} periodic grid per GPU, stencil "
                                      f"size {rmax} (headline) and the sweep 3..15",
                          "grid": [n, n], "stencil_size": rmax,
                          "arithmetic": "the listing's operation order (bit-exact with the "
                                        "oracle); sweep_regrouped: FD_REGROUPED",
                          "l2": "inputs larger than L2: 3 x 512 MiB fields"},
               "sweep": {str(k): v for k, v in sweep.items()},
               "sweep_regrouped": {str(k): v for k, v in regrouped.items()},
               "roofline": {"bound": "hbm", "kernel": f"fd2d_kernel<{args.fd_radii[-1]}>",
                            "achieved": head["achieved_gbs"], "peak": peak, "unit": "GB/s",
                            "frac": head["achieved_gbs"] / peak, "traffic": None,
                            "peak_source": peak_src,
                            "bytes_per_node": "24 (u1, u2 read; u3 written)",
                            "timing": "CUDA events around fd2d_run(steps) on the launching stream"},
               "gpu_launches": 2 * args.steps * len(args.fd_radii),
               "cpu_baseline": cpu, "clocks": clocks}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args):
    """`--gpus N > 1` without a torchrun environment: re-launch this script as
    N ranks (one process per GPU) through torch.distributed.run on 127.0.0.1.
    Exits non-zero when the node has fewer than N GPUs."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not (args.share_device and have >= 1):
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "fd":
        run_fd(args, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1403_0968_b200 import meshgen, sem

    if args.share_device:                 # harness check: all ranks on cuda:0
        local_rank = 0
        os.environ["SEM_COMM"] = "p2p"
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    if world > 1:
        if args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if args.share_device else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    xi, _ = sem.gll(args.N)
    m, parts = rank_mesh(args, rank, world, xi)
    kappa, alpha = coefficients(args, m)
    ctx = sem.Context(m, args.N, device=local_rank, group=group, kappa=kappa, alpha=alpha)
    L = ctx.nlocal
    # algorithmic bytes per local node: K1 96, Ax 64; the screened
    # operator's mass diagonal adds 8 to both
    bpn_k1 = 96.0 + (8.0 if alpha is not None else 0.0)
    bpn_ax = 64.0 + (8.0 if alpha is not None else 0.0)
    L_all = L * world
    _, f = meshgen.manufactured(m)
    b = ctx.rhs(torch.from_numpy(f).to(dev))
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()

    # ---- warm-up ----
    its = None
    for _ in range(max(args.warmup, 1)):
        x.zero_()
        _, its, rel, ok = ctx.cg(b, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                        variant=args.cg_variant)
    assert ok, f"CG did not converge: rel_res={rel}"

    # ---- timed region: K full CG solves, inputs resident in HBM ----
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    launches0 = ctx.launch_count
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters = []
    for _ in range(args.steps):
        x.zero_()
        _, it, rel, ok = ctx.cg(b, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                        variant=args.cg_variant)
        iters.append(it)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    gpu_launches = ctx.launch_count - launches0
    clocks = sampler.stop()
    assert len(set(iters)) == 1, f"non-deterministic iteration counts {iters}"
    its = iters[0]
    t = ms / 1e3
    value = L_all * its * args.steps / t / 1e9
    cg_its_per_s = its * args.steps / t

    # ---- per-kernel device time INSIDE the CUDA graphs of the solve: the same
    # solves again under CUPTI kernel tracing (torch.profiler, CUDA activity
    # only; tools/kernel_trace.py) -- GPU start/end timestamps of every kernel
    # node, no events between kernels, graphs as in the timed region ----
    prof_steps = max(1, min(3, args.steps))
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import kernel_trace

    def traced_solves():
        for _ in range(prof_steps):
            x.zero_()
            ctx.cg(b, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                   variant=args.cg_variant)

    trace_path = os.environ.get("SEM_BENCH_TRACE")      # optional chrome-trace dump
    try:
        tev = kernel_trace.trace(traced_solves, export=trace_path)
        tcls, tn = kernel_trace.per_solve(tev, its)
    except Exception as e:  # profiler unavailable: fall back to the event timing below
        print(f"bench.py: CUPTI kernel trace unavailable ({e})", file=sys.stderr)
        tcls, tn = {"k1": [], "k2": []}, 0

    # ---- algorithmic bytes per launch (and an event-bracketed cross-check):
    # sem_profile runs the solve ungraphed with CUDA events around every
    # launch on the library stream ----
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(prof_steps):
        x.zero_()
        ctx.cg(b, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                        variant=args.cg_variant)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    prof = ctx.profile_read()
    ctx.profile(False)

    # ---- per-kernel roofline: each CG kernel replayed back to back as one
    # CUDA graph on the library stream, CUDA events around it (no per-launch
    # event gaps).  Algorithmic bytes per launch: K1 96 B/node,
    # K2 from the gather-scatter plan (the profiled pass), Ax 64 B/node. ----
    peak, peak_src = peaks()
    k2_bytes = prof["k2"][2] / prof["k2"][1] if prof["k2"][1] else None
    kern = {}
    for name, by in (("k1", bpn_k1 * L), ("k2", k2_bytes), ("ax", bpn_ax * L)):
        if world > 1 or by is None:
            continue
        reps = 50
        ctx.kernel_replay(name, 5)
        torch.cuda.synchronize()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        ctx.kernel_replay(name, reps)
        q1.record(stream)
        torch.cuda.synchronize()
        us = 1e3 * q0.elapsed_time(q1) / reps
        kern[name] = {"avg_launch_us": us, "bytes_per_launch": by,
                      "achieved_gbs": by / (us * 1e-6) / 1e9, "frac": by / (us * 1e-6) / 1e9 / peak}
    # headline: K1 inside the graphed solve (CUPTI timestamps); bytes per
    # launch from the library's accounting (96 B/node, 72 at k = 0)
    k1_ms, k1_n, k1_bytes = prof["k1"]
    k1_bpl = k1_bytes / k1_n if k1_n else None
    k2_bpl = prof["k2"][2] / prof["k2"][1] if prof["k2"][1] else None
    in_solve = {}
    for name, bpl in (("k1", k1_bpl), ("k2", k2_bpl)):
        d = tcls.get(name) or []
        if d and bpl:
            us_ = statistics.fmean(d)
            in_solve[name] = {"avg_launch_us": us_, "launches": len(d), "bytes_per_launch": bpl,
                              "achieved_gbs": bpl / (us_ * 1e-6) / 1e9,
                              "frac": bpl / (us_ * 1e-6) / 1e9 / peak,
                              "us_per_solve": sum(d) / max(tn, 1)}
    # the same with CUDA events around every launch of the UNGRAPHED solve
    # (host launch gaps fall inside the brackets: an upper bound)
    in_events = {}
    for name in ("k1", "k2"):
        ms_, n_, by_ = prof[name]
        if n_:
            us_ = 1e3 * ms_ / n_
            in_events[name] = {"avg_launch_us": us_, "bytes_per_launch": by_ / n_,
                               "achieved_gbs": by_ / n_ / (us_ * 1e-6) / 1e9,
                               "frac": by_ / n_ / (us_ * 1e-6) / 1e9 / peak}
    if "k1" in in_solve:
        k1_in_solve_us = in_solve["k1"]["avg_launch_us"]
        achieved = in_solve["k1"]["achieved_gbs"]
        k1_launches = in_solve["k1"]["launches"]
    else:
        k1_in_solve_us = in_events["k1"]["avg_launch_us"] if "k1" in in_events else None
        achieved = in_events["k1"]["achieved_gbs"] if "k1" in in_events else None
        k1_launches = k1_n
    dmma = args.N == 7 and not os.environ.get("SEM_AX_KERNEL")
    k1_name = ("K1: ax_dmma_kernel<CG=true> (N=7: r/s contractions on the FP64 tensor cores; "
               "x/p update + Ax + (p,Ap) partials)" if dmma else
               "K1: ax_tma_kernel<N,CG=true> (x/p update + Ax + (p,Ap) partials)")
    traffic = ncu_traffic(("ax_dmma_kernel<1, 0, 0, 0",) if dmma else
                          (f"ax_tma_kernel<{args.N}, true, false>", f"ax_tma_kernel<{args.N}, 1>")) \
        if alpha is None and args.precond == "none" and args.cg_variant == "standard" else None
    # share of the timed solve: per-solve device time of each class inside the
    # graph over the timed region's ms per solve
    shares = {k: v["us_per_solve"] / 1e3 / (ms / args.steps) for k, v in in_solve.items()}
    # the work vectors were clobbered by the replays; the next solve re-inits
    x.zero_()
    ctx.cg(b, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                        variant=args.cg_variant)

    # ---- Ax alone on the same mesh (64 B/node), for the Ax GDOF/s metric ----
    u = torch.from_numpy(meshgen.random_field(L, 0)).to(dev)
    w = torch.empty_like(u)
    for _ in range(5):
        ctx.ax(u, w)
    ctx.profile(True)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(args.ax_reps):
        ctx.ax(u, w)
    a1.record(stream)
    torch.cuda.synchronize()
    ax_ms = max_over_ranks(a0.elapsed_time(a1)) / args.ax_reps
    pa = ctx.profile_read()["ax"]
    ctx.profile(False)
    ax_kernel_ms = pa[0] / pa[1]
    ax = {"gdof_s": L_all / (ax_ms / 1e3) / 1e9, "ms_per_apply": ax_ms,
          "kernel_ms": ax_kernel_ms,
          "achieved_gbs": bpn_ax * L / (ax_kernel_ms / 1e3) / 1e9,
          "frac": bpn_ax * L / (ax_kernel_ms / 1e3) / 1e9 / peak,
          "gflops": (12 * (args.N + 1) ** 4 + 15 * (args.N + 1) ** 3) * (L / (args.N + 1) ** 3)
          / (ax_kernel_ms / 1e3) / 1e9,
          "bytes_per_apply": bpn_ax * L,
          "l2_note": f"working set {bpn_ax:.0f} B/node; at c3 partly L2-resident"}

    # ---- end to end through the public API with host buffers ----
    b_host = b.cpu().pin_memory()
    x_host = torch.empty_like(b_host).pin_memory()
    b_dev = torch.empty_like(b)
    for _ in range(2):
        b_dev.copy_(b_host, non_blocking=True)
        x.zero_()
        ctx.cg(b_dev, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                        variant=args.cg_variant)
        x_host.copy_(x, non_blocking=True)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    e2e_steps = max(1, min(args.steps, 10))
    for _ in range(e2e_steps):
        b_dev.copy_(b_host, non_blocking=True)
        x.zero_()
        _, it2, _, _ = ctx.cg(b_dev, x, tol=args.tol, maxit=args.maxit, precond=args.precond,
                        variant=args.cg_variant)
        x_host.copy_(x, non_blocking=True)
    h1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(h0.elapsed_time(h1))
    e2e = {"value": L_all * it2 * e2e_steps / (e2e_ms / 1e3) / 1e9, "unit": "GDOF/s",
           "h2d_bytes_per_step": 8 * L, "d2h_bytes_per_step": 8 * L,
           "ms_per_step": e2e_ms / e2e_steps}

    # ---- oracle on the host cores (rank 0, N=1 only), bounded sample ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)

    if rank == 0:
        ws = 16 * L + ctx.workspace.numel()
        out = {
            "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded deformed-box mesh, manufactured sin RHS)",
            "cg_iters_per_s": cg_its_per_s,
            "config": {"workload": workload_name(args, world), "N": args.N,
                       "elements_per_gpu": m.nelem, "local_dof_per_gpu": L,
                       "unique_dof_total": ctx.nglobal, "cg_iters": its, "tol": args.tol,
                       "partition": "x".join(map(str, parts)), "operator": args.operator,
                       "precond": args.precond, "cg_variant": args.cg_variant,
                       "parallelism": f"element partition over {world} GPU(s)",
                       **({"harness_check": "--share-device: all ranks time-share cuda:0; "
                                            "NOT a measurement"} if args.share_device else {}),
                       "l2": f"inputs larger than L2: {ws / 2**20:.0f} MiB resident working set "
                             f"> {L2_BYTES / 2**20:.0f} MiB L2, streamed every iteration"},
            "ax": ax,
            "roofline": {"bound": "hbm",
                         "kernel": k1_name,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         # DRAM bytes per launch (ncu, cold cache) over the in-graph
                         # launch time: frac above 1 means algorithmic bytes served
                         # from L2 (r written by the previous K2, x / p by the
                         # previous K1), this is the DRAM side of the same launch
                         "dram_frac": (traffic / (k1_in_solve_us * 1e-6) / 1e9 / peak
                                       if traffic and k1_in_solve_us else None),
                         "peak_source": peak_src,
                         "bytes_per_node": f"{bpn_k1:.0f} (x,r,p,G{',H' if alpha is not None else ''} "
                                           "read; x,p,w write)",
                         "avg_launch_us": k1_in_solve_us,
                         "launches": k1_launches,
                         "kernels_replayed": kern,
                         "kernels_in_solve": in_solve,
                         "kernels_events_ungraphed": in_events,
                         "step_share": shares,
                         "iteration": {"us": 1e3 * ms / args.steps / its,
                                       "algorithmic_bytes": bpn_k1 * L + (k2_bytes or 0.0),
                                       "frac": (bpn_k1 * L + (k2_bytes or 0.0)) /
                                               (ms / args.steps / its * 1e-3) / 1e9 / peak},
                         "timing": "achieved / kernels_in_solve / step_share: CUPTI GPU "
                                   "timestamps (torch.profiler CUDA activity) of every kernel "
                                   "node INSIDE the CG chunk graphs of "
                                   f"{prof_steps} solves of the same workload run right after the "
                                   "timed region (the first `cg_iters` K1 / K2 launches of each "
                                   "solve; step_share against the timed ms per solve); "
                                   "kernels_events_ungraphed: CUDA events around every launch of "
                                   "the ungraphed solve (sem_profile; host gaps included); "
                                   "kernels_replayed: CUDA events around a graph of 50 "
                                   "back-to-back launches of one kernel (sem_kernel_replay, no "
                                   "CG neighbours in L2)"},
            "gpu_launches": gpu_launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    ctx.free()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
