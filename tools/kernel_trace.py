"""Per-kernel device timing INSIDE CUDA graphs via CUPTI (torch.profiler /
kineto, CUDA activity only): every kernel libsem launches -- directly or as a
node of a CG chunk graph -- with its GPU start/end timestamps.  Used by
bench.py for the in-solve kernel times and step shares, and to dump a
chrome-trace timeline (the nsys substitute of SURVEY.md §8(d); nsys is not in
this image).  Measurement infrastructure, not product code."""
from __future__ import annotations


def trace(fn, export: str | None = None):
    """Run fn() under the CUDA activity profiler; return a list of
    (name, start_us, dur_us, stream) for every GPU kernel, in start order."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    if export:
        prof.export_chrome_trace(export)
    out = []
    for e in prof.events():
        if getattr(e, "device_type", None) != torch.autograd.DeviceType.CUDA:
            continue
        if e.name.startswith("Memcpy") or e.name.startswith("Memset"):
            continue
        tr = e.time_range
        out.append((e.name, float(tr.start), float(tr.end - tr.start), getattr(e, "device_resource_id", None)))
    out.sort(key=lambda t: t[1])
    return out


def _targs(name: str):
    """Template arguments of a demangled kernel name ('a<7, true, false>(...)')."""
    i = name.find("<")
    if i < 0:
        return []
    depth, j = 0, i
    for j in range(i, len(name)):
        if name[j] == "<":
            depth += 1
        elif name[j] == ">":
            depth -= 1
            if depth == 0:
                break
    return [t.strip() for t in name[i + 1:j].split(",")]


def classify(name: str) -> str:
    """Kernel class inside the CG loop: 'k1' = the operator kernel of an
    iteration (ax_*_kernel with CG = true, or the single-reduction KA with
    DOT = true), 'k2' = the gather-scatter + update kernel (k2_kernel with
    INIT = false, the pipelined k2p_kernel, kb_sr_kernel), else 'other'
    (plain Ax, CG start/finish, ...)."""
    args = _targs(name)
    bools = [a for a in args if a in ("true", "false")]
    if "ax_" in name and "_kernel<" in name:
        # ax_dmma_kernel<CG, MASS, PC, DOT>, ax_tma/hi_kernel<N, CG, MASS, PC, DOT>
        cg = bools[0] == "true" if bools else False
        dot = len(bools) >= 4 and bools[3] == "true"
        return "k1" if (cg or dot) else "other"
    if "k2_kernel<" in name:
        return "k2" if len(bools) >= 1 and bools[0] == "false" else "other"
    if "kb_sr_kernel<" in name or "k2p_kernel<" in name:
        return "k2"
    return "other"


def per_solve(events, its):
    """Split a trace of consecutive CG solves at cg_init_kernel / sr_init_kernel
    and keep, per solve, the first `its` K1 and K2 launches (later launches of
    the last chunk are no-ops after the stop).  Returns {class: [us, ...]} and
    the number of solves seen."""
    out = {"k1": [], "k2": []}
    nsolve = 0
    cnt = {"k1": 0, "k2": 0}
    for name, _, d, _ in events:
        if "cg_init_kernel" in name or "sr_init_kernel" in name:
            nsolve += 1
            cnt = {"k1": 0, "k2": 0}
            continue
        c = classify(name)
        if c in cnt and nsolve > 0 and cnt[c] < its:
            cnt[c] += 1
            out[c].append(d)
    return out, nsolve


def summarize(events, ncalls: int = 1):
    """{class: {"n": launches, "us": total device us per call}} plus the span."""
    if not events:
        return {}, 0.0
    span = max(s + d for _, s, d, _ in events) - min(s for _, s, _, _ in events)
    agg = {}
    for name, _, d, _ in events:
        c = classify(name)
        a = agg.setdefault(c, {"n": 0, "us": 0.0, "names": set()})
        a["n"] += 1
        a["us"] += d
        a["names"].add(name)
    for a in agg.values():
        a["n"] //= ncalls
        a["us"] /= ncalls
        a["names"] = sorted(a["names"])
    return agg, span / ncalls
