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


def classify(name: str) -> str:
    """Kernel class of a libsem kernel name (K1 = the CG operator kernel,
    K2 = gather-scatter + residual update)."""
    n = name
    if "k2_kernel" in n or "kb_sr_kernel" in n:
        return "k2"
    if ("ax_dmma_kernel" in n or "ax_tma_kernel" in n or "ax_hi_kernel" in n or
            "ax_dmmag_kernel" in n or "ax_kernel" in n):
        return "ax"
    return "other"


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
