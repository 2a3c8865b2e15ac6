#!/usr/bin/env python
"""Summarise ncu output into profiles/ (committed evidence).

  python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches.csv \
      --full gpurun_out/prof.ncu-rep [--kernel-regex ax_tma_kernel<7, true>]

Writes profiles/ncu_summary_<tag>.json and profiles/ncu_summary_<tag>.md:
  * launch list (gpu__time_duration.sum per launch, --clock-control none):
    per-kernel count, mean/median duration and share of all device time;
  * the `--set full` capture of the dominant kernel: DRAM bytes per launch,
    duration, occupancy, stall reasons, pipe utilisation.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import statistics
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name].append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "mean_ns": sum(v) / len(v),
                    "median_ns": statistics.median(v), "share": sum(v) / tot})
    return out


def full(path, regex=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        if regex and regex not in d["kernel"]:
            continue
        for m in FULL_METRICS:
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[m] = v
                d[m + "__unit"] = units[hdr.index(m)]
        res.append(d)
    return res


def to_bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                "GB": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--kernel-regex")
    ap.add_argument("--algorithmic-bytes", type=float,
                    help="algorithmic bytes per launch of the dominant kernel")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    out = {"tag": a.tag, "note": a.note}
    if a.launches:
        out["launch_list"] = launches(a.launches)
        out["launch_list_source"] = ("ncu --metrics gpu__time_duration.sum --clock-control none "
                                     "(cold-cache, serialised launches: compare shares)")
    if a.full:
        caps = full(a.full, a.kernel_regex)
        out["full_capture"] = caps
        if caps:
            c = caps[-1]
            rd = to_bytes(c["dram__bytes_read.sum"], c["dram__bytes_read.sum__unit"])
            wr = to_bytes(c["dram__bytes_write.sum"], c["dram__bytes_write.sum__unit"])
            dom = {"kernel": c["kernel"], "dram_bytes_per_launch": rd + wr,
                   "dram_read_bytes": rd, "dram_write_bytes": wr,
                   "duration_ns": to_bytes(c["gpu__time_duration.sum"], "byte") *
                   {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6}.get(
                       c["gpu__time_duration.sum__unit"], 1)}
            if a.algorithmic_bytes:
                dom["algorithmic_bytes_per_launch"] = a.algorithmic_bytes
                dom["traffic_over_algorithmic"] = (rd + wr) / a.algorithmic_bytes
            out["dominant"] = dom
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    jp = os.path.join(ROOT, "profiles", f"ncu_summary_{a.tag}.json")
    json.dump(out, open(jp, "w"), indent=1)
    md = [f"# ncu summary {a.tag}", "", a.note, ""]
    if "launch_list" in out:
        md += ["## Launch list (" + out["launch_list_source"] + ")", "",
               "| kernel | launches | mean us | median us | share |", "|---|---|---|---|---|"]
        for r in out["launch_list"][:15]:
            md.append(f"| `{r['kernel']}` | {r['launches']} | {r['mean_ns'] / 1e3:.1f} | "
                      f"{r['median_ns'] / 1e3:.1f} | {r['share']:.3f} |")
        md.append("")
    if "full_capture" in out:
        md += ["## --set full capture", ""]
        for c in out["full_capture"]:
            md.append(f"### `{c['kernel']}`")
            md.append("")
            md.append("| metric | value | unit |")
            md.append("|---|---|---|")
            for m in FULL_METRICS:
                if m in c:
                    md.append(f"| {m} | {c[m]} | {c.get(m + '__unit', '')} |")
            md.append("")
    if "dominant" in out:
        md += ["## Dominant kernel", "", "```", json.dumps(out["dominant"], indent=1), "```", ""]
    open(os.path.join(ROOT, "profiles", f"ncu_summary_{a.tag}.md"), "w").write("\n".join(md))
    print(jp)


if __name__ == "__main__":
    main()
