#!/usr/bin/env python
"""Summarise an ncu report (or a launch-list CSV) into small committed files under profiles/.

    python tools/ncu_summary.py full   gpurun_out/prof.ncu-rep  profiles/r01_ncu_full.csv  [--traffic profiles/traffic.json]
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launch_shares.csv

`full`: one row per profiled launch -- duration, DRAM bytes read/write, DRAM / SM throughput,
occupancy, issue activity and the top stall reasons; --traffic writes the per-kernel DRAM bytes
per launch (mean over the launches captured) that bench.py reports as roofline.traffic.
`launches`: per-kernel totals and SHARES of the device time from the
`--metrics gpu__time_duration.sum` pass (cold-cache, serialised: compare shares, not absolutes).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys

NCU = "ncu"


def _csv(args):
    out = subprocess.run([NCU, *args], capture_output=True, text=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)
    return name.replace("queen::", "")


def full(rep: str, out: str, traffic: str | None):
    raw = _csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units, rows = raw[0], raw[1], raw[2:]
    want = {
        "gpu__time_duration.sum": "duration",
        "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "sm__inst_executed.avg.per_cycle_active": "ipc",
        "launch__registers_per_thread": "regs",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    }
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
             "ns": 1e-3, "us": 1, "ms": 1e3}
    ki = hdr.index("Kernel Name")
    cols = {w: hdr.index(k) for k, w in want.items() if k in hdr}
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and
                  h.endswith("_per_issue_active.ratio")]
    recs = []
    for r in rows:
        d = {"kernel": short(r[ki])}
        for w, i in cols.items():
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                v = None
            u = units[i]
            if v is not None and w in ("duration", "dram_read", "dram_write"):
                v = v * scale.get(u, 1)  # duration -> us, bytes -> bytes
            d[w] = v
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(r[i]), hdr[i]))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        d["top_stalls"] = "; ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in stalls[:3])
        recs.append(d)
    keys = ["kernel", "duration", "dram_read", "dram_write", "dram_pct", "sm_pct", "occupancy_pct", "ipc", "regs",
            "fma_pipe_pct", "xu_pipe_pct", "top_stalls"]
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=keys, extrasaction="ignore")
        w.writeheader()
        for d in recs:
            w.writerow({k: (f"{d[k]:.4g}" if isinstance(d.get(k), float) else d.get(k)) for k in keys})
    if traffic:
        agg = collections.defaultdict(list)
        for d in recs:
            if d.get("dram_read") is not None and d.get("dram_write") is not None:
                agg[d["kernel"]].append(d["dram_read"] + d["dram_write"])
        try:
            prev = json.load(open(traffic))
        except Exception:
            prev = {}
        prev.update({k: sum(v) / len(v) for k, v in agg.items()})
        json.dump(prev, open(traffic, "w"), indent=1, sort_keys=True)
    print(f"wrote {out} ({len(recs)} launches)")


def launches(src: str, out: str):
    txt = open(src).read().splitlines()
    start = [i for i, ln in enumerate(txt) if ln.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    scale = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}
    agg = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            agg[short(r["Kernel Name"])].append(float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]])
    tot = sum(sum(v) for v in agg.values())
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "mean_us", "total_us", "share"])
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            w.writerow([k, len(v), f"{sum(v) / len(v):.2f}", f"{sum(v):.1f}", f"{sum(v) / tot:.4f}"])
    print(f"wrote {out} ({len(rows)} launches)")


if __name__ == "__main__":
    mode, src, out = sys.argv[1:4]
    tr = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    full(src, out, tr) if mode == "full" else launches(src, out)
