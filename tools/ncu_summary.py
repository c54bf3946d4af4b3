#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: key metrics of a --set full report and
the per-kernel share of a gpu__time_duration launch list.

    python tools/ncu_summary.py report.ncu-rep [--label NAME] [--launches launches.csv]
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
    "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        kernels.append(d)
    return kernels


def summarise(rep, label):
    res = []
    for d in raw(rep):
        k = {"kernel": d.get("Kernel Name", ("?", ""))[0][:120], "label": label}
        for key in KEYS:
            if key in d:
                k[key] = f"{d[key][0]} {d[key][1]}".strip()
        stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): v
                  for h, (v, u) in d.items()
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")}
        k["stalls_per_issue"] = {s: v for s, v in sorted(stalls.items(), key=lambda x: -float(x[1] or 0))[:8]}
        res.append(k)
    return res


def launches(path):
    lines = open(path).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[i:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi:
            d[r[ki][:90]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    return [{"kernel": k, "launches": len(v), "mean_ns": sum(v) / len(v), "share_pct": 100 * sum(v) / tot}
            for k, v in sorted(d.items(), key=lambda x: -sum(x[1]))]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--label", default="")
    ap.add_argument("--launches")
    a = ap.parse_args()
    out = {}
    if a.report:
        out["full"] = summarise(a.report, a.label)
    if a.launches:
        out["launches"] = launches(a.launches)
    json.dump(out, sys.stdout, indent=1)
    print()
