#!/usr/bin/env python3
"""Summarise ncu reports / launch lists into markdown for profiles/.

  scripts/ncu_summary.py report REP.ncu-rep [--title T]      -> key metrics per kernel
  scripts/ncu_summary.py launches LAUNCHES.csv [--title T]   -> per-kernel time shares
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Compute (SM) Throughput", "Issue Slots Busy", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Achieved Occupancy",
        "Registers Per Thread", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate",
        "L2 Cache Throughput", "DRAM Throughput", "Mem Pipes Busy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed_op_global_red.sum"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(rep, title):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    kern = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            kern.setdefault(d["Kernel Name"].split("(")[0].replace("<unnamed>::", ""), {})[d["Metric Name"]] = (
                f"{d['Metric Value']} {d['Metric Unit']}".strip())
    raw = ncu_csv(rep, "raw")
    rh = raw[0]
    for r in raw[2:]:
        d = dict(zip(rh, r))
        k = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        for m in RAW:
            if m in d and d[m] not in ("", "n/a"):
                kern.setdefault(k, {})[m] = f"{d[m]} {raw[1][rh.index(m)]}".strip()
    print(f"## {title}\n")
    print(f"Source: `{rep}` (ncu --set full --clock-control none; one capture per kernel).\n")
    names = list(kern)
    print("| metric | " + " | ".join(f"`{n}`" for n in names) + " |")
    print("|---|" + "---|" * len(names))
    for m in KEYS + RAW:
        if any(m in kern[n] for n in names):
            print(f"| {m} | " + " | ".join(kern[n].get(m, "") for n in names) + " |")
    print()


def launches(path, title):
    rows = [r for r in csv.reader(open(path)) if r]
    h, agg = None, {}
    for r in rows:
        if r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            k = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
            v = float(d["Metric Value"])
            unit = d.get("Metric Unit", "ns")
            scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"## {title}\n")
    print(f"Source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache,"
          " serialised launches: compare shares, not absolute times).\n")
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if v / tot >= 0.0005:
            print(f"| `{k[:60]}` | {n} | {v:.1f} | {100 * v / tot:.1f}% |")
    print()


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    title = sys.argv[sys.argv.index("--title") + 1] if "--title" in sys.argv else path
    (report if mode == "report" else launches)(path, title)
