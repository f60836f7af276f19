#!/usr/bin/env python3
"""Summarise ncu reports / launch lists into markdown for profiles/.

  scripts/ncu_summary.py report REP.ncu-rep [--title T]      -> key metrics per kernel
  scripts/ncu_summary.py launches LAUNCHES.csv [--title T]   -> per-kernel time shares
  scripts/ncu_summary.py stalls REP.ncu-rep [--title T] [--top N] -> stall samples per SASS line
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


STALLS = ["stall_long_sb", "stall_wait", "stall_math", "stall_branch_resolving", "stall_no_inst",
          "stall_dispatch", "stall_lg", "stall_short_sb", "stall_selected", "stall_not_selected"]


def stalls(rep, title, top=15):
    """Warp-stall samples attributed to SASS instructions (source page of a --set full
    capture taken with --import-source on)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h)]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(int(r[ix[key]] or 0) for r in data) or 1
    print(f"## {title}\n")
    print(f"Source: `{rep}` (source page, SASS view). {tot} stall samples.\n")
    print("| reason | share of samples |\n|---|---|")
    for c in STALLS:
        print(f"| {c[6:]} | {100 * sum(int(r[ix[c]] or 0) for r in data) / tot:.1f}% |")
    print(f"\nTop {top} instructions by samples:\n")
    print("| share | executed | SASS | main reasons |\n|---|---|---|---|")
    for r in sorted(data, key=lambda r: -int(r[ix[key]] or 0))[:top]:
        why = sorted(((int(r[ix[c]] or 0), c[6:]) for c in STALLS), reverse=True)[:2]
        print(f"| {100 * int(r[ix[key]]) / tot:.1f}% | {r[ix['Instructions Executed']]} | "
              f"`{r[1].strip()[:56]}` | " + ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in why) + " |")
    print()


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    title = sys.argv[sys.argv.index("--title") + 1] if "--title" in sys.argv else path
    if mode == "stalls":
        stalls(path, title, int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15)
    else:
        (report if mode == "report" else launches)(path, title)
