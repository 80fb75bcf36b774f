#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, no GPU).

  python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep   > profiles/rNN_..._ncu_full.txt
  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_..._launches.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"# kernel {d.get('Kernel Name', '?')[:90]}  id={d.get('ID')}")
        for k in KEYS + sorted(x for x in h if x.startswith("nvl") and x not in KEYS):
            if k in d:
                print(f"{k:60s} {d[k]:>16s} {units[h.index(k)]}")
        print()


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    tot = 0.0
    by = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(d["Metric Value"].replace(",", ""))
        name = d["Kernel Name"].split("(")[0][:60]
        by.setdefault(name, []).append(ns)
        tot += ns
    print(f"# {sum(len(v) for v in by.values())} launches, {tot / 1e3:.1f} us total (cold-cache, serialised)")
    for name, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name:62s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:10.2f} us  share={sum(v) / tot:6.1%}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
