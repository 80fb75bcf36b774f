#!/usr/bin/env python
"""Summarise graph-mode sweeps (tools/sweep.py --graph) for DESIGN.md §7.1: per collective,
1 KB latency, 64 MiB and 1 GiB busbw of the default set ('auto', else the best schedule) next
to NCCL, and the min-max speedup over NCCL across the sweep.

  python tools/results_table.py profiles/r01_sweep_n2_graph.jsonl profiles/r01_sweep_n4_graph.jsonl"""
import json
import sys

for path in sys.argv[1:]:
    rows = [json.loads(l) for l in open(path)]
    n = rows[0]["n"]
    print(f"## n={n} ({path})")
    print("| coll | 1 KB us (NCCL) | 64 MiB busbw (NCCL) | 1 GiB busbw (NCCL) | default vs NCCL min-max (size of min) |")
    print("|---|---|---|---|---|")
    for c in ("allgather", "alltoall", "allreduce", "reducescatter"):
        rs = [r for r in rows if r["coll"] == c]
        if not rs:
            continue
        key = "auto" if f"taccl_auto_us" in rs[0] else rs[0]["taccl_best"]

        def us(r):
            return r.get(f"taccl_{key}_us", r["taccl_best_us"])

        def bw(r):
            return r.get(f"taccl_{key}_busbw", r["taccl_best_busbw"])
        by = {r["S"]: r for r in rs}
        sp = [(r["nccl_us"] / us(r), r["S"]) for r in rs if "nccl_us" in r]
        lo = min(sp)
        f = lambda S, g: f"{g(by[S]):.1f} ({by[S]['nccl_' + ('us' if g is us else 'busbw')]:.1f})" if S in by else "-"
        print(f"| {c} | {f(1024, us)} | {f(1 << 26, bw)} | {f(1 << 30, bw)} | {lo[0]:.2f} ({lo[1]} B) - {max(sp)[0]:.2f} |")
