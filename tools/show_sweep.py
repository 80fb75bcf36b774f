#!/usr/bin/env python
"""Print a sweep JSONL (tools/sweep.py output) as a table."""
import json
import sys

for path in sys.argv[1:]:
    for l in open(path):
        r = json.loads(l)
        algs = "/".join(f"{k[6:-3]}={v:.1f}" for k, v in r.items() if k.startswith("taccl_") and k.endswith("_us") and k != "taccl_best_us")
        print(f"{r['coll']:10s} n={r['n']} {r['S']:>11d} {algs:32s} best_bw={r['taccl_best_busbw']:7.1f} "
              f"nccl={r.get('nccl_us', 0):8.1f}us {r.get('nccl_busbw', 0):7.1f} x{r.get('speedup_vs_nccl', 0):5.2f}")
