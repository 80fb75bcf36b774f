#!/usr/bin/env python
"""alpha-beta profile of NVLink 5 through this executor (the paper's
profiler, Table 1).

Fits t = alpha + beta * m per (collective, algorithm, protocol range) from sweep JSONL rows
(tools/sweep.py), where m is the MB each connection carries in one call:
  AG / A2A direct at n ranks: n-1 concurrent connections per GPU, m = S/n per connection;
  AG ring: 1 connection per GPU, m = S/n per hop, n-1 hops (t = (n-1)(alpha + beta m)).
Two ranges are fitted separately: LL (S <= 1 MiB) and direct (S >= 8 MiB).
The multi-connection comparison ("fig:multiconnection") is the ratio of
per-connection beta for direct (n-1 connections) vs ring (1 connection).

  python tools/alphabeta.py profiles/r01_sweep_n4_graph.jsonl [...] > profiles/r01_alphabeta.json
"""
import json
import sys

import numpy as np


def fit(xs, ys):
    A = np.vstack([np.ones(len(xs)), xs]).T
    (a, b), *_ = np.linalg.lstsq(A, ys, rcond=None)
    return float(a), float(b)


def main(paths):
    out = []
    for path in paths:
        rows = [json.loads(l) for l in open(path)]
        for coll in ("allgather", "alltoall"):
            for algo in ("direct", "ring"):
                for rng, lo, hi in (("ll", 0, 1 << 20), ("direct", 8 << 20, 1 << 40)):
                    pts = [(r["S"], r[f"taccl_{algo}_us"]) for r in rows
                           if r["coll"] == coll and f"taccl_{algo}_us" in r and lo <= r["S"] <= hi]
                    if len(pts) < 3:
                        continue
                    n = rows[0]["n"]
                    hops = (n - 1) if algo == "ring" else 1
                    m = np.array([s / n / (1 << 20) for s, _ in pts])
                    t = np.array([us / hops for _, us in pts])
                    a, b = fit(m, t)
                    out.append({"source": path, "coll": coll, "algo": algo, "n": n, "range": rng,
                                "connections_per_gpu": 1 if algo == "ring" else n - 1,
                                "alpha_us": round(a, 3), "beta_us_per_MB": round(b, 4),
                                "per_connection_GBps": round((1 << 20) / (b * 1e-6) / 1e9, 1) if b > 0 else None,
                                "points": len(pts)})
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1:])
