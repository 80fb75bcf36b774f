#!/usr/bin/env python
"""Synthesis report of the three-stage MILP synthesizer (generator/milp.py) next to the greedy
stand-in, on the BASELINE configs' topologies (the paper reports synthesis times per sketch,
PAPER.md:1110-1130): per case the Stage-1 relaxed optimum, the Stage-2 ordering's makespan,
the Stage-3 exact optimum, the greedy makespan (same alpha-beta model, us) and the solver wall
time. CPU only.

  python tools/milp_report.py > profiles/r01_milp_synthesis.txt
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04867_b200.generator import greedy, milp  # noqa: E402

CASES = [  # (label, coll, n, p, kwargs)
    ("C2 AG nvswitch", "allgather", 8, 1, {"size": 1 << 20}),
    ("C2 AG nvswitch p=2", "allgather", 8, 2, {"size": 1 << 20}),
    ("C2 AG nvswitch uc-min", "allgather", 8, 1, {"size": 1 << 20, "policy": "uc-min"}),
    ("C3 A2A nvswitch", "alltoall", 8, 1, {"size": 1 << 20}),
    ("C3 A2A nvswitch p=2", "alltoall", 8, 2, {"size": 1 << 20}),
    ("C3 A2A nvswitch p=2 64KB", "alltoall", 8, 2, {"size": 1 << 16}),
    ("C5 AG 2x4 (dgx2-sk-2-like)", "allgather", 8, 1, {"topology": "2x4", "size": 1 << 16}),
    ("C5 AG 2x4 p=2", "allgather", 8, 2, {"topology": "2x4", "size": 1 << 16}),
    ("C5 A2A 2x4", "alltoall", 8, 1, {"topology": "2x4", "size": 1 << 16}),
    ("C5 A2A 2x4 1MB", "alltoall", 8, 1, {"topology": "2x4", "size": 1 << 20}),
]

print(f"{'case':30s} {'routing':>9s} {'ordering':>9s} {'exact':>9s} {'greedy':>9s} {'MILP/greedy':>11s} {'solve s':>8s}  status")
for label, coll, n, p, kw in CASES:
    info = {}
    t0 = time.time()
    alg = milp.synthesize(coll, n, p, info=info, time_limit=60.0, **kw)
    dt = time.time() - t0
    g = greedy.synthesize(coll, n, p, **kw)
    st = info["stages"][0]
    tg = greedy.schedule_time(g.transfers)
    tm = greedy.schedule_time(alg.transfers)
    status = "optimal" if st["exact_status"] == 0 else "time limit (best found)"
    print(f"{label:30s} {st['routing_time']:9.3f} {st['ordering_time']:9.3f} {tm:9.3f} {tg:9.3f} {tm / tg:11.3f} {dt:8.1f}  {status}")
