#!/usr/bin/env python
"""Link bytes a schedule moves vs the collective's algorithmic bytes (relays
of hierarchical / greedy schedules move more than (n-1)/n * S per rank).

  python tools/schedule_bytes.py                  # table for the generator's schedules
Per rank: link bytes = sum over its `s` steps of cnt x chunk bytes, with chunk bytes =
S / N_out for AG (S = output bytes), S / (n p) for A2A (S = per-rank send bytes), S / (n p)
for AR (S = buffer bytes) and RS (S = send bytes). Algorithmic bytes per rank: (n-1)/n S
for AG / A2A / RS, 2 (n-1)/n S for AR. Reported as the max over ranks / algorithmic."""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2111_04867_b200.generator import generate  # noqa: E402


def link_ratio(text):
    head = re.search(r'<algo [^>]*coll="(\w+)" nranks="(\d+)" chunks_per_rank="(\d+)"', text)
    coll, n, p = head.group(1), int(head.group(2)), int(head.group(3))
    chunk_frac = 1.0 / (n * p)  # chunk bytes / S in every convention above
    per_rank = []
    for g in re.split(r"<gpu ", text)[1:]:
        sent = sum(int(c) for c in re.findall(r'type="s"[^>]*cnt="(\d+)"', g))
        per_rank.append(sent * chunk_frac)
    algo = (2.0 if coll == "allreduce" else 1.0) * (n - 1) / n
    return coll, n, p, max(per_rank) / algo


if __name__ == "__main__":
    rows = [("allgather", "direct", 8, {}), ("allgather", "ring", 8, {}), ("allgather", "hier", 8, {}),
            ("allgather", "greedy", 8, {"topology": "2x4"}), ("alltoall", "direct", 8, {}),
            ("alltoall", "hier", 8, {}), ("alltoall", "greedy", 8, {"topology": "2x4"}),
            ("allreduce", "direct", 8, {}), ("allreduce", "ring", 8, {}), ("allreduce", "oneshot", 8, {}),
            ("reducescatter", "direct", 8, {}), ("allgather", "hier", 4, {}), ("alltoall", "hier", 4, {})]
    print(f"{'coll':14s} {'algo':8s} {'n':>2s} {'p':>2s}  link/algorithmic bytes (max over ranks)")
    for coll, algo, n, kw in rows:
        for p in (1, 2):
            c, nn, pp, r = link_ratio(generate(coll, algo, n, p, 1, **kw))
            print(f"{coll:14s} {algo:8s} {nn:2d} {pp:2d}  {r:.3f}  {kw if kw else ''}")
