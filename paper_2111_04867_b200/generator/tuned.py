"""Size-specialised default schedule sets (TACCL keeps
several algorithms per collective and uses the best one for each buffer size).

Each entry is (algorithm, [minBytes, maxBytes)) in the runtime's selection convention
(include/taccl.h taccl_run: S = AG output bytes, A2A per-rank send bytes, AR buffer bytes,
RS send bytes). Crossovers come from the graph-mode sweeps on B200 in profiles/
(r01_sweep_n2_graph.jsonl, r01_sweep_n4_graph.jsonl, r01_small_sweep_n4.jsonl); n = 8 is
unmeasured (the pool offers <= 4 GPUs) and extrapolated from n = 4.
"""
from __future__ import annotations

import math

MiB = 1 << 20
INF = math.inf


def ranges(coll: str, n: int):
    """[(algo, min_bytes, max_bytes)] covering [0, inf) for `coll` at n ranks; algo may carry
    a chunk-partitioning suffix `_pK` (K chunks per rank)."""
    if n == 1:
        return [("direct", 0, INF)]
    if coll == "allgather":
        return [("direct", 0, INF)] if n == 2 else [("direct", 0, 128 * MiB), ("ring", 128 * MiB, INF)]
    if coll == "alltoall":
        return [("direct", 0, INF)]
    # rings round every hop's bf16 partial (reading R4): at n >= 8 that reaches 1.2e-2 relative
    # error on U[1,2) inputs, above the north star's 1e-2, so large-n sets keep the direct
    # (one rounding per element) schedules
    if coll == "allreduce":
        if n == 2:
            return [("oneshot", 0, 16 * MiB), ("direct", 16 * MiB, INF)]
        small = MiB // 2 if n <= 4 else MiB // 4
        if n >= 8:
            return [("oneshot", 0, small), ("direct", small, INF)]
        # below 128 MiB the direct schedule (multi-input reduce with every load in flight) is
        # ahead of the ring (r01_sweep_n4_graph.jsonl: 64 MiB 185 vs 203 us); at 128-256 MiB
        # the plain ring is (two boxes: 128 MiB 342-344 vs ring_p2 354-369 us, 256 MiB 633-641
        # vs 649-672); from 512 MiB 2 chunks per rank pipeline the ring's 2(n-1) hops better
        # (512 MiB 1226 vs 1237-1259 us; profiles/r01_ar_variants_n4.txt)
        return [("oneshot", 0, small), ("direct", small, 128 * MiB), ("ring", 128 * MiB, 512 * MiB),
                ("ring_p2", 512 * MiB, INF)]
    if coll == "reducescatter":
        if n == 2 or n >= 8:
            return [("direct", 0, INF)]
        return [("direct", 0, 32 * MiB), ("ring", 32 * MiB, INF)]
    raise ValueError(coll)


def default_schedules(coll: str, n: int):
    """EF texts of the default set for (coll, n), each carrying its size range."""
    from . import generate
    out = []
    for algo, lo, hi in ranges(coll, n):
        name, _, p = algo.partition("_p")
        out.append(generate(coll, name, n, int(p) if p else 1, 1, min_bytes=lo, max_bytes=hi))
    return out
