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


BF16 = ("bfloat16",)
WIDE = ("int32", "float32")


def ranges(coll: str, n: int):
    """[(algo, min_bytes, max_bytes[, dtypes])] covering [0, inf) for `coll` at n ranks, for
    every element type; algo may carry a chunk-partitioning suffix `_pK` (K chunks per rank,
    PAPER.md:702-711), then `_split` (sends and receives lowered into separate threadblocks,
    generate(pair=False)) and then `_ovl` (the overlap="1" execution hint: warp-specialised send +
    receive-reduce pairs); an entry with a dtypes tuple is selected only for those types."""
    if n == 1:
        return [("direct", 0, INF)]
    if coll == "allgather":
        return [("direct", 0, INF)] if n == 2 else [("direct", 0, 128 * MiB), ("ring", 128 * MiB, INF)]
    if coll == "alltoall":
        return [("direct", 0, INF)]
    if coll == "allreduce":
        if n == 2:
            return [("oneshot", 0, 16 * MiB), ("direct", 16 * MiB, INF)]
        small = MiB // 2 if n <= 4 else MiB // 4
        if n >= 8:  # extrapolated from n = 4 (no 8-GPU box): overlap pairs from 64 MiB
            return [("oneshot", 0, small), ("direct", small, 64 * MiB), ("direct_ovl", 64 * MiB, INF)]
        # below 64 MiB the direct schedule (multi-input reduce with every load in flight) is
        # ahead of the ring (r01_sweep_n4_graph.jsonl: 64 MiB 185 vs 203 us). bf16: a ring
        # carries fp32 partials on its n-2 middle hops (reading R6; 2x those bytes), so rings
        # are out (profiles/r02_sweep_ar_ring_ab_n4.txt: 128 MiB 366 vs 463 us, 512 MiB 1356 vs
        # 1723). From 64 MiB the overlap hint (each paired send and the receive-reduce after it
        # run at once on the two halves of every CTA, the reduce consuming stripes as they land)
        # removes the reduce tail between the two phases (profiles/r02_knob_scan_overlap_n4.txt:
        # bf16 64 MiB 181 vs 187 us, 128 MiB 327 vs 357, 1 GiB 2381 vs 2557); from 256 MiB the
        # all-pairs RS + ring AG ("dring": one AG connection per GPU) with the hint is ahead
        # (512 MiB 1180 vs 1208, 1 GiB 2358 vs 2381); fp32/int32 the same shape from 128 MiB
        # (fp32 512 MiB 1189 vs ring 1209 and direct+hint 1211)
        return [("oneshot", 0, small), ("direct", small, 64 * MiB), ("direct_ovl", 64 * MiB, 256 * MiB, BF16),
                ("dring_ovl", 256 * MiB, INF, BF16), ("direct_ovl", 64 * MiB, 128 * MiB, WIDE),
                ("dring_ovl", 128 * MiB, INF, WIDE)]
    if coll == "reducescatter":
        if n == 2:
            # from 256 MiB the split lowering's streamed push reduce beats the paired schedule's
            # in-place pull (1 GiB 800 vs 833 us, 256 MiB 221 vs 223; profiles/r02_knob_scan_split_n2.txt);
            # the overlap hint loses at n=2 (1 GiB 877 us, r02_knob_scan_overlap_n4.txt)
            return [("direct", 0, 256 * MiB), ("direct_split", 256 * MiB, INF)]
        if n >= 8:  # extrapolated from n = 4 (no 8-GPU box)
            return [("direct", 0, 80 * MiB), ("direct_ovl", 80 * MiB, INF)]
        # bf16 rings carry fp32 partials on n-2 of n-1 hops (reading R6): 0.58-0.72x NCCL at
        # 32 MiB-1 GiB (profiles/r02_sweep_n4_graph.txt), so bf16 stays all-pairs; from 80 MiB
        # with the overlap hint (warp-specialised send + streamed reduce pairs; profiles/
        # r02_knob_scan_overlap_n4.txt: 96 MiB 147 vs 155 us, 128 MiB 186 vs 203, 1 GiB 1231 vs
        # 1372; the split lowering's streamed reduces 147 / 187 / 1279). int32/fp32 keep round
        # 1's relay-first ring from 32 MiB up to 512 MiB, the hinted all-pairs schedule above
        # (fp32 768 MiB 935 vs 953 us, 1 GiB 1232 vs 1266)
        return [("direct", 0, 32 * MiB), ("direct", 32 * MiB, 80 * MiB, BF16), ("direct_ovl", 80 * MiB, INF, BF16),
                ("ring", 32 * MiB, 512 * MiB, WIDE), ("direct_ovl", 512 * MiB, INF, WIDE)]
    raise ValueError(coll)


def multicast_ranges(coll: str, n: int):
    """Multicast-reduce (NVLink SHARP) entries, loaded after the partition so they win their
    range whenever a call can run them (both buffers in the symmetric pool, 16-byte chunks;
    otherwise the runtime falls back to the partition's entry). At n = 2 the switch saves no
    bytes and costs a round trip (round 1 probe: 394 vs 700 GB/s busbw); from n = 4 it moves
    ~S per GPU each way instead of 1.5 S (profiles/r01_nvls_probe.txt). int32 has no vector
    form in the switch (scalar adds), so floats only."""
    if coll != "allreduce" or n < 4:
        return []
    # n = 4 (profiles/r02_nvls_lean_scan_n4.txt, lean multicast kernel): ahead of direct from
    # 4 MiB (4 MiB 31.8 vs 35.3 us, 8 MiB 41.9 vs 44.4, 64 MiB 170.6 vs 184); fp32 until the
    # relay-first ring takes over at 128 MiB
    return [("nvls", 4 * MiB, INF, ("bfloat16",)), ("nvls", 4 * MiB, 128 * MiB, ("float32",))]


def default_schedules(coll: str, n: int, multicast: bool = True):
    """EF texts of the default set for (coll, n), each carrying its size range; multicast
    entries (multicast_ranges) last."""
    from . import generate
    out = []
    extra = multicast_ranges(coll, n) if multicast else []
    for algo, lo, hi, *dt in ranges(coll, n) + extra:
        ovl = algo.endswith("_ovl")
        algo = algo.removesuffix("_ovl")
        split = algo.endswith("_split")
        name, _, p = algo.removesuffix("_split").partition("_p")
        out.append(generate(coll, name, n, int(p) if p else 1, 1, min_bytes=lo, max_bytes=hi,
                            pair=not split, dtypes=dt[0] if dt else None, overlap=ovl))
    return out
