"""Element-wise full-size comparison against the oracle's definitions (test helper).

All four collectives act element-wise along `count` ("the same data index"
for Allreduce; Allgather/Alltoall move whole ranges), so the columns [c0, c1) of every input
row form a valid problem of count c1 - c0 whose result is the same columns of every output
row. The full-size tests walk ALL columns block by block — every output element is compared
with the oracle's definition — while host memory stays bounded by one block.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle

VIEW = {"int32": (torch.int32, np.int32), "float32": (torch.float32, np.float32), "bfloat16": (torch.int16, np.uint16)}
TOL = {"float32": 1e-6, "bfloat16": 1e-2}  # north star: relative to the fp64 sum


def rows(coll, n):
    rows_in = n if coll in ("alltoall", "reducescatter") else 1
    rows_out = n if coll in ("allgather", "alltoall") else 1
    return rows_in, rows_out


def _host(t, dtype):
    tv, nv = VIEW[dtype]
    return t.view(tv).cpu().numpy().view(nv)


def check_blocked(coll, n, count, dtype, exact, inputs, outputs, block=1 << 23):
    """inputs: n device tensors (rank order); outputs: {rank: device tensor}. exact: compare
    bits with oracle.expected_outputs (AG/A2A any dtype, int32 AR/RS); else float AR/RS within
    TOL of oracle's fp64 sum. Returns (ok, detail)."""
    rows_in, rows_out = rows(coll, n)
    vd = "int32" if (exact and dtype == "float32") else dtype  # exact checks compare raw bits
    worst = 0.0
    for c0 in range(0, count, block):
        c1 = min(count, c0 + block)
        sub = [np.concatenate([_host(x[r * count + c0:r * count + c1], vd) for r in range(rows_in)]) for x in inputs]
        k = c1 - c0
        if exact:
            want = oracle.expected_outputs(coll, sub, vd)
        elif coll == "allreduce":
            ref = oracle.expected_allreduce_f64(sub, dtype)
            want = [ref] * n
        else:
            want = oracle.expected_reducescatter_f64(sub, dtype)
        for r, out in outputs.items():
            got = np.concatenate([_host(out[q * count + c0:q * count + c1], vd) for q in range(rows_out)])
            if exact:
                w = want[r].view(got.dtype)
                if not np.array_equal(got, w):
                    bad = np.nonzero(got != w)[0]
                    return False, f"rank {r}: {bad.size} mismatches in columns [{c0}, {c1}), first {bad[:4]} (of {rows_out}x{k})"
            else:
                rel = np.abs(oracle.collectives.to_f64(got, dtype) - want[r]) / np.abs(want[r])
                worst = max(worst, float(rel.max()))
                if rel.max() > TOL[dtype]:
                    return False, f"rank {r}: relative error {rel.max():.3e} > {TOL[dtype]} in columns [{c0}, {c1})"
    return True, f"max rel {worst:.3e}" if not exact else "bit-exact"
