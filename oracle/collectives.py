"""Collective definitions for the oracle (test infrastructure; see oracle/__init__.py).

PAPER.md:218–225 (§2): "In Allgather, every GPU receives the data buffers of all other
GPUs. In Alltoall, every GPU receives different parts, or chunks, of the data buffers
present on all GPUs. This effectively transposes the data chunk from buffer index to GPU
index ... In Allreduce, every GPU ends up with a data buffer that has the results of
performing a point-wise computation (e.g. sum ...) over the same data index of all GPUs."
ReduceScatter (§5.3): Allreduce's point-wise sum of which each GPU
keeps only its own part (NCCL convention: rank r keeps elements [r·count, (r+1)·count)).
Chunk-level pre/postconditions: App. B; chunk-id layout SPEC.md:142.
"""
from __future__ import annotations

import numpy as np

from .ef import ScheduleError

DTYPES = {
    # name: (numpy storage dtype, element bytes)
    "int32": (np.int32, 4),
    "float32": (np.float32, 4),
    "bfloat16": (np.uint16, 2),  # raw bf16 bit patterns
}


def buffer_chunks(coll: str, n: int, p: int):
    """(N_in, N_out) chunk counts the collective fixes for a rank (docs/SCHEDULE.md)."""
    if coll == "allgather":
        return p, n * p
    if coll in ("alltoall", "allreduce"):
        return n * p, n * p
    if coll == "reducescatter":
        return n * p, p
    raise ScheduleError("syntax", f"unknown collective {coll}")


def input_elems(coll: str, n: int, count: int) -> int:
    """E_in: elements of the input buffer for NCCL-style `count` (reading G8)."""
    return n * count if coll in ("alltoall", "reducescatter") else count


def output_elems(coll: str, n: int, count: int) -> int:
    return count if coll in ("allreduce", "reducescatter") else n * count


def chunk_elems(coll: str, n: int, p: int, count: int) -> int:
    """c_e = E_in / N_in; all chunks of all buffers have this size."""
    n_in, _ = buffer_chunks(coll, n, p)
    e_in = input_elems(coll, n, count)
    if e_in % n_in:
        raise ValueError(f"count={count} not divisible into {n_in} equal chunks (reading G2)")
    return e_in // n_in


# --- chunk-level pre/postconditions (App. B) -------------

def precondition(coll: str, n: int, p: int):
    """{rank: {input chunk index: token}}; AG/A2A tokens are global chunk ids,
    AR/RS tokens are (chunk index, contribution counts per rank)."""
    pre = {}
    for r in range(n):
        if coll == "allgather":
            pre[r] = {k: r * p + k for k in range(p)}
        elif coll == "alltoall":
            pre[r] = {d * p + k: (r * n + d) * p + k for d in range(n) for k in range(p)}
        else:
            pre[r] = {k: (k, tuple(1 if s == r else 0 for s in range(n))) for k in range(n * p)}
    return pre


def postcondition(coll: str, n: int, p: int):
    """{rank: {output chunk index: required token}}."""
    post = {}
    for r in range(n):
        if coll == "allgather":
            post[r] = {g: g for g in range(n * p)}
        elif coll == "alltoall":
            post[r] = {s * p + k: (s * n + r) * p + k for s in range(n) for k in range(p)}
        elif coll == "reducescatter":
            post[r] = {k: (r * p + k, tuple([1] * n)) for k in range(p)}
        else:
            post[r] = {k: (k, tuple([1] * n)) for k in range(n * p)}
    return post


# --- element-level definitions ----------------------------------------

def expected_outputs(coll: str, inputs, dtype: str):
    """The collective's result for host inputs (one 1-D array per rank).

    AG: out_r = in_0 ++ in_1 ++ ... ++ in_{n-1}.
    A2A: out_r[s*count + i] = in_s[r*count + i].
    AR (int32 only here; floats use expected_allreduce_f64): out_r[i] = sum_s in_s[i] mod 2^32.
    RS (int32 only): out_r[i] = sum_s in_s[r*count + i] mod 2^32.
    """
    n = len(inputs)
    if coll == "allgather":
        out = np.concatenate(inputs)
        return [out.copy() for _ in range(n)]
    if coll == "alltoall":
        count = inputs[0].size // n
        outs = []
        for r in range(n):
            outs.append(np.concatenate([inputs[s][r * count:(r + 1) * count] for s in range(n)]))
        return outs
    if coll == "allreduce":
        if dtype != "int32":
            raise ValueError("float allreduce has no single exact result; use expected_allreduce_f64")
        acc = np.zeros(inputs[0].size, dtype=np.int64)
        for x in inputs:
            acc += x.astype(np.int64)
        out = (acc & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        return [out.copy() for _ in range(n)]
    if coll == "reducescatter":
        if dtype != "int32":
            raise ValueError("float reducescatter has no single exact result; use expected_reducescatter_f64")
        count = inputs[0].size // n
        outs = []
        for r in range(n):
            acc = np.zeros(count, dtype=np.int64)
            for x in inputs:
                acc += x[r * count:(r + 1) * count].astype(np.int64)
            outs.append((acc & 0xFFFFFFFF).astype(np.uint32).view(np.int32))
        return outs
    raise ValueError(coll)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> float64 (exact: bf16 is the top half of a binary32)."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def to_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bfloat16":
        return bf16_to_f64(x)
    return x.astype(np.float64)


def expected_allreduce_f64(inputs, dtype: str) -> np.ndarray:
    """fp64 reference sum_s (double) in_s[i] for float allreduce (north star tolerance)."""
    acc = np.zeros(inputs[0].size, dtype=np.float64)
    for x in inputs:
        acc += to_f64(x, dtype)
    return acc


def expected_reducescatter_f64(inputs, dtype: str):
    """fp64 reference for float reducescatter: out_r[i] = sum_s (double) in_s[r*count + i]."""
    n = len(inputs)
    count = inputs[0].size // n
    full = expected_allreduce_f64(inputs, dtype)
    return [full[r * count:(r + 1) * count].copy() for r in range(n)]
