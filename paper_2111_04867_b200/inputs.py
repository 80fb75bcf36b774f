"""Seeded synthetic inputs shared by tests and bench.py (no method arithmetic here).

Recipe: PCG64 with seed = 211104867 + 1000*config +
rank. Allgather/Alltoall use random 16-bit (or 32-bit) patterns compared as raw bits;
Allreduce uses U[1,2), integer-valued floats (exact under any summation order) and N(0,1).
bf16 values are returned as uint16 bit patterns (torch's float32 -> bfloat16 conversion).
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 211104867


def rng(config: int, rank: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(BASE_SEED + 1000 * config + rank))


def _to_bf16_bits(f32: np.ndarray) -> np.ndarray:
    import torch
    return torch.from_numpy(np.ascontiguousarray(f32, np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def random_bits(n: int, dtype: str, config: int, rank: int) -> np.ndarray:
    g = rng(config, rank)
    if dtype == "bfloat16":
        return g.integers(0, 1 << 16, n, dtype=np.uint16)
    if dtype == "int32":
        return g.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    if dtype == "float32":
        return g.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    raise ValueError(dtype)


def allreduce_input(n: int, dtype: str, kind: str, config: int, rank: int) -> np.ndarray:
    """kind: 'uniform' U[1,2) | 'intval' integer-valued | 'normal' N(0,1) | 'bits' (int32)."""
    g = rng(config, rank)
    if dtype == "int32":
        return g.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    if kind == "uniform":
        f = g.uniform(1.0, 2.0, n).astype(np.float32)
    elif kind == "intval":
        lim = 16 if dtype == "bfloat16" else 1 << 20
        f = g.integers(-lim, lim, n).astype(np.float32)
    elif kind == "normal":
        f = g.standard_normal(n).astype(np.float32)
    else:
        raise ValueError(kind)
    return _to_bf16_bits(f) if dtype == "bfloat16" else f
