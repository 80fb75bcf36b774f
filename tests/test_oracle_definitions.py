"""Pins for oracle/collectives.py and the oracle's arithmetic (no GPU).

Each test checks the oracle against something other than itself: per-element index
definitions, an algebraic property (Alltoall is an involution),
Python big-integer sums, math.fsum, exact rational rounding, hand-worked bf16 sums
(tests/golden/bf16_add.txt) and torch's CPU bf16 conversion (a library routine).
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import collectives as C
from oracle.simulate import add, bf16_round
from conftest import GOLDEN


def _rand(n, count, seed, dtype=np.int32):
    rng = np.random.default_rng(seed)
    return [rng.integers(-2**31, 2**31, count, dtype=np.int64).astype(dtype) for _ in range(n)]


@pytest.mark.parametrize("n,count", [(1, 5), (2, 7), (3, 4), (8, 3)])
def test_allgather_definition_elementwise(n, count):
    # "every GPU receives the data buffers of all other GPUs"
    ins = _rand(n, count, 1)
    outs = C.expected_outputs("allgather", ins, "int32")
    for r in range(n):
        for s in range(n):
            for i in range(count):
                assert outs[r][s * count + i] == ins[s][i]


@pytest.mark.parametrize("n,count", [(1, 3), (2, 5), (4, 2), (8, 3)])
def test_alltoall_definition_elementwise(n, count):
    # "transposes the data chunk from buffer index to GPU index"
    ins = _rand(n, n * count, 2)
    outs = C.expected_outputs("alltoall", ins, "int32")
    for r in range(n):
        for s in range(n):
            for i in range(count):
                assert outs[r][s * count + i] == ins[s][r * count + i]


@pytest.mark.parametrize("n,count", [(2, 3), (4, 5), (8, 2)])
def test_alltoall_is_an_involution(n, count):
    ins = _rand(n, n * count, 3)
    twice = C.expected_outputs("alltoall", C.expected_outputs("alltoall", ins, "int32"), "int32")
    for a, b in zip(twice, ins):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_allreduce_int32_wraps_like_bigint(n):
    ins = _rand(n, 64, 4)
    ins[0][0] = 2**31 - 1
    if n > 1:
        ins[1][0] = 1  # forces a wrap at element 0
    outs = C.expected_outputs("allreduce", ins, "int32")
    for i in range(64):
        s = sum(int(x[i]) for x in ins) % 2**32
        s = s - 2**32 if s >= 2**31 else s
        for o in outs:
            assert int(o[i]) == s


@pytest.mark.parametrize("n,count", [(1, 4), (2, 3), (3, 5), (8, 2)])
def test_reducescatter_definition_elementwise(n, count):
    # ReduceScatter: rank r keeps the point-wise sum of part r,
    # written out with Python big integers and reduced mod 2^32 (reading G13)
    ins = _rand(n, n * count, 6)
    outs = C.expected_outputs("reducescatter", ins, "int32")
    for r in range(n):
        assert outs[r].size == count
        for i in range(count):
            s = sum(int(x[r * count + i]) for x in ins) % 2**32
            assert int(outs[r][i]) == (s - 2**32 if s >= 2**31 else s)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_allgather_of_reducescatter_is_allreduce(n):
    # Allreduce = ReduceScatter followed by Allgather
    ins = _rand(n, n * 3, 7)
    rs = C.expected_outputs("reducescatter", ins, "int32")
    ag = C.expected_outputs("allgather", rs, "int32")
    ar = C.expected_outputs("allreduce", ins, "int32")
    for a, b in zip(ag, ar):
        assert np.array_equal(a, b)


def test_reducescatter_f64_matches_fsum():
    rng = np.random.default_rng(8)
    n, count = 4, 25
    ins = [rng.standard_normal(n * count).astype(np.float32) for _ in range(n)]
    ref = C.expected_reducescatter_f64(ins, "float32")
    for r in range(n):
        for i in range(count):
            assert ref[r][i] == pytest.approx(math.fsum(float(x[r * count + i]) for x in ins), rel=1e-15, abs=1e-15)


def test_allreduce_f64_matches_fsum():
    rng = np.random.default_rng(5)
    ins = [rng.standard_normal(100).astype(np.float32) for _ in range(8)]
    ref = C.expected_allreduce_f64(ins, "float32")
    for i in range(100):
        assert ref[i] == pytest.approx(math.fsum(float(x[i]) for x in ins), rel=1e-15, abs=1e-15)


def test_chunk_geometry_table():
    # docs/SCHEDULE.md table; SPEC.md:127-135 chunk_size examples
    assert C.buffer_chunks("allgather", 16, 2) == (2, 32)
    assert C.buffer_chunks("alltoall", 16, 1) == (16, 16)
    assert C.chunk_elems("allgather", 16, 2, 1 << 20) == 1 << 19     # 1 MB input, p=2 -> 0.5 MB
    assert C.chunk_elems("alltoall", 16, 1, 1 << 20) == 1 << 20      # per-peer count = chunk
    assert C.chunk_elems("allreduce", 8, 1, 8 * 1000) == 1000
    with pytest.raises(ValueError):
        C.chunk_elems("allreduce", 8, 1, 1001)
    # ReduceScatter: input n*count (n*p chunks), output count (the rank's p chunks)
    assert C.buffer_chunks("reducescatter", 8, 2) == (16, 2)
    assert C.chunk_elems("reducescatter", 8, 2, 1000) == 500
    assert C.postcondition("reducescatter", 4, 2)[3] == {0: (6, (1, 1, 1, 1)), 1: (7, (1, 1, 1, 1))}


def test_pre_and_postconditions_shapes():
    # SPEC.md:123-125 build_collective examples
    pre = C.precondition("allgather", 4, 1)
    post = C.postcondition("allgather", 4, 1)
    assert all(pre[r] == {0: r} for r in range(4))
    assert all(post[r] == {g: g for g in range(4)} for r in range(4))
    # alltoall (2, 1): chunk from rank 0 slot 1 must end on rank 1
    pre = C.precondition("alltoall", 2, 1)
    post = C.postcondition("alltoall", 2, 1)
    assert pre[0][1] == 1 and post[1][0] == 1
    assert sorted(t for r in range(2) for t in pre[r].values()) == [0, 1, 2, 3]


# ---------------------------------------------------------------- bf16 arithmetic pins

def _bf16_value(bits):
    bits = int(bits)
    sign = -1 if bits & 0x8000 else 1
    e = (bits >> 7) & 0xFF
    f = bits & 0x7F
    if e == 0:
        return sign * Fraction(f, 128) * Fraction(2) ** -126
    return sign * (1 + Fraction(f, 128)) * Fraction(2) ** (e - 127)


def _exact_rne_bf16(x: Fraction):
    """Correct RNE of a finite rational to bf16 bits, by searching the two neighbours."""
    if x == 0:
        return 0
    sign = 0x8000 if x < 0 else 0
    ax = abs(x)
    # non-negative finite bf16 bit patterns 0..0x7F7F are monotone in value: bisect for the
    # first pattern >= |x|, then pick the nearer neighbour (ties: even pattern)
    lo_b, hi_b = 0, 0x7F80
    while lo_b < hi_b:
        mid = (lo_b + hi_b) // 2
        if _bf16_value(mid) >= ax:
            hi_b = mid
        else:
            lo_b = mid + 1
    if lo_b == 0x7F80:
        # above max finite: RNE overflows to inf past max + half an ulp
        half = (_bf16_value(0x7F7F) - _bf16_value(0x7F7E)) / 2
        return sign | (0x7F80 if ax >= _bf16_value(0x7F7F) + half else 0x7F7F)
    hi, lo = lo_b, lo_b - 1
    dhi, dlo = _bf16_value(hi) - ax, ax - _bf16_value(lo)
    best = hi if (dhi < dlo or (dhi == dlo and hi % 2 == 0)) else lo
    return sign | best


def test_bf16_add_hand_worked_cases():
    with open(os.path.join(GOLDEN, "bf16_add.txt")) as f:
        rows = [l.split("#")[0].split() for l in f if l.strip() and not l.startswith("#")]
    a = np.array([int(r[0], 16) for r in rows], np.uint16)
    b = np.array([int(r[1], 16) for r in rows], np.uint16)
    want = np.array([int(r[2], 16) for r in rows], np.uint16)
    got = add(a, b, "bfloat16")
    assert [hex(x) for x in got] == [hex(x) for x in want]
    nan = add(np.array([0x7F80], np.uint16), np.array([0xFF80], np.uint16), "bfloat16")
    assert (nan[0] & 0x7F80) == 0x7F80 and (nan[0] & 0x7F) != 0


def test_bf16_add_matches_exact_rational_rounding():
    rng = np.random.default_rng(6)
    # finite normal values spanning a few binades, both signs; includes exponent gaps > 15
    a = rng.integers(0x3000, 0x4400, 300).astype(np.uint16) | (rng.integers(0, 2, 300) << 15).astype(np.uint16)
    b = rng.integers(0x3000, 0x4400, 300).astype(np.uint16) | (rng.integers(0, 2, 300) << 15).astype(np.uint16)
    got = add(a, b, "bfloat16")
    # table of all finite bf16 values for the neighbour search
    for x, y, g in zip(a, b, got):
        assert int(g) == _exact_rne_bf16(_bf16_value(x) + _bf16_value(y)), (hex(x), hex(y))


def test_bf16_round_matches_torch_conversion():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    f = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 1e3,
                        rng.uniform(1, 2, 20000).astype(np.float32),
                        np.array([0.0, -0.0, np.inf, -np.inf, 3.4e38, 1e-40], np.float32)])
    ours = bf16_round(f)
    theirs = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, theirs)


def test_int32_add_wraps():
    a = np.array([2**31 - 1, -2**31, -1], np.int32)
    b = np.array([1, -1, 1], np.int32)
    assert add(a, b, "int32").tolist() == [-2**31, 2**31 - 1, 0]


def test_float32_add_is_single_rounding():
    rng = np.random.default_rng(8)
    a = rng.standard_normal(1000).astype(np.float32)
    b = rng.standard_normal(1000).astype(np.float32) * 1e-4
    got = add(a, b, "float32")
    for x, y, g in zip(a, b, got):
        # float64 sum of two float32 is exact here; one rounding to float32 must match
        assert g == np.float32(np.float64(x) + np.float64(y))


# ---------------------------------------------------------------- bf16 -> fp64 conversion
# oracle.collectives.bf16_to_f64 / to_f64 convert BOTH the fp64 reference inputs and the GPU
# outputs in every bf16 tolerance check, so a wrong shift or half would distort both alike.
# Pinned to hand-decoded values (bf16 = the top 16 bits of an IEEE binary32: 1 sign, 8
# exponent, 7 fraction bits) and to torch's own bf16 -> float64 conversion.
BF16_HAND = [  # bits, value (decoded by hand from sign/exponent/fraction)
    (0x3F80, 1.0), (0xC000, -2.0), (0x0001, 2.0 ** -133), (0x0080, 2.0 ** -126),
    (0x7F80, math.inf), (0xFF80, -math.inf), (0x8000, -0.0), (0x0000, 0.0),
    (0x3FC0, 1.5), (0x4049, 3.140625), (0x7F7F, (2 - 2.0 ** -7) * 2.0 ** 127), (0xBF81, -(1 + 2.0 ** -7)),
]


def test_bf16_to_f64_hand_values():
    from oracle.collectives import bf16_to_f64, to_f64
    bits = np.array([b for b, _ in BF16_HAND], np.uint16)
    want = [v for _, v in BF16_HAND]
    for f in (bf16_to_f64(bits), to_f64(bits, "bfloat16")):
        assert f.dtype == np.float64
        assert f.tolist() == want
        assert [math.copysign(1, x) for x in f] == [math.copysign(1, x) for x in want]  # -0.0 keeps its sign
    nan = bf16_to_f64(np.array([0x7FC0, 0xFFC1], np.uint16))
    assert np.isnan(nan).all()


def test_bf16_to_f64_matches_torch_on_every_pattern():
    torch = pytest.importorskip("torch")
    from oracle.collectives import bf16_to_f64
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)  # all 65536 bf16 patterns
    ours = bf16_to_f64(bits)
    theirs = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    both_nan = np.isnan(ours) & np.isnan(theirs)
    assert np.array_equal(ours[~both_nan], theirs[~both_nan])
    assert np.array_equal(np.isnan(ours), np.isnan(theirs))
    assert np.array_equal(np.signbit(ours[~both_nan]), np.signbit(theirs[~both_nan]))


def test_to_f64_other_dtypes_are_plain_widening():
    from oracle.collectives import to_f64
    f = np.array([1.5, -0.1, 3.4e38, 1e-45], np.float32)
    assert to_f64(f, "float32").tolist() == [float(x) for x in f]  # exact widening of binary32
    i = np.array([-2**31, 2**31 - 1, 0], np.int32)
    assert to_f64(i, "int32").tolist() == [-2.0 ** 31, 2.0 ** 31 - 1, 0.0]
