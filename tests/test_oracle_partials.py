"""Pins of the oracle's bf16 "partials" reduction mode (oracle/simulate.py run(bf16=...);
DESIGN.md reading R6): an rrc's result keeps its fp32 accumulator, later rrcs read fp32
partials (local source or a send's message) when the whole range holds them, a receive (r)
or copy drops them, every rrc adds in fp32 with RNE. Pinned against values worked by hand,
against exact rational arithmetic (where every fp32 sum is exact, the mode must return the
correctly rounded bf16 of the exact sum for EVERY schedule), and against the per-step mode
where no intermediate rounding occurs.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import golden
from paper_2111_04867_b200.generator import generate
from test_oracle_definitions import _bf16_value, _exact_rne_bf16

ONE, E8, ZERO = 0x3F80, 0x3B80, 0x0000  # 1.0, 2^-8, +0.0 as bf16 bits


def _relay_inputs(vals):
    # rs_relay_n4: chunk d is reduced as o_d = (i_d[d] + i_{d+1}[d]) + bf16(i_{d+2}[d] + i_{d+3}[d]);
    # vals[k] is the value every rank x contributes to chunk c with (x - c) mod 4 == k
    return [np.array([vals[(x - c) % 4] for c in range(4)], np.uint16) for x in range(4)]


def test_relay_receive_drops_the_partial():
    # relay = i_{d+2} + i_{d+3} = 1 + 2^-8: fp32 partial 1+2^-8, bf16 bits RNE -> 1.0 (tie to
    # even). The plain receive on d+1 keeps only the bits, so d computes
    # (2^-8 + 0) + 1.0 = 1 + 2^-8 -> RNE 1.0 = 0x3F80. (Had the partial survived the relay:
    # 2^-8 + 1 + 2^-8 = 1 + 2^-7 = 0x3F81.)
    prog = oracle.parse(golden("rs_relay_n4.xml"))
    outs = oracle.run(prog, _relay_inputs({0: E8, 1: ZERO, 2: ONE, 3: E8}), "bfloat16", bf16="partials")
    assert [int(o[0]) for o in outs] == [0x3F80] * 4


def test_local_chain_keeps_fp32_partial():
    # i_d = 1.0, i_{d+1} = 2^-8, relay = bf16(2^-8 + 0) = 2^-8. Partials: the rrc chain on d
    # sums 1 + 2^-8 (fp32, exact) + 2^-8 = 1 + 2^-7 -> 0x3F81 (= the exact sum). Per-step:
    # bf16(1 + 2^-8) = 1.0 (tie to even), then bf16(1 + 2^-8) = 1.0 -> 0x3F80.
    prog = oracle.parse(golden("rs_relay_n4.xml"))
    ins = _relay_inputs({0: ONE, 1: E8, 2: E8, 3: ZERO})
    assert [int(o[0]) for o in oracle.run(prog, ins, "bfloat16", bf16="partials")] == [0x3F81] * 4
    assert [int(o[0]) for o in oracle.run(prog, ins, "bfloat16", bf16="per_step")] == [0x3F80] * 4


@pytest.mark.parametrize("algo", ["ring", "direct", "oneshot"])
def test_tie_case_every_schedule(algo):
    # three ranks contribute 1, 2^-8, 2^-8 to every element: the exact sum 1 + 2^-7 is a bf16
    # value (0x3F81) and every fp32 association is exact, so partials give 0x3F81 on every
    # rank whatever the schedule's order; per-step rounding gives 0x3F80 whenever the chain
    # adds 1 + 2^-8 first (a tie that rounds to even)
    n, count = 3, 3 * 5
    prog = oracle.parse(generate("allreduce", algo, n, 1, 1))
    ins = [np.full(count, v, np.uint16) for v in (ONE, E8, E8)]
    for o in oracle.run(prog, ins, "bfloat16", bf16="partials"):
        assert (o == 0x3F81).all()


def _exact_sum_inputs(n, count, seed):
    # bf16 values +-k * 2^e with 8-bit significands k in [128, 256) and e in [-13, -6]: every
    # partial sum of up to 8 of them is a multiple of 2^-13 below 2^6, i.e. fits in 19 < 24
    # significand bits, so EVERY fp32 association is exact; the bf16 rounding of the total is not
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        k = rng.integers(128, 256, count)
        e = rng.integers(-13, -5, count)
        f = (k * np.exp2(e.astype(np.float64))) * rng.choice([-1.0, 1.0], count)
        bits = (f.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)  # exact: 8-bit significands
        assert np.array_equal((bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64), f)
        out.append(bits)
    return out


SCHEDS = [("allreduce", "ring", 8, 1, {}), ("allreduce", "direct", 8, 1, {}), ("allreduce", "oneshot", 8, 1, {}),
          ("allreduce", "greedy", 8, 1, {"policy": "uc-min"}), ("allreduce", "greedy", 4, 2, {"policy": "uc-max"}),
          ("allreduce", "milp", 4, 2, {}), ("allreduce", "ring", 4, 2, {}),
          ("reducescatter", "ring", 8, 1, {}), ("reducescatter", "direct", 8, 1, {}),
          ("reducescatter", "milp", 8, 1, {"topology": "2x4", "size": 1 << 16})]


@pytest.mark.parametrize("coll,algo,n,p,kw", SCHEDS)
def test_exact_fp32_sums_round_once_for_every_schedule(coll, algo, n, p, kw):
    # where fp32 never rounds, the partials mode must return the correctly rounded bf16 of the
    # exact rational sum (the collective's definition, rounded once) — for
    # every schedule, whatever its association order or hop structure
    prog = oracle.parse(generate(coll, algo, n, p, 1, **kw))
    count = n * p * 7 if coll == "allreduce" else p * 7
    e_in = n * count if coll == "reducescatter" else count
    ins = _exact_sum_inputs(n, e_in, 41)
    exact = [_exact_rne_bf16(sum((_bf16_value(x[i]) for x in ins), Fraction(0))) for i in range(e_in)]
    outs = oracle.run(prog, ins, "bfloat16", bf16="partials")
    for r, o in enumerate(outs):
        want = exact if coll == "allreduce" else exact[r * count:(r + 1) * count]
        assert [int(v) for v in o] == want, (r, algo)


def test_per_step_mode_fails_the_exact_pin_on_a_ring():
    # the pin above has teeth: per-step bf16 rounding along an 8-rank ring differs from the
    # once-rounded exact sum on these inputs
    prog = oracle.parse(generate("allreduce", "ring", 8, 1, 1))
    ins = _exact_sum_inputs(8, 8 * 7, 41)
    exact = [_exact_rne_bf16(sum((_bf16_value(x[i]) for x in ins), Fraction(0))) for i in range(8 * 7)]
    o = oracle.run(prog, ins, "bfloat16", bf16="per_step")[0]
    assert [int(v) for v in o] != exact


@pytest.mark.parametrize("algo,n", [("ring", 8), ("direct", 4), ("oneshot", 4)])
def test_modes_agree_without_rounding(algo, n):
    # integer-valued bf16 in [-16, 16): every partial sum is exact in bf16 too, so the two
    # modes (and the int-like definition) coincide
    from paper_2111_04867_b200.inputs import allreduce_input
    prog = oracle.parse(generate("allreduce", algo, n, 1, 1))
    ins = [allreduce_input(n * 33, "bfloat16", "intval", 42, r) for r in range(n)]
    a = oracle.run(prog, ins, "bfloat16", bf16="partials")
    b = oracle.run(prog, ins, "bfloat16", bf16="per_step")
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("dtype", ["int32", "float32"])
def test_bf16_mode_leaves_other_dtypes_alone(dtype):
    from paper_2111_04867_b200.inputs import allreduce_input
    prog = oracle.parse(generate("allreduce", "ring", 4, 1, 1))
    ins = [allreduce_input(4 * 50, dtype, "uniform" if dtype == "float32" else "bits", 43, r) for r in range(4)]
    a = oracle.run(prog, ins, dtype, bf16="partials")
    b = oracle.run(prog, ins, dtype, bf16="per_step")
    assert all(np.array_equal(x.view(np.uint32), y.view(np.uint32)) for x, y in zip(a, b))


def test_partials_meet_the_north_star_bound_where_per_step_does_not():
    # north star: bf16 Allreduce within 1e-2 relative of the fp64 sum. U[1,2) on 8 ranks through
    # an 8-rank ring: per-hop rounding reaches ~1.24e-2; fp32 partials round once (~4e-3)
    from paper_2111_04867_b200.inputs import allreduce_input
    n, count = 8, 8 * 4000
    prog = oracle.parse(generate("allreduce", "ring", n, 1, 1))
    ins = [allreduce_input(count, "bfloat16", "uniform", 6, r) for r in range(n)]
    ref = oracle.expected_allreduce_f64(ins, "bfloat16")
    rel = {m: max(float((np.abs(oracle.collectives.to_f64(o, "bfloat16") - ref) / ref).max())
                  for o in oracle.run(prog, ins, "bfloat16", bf16=m)) for m in ("partials", "per_step")}
    assert rel["partials"] <= 2 ** -8 * 1.01  # one RNE: at most half an ulp (2^-8 relative)
    assert rel["per_step"] > 1e-2
