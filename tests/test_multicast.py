"""CPU tests of the multicast-reduce step (`mr`, NVLink SHARP; reading N1): both
validators accept the generator's schedules and reject the same broken ones with the same
class; the oracle's `mr` computes the Allreduce definition — exactly for
int32, and for bf16 the once-rounded exact sum wherever fp32 accumulation is exact; the
barrier ordering is what the race check enforces."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2111_04867_b200 import taccl
from paper_2111_04867_b200.generator import generate
from paper_2111_04867_b200.inputs import allreduce_input
from test_oracle_definitions import _bf16_value, _exact_rne_bf16


def both(text):
    v = oracle.validate(text)
    ok, kind, _ = taccl.validate(text, True)
    return (v.ok, v.kind), (ok, kind)


@pytest.mark.parametrize("n,p", [(2, 1), (4, 1), (4, 2), (8, 1), (8, 4)])
def test_nvls_schedules_valid_and_exact(n, p):
    text = generate("allreduce", "nvls", n, p, 1)
    (ok1, _), (ok2, _) = both(text)
    assert ok1 and ok2
    ins = [allreduce_input(n * p * 9, "int32", "bits", 70, r) for r in range(n)]
    outs = oracle.run(oracle.parse(text), ins, "int32")
    assert all(np.array_equal(a, b) for a, b in zip(outs, oracle.expected_outputs("allreduce", ins, "int32")))


def test_nvls_bf16_rounds_the_exact_sum_once():
    # U[1,2)-like bf16 values (8-bit significands, one binade): every fp32 partial sum of <= 8
    # is exact, so the switch's fp32 accumulation (any order) rounds the exact sum once
    n = 8
    text = generate("allreduce", "nvls", n, 1, 1)
    rng = np.random.default_rng(71)
    ins = [(0x3F80 | rng.integers(0, 128, n * 40)).astype(np.uint16) for _ in range(n)]
    want = [_exact_rne_bf16(sum((_bf16_value(x[i]) for x in ins), Fraction(0))) for i in range(n * 40)]
    for o in oracle.run(oracle.parse(text), ins, "bfloat16"):
        assert [int(v) for v in o] == want


def _edit(text, rank, old, new):
    head, sep, rest = text.partition(f'<gpu id="{rank}"')
    body, sep2, tail = rest.partition("</gpu>")
    assert old in body
    return head + sep + body.replace(old, new, 1) + sep2 + tail


def test_missing_member_is_a_match_error():
    text = generate("allreduce", "nvls", 4, 1, 1)
    bad = _edit(text, 2, '<step s="0" type="mr" srcbuf="i" srcoff="2" dstbuf="o" dstoff="2" cnt="1" deps=""/>', "")
    assert both(bad) == ((False, "match"), (False, "match"))


def test_overlapping_shares_race():
    # rank 1 reduces rank 0's share as well: two members of one group write o[0] unordered
    text = generate("allreduce", "nvls", 4, 1, 1)
    bad = _edit(text, 1, 'srcoff="1" dstbuf="o" dstoff="1"', 'srcoff="0" dstbuf="o" dstoff="0"')
    assert both(bad) == ((False, "race"), (False, "race"))


def test_mr_needs_a_peerless_threadblock_and_a_reduction():
    text = generate("allreduce", "nvls", 2, 1, 1)
    bad = _edit(text, 0, '<tb id="0" send="-1" recv="-1"', '<tb id="0" send="1" recv="-1"')
    assert both(bad) == ((False, "structure"), (False, "structure"))


def test_barrier_orders_later_steps_on_every_rank():
    # a copy of another rank's share after the group is ordered by the barrier (valid); the
    # same copy placed in a concurrent threadblock without a dependency races with the group
    n = 2
    text = generate("allreduce", "nvls", n, 1, 1)
    after = text.replace('cnt="1" deps=""/>\n  </tb>', 'cnt="1" deps=""/>\n   <step s="1" type="nop" deps=""/>\n  </tb>')
    assert both(after) == ((True, None), (True, None))
    # rank 0 reads o[1] (written by rank 1's member) in a second, unordered threadblock
    racy = _edit(text, 0, "  </tb>\n", '  </tb>\n  <tb id="1" send="-1" recv="-1" chan="0">\n'
                 '   <step s="0" type="cpy" srcbuf="i" srcoff="1" dstbuf="o" dstoff="1" cnt="1" deps=""/>\n  </tb>\n')
    assert both(racy)[0] == (False, "race") and both(racy)[1] == (False, "race")
