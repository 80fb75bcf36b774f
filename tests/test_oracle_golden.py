"""Oracle pins on the hand-written golden programs (tests/golden/README.md)."""
import numpy as np
import pytest

import oracle
from oracle.ef import serialize
from conftest import golden
import mutate


def test_c1_worked_example_numeric():
    # in_r[i] = (r<<16)+i, 512 int32 per rank -> out[j] = ((j>>9)<<16)+(j&511)
    prog = oracle.parse(golden("c1_ag_ring_n2_p2.xml"))
    assert oracle.validate(prog).ok
    ins = [((r << 16) + np.arange(512)).astype(np.int32) for r in range(2)]
    outs = oracle.run(prog, ins, "int32")
    j = np.arange(1024)
    want = ((j >> 9) << 16) + (j & 511)
    for o in outs:
        assert o.tolist() == want.tolist()
    assert outs[0][0] == 0 and outs[0][511] == 511 and outs[0][512] == 65536 and outs[0][1023] == 66047


def test_c1_symbolic():
    prog = oracle.parse(golden("c1_ag_ring_n2_p2.xml"))
    outs = oracle.run_symbolic(prog)
    assert outs == [[0, 1, 2, 3], [0, 1, 2, 3]]


def test_gar_numeric_and_symbolic():
    prog = oracle.parse(golden("ar_rsag_n2_p1.xml"))
    assert oracle.validate(prog).ok
    rng = np.random.default_rng(9)
    ins = [rng.integers(-1000, 1000, 6).astype(np.int32) for _ in range(2)]
    outs = oracle.run(prog, ins, "int32")
    for o in outs:
        assert o.tolist() == (ins[0] + ins[1]).tolist()
    sym = oracle.run_symbolic(prog)
    assert sym[0] == [(0, (1, 1)), (1, (1, 1))]


def test_serialize_parse_roundtrip_is_identical():
    # serialize -> parse -> serialize is byte-identical
    for f in ("c1_ag_ring_n2_p2.xml", "ar_rsag_n2_p1.xml"):
        t1 = serialize(oracle.parse(golden(f)))
        assert serialize(oracle.parse(t1)) == t1


MUTS = mutate.load_mutations(golden("mutations.txt"))


@pytest.mark.parametrize("f,op,sem,direct,cite", MUTS, ids=[f"{m[0]}:{m[1]}" for m in MUTS])
def test_named_mutations(f, op, sem, direct, cite):
    prog = mutate.apply(oracle.parse(golden(f)), op)
    for mode, want in (("semantic", sem), ("direct", direct)):
        v = oracle.validate(prog, mode=mode)
        got = "ok" if v.ok else v.kind
        assert got == want, f"{mode}: {v.msg} ({cite})"


def test_mutation_messages_name_the_failure():
    prog = oracle.parse(golden("ar_rsag_n2_p1.xml"))
    v = oracle.validate(mutate.apply(prog, "set 0 0 0 deps 0:3"))
    assert "r0:tb0:s0" in v.msg and "r0:tb0:s3" in v.msg          # names the cycle
    v = oracle.validate(mutate.apply(prog, "set 1 0 1 type r"))
    assert "(chunk 1, rank 0)" in v.msg and "missing contributions from ranks [1]" in v.msg
    c1 = oracle.parse(golden("c1_ag_ring_n2_p2.xml"))
    v = oracle.validate(mutate.apply(c1, "delete 0 1 0"))
    assert "(chunk 0, rank 0) missing" in v.msg


def test_syntax_errors():
    for bad in ("<algo", "<x/>", golden("c1_ag_ring_n2_p2.xml").replace('type="cpy"', 'type="mov"'),
                golden("c1_ag_ring_n2_p2.xml").replace('coll="allgather"', 'coll="bcast"')):
        v = oracle.validate(bad)
        assert not v.ok and v.kind == "syntax"
