"""CPU tests of the boundary: libtaccl.so loads, exports every symbol include/taccl.h
declares, and its C++ validator agrees with the oracle on golden programs, generated
schedules and a corpus of >1000 random mutations."""
import ctypes
import os
import random
import re

import pytest

import oracle
from oracle.ef import serialize
from paper_2111_04867_b200 import taccl
from paper_2111_04867_b200.generator import generate
from conftest import ROOT, golden
import mutate


def header_functions():
    text = open(os.path.join(ROOT, "include", "taccl.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|taccl_result_t|uint64_t)\s+(taccl_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(taccl.LIB_PATH)
    names = header_functions()
    assert len(names) >= 17
    for name in names:
        assert hasattr(lib, name), name


def test_no_compute_calls_needed_for_validation():
    ok, kind, msg = taccl.validate(golden("c1_ag_ring_n2_p2.xml"))
    assert ok, msg


@pytest.mark.parametrize("f", ["c1_ag_ring_n2_p2.xml", "ar_rsag_n2_p1.xml", "ag_relay_cpy_n2.xml"])
def test_golden_programs_pass_both_validators(f):
    text = golden(f)
    assert oracle.validate(oracle.parse(text)).ok
    for direct in (True, False):
        ok, kind, msg = taccl.validate(text, direct)
        assert ok, (f, direct, kind, msg)


MUTS = mutate.load_mutations(golden("mutations.txt"))


@pytest.mark.parametrize("f,op,sem,direct,cite", MUTS, ids=[f"{m[0]}:{m[1]}" for m in MUTS])
def test_named_mutations_cpp(f, op, sem, direct, cite):
    text = serialize(mutate.apply(oracle.parse(golden(f)), op))
    for is_direct, want in ((False, sem), (True, direct)):
        ok, kind, msg = taccl.validate(text, is_direct)
        assert ("ok" if ok else kind) == want, f"{msg} ({cite})"


GEN = [(c, a, n, p) for c, a in [("allgather", "ring"), ("allgather", "direct"), ("alltoall", "direct"),
                                 ("allreduce", "ring"), ("allreduce", "direct"), ("allgather", "hier"),
                                 ("alltoall", "hier"), ("reducescatter", "ring"), ("reducescatter", "direct"),
                                 ("allreduce", "oneshot")]
       for n in (2, 4, 8) for p in (1, 2)]


@pytest.mark.parametrize("coll,algo,n,p", GEN)
def test_generated_schedules_pass_both_validators(coll, algo, n, p):
    text = generate(coll, algo, n, p, 1)
    assert oracle.validate(text).ok
    ok, kind, msg = taccl.validate(text)
    assert ok, f"{kind}: {msg}"


def _random_mutation(prog, rnd):
    """A random single mutation of a program (oracle Program objects)."""
    r = rnd.randrange(prog.nranks)
    g = prog.gpus[r]
    t = rnd.randrange(len(g.tbs))
    tb = g.tbs[t]
    if not tb.steps:
        return f"settb {r} {t} chan {rnd.randrange(2)}"
    k = rnd.randrange(len(tb.steps))
    st = tb.steps[k]
    choice = rnd.randrange(9)
    if choice == 0:
        return f"delete {r} {t} {k}"
    if choice == 1 and len(tb.steps) > 1:
        k2 = rnd.randrange(len(tb.steps))
        return f"swap {r} {t} {k} {k2}"
    if choice == 2:
        dt = rnd.randrange(len(g.tbs))
        if g.tbs[dt].steps:
            return f"set {r} {t} {k} deps {dt}:{rnd.randrange(len(g.tbs[dt].steps))}"
        return f"set {r} {t} {k} deps -"
    if choice == 3:
        return f"set {r} {t} {k} deps -"
    if choice == 4 and st.type != "nop":
        return f"set {r} {t} {k} cnt {max(1, st.cnt + rnd.choice([-1, 1]))}"
    if choice == 5 and st.dstbuf is not None:
        return f"set {r} {t} {k} dstoff {max(0, st.dstoff + rnd.choice([-1, 1]))}"
    if choice == 6 and st.srcbuf is not None:
        return f"set {r} {t} {k} srcoff {max(0, st.srcoff + rnd.choice([-1, 1]))}"
    if choice == 7:
        return f"settb {r} {t} {rnd.choice(['send', 'recv'])} {rnd.randrange(-1, prog.nranks)}"
    if st.type in ("r", "rrc"):
        return f"set {r} {t} {k} type {'rrc' if st.type == 'r' else 'r'}"
    return f"set {r} {t} {k} deps -"


def test_mutation_corpus_verdicts_agree():
    rnd = random.Random(211104867)
    bases = [golden("c1_ag_ring_n2_p2.xml"), golden("ar_rsag_n2_p1.xml")]
    for c, a, n, p in [("allgather", "ring", 3, 1), ("allgather", "direct", 3, 2), ("alltoall", "direct", 3, 1),
                       ("allreduce", "ring", 3, 1), ("allreduce", "direct", 4, 1), ("alltoall", "hier", 4, 1),
                       ("allgather", "hier", 4, 1), ("reducescatter", "ring", 3, 1), ("reducescatter", "direct", 3, 2)]:
        bases.append(generate(c, a, n, p, 1))
    total, kinds = 0, {}
    for base in bases:
        prog = oracle.parse(base)
        for _ in range(160):
            op = _random_mutation(prog, rnd)
            try:
                mp = mutate.apply(prog, op)
            except (IndexError, ValueError):
                continue
            if op.startswith("set") and " type " in op and mp.gpus[int(op.split()[1])].tbs[int(op.split()[2])].steps[int(op.split()[3])].srcbuf is None \
                    and "rrc" in op:
                continue  # r -> rrc needs a source operand; not a well-formed mutation
            text = serialize(mp)
            for direct in (True, False):
                v = oracle.validate(text, mode="direct" if direct else "semantic")
                ok, kind, msg = taccl.validate(text, direct)
                want = "ok" if v.ok else v.kind
                got = "ok" if ok else kind
                assert got == want, f"{op} on {prog.name} (direct={direct}): oracle {want} [{v.msg}] vs C++ {got} [{msg}]"
                kinds[want] = kinds.get(want, 0) + 1
            total += 1
    assert total >= 1000
    # the corpus exercises every failure class
    for k in ("ok", "structure", "match", "cycle", "race", "uninit", "postcondition"):
        assert kinds.get(k, 0) > 0, kinds
