"""Oracle pins that hold for any schedule: determinism over every linearisation (brute force
on tiny programs), symbolic/numeric agreement, and the instance invariant.
Programs come from tests/golden and from the product's generator (its text is an input here;
the oracle checks it against the collective's definition)."""
import functools
import itertools

import numpy as np
import pytest

import oracle
from oracle.validate import build_graph, topo_order
from conftest import golden


def linear_extensions(graph, limit):
    """All topological orders (DFS), or None if there are more than `limit`."""
    n = len(graph.nodes)
    pred_mask = [0] * n
    for u, vs in enumerate(graph.succ):
        for v in vs:
            pred_mask[v] |= 1 << u

    @functools.lru_cache(maxsize=None)
    def count(done):
        if done == (1 << n) - 1:
            return 1
        return sum(count(done | (1 << v)) for v in range(n)
                   if not (done >> v) & 1 and (pred_mask[v] & ~done) == 0)

    total = count(0)
    if total > limit:
        return None, total
    out = []

    def rec(done, order):
        if len(order) == n:
            out.append(list(order))
            return
        for v in range(n):
            if not (done >> v) & 1 and (pred_mask[v] & ~done) == 0:
                order.append(v)
                rec(done | (1 << v), order)
                order.pop()
    rec(0, [])
    return out, total


def _inputs(prog, count, dtype, seed):
    rng = np.random.default_rng(seed)
    n = prog.nranks
    e_in = n * count if prog.coll in ("alltoall", "reducescatter") else count
    if dtype == "int32":
        return [rng.integers(-2**31, 2**31, e_in, dtype=np.int64).astype(np.int32) for _ in range(n)]
    return [rng.integers(0, 1 << 16, e_in).astype(np.uint16) for _ in range(n)]


def _check_all_orders(prog, count, dtype, limit=100000):
    graph = build_graph(prog)
    orders, total = linear_extensions(graph, limit)
    assert orders is not None, f"{total} linear extensions"
    ins = _inputs(prog, count, dtype, 11)
    ref = oracle.run(prog, ins, dtype, graph=graph, order=topo_order(graph))
    sym_ref = oracle.run_symbolic(prog, graph=graph, order=topo_order(graph))
    for order in orders:
        outs = oracle.run(prog, ins, dtype, graph=graph, order=order)
        assert all(np.array_equal(a, b) for a, b in zip(outs, ref))
        assert oracle.run_symbolic(prog, graph=graph, order=order) == sym_ref
    return total


def test_all_linearisations_c1():
    total = _check_all_orders(oracle.parse(golden("c1_ag_ring_n2_p2.xml")), 8, "int32")
    assert total > 1


def test_all_linearisations_gar():
    total = _check_all_orders(oracle.parse(golden("ar_rsag_n2_p1.xml")), 6, "int32")
    assert total > 1


@pytest.mark.parametrize("algo,n", [("ring", 3), ("direct", 2)])
def test_all_linearisations_reducescatter(algo, n):
    # generator text is only an input here: every order must give the definition's result
    from paper_2111_04867_b200.generator import generate
    prog = oracle.parse(generate("reducescatter", algo, n, 1, 1))
    total = _check_all_orders(prog, 4, "int32")
    assert total > 1
    ins = _inputs(prog, 4, "int32", 11)
    want = oracle.expected_outputs("reducescatter", ins, "int32")
    assert all(np.array_equal(a, b) for a, b in zip(oracle.run(prog, ins, "int32"), want))


def test_allgather_output_matches_definition_on_golden():
    prog = oracle.parse(golden("c1_ag_ring_n2_p2.xml"))
    ins = _inputs(prog, 10, "bfloat16", 12)
    outs = oracle.run(prog, ins, "bfloat16")
    want = oracle.expected_outputs("allgather", ins, "bfloat16")
    assert all(np.array_equal(a, b) for a, b in zip(outs, want))


def test_symbolic_numeric_agree_on_chunk_id_encoding():
    # numeric run with every element = chunk id * 1000 + offset decodes to the symbolic tokens
    prog = oracle.parse(golden("c1_ag_ring_n2_p2.xml"))
    ce = 7
    ins = [np.array([(r * 2 + k) * 1000 + e for k in range(2) for e in range(ce)], np.int32)
           for r in range(2)]
    outs = oracle.run(prog, ins, "int32")
    sym = oracle.run_symbolic(prog)
    for o, s in zip(outs, sym):
        for k, tok in enumerate(s):
            assert (o[k * ce:(k + 1) * ce] // 1000 == tok).all()


def test_instance_expansion_invariant_on_golden():
    for f, dtype, count in (("c1_ag_ring_n2_p2.xml", "int32", 24), ("ar_rsag_n2_p1.xml", "int32", 24)):
        prog = oracle.parse(golden(f))
        for m in (2, 3, 4):
            prog.instances = m
            exp = oracle.expand_instances(prog)
            assert exp.instances == 1 and exp.chunks_per_rank == prog.chunks_per_rank * m
            assert sum(len(t.steps) > 0 for t in exp.gpus[0].tbs) == m * sum(
                len(t.steps) > 0 for t in prog.gpus[0].tbs)
            assert oracle.validate(exp).ok
            ins = _inputs(prog, count, dtype, 13)
            a = oracle.run(prog, ins, dtype)
            b = oracle.run(exp, ins, dtype)
            assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_instance_subchunk_floor_split_by_hand():
    # reading G3 / docs/SCHEDULE.md: subchunk j of a chunk of c_e elements is
    # [floor(j*c_e/m), floor((j+1)*c_e/m)). c_e = 4, m = 3 -> [0,1), [1,2), [2,4): instance 2
    # carries two elements of every chunk. C1's AG ring (p=2) on count 8 (c_e = 4): an input
    # element lands in the output exactly where the Allgather definition puts it, and every
    # one of the 3 instances moves its own subchunk (tagged by instance through a poisoned copy).
    prog = oracle.parse(golden("c1_ag_ring_n2_p2.xml"))
    prog.instances = 3
    exp = oracle.expand_instances(prog)
    assert exp.subchunks == 3 and exp.chunks_per_rank == 6
    ins = [np.arange(8, dtype=np.int32) + 100 * r for r in range(2)]
    outs = oracle.run(exp, ins, "int32")
    for o in outs:
        assert o.tolist() == list(range(8)) + list(range(100, 108))
    # the element ranges the expanded chunks name (chunk q' = subchunk q' % 3 of chunk q' // 3)
    from oracle import simulate
    seen = []
    orig_read = simulate._execute

    def spy(prog_, graph, order, bufs, read, write, reduce, *rest):
        def w(buf, off, cnt, vals):
            seen.append((off, len(vals)))
            return write(buf, off, cnt, vals)
        return orig_read(prog_, graph, order, bufs, read, w, reduce, *rest)
    simulate._execute = spy
    try:
        oracle.run(exp, ins, "int32")
    finally:
        simulate._execute = orig_read
    sizes = {off % 3: n for off, n in seen}
    assert sizes == {0: 1, 1: 1, 2: 2}


@pytest.mark.parametrize("coll,algo,n,p,m,count", [
    ("allgather", "ring", 4, 1, 3, 10), ("allgather", "direct", 3, 2, 4, 2 * 7),
    ("alltoall", "direct", 4, 1, 3, 5), ("allreduce", "ring", 4, 1, 3, 4 * 5),
    ("allreduce", "direct", 3, 2, 4, 3 * 2 * 3), ("reducescatter", "ring", 3, 1, 2, 7)])
def test_instance_expansion_invariant_ragged(coll, algo, n, p, m, count):
    # expanded (m instances, floor split; c_e not a multiple of m) == unexpanded, bit for bit,
    # on generated programs; and both equal the collective's definition (int32)
    from paper_2111_04867_b200.generator import generate
    from paper_2111_04867_b200.inputs import allreduce_input
    prog = oracle.parse(generate(coll, algo, n, p, m))
    ce = oracle.chunk_elems(coll, n, p, count)
    assert ce % m != 0
    exp = oracle.expand_instances(prog)
    assert oracle.validate(exp).ok
    e_in = n * count if coll in ("alltoall", "reducescatter") else count
    ins = [allreduce_input(e_in, "int32", "bits", 31, r) for r in range(n)]
    a, b = oracle.run(prog, ins, "int32"), oracle.run(exp, ins, "int32")
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert all(np.array_equal(x, y) for x, y in zip(a, oracle.expected_outputs(coll, ins, "int32")))
