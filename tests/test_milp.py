"""CPU tests of the three-stage MILP synthesizer (generator/milp.py; App. B).

Pins: every synthesized program is checked by the oracle against the collective's definition;
the Stage-1 optimum equals the relaxed bound that closed forms give for switch topologies
(eq. link1 / switch1s1 / switch1r1 with shortest paths); Stage 3 reproduces the paper's
contiguity example (two 32 KB chunks over IB together: 8.325 us vs 10.025 us apart,
PAPER.md:549–551); the final schedule is never slower than the Stage-2 ordering it refines
(Stage 3 can always pick 'nothing together', which is that ordering's schedule)."""
import numpy as np
import pytest

import oracle
from paper_2111_04867_b200.generator import generate, milp
from paper_2111_04867_b200.generator.greedy import schedule_time
from paper_2111_04867_b200.generator.topology import (
    IB_ALPHA_US, IB_BETA_US_PER_MB, NVLINK_ALPHA_US, NVLINK5_BETA_US_PER_MB, Sketch, multinode, rotate)

CASES = [("allgather", 4, 1, {}), ("allgather", 8, 2, {}), ("alltoall", 4, 2, {}), ("alltoall", 8, 1, {}),
         ("allgather", 8, 1, {"policy": "uc-min"}), ("allreduce", 4, 1, {}), ("reducescatter", 4, 2, {}),
         ("allgather", 8, 1, {"topology": "2x4", "size": 1 << 16}),
         ("alltoall", 8, 1, {"topology": "2x4", "size": 1 << 16}),
         ("allreduce", 8, 1, {"topology": "2x4", "size": 1 << 16})]


@pytest.mark.parametrize("coll,n,p,kw", CASES, ids=[f"{c[0]}-n{c[1]}-p{c[2]}-{c[3]}" for c in CASES])
def test_milp_schedule_is_correct(coll, n, p, kw):
    text = generate(coll, "milp", n, p, 1, **kw)
    v = oracle.validate(text)
    assert v.ok, f"{v.kind}: {v.msg}"
    rng = np.random.default_rng(7 * n + p)
    count = (n * p if coll != "allgather" else p) * 5
    e_in = n * count if coll in ("alltoall", "reducescatter") else count
    ins = [rng.integers(-1000, 1000, e_in).astype(np.int32) for _ in range(n)]
    outs = oracle.run(oracle.parse(text), ins, "int32")
    assert all(np.array_equal(a, b) for a, b in zip(outs, oracle.expected_outputs(coll, ins, "int32")))


@pytest.mark.parametrize("n", [3, 4, 8])
def test_routing_optimum_on_a_switch_is_the_port_bound(n):
    # Allgather on one switch: shortest paths are the direct links, every rank must receive
    # n-1 chunks through its switch port -> relaxed optimum (n-1)*lat (eq. switch1r1), and the
    # exact schedule reaches it (a rotation: step k sends to rank r+k)
    size = 1 << 20
    info = {}
    alg = milp.synthesize("allgather", n, 1, size=size, info=info)
    lat = NVLINK_ALPHA_US + NVLINK5_BETA_US_PER_MB * size / (1 << 20)
    st = info["stages"][0]
    assert st["routing_time"] == pytest.approx((n - 1) * lat, rel=1e-6)
    if n > 3:  # at n = 3 the Stage-2 tie-breaks (lowest chunk, then destination) collide on a port
        assert st["exact_time"] == pytest.approx((n - 1) * lat, rel=1e-6)
        assert schedule_time(alg.transfers) == pytest.approx((n - 1) * lat, rel=1e-6)
    assert {(t.src, t.dst) for t in alg.transfers} == {(u, v) for u in range(n) for v in range(n) if u != v}


def test_contiguity_stage_sends_two_ib_chunks_together():
    # two 32 KB chunks over IB: apart 2*(1.7+3.3125) = 10.025 us, together
    # 1.7 + 6.625 = 8.325 us. Two single-GPU nodes, Allgather with 2 chunks per rank of 32 KB.
    topo = multinode(2, 1)
    info = {}
    alg = milp.synthesize("allgather", 2, 2, topology=topo, size=64 << 10, info=info)
    assert all(len(t.chunks) == 2 for t in alg.transfers) and len(alg.transfers) == 2
    assert schedule_time(alg.transfers) == pytest.approx(8.325, abs=1e-6)
    assert info["stages"][0]["exact_time"] == pytest.approx(8.325, abs=1e-6)
    ib = IB_ALPHA_US + IB_BETA_US_PER_MB * 32 / 1024
    assert info["stages"][0]["ordering_time"] == pytest.approx(2 * ib, abs=1e-6)  # Stage 2 alone


def test_contiguity_declined_when_pipelining_wins():
    # large chunks through a relay: sending them one by one lets the second hop start after
    # one chunk (pipelining), so the optimum keeps them apart on the first hop
    from paper_2111_04867_b200.generator.topology import Link, Topology
    t = Topology("line3", 3, [0, 0, 0])
    for (u, v) in ((0, 1), (1, 2)):
        t.links[(u, v)] = Link(0.1, 10.0, "nvlink")
    sk = Sketch(input_chunkup=2, input_size=2 << 20)
    from paper_2111_04867_b200.generator.milp import contiguity, route
    chunks = [(0, 0, [2]), (1, 0, [2])]
    trees, t1, _ = route("allgather", t, sk, chunks, 1.0)
    assert trees[0] == [(0, 1), (1, 2)]
    ordered = [(0.0, 10.1, (0,), 0, 1), (10.1, 20.2, (1,), 0, 1), (10.1, 20.2, (0,), 1, 2), (20.2, 30.3, (1,), 1, 2)]
    xf, t3, _ = contiguity(t, ordered, 1.0, {0: 0, 1: 0}, [(0, 2), (1, 2)])
    assert t3 == pytest.approx(30.3, abs=1e-6)  # together would cost 20.1 + 20.1 = 40.2
    assert all(len(x[2]) == 1 for x in xf)


@pytest.mark.parametrize("coll,n,p,kw", [("allgather", 8, 2, {}), ("alltoall", 8, 2, {}),
                                         ("allgather", 8, 2, {"topology": "2x4", "size": 1 << 16}),
                                         ("alltoall", 8, 1, {"topology": "2x4", "size": 1 << 16})])
def test_exact_schedule_never_slower_than_its_ordering(coll, n, p, kw):
    info = {}
    alg = milp.synthesize(coll, n, p, info=info, **kw)
    st = info["stages"][0]
    # (Stage 1 is no lower bound here: it prices every chunk alone, Stage 3 may merge them)
    assert st["exact_time"] <= st["ordering_time"] + 1e-6
    assert schedule_time(alg.transfers) == pytest.approx(st["exact_time"], abs=1e-5)


def test_symmetry_constraints_give_a_rotation_symmetric_schedule():
    # App. B.1 symmetry rows: with offset (1, 4) every transfer's rotation is a transfer
    sk = Sketch(symmetry_offsets=[(1, 4)])
    alg = milp.synthesize("allgather", 4, 1, sketch=sk, size=1 << 20)
    xs = {(t.chunks, t.src, t.dst) for t in alg.transfers}
    for (cs, u, v) in xs:
        assert (tuple(rotate(c, 1, 4) for c in cs), rotate(u, 1, 4), rotate(v, 1, 4)) in xs


def test_relay_map_routes_inter_node_hops_through_the_relay():
    # Listing 1 chunk_to_relay_map: with (4, 1) on 2x4 every inter-node hop of
    # a chunk from rank s leaves from rank (s // 4) * 4 + 1
    sk = Sketch(chunk_to_relay=(4, 1), internode_conn={i: [i] for i in range(4)})
    alg = milp.synthesize("allgather", 8, 1, topology="2x4", sketch=sk, size=1 << 16)
    for t in alg.transfers:
        if t.src // 4 != t.dst // 4:
            for c in t.chunks:
                assert t.src == (c // 4) * 4 + 1
    text = generate("allgather", "milp", 8, 1, 1, topology="2x4", sketch=sk, size=1 << 16)
    assert oracle.validate(text).ok


def test_milp_is_deterministic():
    a = generate("alltoall", "milp", 8, 1, 1, topology="2x4", size=1 << 16)
    assert a == generate("alltoall", "milp", 8, 1, 1, topology="2x4", size=1 << 16)
