"""CPU tests of the offline schedule generator (templates, greedy stand-in, lowering).
Every generated program is checked by the oracle against the collective's definition;
structural facts are pinned to the paper's statements and SPEC.md's examples."""
import math

import numpy as np
import pytest

import oracle
from paper_2111_04867_b200.generator import generate, templates
from paper_2111_04867_b200.generator.greedy import synthesize, schedule_time
from paper_2111_04867_b200.generator.topology import (
    IB_ALPHA_US, IB_BETA_US_PER_MB, Link, Sketch, apply_sketch, multinode, nvswitch, parse_sketch,
    relay_for_chunk, rotate)

MATRIX = [(c, a, n, p, kw)
          for c in ("allgather", "alltoall", "allreduce")
          for a, kw in (("ring", {}), ("direct", {}), ("greedy", {"policy": "uc-max"}),
                        ("greedy", {"policy": "uc-min"}))
          for n in (2, 3, 4, 8) for p in (1, 2)
          if (c, a) != ("alltoall", "ring")]
MATRIX += [(c, "hier", n, p, {}) for c in ("allgather", "alltoall") for n in (4, 8) for p in (1, 2)]
MATRIX += [(c, "greedy", 8, p, {"topology": "2x4"}) for c in ("allgather", "alltoall", "allreduce") for p in (1, 2)]
MATRIX += [("reducescatter", a, n, p, kw) for a, kw in (("ring", {}), ("direct", {}), ("greedy", {"policy": "uc-max"}),
                                                        ("greedy", {"policy": "uc-min"}))
           for n in (2, 3, 4, 8) for p in (1, 2)]
MATRIX += [("reducescatter", "direct", 1, p, {}) for p in (1, 2)]
MATRIX += [("allreduce", "oneshot", n, p, {}) for n in (1, 2, 3, 4, 8) for p in (1, 2)]
MATRIX += [("reducescatter", "greedy", 8, p, {"topology": "2x4"}) for p in (1, 2)]


@pytest.mark.parametrize("coll,algo,n,p,kw", MATRIX, ids=[f"{m[0]}-{m[1]}-n{m[2]}-p{m[3]}-{m[4]}" for m in MATRIX])
def test_generated_schedule_is_correct(coll, algo, n, p, kw):
    text = generate(coll, algo, n, p, 1, **kw)
    v = oracle.validate(text)
    assert v.ok, f"{v.kind}: {v.msg}"
    # numeric spot check against the collective's definition
    prog = oracle.parse(text)
    rng = np.random.default_rng(n * 100 + p)
    count = (n * p if coll != "allgather" else p) * 3
    e_in = n * count if coll in ("alltoall", "reducescatter") else count
    ins = [rng.integers(-1000, 1000, e_in).astype(np.int32) for _ in range(n)]
    outs = oracle.run(prog, ins, "int32")
    want = oracle.expected_outputs(coll, ins, "int32")
    assert all(np.array_equal(a, b) for a, b in zip(outs, want))


def test_generation_is_deterministic():
    for args in (("allreduce", "greedy", 8, 2, 1), ("alltoall", "hier", 8, 2, 4)):
        assert generate(*args) == generate(*args)


def test_ring_has_n_minus_1_transfer_steps_per_chunk():
    # "this algorithm requires n-1 link transfer steps per data chunk"
    for n in (2, 4, 8):
        alg = templates.ring_allgather(n, 2)
        per_chunk = {}
        for t in alg.transfers:
            for c in t.chunks:
                per_chunk[c] = per_chunk.get(c, 0) + 1
        assert set(per_chunk.values()) == {n - 1}


def test_uc_min_on_a_3_rank_switch_is_a_ring_uc_max_uses_all_links():
    # SPEC.md acceptance 8 / PAPER.md:445-452: uc-min -> 3 utilised links forming a cycle,
    # uc-max -> 6
    mn = synthesize("allgather", 3, 1, policy="uc-min")
    mx = synthesize("allgather", 3, 1, policy="uc-max")
    lmin = {(t.src, t.dst) for t in mn.transfers}
    lmax = {(t.src, t.dst) for t in mx.transfers}
    assert len(lmin) == 3 and len(lmax) == 6
    succ = dict(lmin)
    x, seen = 0, []
    for _ in range(3):
        seen.append(x)
        x = succ[x]
    assert x == 0 and sorted(seen) == [0, 1, 2]


@pytest.mark.parametrize("n", [4, 8])
def test_ring_identity_time(n):
    # SPEC.md acceptance 2: a uniform ring Allgather takes (n-1)(alpha + beta*s)
    size = 1 << 20
    alg = synthesize("allgather", n, 1, policy="uc-min", size=size)
    lat = Link(0.7, (1 << 20) / 900e9 * 1e6, "nvlink").cost(size / (1 << 20))
    assert schedule_time(alg.transfers) == pytest.approx((n - 1) * lat, rel=1e-12)


@pytest.mark.parametrize("size", [1 << 10, 1 << 20, 1 << 28])
def test_greedy_never_slower_than_ring_baseline(size):
    # SPEC.md acceptance 9 (under the same cost model, on a switch)
    ring = synthesize("allgather", 8, 1, policy="uc-min", size=size)
    best = min(schedule_time(synthesize("allgather", 8, 1, policy=pol, size=size).transfers)
               for pol in ("uc-max", "uc-min"))
    assert best <= schedule_time(ring.transfers) + 1e-9


def test_contiguity_saving_matches_the_paper():
    # PAPER.md:549-551 / SPEC.md acceptance 1: two 32 KB chunks over IB together are ~17% faster
    ib = Link(IB_ALPHA_US, IB_BETA_US_PER_MB, "ib")
    apart, together = 2 * ib.cost(32 / 1024), ib.cost(32 / 1024, 2)
    assert apart == pytest.approx(10.025) and together == pytest.approx(8.325)
    assert (apart - together) / apart == pytest.approx(0.1696, abs=5e-4)


def test_greedy_merges_chunks_on_ib_links():
    alg = synthesize("alltoall", 8, 2, topology="2x4", size=1 << 16)
    ib = [t for t in alg.transfers if t.src // 4 != t.dst // 4]
    assert ib and max(len(t.chunks) for t in ib) > 1
    assert all(t.src % 4 == t.dst % 4 for t in ib)  # dgx2-sk-2: GPU i <-> GPU i only


def test_relay_map_examples():
    # (r1, r2) = (2, 1): rp=4 -> 5, rp=5 -> 5, rp=0 -> 1
    sk = Sketch(chunk_to_relay=(2, 1))
    assert [relay_for_chunk(sk, rp) for rp in (4, 5, 0)] == [5, 5, 1]


def test_rotational_symmetry_examples():
    # SPEC.md:207-209 and PAPER.md:469-473
    assert rotate(0, 2, 16) == 2 and rotate(1, 2, 16) == 3
    assert rotate(0, 16, 32) == 16 and rotate(16, 16, 32) == 0
    assert rotate(0, 8, 16) == 8 and rotate(8, 8, 16) == 0    # Example 3: 0->1 implies 8->9
    for o, g in ((2, 16), (16, 32), (3, 8)):
        r = 5
        for _ in range(g // math.gcd(o, g)):
            r = rotate(r, o, g)
        assert r == 5


LISTING1 = """{
    // sketch for intra-node policy
    "intranode_sketch": {"strategy": "switch", "switches": [[0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15]],
                         "switch_hyperedge_strategy": ["uc-min"]},
    "internode_sketch": {"strategy": "relay",
        "internode_conn": {"1" : [0], "3" : [2], "5" : [4], "7" : [6], "9" : [8], "11" : [10], "13" : [12], "15" : [14]},
        "beta_split": {"1": 1, "3": 1, "5": 1, "7" : 1, "9" : 1, "11" : 1, "13" : 1, "15" : 1},
        "chunk_to_relay_map": [2,1]},
    "symmetry_offsets": [[2, 16], [16, 32]],
    "hyperparameters": {"input_chunkup": 2, "input_size": "1M"}
}"""


def test_listing1_sketch_parses_and_prunes():
    # PAPER.md:1289-1315
    sk = parse_sketch(LISTING1)
    assert sk.policy == "uc-min" and sk.input_chunkup == 2 and sk.input_size == 1 << 20
    assert sk.internode_conn[1] == [0] and sk.chunk_to_relay == (2, 1)
    assert sk.symmetry_offsets == [(2, 16), (16, 32)]
    lt = apply_sketch(multinode(2, 16), sk)
    inter = [(u, v) for (u, v) in lt.links if u // 16 != v // 16]
    senders = {u for u, _ in inter}
    assert len([u for u in senders if u < 16]) == 8 and all(u % 2 == 1 for u in senders)
    assert all(sum(1 for (a, _) in inter if a == u) == 1 for u in senders)
    with pytest.raises(ValueError):
        parse_sketch('{"symmetry_offsets": [[0, 16]]}')


def test_listing1_sketch_synthesizes_a_correct_allgather():
    sk = parse_sketch(LISTING1)
    alg = synthesize("allgather", 32, 2, topology=multinode(2, 16), sketch=sk)
    from paper_2111_04867_b200.generator.lowering import lower
    v = oracle.validate(lower(alg))
    assert v.ok, v.msg
    inter = [t for t in alg.transfers if t.src // 16 != t.dst // 16]
    assert all(t.src % 2 == 1 and t.dst % 2 == 0 for t in inter)   # relays: odd -> even
    # symmetric routing: every chunk crosses nodes exactly once
    crossings = {}
    for t in inter:
        for c in t.chunks:
            crossings[c] = crossings.get(c, 0) + 1
    assert set(crossings.values()) == {1} and len(crossings) == 64


def test_lowering_threadblock_rule_and_own_copy():
    # PAPER.md:750, 781-783 (one send peer, one recv peer per tb) and 768-769 (own copy)
    prog = oracle.parse(generate("allgather", "greedy", 8, 2, 1))
    for g in prog.gpus:
        cpy = [s for tb in g.tbs for s in tb.steps if s.type == "cpy"]
        assert len(cpy) == 1 and cpy[0].srcbuf == "i" and cpy[0].dstoff == g.id * 2
        for tb in g.tbs:
            assert all(s.type != "s" or tb.send >= 0 for s in tb.steps)


def test_instances_double_threadblocks_and_halve_chunks():
    # n=2 instances -> tb count doubles, per-step chunk size halves
    prog = oracle.parse(generate("allgather", "ring", 4, 1, 2))
    exp = oracle.expand_instances(prog)
    assert len(exp.gpus[0].tbs) == 2 * len(prog.gpus[0].tbs)
    assert exp.gpus[0].o_chunks == 2 * prog.gpus[0].o_chunks
    ins = [np.arange(8, dtype=np.int32) + 100 * r for r in range(4)]
    a, b = oracle.run(prog, ins, "int32"), oracle.run(exp, ins, "int32")
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_measured_profile_topology_synthesizes_correct_schedules():
    # the profiled B200 alpha-beta (tools/alphabeta.py) plugs into the greedy synthesizer
    from paper_2111_04867_b200.generator.topology import nvswitch_measured
    for coll in ("allgather", "alltoall"):
        alg = synthesize(coll, 4, 2, topology=nvswitch_measured(4))
        from paper_2111_04867_b200.generator.lowering import lower
        assert oracle.validate(lower(alg)).ok


@pytest.mark.parametrize("coll", ["allgather", "alltoall", "allreduce", "reducescatter"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_default_sets_cover_all_sizes_once(coll, n):
    # size-specialised sets: contiguous, disjoint, [0, inf)
    from paper_2111_04867_b200.generator.tuned import default_schedules, ranges
    for dt in ("int32", "float32", "bfloat16"):  # every element type sees a partition of [0, inf)
        rs = [r[:3] for r in ranges(coll, n) if len(r) == 3 or dt in r[3]]
        assert rs[0][1] == 0 and rs[-1][2] == math.inf
        for (_, _, hi), (_, lo, _) in zip(rs, rs[1:]):
            assert hi == lo
    from paper_2111_04867_b200 import taccl
    for text in default_schedules(coll, n):
        v = oracle.validate(text)
        assert v.ok, f"{v.kind}: {v.msg}"
        assert taccl.validate(text, True)[0]  # the C++ loader's checks too (overlap hints included)


# ---------------------------------------------------------------- contiguity (lowering.coalesce)

def _steps(text, rank=0):
    prog = oracle.parse(text)
    return [st for tb in prog.gpus[rank].tbs for st in tb.steps]


@pytest.mark.parametrize("n,p", [(2, 4), (4, 2), (8, 4)])
def test_direct_alltoall_chunks_travel_together(n, p):
    # chunks sent consecutively over a link may be sent together. A direct
    # Alltoall's p chunks per peer are final deliveries from the input: one cnt=p send and one
    # cnt=p receive per peer (`s r s r s r s r` for n=2, p=4 before)
    st = _steps(generate("alltoall", "direct", n, p, 1))
    assert sorted(s.type for s in st) == sorted(["s"] * (n - 1) + ["r"] * (n - 1) + ["cpy"])
    assert all(s.cnt == p for s in st)
    unmerged = _steps(generate("alltoall", "direct", n, p, 1, merge=False))
    assert len(unmerged) == 2 * (n - 1) * p + 1


def test_ring_hops_keep_their_pipelining():
    # a ring forwards every chunk: merging the p chunks of a hop would delay the first one's
    # forward, so a p=2 ring keeps one step per chunk and hop
    n, p = 4, 2
    st = _steps(generate("allgather", "ring", n, p, 1))
    assert sum(s.type == "s" for s in st) == (n - 1) * p and all(s.cnt == 1 for s in st if s.type == "s")


def test_merged_schedules_compute_the_same_result():
    from paper_2111_04867_b200.inputs import allreduce_input
    for coll, algo, n, p in [("alltoall", "direct", 4, 4), ("reducescatter", "direct", 4, 2),
                             ("allreduce", "direct", 4, 2), ("alltoall", "hier", 8, 2)]:
        count = n * p * 5 if coll in ("allreduce",) else p * 5
        e_in = n * count if coll in ("alltoall", "reducescatter") else count
        ins = [allreduce_input(e_in, "int32", "bits", 60, r) for r in range(n)]
        a = oracle.run(oracle.parse(generate(coll, algo, n, p, 1)), ins, "int32")
        b = oracle.run(oracle.parse(generate(coll, algo, n, p, 1, merge=False)), ins, "int32")
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        assert all(np.array_equal(x, y) for x, y in zip(a, oracle.expected_outputs(coll, ins, "int32")))


def test_rounds_variant_orders_sends_by_round():
    # generate(..., "rounds"): the split all-pairs schedule where the send of round d waits for
    # the receive of round d - 1 (both validators accept it; deps only on this rank's receives)
    import re
    from paper_2111_04867_b200 import taccl
    for coll, n in (("alltoall", 4), ("allgather", 8)):
        text = generate(coll, "rounds", n, 1, 1)
        assert oracle.validate(text).ok and taccl.validate(text, True)[0]
        for r in range(n):
            body = text[text.index(f'<gpu id="{r}"'):]
            body = body[:body.index("</gpu>")]
            recv_tb = {int(b): int(a) for a, b in re.findall(r'<tb id="(\d+)" send="-1" recv="(\d+)"', body)}
            for t, peer, deps in re.findall(r'<tb id="(\d+)" send="(\d+)" recv="-1"[^>]*>\s*<step s="0" type="s"[^>]*deps="([^"]*)"', body):
                d = (int(peer) - r) % n
                want = "" if d < 2 else f"{recv_tb[(r - (d - 1)) % n]}:0"
                assert deps == want, (coll, r, t, deps, want)


def test_default_sets_use_the_measured_variants():
    # generator/tuned.py choices pinned to the measurements they cite (profiles/r02_*):
    # overlap pairs for RS n=4 bf16 from 80 MiB and AR n=4 from 64 MiB, the streamed split RS at
    # n=2 from 256 MiB, the fp32 ring RS up to 512 MiB
    from paper_2111_04867_b200.generator.tuned import ranges
    MiB = 1 << 20

    def pick(coll, n, S, dt):
        return next(r[0] for r in ranges(coll, n) if r[1] <= S < r[2] and (len(r) == 3 or dt in r[3]))
    assert pick("reducescatter", 4, 64 * MiB, "bfloat16") == "direct"
    assert pick("reducescatter", 4, 80 * MiB, "bfloat16") == "direct_ovl"
    assert pick("reducescatter", 4, 256 * MiB, "float32") == "ring"
    assert pick("reducescatter", 4, 512 * MiB, "float32") == "direct_ovl"
    assert pick("reducescatter", 2, 128 * MiB, "bfloat16") == "direct"
    assert pick("reducescatter", 2, 256 * MiB, "bfloat16") == "direct_split"
    assert pick("allreduce", 4, 32 * MiB, "bfloat16") == "direct"
    assert pick("allreduce", 4, 64 * MiB, "bfloat16") == "direct_ovl"
    assert pick("allreduce", 4, 256 * MiB, "bfloat16") == "dring_ovl"
    assert pick("allreduce", 4, 128 * MiB, "int32") == "dring_ovl"
    assert 'overlap="1"' in generate("reducescatter", "direct", 4, 1, 1, overlap=True)
