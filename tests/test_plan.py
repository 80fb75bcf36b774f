"""CPU tests of the plan builder (csrc/plan.cpp) through the host-only taccl_plan_dump: the
transformations the executor relies on — rrc chain fusion, rrc+send fusion, pull-mode marking
(both sides of a connection must agree), minimal chain dependencies and post-dependency
elision. The GPU parity tests prove the results; these pin the shapes."""
import re

import pytest

from paper_2111_04867_b200 import taccl
from paper_2111_04867_b200.generator import generate

STEP = re.compile(r"\s+(\d+) (\w+) src=(\w+):(\d+) dst=(\w+):(\d+) cnt=(\d+) seq=(\d+) poff=(-?\d+) "
                  r"deps=([\d:,]*) post=([\d:,]*) part=(\d+)/(\d+) fuse=(\d+) fwd=(\d+) pf=(\d+)( prog2?)?")
TB = re.compile(r"tb (\d+) send=(-?\d+) recv=(-?\d+) chan=(\d+) indep=(\d)")


def plan(text, rank, ll=False):
    tbs = []
    for line in taccl.plan_dump(text, rank, ll).splitlines():
        if line.startswith("order"):
            continue
        m = TB.match(line)
        if m:
            tbs.append({"send": int(m[2]), "recv": int(m[3]), "chan": int(m[4]), "steps": []})
            continue
        m = STEP.match(line)
        assert m, line
        tbs[-1]["steps"].append({"op": m[2], "src": (m[3], int(m[4])), "dst": (m[5], int(m[6])), "cnt": int(m[7]),
                                 "seq": int(m[8]), "poff": int(m[9]), "deps": [d for d in m[10].split(",") if d],
                                 "post": [d for d in m[11].split(",") if d], "part": int(m[12]), "nparts": int(m[13]),
                                 "fuse": int(m[14]), "pf": int(m[16]), "prog": 0 if not m[17] else 2 if m[17].endswith("2") else 1})
    return tbs


def test_rs_n2_plain_rrc_is_pulled_on_both_sides():
    text = generate("reducescatter", "direct", 2, 1, 1)
    for r in range(2):
        (tb,) = plan(text, r)
        send, rrc = tb["steps"]
        assert send["op"] == "SEND" and rrc["op"] == "RRC"
        # the receiver reads the peer's input chunk r in place; the sender marks the same send
        assert rrc["poff"] == r and send["poff"] == 1 - r


def test_ar_n2_rrc_fused_with_its_send_and_not_pulled_by_default():
    text = generate("allreduce", "direct", 2, 1, 1)
    (tb,) = plan(text, 0)
    assert [s["op"] for s in tb["steps"]] == ["SEND", "RRCS", "SENT", "RECV"]
    assert all(s["poff"] == -1 for s in tb["steps"])


def test_pull_kinds_env_marks_rrcs_and_chains(monkeypatch):
    monkeypatch.setenv("TACCL_PULL_KINDS", "7")
    (tb,) = plan(generate("allreduce", "direct", 2, 1, 1), 1)
    assert tb["steps"][1]["op"] == "RRCS" and tb["steps"][1]["poff"] == 1 and tb["steps"][0]["poff"] == 0
    tbs = plan(generate("reducescatter", "direct", 4, 1, 1), 2)
    assert all(t["steps"][0]["poff"] >= 0 for t in tbs)   # every chain input pulled -> sends marked


@pytest.mark.parametrize("n", [3, 4, 8])
def test_rs_chain_members_have_no_dependencies_and_no_post_wait(n):
    # all-pairs RS: rank r's n-1 rrcs into o[0] form one chain; nothing conflicting precedes
    # it and nothing follows it, so no member waits on another CTA at all
    tbs = plan(generate("reducescatter", "direct", n, 1, 1), 0)
    members = [t["steps"][1] for t in tbs if len(t["steps"]) > 1]
    assert len(members) == n - 1
    assert all(m["op"] == "RRC_FUSED" and m["fuse"] == n - 1 and m["nparts"] == n - 1 for m in members)
    assert sorted(m["part"] for m in members) == list(range(n - 1))
    assert all(m["deps"] == [] and m["post"] == [] for m in members)


def test_pulled_chain_keeps_post_wait(monkeypatch):
    # with pulled chains (TACCL_PULL_KINDS=7) the last member acks every input for all
    # members, so it must wait for their portions even when nothing follows the chain
    monkeypatch.setenv("TACCL_PULL_KINDS", "7")
    tbs = plan(generate("reducescatter", "direct", 4, 1, 1), 0)
    members = [t["steps"][1] for t in tbs]
    last = max(members, key=lambda m: m["part"])
    assert len(last["post"]) == 2 and all(m["deps"] == [] for m in members)


def test_ar_chain_keeps_post_wait_when_a_send_follows():
    # direct AR: the chain's last member is followed by the AG-phase send of the reduced chunk,
    # so it must still wait for the other members' portions before that send may read o[r]
    tbs = plan(generate("allreduce", "direct", 4, 1, 1), 0)
    members = [(i, t["steps"][1]) for i, t in enumerate(tbs) if t["steps"][1]["op"] == "RRC_FUSED"]
    last = max(members, key=lambda x: x[1]["part"])
    others = sorted(f"{i}:1" for i, _ in members if i != last[0])
    assert sorted(last[1]["post"]) == others
    assert all(m["deps"] == [] for _, m in members)


def test_old_deps_knob_restores_every_incoming_edge(monkeypatch):
    # A/B knob TACCL_CHAIN_OLDDEPS=1 restores "every incoming edge of X_1": the members then
    # wait on X_1's threadblock predecessor (the send) — the edge the trimming removes
    monkeypatch.setenv("TACCL_CHAIN_OLDDEPS", "1")
    tbs = plan(generate("reducescatter", "direct", 4, 1, 1), 0)
    members = [t["steps"][1] for t in tbs]
    assert sum(1 for m in members if m["deps"]) == 2   # the two non-head members
    assert any(m["post"] for m in members)


def test_ring_relays_fuse_recv_copy_send():
    # ring AG at n=4: the relays' receive + forward of the same chunk become one RCS step
    tbs = plan(generate("allgather", "ring", 4, 1, 1), 0)
    ops = [s["op"] for t in tbs for s in t["steps"]]
    assert "RCS" in ops and "SENT" in ops


def test_plan_dump_errors():
    with pytest.raises(taccl.TacclError):
        taccl.plan_dump("<algo", 0)
    with pytest.raises(taccl.TacclError):
        taccl.plan_dump(generate("allgather", "ring", 2, 1, 1), 5)


# ---------------------------------------------------------------- bf16 partials (reading R6)
P_SRC, P_IN, P_KEEP, P_OUT, P_MIX = 1, 2, 4, 8, 16


def test_ring_partial_flags_by_hand():
    # ring AR n=3, rank 0 (generator/templates.py): tb1 receives chunk 2 from rank 1 and
    # reduces it into o[2] (its first rrc: both operands bf16 -> no P_IN / P_SRC); tb0 sends o[2]
    # on to rank 2, whose receive is an rrc -> the send is fp32 (P_OUT) from the shadow that the
    # rrc keeps (P_KEEP). tb1's second rrc (chunk 0) receives rank 1's partial (P_IN); it is
    # fused with the send of the finished chunk to a plain receive: bf16 forward, nothing kept.
    text = generate("allreduce", "ring", 3, 1, 1)
    for ll in (False, True):
        tb0, tb1 = plan(text, 0, ll)
        assert [(x["op"], x["pf"]) for x in tb1["steps"]] == [("RRC", P_KEEP), ("RRCS", P_IN), ("SENT", 0), ("SEND", 0)]
        assert [(x["op"], x["pf"]) for x in tb0["steps"]] == [("SEND", 0), ("SEND", P_OUT), ("RECV", 0), ("RECV", 0)]


def test_relay_and_direct_schedules_carry_no_partials():
    # a reduced value relayed through a plain receive is rounded there; all-pairs (direct)
    # reductions are one fused chain per chunk whose inputs are the peers' inputs
    from conftest import golden
    for text, n in ((golden("rs_relay_n4.xml"), 4), (generate("allreduce", "direct", 4, 1, 1), 4),
                    (generate("allreduce", "oneshot", 4, 1, 1), 4)):
        for r in range(n):
            assert all(x["pf"] == 0 for tb in plan(text, r) for x in tb["steps"])


def test_ring_rs_middle_hops_move_fp32():
    # ring RS n=4: chunk d is reduced along d+1 -> d+2 -> d+3 -> d; every hop after the first
    # sends a partial (P_OUT on the sender, P_IN on the receiving rrc); rrc+send fusions forward
    # their fp32 accumulator directly and keep no shadow
    text = generate("reducescatter", "ring", 4, 1, 1)
    for r in range(4):
        steps = [x for tb in plan(text, r) for x in tb["steps"]]
        ins = [x for x in steps if x["op"] in ("RRC", "RRCS")]
        assert sum(1 for x in ins if x["pf"] & P_IN) == 2  # 3 receive-reduces, the first is bf16
        assert all(x["pf"] & P_OUT for x in steps if x["op"] == "RRCS")
        assert not any(x["pf"] & P_KEEP for x in steps if x["op"] == "RRCS")


PARTIAL_SCHEDS = [("allreduce", "ring", 4, 1, {}), ("allreduce", "ring", 8, 2, {}), ("allreduce", "direct", 4, 2, {}),
                  ("allreduce", "oneshot", 4, 1, {}), ("allreduce", "greedy", 8, 1, {"policy": "uc-min"}),
                  ("allreduce", "greedy", 4, 2, {"policy": "uc-max"}), ("allreduce", "milp", 4, 2, {}),
                  ("reducescatter", "ring", 8, 1, {}), ("reducescatter", "greedy", 8, 2, {}),
                  ("reducescatter", "milp", 8, 1, {"topology": "2x4", "size": 1 << 16}),
                  ("allreduce", "ring", 4, 1, {"pair": "peer"})]


@pytest.mark.parametrize("coll,algo,n,p,kw", PARTIAL_SCHEDS)
def test_static_partial_flags_match_the_oracles_dynamic_rule(coll, algo, n, p, kw, monkeypatch):
    # two independent implementations of reading R6: the plan's last-writer analysis (C++,
    # static, per step) and the oracle's partials mode (Python, dynamic, per message). For
    # every receive-reduce the oracle executes, the operands it read as fp32 partials must be
    # exactly the ones the plan flags (P_SRC: local source; P_IN: the matched send's message)
    import numpy as np
    import oracle
    from oracle import simulate
    from paper_2111_04867_b200.inputs import allreduce_input
    text = generate(coll, algo, n, p, 1, **kw)
    seen = {}
    orig = simulate._execute

    def spy(prog_, graph, order, bufs, read, write, reduce, *rest):
        def red(mine, got, where):
            seen[where] = (mine.part is not None, got.part is not None)
            return reduce(mine, got, where)
        return orig(prog_, graph, order, bufs, read, write, red, *rest)
    monkeypatch.setattr(simulate, "_execute", spy)
    count = n * p * 3 if coll == "allreduce" else p * 3
    e_in = n * count if coll == "reducescatter" else count
    oracle.run(oracle.parse(text), [allreduce_input(e_in, "bfloat16", "uniform", 3, r) for r in range(n)], "bfloat16")
    monkeypatch.setenv("TACCL_NO_FUSE", "1")  # the flags of the original steps, before fusions
    monkeypatch.setenv("TACCL_NO_RRCS", "1")
    assert seen
    for r in range(n):
        for t, tb in enumerate(plan(text, r)):
            for k, x in enumerate(tb["steps"]):
                if x["op"] != "RRC":
                    continue
                src32, in32 = seen[(r, t, k)]
                assert bool(x["pf"] & P_SRC) == src32 and bool(x["pf"] & P_IN) == in32, (r, t, k, x["pf"], seen[(r, t, k)])


@pytest.mark.parametrize("coll,n", [("reducescatter", 4), ("allreduce", 4), ("allreduce", 8), ("reducescatter", 2)])
def test_streamed_marks_split_reduces_and_their_sends(coll, n):
    # split direct (sends and receive-reduces in separate tbs): every chain member is its tb's
    # first step and every input comes from a plain send -> the chain and exactly the sends
    # that feed it stream (seq 0 on each connection); the Allreduce's second phase (plain
    # receives) does not. Paired send+rrc threadblocks stream nothing.
    split, paired = generate(coll, "direct", n, 1, 1, pair=False), generate(coll, "direct", n, 1, 1)
    for r in range(n):
        steps = [x for tb in plan(split, r) for x in tb["steps"]]
        red = [x for x in steps if x["op"] in ("RRC", "RRC_FUSED")]
        assert red and all(x["prog"] for x in red)
        assert all(x["prog"] == (x["seq"] == 0) for x in steps if x["op"] == "SEND")
        assert not any(x["prog"] for x in steps if x["op"] not in ("SEND", "RRC", "RRC_FUSED"))
        assert not any(x["prog"] for tb in plan(paired, r) for x in tb["steps"])


def test_streamed_skips_partials_and_forwarded_messages():
    # ring AR: its receive-reduces carry bf16 partial flags or are fused with their send
    # (K_RRCS), and the sends feeding them are forwards -> nothing streams, split or paired
    for pair in (True, False):
        text = generate("allreduce", "ring", 4, 1, 1, pair=pair)
        for r in range(4):
            assert not any(x["prog"] for tb in plan(text, r) for x in tb["steps"])


ORDER_SCHEDS = [("alltoall", "direct", 4, {}), ("allgather", "ring", 4, {}), ("allreduce", "direct", 8, {}),
                ("allreduce", "ring", 3, {}), ("reducescatter", "direct", 4, {"pair": False}),
                ("allreduce", "dring", 4, {}), ("allgather", "greedy", 8, {}), ("alltoall", "hier", 4, {})]


@pytest.mark.parametrize("coll,algo,n,kw", ORDER_SCHEDS)
def test_merged_order_is_a_level_order(coll, algo, n, kw):
    # merged execution (plan.cpp merged_order): every step exactly once and each threadblock's
    # steps in program order (cross-rank consistency is what the GPU tests exercise: a wrong
    # order deadlocks and surfaces as a watchdog timeout)
    text = generate(coll, algo, n, 1, 1, **kw)
    for r in range(n):
        dump = taccl.plan_dump(text, r)
        order = [tuple(map(int, x.split(":"))) for x in next(l for l in dump.splitlines() if l.startswith("order")).split()[1:]]
        tbs = plan(text, r)
        assert sorted(order) == sorted((t, k) for t, tb in enumerate(tbs) for k in range(len(tb["steps"])))
        for t in range(len(tbs)):
            ks = [k for (tt, k) in order if tt == t]
            assert ks == sorted(ks)


def test_merged_order_puts_a2a_sends_before_receives():
    # all-pairs Alltoall: the three sends (one per peer, level 0) come first, then the receives
    text = generate("alltoall", "direct", 4, 1, 1)
    tbs = plan(text, 0)
    dump = taccl.plan_dump(text, 0)
    order = [tuple(map(int, x.split(":"))) for x in next(l for l in dump.splitlines() if l.startswith("order")).split()[1:]]
    ops = [tbs[t]["steps"][k]["op"] for t, k in order]
    first_recv = ops.index("RECV")
    assert all(o != "RECV" for o in ops[:first_recv]) and all(o in ("RECV", "NOP") for o in ops[first_recv:])


def test_streamed_plain_rrc_is_not_pulled():
    # RS n=2: the paired schedule's plain rrc reads the peer's input in place (pull); the split
    # lowering streams it instead, and then neither end pulls (plan.cpp mark_streamed)
    paired, split = generate("reducescatter", "direct", 2, 1, 1), generate("reducescatter", "direct", 2, 1, 1, pair=False)
    for r in range(2):
        steps = [x for tb in plan(paired, r) for x in tb["steps"]]
        assert any(x["op"] == "RRC" and x["poff"] >= 0 and not x["prog"] for x in steps)
        steps = [x for tb in plan(split, r) for x in tb["steps"]]
        rrc = [x for x in steps if x["op"] == "RRC"]
        send = [x for x in steps if x["op"] == "SEND"]
        assert rrc and all(x["prog"] and x["poff"] == -1 for x in rrc)
        assert send and all(x["prog"] and x["poff"] == -1 for x in send)


def test_overlap_hint_pairs_sends_with_their_receive_reduces(monkeypatch):
    # overlap="1" (docs/SCHEDULE.md): the paired direct schedules' receive-reduces run beside
    # the send before them (prog 2) and their input sends stream; without the hint nothing
    # streams; TACCL_WARPSPEC=0 turns the hint off, =1 forces it on
    monkeypatch.delenv("TACCL_WARPSPEC", raising=False)
    for coll, n in (("reducescatter", 4), ("allreduce", 4), ("reducescatter", 8)):
        hinted, plain = generate(coll, "direct", n, 1, 1, overlap=True), generate(coll, "direct", n, 1, 1)
        assert 'overlap="1"' in hinted and "overlap" not in plain
        red = [x for tb in plan(hinted, 0) for x in tb["steps"] if x["op"] == "RRC_FUSED"]
        assert red and all(x["prog"] == 2 for x in red)
        assert not any(x["prog"] for tb in plan(plain, 0) for x in tb["steps"])
        monkeypatch.setenv("TACCL_WARPSPEC", "0")
        assert not any(x["prog"] == 2 for tb in plan(hinted, 0) for x in tb["steps"])
        monkeypatch.setenv("TACCL_WARPSPEC", "1")
        assert any(x["prog"] == 2 for tb in plan(plain, 0) for x in tb["steps"])
        monkeypatch.delenv("TACCL_WARPSPEC")


def test_overlap_attribute_is_validated_by_both_checkers():
    import oracle
    text = generate("reducescatter", "direct", 4, 1, 1, overlap=True)
    assert oracle.validate(text).ok and taccl.validate(text, True)[0]
    bad = text.replace('overlap="1"', 'overlap="2"')
    assert oracle.validate(bad).kind == "syntax" and taccl.validate(bad, True)[:2] == (False, "syntax")
