"""Lowering an abstract algorithm to EF v1 text (§6.2).

The passes, in the paper's order:

* Buffer allocation: user input/output, runtime scratch; chunks are
  indices into them; a rank's own chunks are copied input -> output "at the end" (one
  `cpy` threadblock that runs concurrently, reading G9).
* Contiguity: final deliveries on the same link are merged into one
  multi-chunk transfer (`coalesce`), so they become one cnt > 1 step.
* Instruction generation: every transfer becomes a send on the sender and
  a receive (`r`, or `rrc` when it reduces) on the receiver, on concrete buffer indices.
  Transfers of several chunks stay one instruction (`cnt > 1`) when both sides are
  contiguous; otherwise they are split into contiguous runs.
* Dependency insertion: per buffer index, a step depends on the last
  writer of what it reads and, when it writes, on the last writer and every reader since
  (only cross-threadblock edges are emitted; program order covers the rest).
* Threadblock allocation: each threadblock sends to at most one GPU and
  receives from at most one GPU; steps keep the abstract order. Relay hops first: the peer a
  rank receives chunks from and the peer it forwards them to (at least two such hops) share
  a threadblock, so receive and forward are adjacent steps (fused by the executor); then a
  peer that is both sent to and received from shares one threadblock; leftover send-only and
  receive-only peers are paired in order of first use (a ring lands in one threadblock).
* Instances: written as the header's `instances`; the executor runs the
  m copies (docs/SCHEDULE.md).
"""
from __future__ import annotations

import math

from .algorithm import Algorithm, Transfer, a2a_parts


class LoweringError(Exception):
    pass


def _initial(alg: Algorithm, r: int):
    """rank r's starting location of each chunk it holds (precondition)."""
    n, p = alg.nranks, alg.chunks_per_rank
    if alg.coll == "allgather":
        return {r * p + k: ("i", k) for k in range(p)}
    if alg.coll == "alltoall":
        return {(r * n + d) * p + k: ("i", d * p + k) for d in range(n) for k in range(p)}
    return {k: ("i", k) for k in range(n * p)}  # allreduce, reducescatter


def coalesce(alg: Algorithm) -> Algorithm:
    """Contiguity for the executor (§5.1: chunks sent consecutively over a link
    can be sent together, saving a per-transfer latency). On B200 one executor step costs ~2-4 us
    of flag round trips and CTA work at small sizes (the paper's alpha regime), so transfers on the
    same link are merged into one multi-chunk transfer when that loses no pipelining:
      * both deliver their chunks to their final holder (the receiver forwards none of them:
        a forward's timing could be delayed) and both reduce or neither does;
      * the later one's chunks are already at the sender (strictly) before the earlier one is
        sent, so waiting for them delays nothing.
    The merged transfer leaves at the earlier send time and arrives at the later arrival.
    Lowering then emits it as one cnt > 1 step where both sides are contiguous (_runs)."""
    arrivals, sends = {}, {}  # (rank, chunk) -> arrival times at / send times from the rank
    for t in alg.transfers:
        for c in t.chunks:
            arrivals.setdefault((t.dst, c), []).append(t.arrive_time)
            sends.setdefault((t.src, c), []).append(t.send_time)

    def forwarded(r, c, after):  # the rank sends chunk c (e.g. a partial sum) once it arrived
        return any(x >= after for x in sends.get((r, c), []))

    def ready(r, c, at, by):  # every delivery of c to r before `by` was there before `at`
        return all(x < at for x in arrivals.get((r, c), []) if x <= by)

    out = Algorithm(alg.name, alg.coll, alg.nranks, alg.chunks_per_rank)
    groups = {}  # (src, dst) -> index of the open merged transfer in out.transfers
    for t in sorted(alg.transfers, key=lambda t: (t.send_time, t.src, t.dst)):
        final = not any(forwarded(t.dst, c, t.arrive_time) for c in t.chunks)
        g = groups.get((t.src, t.dst, t.reduce)) if final else None
        if g is not None and all(ready(t.src, c, out.transfers[g].send_time, t.send_time) for c in t.chunks):
            m = out.transfers[g]
            out.transfers[g] = Transfer(tuple(sorted(m.chunks + t.chunks)), m.src, m.dst, m.send_time,
                                        max(m.arrive_time, t.arrive_time), t.reduce)
            continue
        out.transfers.append(t)
        if final:
            groups[(t.src, t.dst, t.reduce)] = len(out.transfers) - 1
    return out


def _dst_locations(alg: Algorithm):
    """Destination (buf, idx) of every chunk of every transfer; allocates scratch."""
    n, p = alg.nranks, alg.chunks_per_rank
    scratch = [dict() for _ in range(n)]
    out = []
    for t in alg.transfers:
        locs = []
        for c in t.chunks:
            if alg.coll == "allgather":
                locs.append(("o", c))
            elif alg.coll == "allreduce":
                locs.append(("o", c))
            elif alg.coll == "reducescatter":
                # the owner (c // p) reduces into its output; relays keep partials in scratch
                if t.dst == c // p:
                    locs.append(("o", c % p))
                else:
                    sl = scratch[t.dst].setdefault(c, len(scratch[t.dst]))
                    locs.append(("s", sl))
            else:
                s, d, k = a2a_parts(c, n, p)
                if t.dst == d:
                    locs.append(("o", s * p + k))
                else:
                    sl = scratch[t.dst].setdefault(c, len(scratch[t.dst]))
                    locs.append(("s", sl))
        out.append(locs)
    return out, [len(s) for s in scratch]


def _runs(*lists):
    """Split parallel location lists into maximal runs contiguous in every list."""
    runs, start, m = [], 0, len(lists[0])
    for q in range(1, m + 1):
        if q == m or not all(l[q][0] == l[q - 1][0] and l[q][1] == l[q - 1][1] + 1 for l in lists):
            runs.append((start, q))
            start = q
    return runs


def _instructions(alg: Algorithm):
    """Per-rank ordered instruction lists (dicts)."""
    n = alg.nranks
    dst_locs, n_scratch = _dst_locations(alg)
    events = [[] for _ in range(n)]
    for i, t in enumerate(alg.transfers):
        events[t.src].append((t.send_time, 1, i))
        events[t.dst].append((t.arrive_time, 0, i))   # a receive at T precedes a send at T
    for ev in events:
        ev.sort()
    # locations evolve per rank in event order; a transfer's source side needs the sender's
    # state at send time and an rrc's local source needs the receiver's state at arrival.
    cur = [_initial(alg, r) for r in range(n)]
    src_locs = [None] * len(alg.transfers)
    rrc_src = [None] * len(alg.transfers)
    # walk all events in global time order so a receive updates the receiver's state before
    # any later send reads it
    merged = sorted((e[0], e[1], e[2], r) for r in range(n) for e in events[r])
    for time, kind, i, r in merged:
        t = alg.transfers[i]
        if kind == 1:
            missing = [c for c in t.chunks if c not in cur[r]]
            if missing:
                raise LoweringError(f"rank {r} sends chunk {missing[0]} it does not hold at t={time}")
            src_locs[i] = [cur[r][c] for c in t.chunks]
        else:
            if t.reduce:
                missing = [c for c in t.chunks if c not in cur[r]]
                if missing:
                    raise LoweringError(f"rank {r} reduces chunk {missing[0]} it does not hold")
                rrc_src[i] = [cur[r][c] for c in t.chunks]
            for c, loc in zip(t.chunks, dst_locs[i]):
                cur[r][c] = loc
    instrs = [[] for _ in range(n)]
    for r in range(n):
        for time, kind, i in events[r]:
            t = alg.transfers[i]
            lists = [src_locs[i], dst_locs[i]] + ([rrc_src[i]] if t.reduce else [])
            for x, y in _runs(*lists):
                cnt = y - x
                if kind == 1:
                    instrs[r].append(dict(type="s", peer=t.dst, src=src_locs[i][x], cnt=cnt,
                                          xfer=(i, x)))
                elif t.reduce:
                    instrs[r].append(dict(type="rrc", peer=t.src, src=rrc_src[i][x],
                                          dst=dst_locs[i][x], cnt=cnt, xfer=(i, x)))
                else:
                    instrs[r].append(dict(type="r", peer=t.src, dst=dst_locs[i][x], cnt=cnt,
                                          xfer=(i, x)))
    # own chunks: input -> output copy "at the end"
    p = alg.chunks_per_rank
    for r in range(n):
        if alg.coll == "allgather":
            instrs[r].append(dict(type="cpy", peer=-1, src=("i", 0), dst=("o", r * p), cnt=p))
        elif alg.coll == "alltoall":
            instrs[r].append(dict(type="cpy", peer=-1, src=("i", r * p), dst=("o", r * p), cnt=p))
        elif n == 1:  # one rank: the reduction of one contribution is a copy
            instrs[r].append(dict(type="cpy", peer=-1, src=("i", 0),
                                  dst=("o", 0), cnt=p))
    return instrs, n_scratch


def _check_pairing(instrs):
    """Both sides of a transfer must be split into the same runs (checked, not assumed)."""
    sends, recvs = {}, {}
    for r, lst in enumerate(instrs):
        for ins in lst:
            if ins["type"] == "s":
                sends[ins["xfer"]] = ins["cnt"]
            elif ins["type"] in ("r", "rrc"):
                recvs[ins["xfer"]] = ins["cnt"]
    if sends != recvs:
        raise LoweringError("sender and receiver split a transfer differently")


def _allocate_tbs(lst, pair=True):
    """Threadblock allocation: returns [(send, recv)] and per-instr tb.
    pair=False keeps sends and receives in separate threadblocks (so a reducing receive
    never stalls the same CTA's sends; used for reduce-scatter)."""
    send_peers, recv_peers = [], []
    for ins in lst:
        if ins["type"] == "s" and ins["peer"] not in send_peers:
            send_peers.append(ins["peer"])
        if ins["type"] in ("r", "rrc") and ins["peer"] not in recv_peers:
            recv_peers.append(ins["peer"])
    tbs, by_send, by_recv = [], {}, {}
    # relays first: a receive from q whose chunks the next instruction sends on to q' (a ring's
    # or a relay path's hop) shares a threadblock with the sends to q', so the two steps are
    # adjacent and the executor runs them as one pass (recv-copy-send / recv-reduce-copy-send,
    # SURVEY.md §8(f) row 1); pairs with the most such hops first, each peer in one pair
    if pair and pair != "peer":  # pair="peer": the same-peer pairing alone (A/B measurements)
        hops = {}
        for a, b in zip(lst, lst[1:]):
            if a["type"] in ("r", "rrc") and b["type"] == "s" and b["src"] == a["dst"] and b["cnt"] == a["cnt"]:
                hops[(a["peer"], b["peer"])] = hops.get((a["peer"], b["peer"]), 0) + 1
        for (qr, qs), c in sorted(hops.items(), key=lambda kv: (-kv[1], kv[0])):
            if qr in by_recv or qs in by_send or c < 2:
                continue
            by_send[qs] = by_recv[qr] = len(tbs)
            tbs.append((qs, qr))
    for q in send_peers:
        if pair and q in recv_peers and q not in by_send and q not in by_recv:
            by_send[q] = by_recv[q] = len(tbs)
            tbs.append((q, q))
    ls = [q for q in send_peers if q not in by_send]
    lr = [q for q in recv_peers if q not in by_recv]
    if not pair:
        for q in ls:
            by_send[q] = len(tbs)
            tbs.append((q, -1))
        for q in lr:
            by_recv[q] = len(tbs)
            tbs.append((-1, q))
        ls, lr = [], []
    for j in range(max(len(ls), len(lr))):
        s = ls[j] if j < len(ls) else -1
        rr = lr[j] if j < len(lr) else -1
        if s != -1:
            by_send[s] = len(tbs)
        if rr != -1:
            by_recv[rr] = len(tbs)
        tbs.append((s, rr))
    copy_tb = None
    assign = []
    for ins in lst:
        if ins["type"] == "s":
            assign.append(by_send[ins["peer"]])
        elif ins["type"] in ("r", "rrc"):
            assign.append(by_recv[ins["peer"]])
        else:
            if copy_tb is None:
                copy_tb = len(tbs)
                tbs.append((-1, -1))
            assign.append(copy_tb)
    return tbs, assign


def _ranges(ins):
    reads, writes = [], []
    if "src" in ins:
        b, o = ins["src"]
        reads = [(b, o + q) for q in range(ins["cnt"])]
    if "dst" in ins:
        b, o = ins["dst"]
        writes = [(b, o + q) for q in range(ins["cnt"])]
    return reads, writes


def lower(alg: Algorithm, instances: int = 1, min_bytes=0, max_bytes=math.inf, name=None, pair=True,
          merge=True, dtypes=None, overlap=False) -> str:
    """Lower `alg` to EF v1 text (docs/SCHEDULE.md). pair: share one threadblock between the
    send to and the receive from the same peer (see _allocate_tbs); merge: coalesce final
    deliveries on a link into multi-chunk transfers (see coalesce)."""
    if instances < 1:
        raise LoweringError("instances must be >= 1")
    if merge:
        alg = coalesce(alg)
    n, p = alg.nranks, alg.chunks_per_rank
    instrs, n_scratch = _instructions(alg)
    _check_pairing(instrs)
    n_in, n_out = {"allgather": (p, n * p), "reducescatter": (n * p, p)}.get(alg.coll, (n * p, n * p))
    mx = "inf" if max_bytes == math.inf else str(int(max_bytes))
    out = [f'<algo name="{name or alg.name}" coll="{alg.coll}" nranks="{n}" chunks_per_rank="{p}" '
           f'instances="{instances}" minBytes="{int(min_bytes)}" maxBytes="{mx}" inplace="0"'
           + (f' dtypes="{",".join(dtypes)}"' if dtypes else "") + (' overlap="1"' if overlap else "") + '>']
    for r in range(n):
        lst = instrs[r]
        tbs, assign = _allocate_tbs(lst, pair)
        steps = [[] for _ in tbs]
        state = {}  # (buf, idx) -> (last writer (tb, k) or None, readers [(tb, k)])
        for ins, t in zip(lst, assign):
            k = len(steps[t])
            reads, writes = _ranges(ins)
            deps = {}
            for loc in reads:
                w, _ = state.get(loc, (None, []))
                if w is not None and w[0] != t:
                    deps[w[0]] = max(deps.get(w[0], -1), w[1])
            for loc in writes:
                w, rd = state.get(loc, (None, []))
                for x in ([w] if w is not None else []) + rd:
                    if x[0] != t:
                        deps[x[0]] = max(deps.get(x[0], -1), x[1])
            for loc in reads:
                w, rd = state.get(loc, (None, []))
                state[loc] = (w, rd + [(t, k)])
            for loc in writes:
                state[loc] = ((t, k), [])
            steps[t].append((ins, sorted(deps.items())))
        out.append(f' <gpu id="{r}" i_chunks="{n_in}" o_chunks="{n_out}" s_chunks="{n_scratch[r]}">')
        for t, (sp, rp) in enumerate(tbs):
            out.append(f'  <tb id="{t}" send="{sp}" recv="{rp}" chan="0">')
            for k, (ins, deps) in enumerate(steps[t]):
                a = [f's="{k}"', f'type="{ins["type"]}"']
                if "src" in ins:
                    a += [f'srcbuf="{ins["src"][0]}"', f'srcoff="{ins["src"][1]}"']
                if "dst" in ins:
                    a += [f'dstbuf="{ins["dst"][0]}"', f'dstoff="{ins["dst"][1]}"']
                a.append(f'cnt="{ins["cnt"]}"')
                a.append('deps="' + ",".join(f"{dt}:{dk}" for dt, dk in deps) + '"')
                out.append("   <step " + " ".join(a) + "/>")
            out.append("  </tb>")
        out.append(" </gpu>")
    out.append("</algo>")
    return "\n".join(out) + "\n"
