"""Schedule checks for the oracle (test infrastructure; see oracle/__init__.py).

Each check restates a rule of the paper or a reading listed in DESIGN.md:

* structure — PAPER.md:742–744 (buffers, equal chunks), 750 ("each threadblock can send to
  and receive from at most one GPU"), 751–752 (dependencies name steps); input read-only
  (NCCL const sendbuff); readings G1, G2.
* match — reading G1: the k-th send on connection (A->B, chan) pairs with the k-th
  receive on B ("split into two instructions for the sender and receiver").
* mr (multicast reduce, the NVLink SHARP step; docs/SCHEDULE.md, reading N1): the
  k-th `mr` of every rank forms group k; member r reduces src[x_r..] over EVERY rank and writes
  the sum to dst[y_r..] of EVERY rank. Every step before any member happens before every
  member, and every member before any step after one (a barrier); its accesses are checked on
  every rank's buffers.
* cycle — steps in a threadblock run sequentially and wait on their dependencies
  (PAPER.md:746–752); a cycle in that relation is a deadlock.
* race — conflicting accesses must be ordered ("dependencies for each
  buffer index are inserted to ensure that the data dependencies ... are honored");
  mode "direct" adds the executor's single-assignment rule (docs/SCHEDULE.md).
* uninit / postcondition — symbolic execution (simulate.run_symbolic) against the
  collective's pre/postcondition (App. B).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

from .collectives import buffer_chunks
from .ef import Program, ScheduleError


@dataclass
class Verdict:
    ok: bool
    kind: str | None = None
    msg: str = ""
    errors: list = field(default_factory=list)


@dataclass
class Graph:
    nodes: list            # list of (rank, tb, step), index = node id
    index: dict            # (rank, tb, step) -> node id
    succ: list             # node id -> list of successor ids
    match: dict            # recv node id -> send node id
    send_to_recv: dict     # send node id -> recv node id
    conns: dict            # (A, B, chan) -> list of (send id, recv id)
    groups: list = field(default_factory=list)  # mr group k -> member node ids (rank order)


# ------------------------------------------------------------------------------ structure

def check_structure(prog: Program):
    errs = []
    n, p = prog.nranks, prog.chunks_per_rank
    n_in, n_out = buffer_chunks(prog.coll, n, p)
    if prog.instances < 1:
        errs.append("instances must be >= 1")
    for g in prog.gpus:
        r = g.id
        if g.i_chunks != n_in or g.o_chunks != n_out:
            errs.append(f"rank {r}: i_chunks/o_chunks = {g.i_chunks}/{g.o_chunks}, "
                        f"{prog.coll} with p={p} needs {n_in}/{n_out} (V5)")
        seen_send, seen_recv = {}, {}
        for tb in g.tbs:
            for peer, what in ((tb.send, "send"), (tb.recv, "recv")):
                if peer != -1 and not (0 <= peer < n):
                    errs.append(f"rank {r} tb {tb.id}: {what} peer {peer} out of range (V1)")
                if peer == r:
                    errs.append(f"rank {r} tb {tb.id}: {what} peer is itself (V1)")
            if tb.chan < 0:
                errs.append(f"rank {r} tb {tb.id}: negative chan")
            if tb.send != -1:
                key = (tb.send, tb.chan)
                if key in seen_send:
                    errs.append(f"rank {r}: tbs {seen_send[key]} and {tb.id} both send to "
                                f"{tb.send} on chan {tb.chan} (V3)")
                seen_send[key] = tb.id
            if tb.recv != -1:
                key = (tb.recv, tb.chan)
                if key in seen_recv:
                    errs.append(f"rank {r}: tbs {seen_recv[key]} and {tb.id} both receive from "
                                f"{tb.recv} on chan {tb.chan} (V3)")
                seen_recv[key] = tb.id
            for st in tb.steps:
                where = f"rank {r} tb {tb.id} step {st.s}"
                if st.type == "s" and tb.send == -1:
                    errs.append(f"{where}: send in a tb with no send peer (V2)")
                if st.type in ("r", "rrc") and tb.recv == -1:
                    errs.append(f"{where}: receive in a tb with no recv peer (V2)")
                if st.type != "nop" and st.cnt < 1:
                    errs.append(f"{where}: cnt must be >= 1")
                if st.type == "mr" and (tb.send != -1 or tb.recv != -1):
                    errs.append(f"{where}: multicast reduce in a tb with a peer (its peer is the switch)")
                if st.type == "mr" and prog.coll not in ("allreduce", "reducescatter"):
                    errs.append(f"{where}: multicast reduce in a non-reducing collective")
                if st.dstbuf == "i":
                    errs.append(f"{where}: writes the input buffer (read-only)")
                for buf, off in ((st.srcbuf, st.srcoff), (st.dstbuf, st.dstoff)):
                    if buf is not None and off + st.cnt > g.nchunks(buf):
                        errs.append(f"{where}: {buf}[{off}:{off + st.cnt}] exceeds "
                                    f"{g.nchunks(buf)} chunks (V4)")
                for (t, k) in st.deps:
                    if t >= len(g.tbs) or k >= len(g.tbs[t].steps):
                        errs.append(f"{where}: dependency {t}:{k} does not exist (V6)")
                    elif t == tb.id and k == st.s:
                        errs.append(f"{where}: depends on itself (V6)")
    return errs


# ------------------------------------------------------------------------------ graph

def build_graph(prog: Program) -> Graph:
    """Nodes, program-order + dependency + matching edges. Raises ScheduleError('match')."""
    nodes, index = [], {}
    for g in prog.gpus:
        for tb in g.tbs:
            for st in tb.steps:
                index[(g.id, tb.id, st.s)] = len(nodes)
                nodes.append((g.id, tb.id, st.s))
    succ = [[] for _ in nodes]
    for g in prog.gpus:
        for tb in g.tbs:
            for st in tb.steps:
                v = index[(g.id, tb.id, st.s)]
                if st.s > 0:
                    succ[index[(g.id, tb.id, st.s - 1)]].append(v)
                for (t, k) in st.deps:
                    succ[index[(g.id, t, k)]].append(v)
    # connections: (A, B, chan) -> ordered send / recv lists (reading G1)
    sends, recvs = {}, {}
    for g in prog.gpus:
        for tb in g.tbs:
            for st in tb.steps:
                if st.type == "s":
                    sends.setdefault((g.id, tb.send, tb.chan), []).append((g.id, tb.id, st.s))
                elif st.type in ("r", "rrc"):
                    recvs.setdefault((tb.recv, g.id, tb.chan), []).append((g.id, tb.id, st.s))
    match, send_to_recv, conns = {}, {}, {}
    for key in sorted(set(sends) | set(recvs)):
        ss, rr = sends.get(key, []), recvs.get(key, [])
        a, b, c = key
        if len(ss) != len(rr):
            raise ScheduleError("match", f"connection {a}->{b} chan {c}: {len(ss)} sends vs "
                                         f"{len(rr)} receives")
        pairs = []
        for q, (s, r) in enumerate(zip(ss, rr)):
            cs = prog.gpus[s[0]].tbs[s[1]].steps[s[2]].cnt
            cr = prog.gpus[r[0]].tbs[r[1]].steps[r[2]].cnt
            if cs != cr:
                raise ScheduleError("match", f"connection {a}->{b} chan {c} message {q}: send "
                                             f"cnt {cs} vs receive cnt {cr}")
            si, ri = index[s], index[r]
            succ[si].append(ri)
            match[ri] = si
            send_to_recv[si] = ri
            pairs.append((si, ri))
        conns[key] = pairs
    # multicast reduce groups: the k-th mr step of every rank (in tb, step order)
    mrs = [[index[(g.id, tb.id, st.s)] for tb in g.tbs for st in tb.steps if st.type == "mr"] for g in prog.gpus]
    groups = []
    if any(mrs):
        if len({len(m) for m in mrs}) != 1:
            raise ScheduleError("match", "multicast reduce: ranks have " + "/".join(str(len(m)) for m in mrs)
                                + " mr steps")
        pred = {v: [] for v in range(len(nodes))}
        for u, vs in enumerate(succ):
            for v in vs:
                pred[v].append(u)
        out = [list(vs) for vs in succ]
        for k in range(len(mrs[0])):
            members = [m[k] for m in mrs]
            cnts = {prog.gpus[nodes[v][0]].tbs[nodes[v][1]].steps[nodes[v][2]].cnt for v in members}
            if len(cnts) != 1:
                raise ScheduleError("match", f"multicast reduce group {k}: cnt differs across ranks")
            for q in members:  # a barrier: preds of any member -> every member -> succs of any
                for r in members:
                    if r != q:
                        succ[r].extend(x for x in out[q] if x not in members)
                        for x in pred[q]:
                            if x not in members:
                                succ[x].append(r)
            groups.append(members)
    return Graph(nodes, index, succ, match, send_to_recv, conns, groups)


def topo_order(graph: Graph):
    """Deterministic Kahn order, ties broken by (rank, tb, step). Raises ScheduleError('cycle')."""
    indeg = [0] * len(graph.nodes)
    for vs in graph.succ:
        for v in vs:
            indeg[v] += 1
    heap = [(graph.nodes[v], v) for v in range(len(graph.nodes)) if indeg[v] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        _, u = heapq.heappop(heap)
        order.append(u)
        for v in graph.succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                heapq.heappush(heap, (graph.nodes[v], v))
    if len(order) != len(graph.nodes):
        raise ScheduleError("cycle", "deadlock: " + _describe_cycle(graph, indeg))
    return order


def _describe_cycle(graph: Graph, indeg):
    """Walk predecessors among the unsorted nodes until one repeats; name that cycle."""
    left = {v for v in range(len(graph.nodes)) if indeg[v] > 0}
    pred = {v: [] for v in left}
    for u in left:
        for v in graph.succ[u]:
            if v in left:
                pred[v].append(u)
    v = min(left, key=lambda x: graph.nodes[x])
    seen, path = {}, []
    while v not in seen:
        seen[v] = len(path)
        path.append(v)
        v = min(pred[v], key=lambda x: graph.nodes[x])
    cyc = list(reversed(path[seen[v]:]))
    return " -> ".join("r%d:tb%d:s%d" % graph.nodes[x] for x in cyc + [cyc[0]])


def reachability(graph: Graph, order):
    """desc[v] = bitset (python int) of nodes reachable from v by >= 1 edge."""
    desc = [0] * len(graph.nodes)
    for u in reversed(order):
        m = 0
        for v in graph.succ[u]:
            m |= desc[v] | (1 << v)
        desc[u] = m
    return desc


# ------------------------------------------------------------------------------ races

def _accesses(prog: Program, graph: Graph, mode: str):
    """(rank, buf, lo, hi, is_write, start node, end node, node) per access."""
    acc = []
    for g in prog.gpus:
        for tb in g.tbs:
            for st in tb.steps:
                v = graph.index[(g.id, tb.id, st.s)]
                if st.type == "mr":  # reads and writes the same ranges on every rank
                    for q in range(prog.nranks):
                        acc.append((q, st.srcbuf, st.srcoff, st.srcoff + st.cnt, False, v, v, v))
                        acc.append((q, st.dstbuf, st.dstoff, st.dstoff + st.cnt, True, v, v, v))
                    continue
                if st.srcbuf is not None:
                    acc.append((g.id, st.srcbuf, st.srcoff, st.srcoff + st.cnt, False, v, v, v))
                if st.dstbuf is not None:
                    start = v
                    if st.type == "r" and mode == "direct":
                        start = graph.match[v]  # bytes land while the peer's send runs
                    acc.append((g.id, st.dstbuf, st.dstoff, st.dstoff + st.cnt, True, start, v, v))
    return acc


def check_races(prog: Program, graph: Graph, desc, mode: str = "direct"):
    """Conflicting accesses a, b (same rank/buffer, overlapping, one writes, different steps)
    must satisfy end(a) ->hb start(b) or end(b) ->hb start(a)."""
    acc = _accesses(prog, graph, mode)
    by_key = {}
    for a in acc:
        by_key.setdefault((a[0], a[1]), []).append(a)
    for (rank, buf), lst in sorted(by_key.items()):
        for i in range(len(lst)):
            a = lst[i]
            for j in range(i + 1, len(lst)):
                b = lst[j]
                if a[7] == b[7] or not (a[4] or b[4]):
                    continue
                if a[3] <= b[2] or b[3] <= a[2]:
                    continue
                if (desc[a[6]] >> b[5]) & 1 or (desc[b[6]] >> a[5]) & 1:
                    continue
                na, nb = graph.nodes[a[7]], graph.nodes[b[7]]
                lo, hi = max(a[2], b[2]), min(a[3], b[3])
                raise ScheduleError("race", f"rank {rank} {buf}[{lo}:{hi}]: steps "
                                            f"tb{na[1]}:s{na[2]} and tb{nb[1]}:s{nb[2]} "
                                            f"are unordered")


# ------------------------------------------------------------------------------ verdict

def validate(prog_or_text, mode: str = "direct") -> Verdict:
    """All checks in the order of docs/SCHEDULE.md; the first failing class is the verdict."""
    from .ef import parse
    from .simulate import run_symbolic
    try:
        prog = parse(prog_or_text) if isinstance(prog_or_text, str) else prog_or_text
        errs = check_structure(prog)
        if errs:
            return Verdict(False, "structure", errs[0], errs)
        graph = build_graph(prog)
        order = topo_order(graph)
        desc = reachability(graph, order)
        check_races(prog, graph, desc, mode)
        run_symbolic(prog, graph=graph, order=order)
    except ScheduleError as e:
        return Verdict(False, e.kind, e.msg, [e.msg])
    return Verdict(True)
