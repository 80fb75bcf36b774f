"""TACCL's three-stage synthesizer with real MILPs (App. B).

The paper solves Stages 1 and 3 with Gurobi; here they are the same encodings solved by
HiGHS through `scipy.optimize.milp` (offline, CPU, not on the timed path). Stage 2 is the
paper's greedy ordering heuristic, shared with the greedy stand-in (`greedy.order`).

* Stage 1 — routing (App. B.1). Variables time, start[c,r], send[c,u,v],
  is_sent[c,u,v], is_util[u,v]. Objective time + gamma * sum(is_util) over switched links
  (gamma < 0 for uc-max, > 0 for uc-min, eq. uc). Constraints: time >= start on the
  postcondition; start = 0 on the precondition; send >= start at the sender (eq. corr);
  is_sent -> start[c,v] = send[c,u,v] + lat(u,v) (eq. relbw, big-M); the relaxed bandwidth
  bounds per link (eq. link1) and per switch port (eq. switch1s1 / switch1r1); is_util
  bounds (eq. and1/and2); rotational symmetry (start, send, is_sent equal on symmetric
  images); at least one inter-node link for chunks that cross nodes; the sketch's
  chunk-to-relay map (inter-node sends of a chunk leave from its relay).
* Stage 2 — heuristic ordering (App. B.2): greedy.order on the Stage-1
  trees, without merging; yields chunk_order per link and the switch send/recv orders.
* Stage 3 — contiguity and exact scheduling (App. B.3). Paths and
  orders fixed; variables send, start, time, is_together[c,o,link]. lat[c,link] =
  alpha + beta * (1 + sum_o is_together[c,o]); start[c,v] = send + lat; is_together ->
  equal send times; not is_together -> strict link order (send[o] >= send[c] + lat[c] for
  o after c); switch ports send to / receive from one switched peer at a time in the
  Stage-2 order.

Readings where App. B is silent ("leaving out other less important constraints",
PAPER.md:1490), listed in DESIGN.md §2 as M1–M4:
  M1 flow: a chunk is sent from u only if it started at u or was sent to u, and every
     postcondition rank receives it (without these, start of an absent chunk is free);
  M2 big-M horizon H = (#chunks + n) * max lat (a sequential schedule always fits);
  M3 is_together is transitive within a link, and symmetric (one variable per pair);
  M4 Stage-1 duplicate receptions are pruned to the in-edge that defines start[c,v].
"""
from __future__ import annotations

import math

import numpy as np

from .algorithm import Algorithm
from .topology import Sketch, apply_sketch, multinode, nvswitch, relay_for_chunk, rotate
from . import greedy, templates


class _Model:
    """A small sparse MILP builder over scipy.optimize.milp (HiGHS)."""

    def __init__(self):
        self.lb, self.ub, self.integ, self.obj = [], [], [], []
        self.rows, self.cols, self.vals, self.clb, self.cub = [], [], [], [], []
        self.nrows = 0

    def var(self, lb=0.0, ub=math.inf, integer=False, obj=0.0):
        self.lb.append(lb)
        self.ub.append(ub)
        self.integ.append(1 if integer else 0)
        self.obj.append(obj)
        return len(self.lb) - 1

    def binary(self, obj=0.0):
        return self.var(0.0, 1.0, True, obj)

    def cons(self, terms, lb=-math.inf, ub=math.inf):
        """lb <= sum(coef * x[var]) <= ub; terms: [(var, coef)]"""
        for v, a in terms:
            self.rows.append(self.nrows)
            self.cols.append(v)
            self.vals.append(a)
        self.clb.append(lb)
        self.cub.append(ub)
        self.nrows += 1

    def solve(self, time_limit=60.0, gap=1e-6):
        from scipy.optimize import Bounds, LinearConstraint, milp
        from scipy.sparse import coo_matrix
        nv = len(self.lb)
        cons = []
        if self.nrows:
            A = coo_matrix((self.vals, (self.rows, self.cols)), shape=(self.nrows, nv)).tocsr()
            cons.append(LinearConstraint(A, np.array(self.clb), np.array(self.cub)))
        res = milp(np.array(self.obj), constraints=cons, integrality=np.array(self.integ),
                   bounds=Bounds(np.array(self.lb), np.array(self.ub)),
                   options={"time_limit": time_limit, "mip_rel_gap": gap, "disp": False})
        if res.x is None:
            raise RuntimeError(f"MILP failed: {res.message}")
        return res


def _switched(lt):
    sw = set()
    for s in lt.switches:
        for a in s:
            for b in s:
                if a != b and (a, b) in lt.links:
                    sw.add((a, b))
    return sw


def _rot_chunk(coll, c, n, p, o, g):
    return greedy._rot_chunk(coll, c, n, p, o, g)


# ---------------------------------------------------------------------------- Stage 1

def route(coll, lt, sk: Sketch, chunks, chunk_mb, time_limit=60.0, gamma=None):
    """Stage 1 (App. B.1): {chunk: [(u, v), ...]} (parents before children), the relaxed
    optimum `time` and the MILP status. chunks: [(c, src, [dst, ...])]."""
    n = lt.n
    p = sk.input_chunkup
    links = sorted(lt.links)
    lat = {l: lt.links[l].cost(chunk_mb) for l in links}
    maxlat = max(lat.values())
    H = (len(chunks) + n) * maxlat  # M2
    switched = _switched(lt)
    # shortest-path restriction: chunk c may use (u, v) only if it lies on
    # a shortest (latency) path from c's source to one of its destinations, over the links the
    # sketch leaves that chunk (the relay map removes inter-node links not leaving its relay)
    def relay_ok(s, u, v):
        return not sk.chunk_to_relay or lt.node_of[u] == lt.node_of[v] or u == relay_for_chunk(sk, s)
    dists = {}
    for s0 in range(n):
        d = [[0.0 if a == b else math.inf for b in range(n)] for a in range(n)]
        for (u, v) in links:
            if relay_ok(s0, u, v):
                d[u][v] = min(d[u][v], lat[(u, v)])
        for k in range(n):
            for a in range(n):
                for b in range(n):
                    if d[a][k] + d[k][b] < d[a][b]:
                        d[a][b] = d[a][k] + d[k][b]
        dists[s0] = d

    def on_shortest(s, ds, u, v):
        d, tol = dists[s], 1e-9 * max(1.0, maxlat)
        return relay_ok(s, u, v) and any(abs(d[s][u] + lat[(u, v)] + d[v][t] - d[s][t]) <= tol for t in ds)
    if gamma is None:  # small against any latency: time dominates, util breaks ties (eq. uc)
        gamma = 1e-3 * min(lat.values()) / max(1, len(switched))
        gamma = -gamma if sk.policy == "uc-max" else gamma
    m = _Model()
    T = m.var(0.0, H, obj=1.0)
    src_of = {c: s for c, s, _ in chunks}
    dsts_of = {c: set(d) for c, _, d in chunks}
    start = {(c, r): m.var(0.0, H) for c, _, _ in chunks for r in range(n)}
    send, x = {}, {}
    for c, s, _ in chunks:
        for l in links:
            u, v = l
            forbidden = v == s or not on_shortest(s, dsts_of[c], u, v)
            send[(c, l)] = m.var(0.0, H)
            x[(c, l)] = m.var(0.0, 0.0 if forbidden else 1.0, True)
    for c, s, ds in chunks:
        m.cons([(start[(c, s)], 1.0)], 0.0, 0.0)                     # precondition
        for d in ds:
            m.cons([(T, 1.0), (start[(c, d)], -1.0)], 0.0)           # time >= start (post)
        for l in links:
            u, v = l
            m.cons([(send[(c, l)], 1.0), (start[(c, u)], -1.0)], 0.0)  # eq. corr
            # eq. relbw: x -> start[c,v] - send[c,l] = lat, as two big-M rows
            m.cons([(start[(c, v)], 1.0), (send[(c, l)], -1.0), (x[(c, l)], H)], -math.inf, lat[l] + H)
            m.cons([(start[(c, v)], 1.0), (send[(c, l)], -1.0), (x[(c, l)], -H)], lat[l] - H)
        # M1 flow
        for v in range(n):
            if v == s:
                continue
            ins = [(x[(c, (u, v))], 1.0) for u in range(n) if (u, v) in lt.links]
            if v in ds:
                m.cons(ins, 1.0)
            for w in range(n):
                if (v, w) in lt.links:
                    m.cons([(x[(c, (v, w))], 1.0)] + [(xv, -1.0) for xv, _ in ins], -math.inf, 0.0)
        # inter-node transfer constraint (App. B.1 last equation)
        for d in ds:
            if lt.node_of[d] != lt.node_of[s]:
                cross = [(x[(c, l)], 1.0) for l in links
                         if lt.node_of[l[0]] == lt.node_of[s] and lt.node_of[l[1]] == lt.node_of[d]]
                m.cons(cross, 1.0)
    # relaxed bandwidth: per link (eq. link1), per switch send / recv port (eq. switch1s1/r1)
    for l in links:
        m.cons([(T, 1.0)] + [(x[(c, l)], -lat[l]) for c, _, _ in chunks], 0.0)
    for r in range(n):
        outs = [l for l in switched if l[0] == r]
        ins_ = [l for l in switched if l[1] == r]
        if outs:
            m.cons([(T, 1.0)] + [(x[(c, l)], -lat[l]) for c, _, _ in chunks for l in outs], 0.0)
        if ins_:
            m.cons([(T, 1.0)] + [(x[(c, l)], -lat[l]) for c, _, _ in chunks for l in ins_], 0.0)
    # is_util (eq. and1 / and2) and its objective weight (eq. uc)
    for l in sorted(switched):
        util = m.binary(obj=gamma)
        for c, _, _ in chunks:
            m.cons([(util, 1.0), (x[(c, l)], -1.0)], 0.0)
        m.cons([(util, 1.0)] + [(x[(c, l)], -1.0) for c, _, _ in chunks], -math.inf, 0.0)
    # rotational symmetry (App. B.1): images share start, send and is_sent
    ids = {c for c, _, _ in chunks}
    for (o, g) in sk.symmetry_offsets:
        for c, _, _ in chunks:
            c2 = _rot_chunk(coll, c, n, p, o, g)
            if c2 not in ids or c2 == c:
                continue
            for r in range(n):
                m.cons([(start[(c, r)], 1.0), (start[(c2, rotate(r, o, g))], -1.0)], 0.0, 0.0)
            for l in links:
                l2 = (rotate(l[0], o, g), rotate(l[1], o, g))
                if l2 in lt.links:
                    m.cons([(send[(c, l)], 1.0), (send[(c2, l2)], -1.0)], 0.0, 0.0)
                    m.cons([(x[(c, l)], 1.0), (x[(c2, l2)], -1.0)], 0.0, 0.0)
    res = m.solve(time_limit)
    xs = res.x
    trees = {}
    for c, s, ds in chunks:
        st = {r: xs[start[(c, r)]] for r in range(n)}
        # M4: one in-edge per reached rank — the one whose arrival defines start[c,v]
        inedge = {}
        for l in links:
            if xs[x[(c, l)]] > 0.5:
                u, v = l
                err = abs(xs[send[(c, l)]] + lat[l] - st[v])
                if v not in inedge or err < inedge[v][0]:
                    inedge[v] = (err, u)
        par = {v: u for v, (_, u) in inedge.items()}
        # keep only edges on a path to a destination
        keep = set()
        for d in ds:
            y = d
            while y != s:
                keep.add((par[y], y))
                y = par[y]
        trees[c] = sorted(keep, key=lambda e: st[e[1]])
    return trees, float(xs[T]), res.status


# ---------------------------------------------------------------------------- Stage 3

def contiguity(lt, ordered, chunk_mb, src_of, posts, time_limit=60.0):
    """Stage 3 (App. B.3). ordered: Stage-2 transfers [(start, end, (c,), u, v)] (one chunk
    each). Returns [(send_time, arrive_time, chunks, u, v)] with chunks sent together grouped,
    the optimum time and the MILP status. posts: [(c, r)] postcondition pairs."""
    switched = _switched(lt)
    lat1 = {l: lt.links[l].alpha + lt.links[l].beta * chunk_mb for l in lt.links}
    H = (len(ordered) + lt.n) * max(lt.links[l].alpha + lt.links[l].beta * chunk_mb * (1 + len(ordered))
                                     for l in lt.links) if ordered else 1.0
    m = _Model()
    T = m.var(0.0, H, obj=1.0)
    per_link = {}
    for (t0, _, cs, u, v) in sorted(ordered):
        per_link.setdefault((u, v), []).append(cs[0])
    start = {}

    def st(c, r):
        if (c, r) not in start:
            start[(c, r)] = m.var(0.0, H)
            if src_of[c] == r:
                m.cons([(start[(c, r)], 1.0)], 0.0, 0.0)
        return start[(c, r)]
    send, latv, tog = {}, {}, {}
    for l, cs in per_link.items():
        u, v = l
        a, b = lt.links[l].alpha, lt.links[l].beta * chunk_mb
        for c in cs:
            send[(c, l)] = m.var(0.0, H)
            latv[(c, l)] = m.var(0.0, H)
            m.cons([(send[(c, l)], 1.0), (st(c, u), -1.0)], 0.0)              # eq. corr
        for i in range(len(cs)):
            for j in range(i + 1, len(cs)):
                tog[(cs[i], cs[j], l)] = m.binary()
        for i, c in enumerate(cs):
            # lat[c] = alpha + beta * (1 + sum_o together[c, o])
            terms = [(latv[(c, l)], 1.0)]
            for j, o in enumerate(cs):
                if j != i:
                    terms.append((tog[(min(c, o, key=cs.index), max(c, o, key=cs.index), l)], -b))
            m.cons(terms, a + b, a + b)
            m.cons([(st(c, v), 1.0), (send[(c, l)], -1.0), (latv[(c, l)], -1.0)], 0.0, 0.0)
        for i in range(len(cs)):
            for j in range(i + 1, len(cs)):
                c, o = cs[i], cs[j]
                t = tog[(c, o, l)]
                # together -> equal send times; not together -> o waits for c (link order)
                m.cons([(send[(o, l)], 1.0), (send[(c, l)], -1.0), (t, H)], -math.inf, H)
                m.cons([(send[(o, l)], 1.0), (send[(c, l)], -1.0), (t, -H)], -H)
                m.cons([(send[(o, l)], 1.0), (send[(c, l)], -1.0), (latv[(c, l)], -1.0), (t, H)], 0.0)
                for k in range(j + 1, len(cs)):  # M3 transitivity over ordered triples
                    q = cs[k]
                    m.cons([(tog[(c, q, l)], 1.0), (t, -1.0), (tog[(o, q, l)], -1.0)], -1.0)
                    m.cons([(t, 1.0), (tog[(c, q, l)], -1.0), (tog[(o, q, l)], -1.0)], -1.0)
                    m.cons([(tog[(o, q, l)], 1.0), (t, -1.0), (tog[(c, q, l)], -1.0)], -1.0)
    # switch ports: one switched peer at a time, in the Stage-2 order (different links only;
    # the link rows above already order a link's own chunks)
    for r in range(lt.n):
        for side in (0, 1):
            seq = [(t0, cs[0], (u, v)) for (t0, _, cs, u, v) in sorted(ordered)
                   if (u, v) in switched and (u, v)[side] == r]
            for i in range(len(seq)):
                for j in range(i + 1, len(seq)):
                    (_, c, l1), (_, o, l2) = seq[i], seq[j]
                    if l1 != l2:
                        m.cons([(send[(o, l2)], 1.0), (send[(c, l1)], -1.0), (latv[(c, l1)], -1.0)], 0.0)
    for (c, r) in posts:
        m.cons([(T, 1.0), (st(c, r), -1.0)], 0.0)
    res = m.solve(time_limit)
    xs = res.x
    out = []
    for l, cs in per_link.items():
        done = set()
        for i, c in enumerate(cs):
            if c in done:
                continue
            grp = [c] + [o for o in cs[i + 1:] if xs[tog[(c, o, l)]] > 0.5]
            done.update(grp)
            s0 = xs[send[(c, l)]]
            out.append((s0, s0 + lt.links[l].cost(chunk_mb, len(grp)), tuple(sorted(grp)), l[0], l[1]))
    return _repair(out, src_of, lt, chunk_mb), float(xs[T]), res.status


def _repair(xfers, src_of, lt, chunk_mb):
    """Snap solver times (feasible up to HiGHS tolerances) to an exactly consistent clock:
    in solver send order, a transfer starts no earlier than its chunks' arrival at the sender
    and the previous transfer on its link; arrival = start + alpha + k*beta*s."""
    avail = {(c, s): 0.0 for c, s in src_of.items()}
    link_free = {}
    out = []
    for (s0, _, cs, u, v) in sorted(xfers, key=lambda t: (round(t[0], 6), t[3], t[4], t[2])):
        s = max([round(s0, 6), link_free.get((u, v), 0.0)] + [avail[(c, u)] for c in cs])
        e = s + lt.links[(u, v)].cost(chunk_mb, len(cs))
        link_free[(u, v)] = e
        for c in cs:
            avail[(c, v)] = e
        out.append((s, e, cs, u, v))
    return out


# ---------------------------------------------------------------------------- driver

def synthesize(coll, nranks, chunks=1, policy="uc-max", topology=None, sketch=None, size=None,
               time_limit=60.0, _reverse=False, info=None, **_):
    """Three-stage MILP synthesis for AG / A2A; RS = inverse AG, AR = RS ++ AG (as greedy).
    `info` (dict) receives each stage's objective and solver status."""
    sk = sketch or Sketch(policy=policy, input_chunkup=chunks)
    sk.input_chunkup = chunks
    if size is not None:
        sk.input_size = size
    if topology is None or topology == "nvswitch":
        topo = nvswitch(nranks)
    elif isinstance(topology, str) and topology.startswith("2x"):
        k = int(topology[2:])
        topo = multinode(2, k)
        if sk.internode_conn is None:
            sk.internode_conn = {i: [i] for i in range(k)}
    else:
        topo = topology
    if topo.n != nranks:
        raise ValueError("topology size != nranks")
    kw = dict(policy=policy, topology=topo, sketch=sk, size=size, time_limit=time_limit, info=info)
    if coll == "allreduce":
        ag = synthesize("allgather", nranks, chunks, **kw)
        ag_rev = synthesize("allgather", nranks, chunks, _reverse=True, **kw)
        return templates.allreduce(templates.invert_allgather(ag_rev), ag, f"ar_milp_{sk.policy}_n{nranks}_p{chunks}")
    if coll == "reducescatter":
        ag_rev = synthesize("allgather", nranks, chunks, _reverse=True, **kw)
        return templates.invert_allgather(ag_rev, f"rs_milp_{sk.policy}_n{nranks}_p{chunks}", coll="reducescatter")
    # the logical topology as for greedy (uc-min keeps a ring through each switch); the
    # switch policy also enters the routing objective as the is_util term (eq. uc)
    lt = apply_sketch(topo, sk)
    if _reverse:
        lt.links = {(v, u): l for (u, v), l in lt.links.items()}
    per_chunk = sk.input_size / (chunks if coll == "allgather" else chunks * nranks)
    mb = per_chunk / (1 << 20)
    cl = greedy._chunks(coll, nranks, chunks)
    trees, t1, s1 = route(coll, lt, sk, cl, mb, time_limit)
    src_of = {c: s for c, s, _ in cl}
    ordered = greedy.order(lt, trees, mb, src_of, merge=False)
    posts = [(c, d) for c, _, ds in cl for d in ds]
    xfers, t3, s3 = contiguity(lt, ordered, mb, src_of, posts, time_limit)
    if info is not None:
        info.setdefault("stages", []).append({"routing_time": t1, "routing_status": int(s1),
                                              "ordering_time": max(e for _, e, *_ in ordered),
                                              "exact_time": t3, "exact_status": int(s3),
                                              "final_time": max(e for _, e, *_ in xfers)})
    alg = Algorithm(f"{'ag' if coll == 'allgather' else 'a2a'}_milp_{sk.policy}_n{nranks}_p{chunks}", coll, nranks, chunks)
    for (s, e, cs, u, v) in sorted(xfers):
        alg.add(cs, u, v, s, arrive=e)
    return alg
