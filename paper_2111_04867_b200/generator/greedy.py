"""Sketch-guided greedy route + order synthesizer: the stand-in for TACCL's MILP stages.

The paper synthesizes in three stages (App. B):
routing (MILP, bandwidth-relaxed), heuristic ordering (greedy) and contiguity/exact
scheduling (MILP). Without a MILP solver this module keeps Stage 2 as the paper describes it
and replaces Stages 1 and 3 by greedy rules (SURVEY.md M14–M16):

* Routing (Stage 1 stand-in): each chunk is routed on a shortest-latency multicast tree
  from its source to its destination set over the sketch's logical topology (the paper
  restricts paths to shortest paths too); ties go to the link with the
  least latency already assigned (the relaxed bandwidth term of eq. link1),
  then to the smallest rank offset from the source (rotation-invariant). Inter-node hops
  must leave from the chunk's relay when the sketch has a chunk_to_relay_map. Chunks in a
  rotational-symmetry orbit reuse the base chunk's rotated
  tree.
* Ordering (Stage 2, App. B.2): candidates are the next unscheduled
  link of every chunk's tree whose chunk is already available at the link's source; each
  round schedules the candidate that can start earliest given the running link time, the
  chunk time and the switch send/recv port times (App. B.3's switch constraints), ties by
  (1) longest remaining path to the chunk's final GPU, (2) shortest path traversed so far,
  (3) lowest chunk id, (4) lowest destination.
* Contiguity (Stage 3 stand-in): on IB links (the paper uses contiguity only there,
  PAPER.md:636–637) every chunk already waiting at the sender when a transfer starts joins
  it: one transfer costing alpha + k*beta*s.
Reduce-scatter / allreduce come from templates.invert_allgather / templates.allreduce.
"""
from __future__ import annotations

import heapq

from .algorithm import Algorithm, a2a_chunk, a2a_parts, ag_chunk
from .topology import Sketch, Topology, apply_sketch, multinode, nvswitch, relay_for_chunk, rotate
from . import templates


def _chunks(coll, n, p):
    """(chunk id, source rank, destination set) per the collective's pre/postcondition."""
    out = []
    for s in range(n):
        for k in range(p):
            if coll == "allgather":
                out.append((ag_chunk(s, k, p), s, [d for d in range(n) if d != s]))
            else:
                for d in range(n):
                    if d != s:
                        out.append((a2a_chunk(s, d, k, n, p), s, [d]))
    return out


def _rot_chunk(coll, c, n, p, o, g):
    if coll == "allgather":
        s, k = divmod(c, p)
        return ag_chunk(rotate(s, o, g), k, p)
    s, d, k = a2a_parts(c, n, p)
    return a2a_chunk(rotate(s, o, g), rotate(d, o, g), k, n, p)


def route(coll, lt: Topology, sk: Sketch, chunks, chunk_mb):
    """Multicast tree per chunk: {chunk: [(u, v), ...]} with parents before children."""
    load = {l: 0.0 for l in lt.links}
    out_adj = {u: [] for u in range(lt.n)}
    for (u, v) in lt.links:
        out_adj[u].append(v)
    trees = {}
    done = set()
    n, p = lt.n, sk.input_chunkup
    for c, src, dsts in chunks:
        if c in done:
            continue
        relay = relay_for_chunk(sk, src) if sk.chunk_to_relay else None

        def allowed(u, v):
            if relay is not None and lt.node_of[u] != lt.node_of[v] and u != relay:
                return False
            return True
        # Dijkstra on latency; among equal-latency parents prefer the least-loaded link,
        # then the smallest rank offset from the source (rotation-invariant)
        dist = {src: 0.0}
        best = {src: (0.0, 0.0, 0)}
        par = {}
        heap = [(0.0, src)]
        seen = set()
        while heap:
            d, u = heapq.heappop(heap)
            if u in seen:
                continue
            seen.add(u)
            for v in sorted(out_adj[u], key=lambda x: (x - src) % n):
                if v == src or not allowed(u, v):
                    continue
                key = (round(d + lt.links[(u, v)].cost(chunk_mb), 9), load[(u, v)], (u - src) % n)
                if v not in best or key < best[v]:
                    best[v] = key
                    dist[v] = key[0]
                    par[v] = u
                    heapq.heappush(heap, (key[0], v))
        edges = set()
        for d in dsts:
            if d not in par and d != src:
                raise ValueError(f"chunk {c}: destination {d} unreachable from {src} in the logical topology")
            x = d
            while x != src:
                edges.add((par[x], x))
                x = par[x]
        ordered = sorted(edges, key=lambda e: dist[e[1]])  # parents before children
        for e in ordered:
            load[e] += lt.links[e].cost(chunk_mb)
        trees[c] = ordered
        done.add(c)
        # symmetric images (rotational offsets) reuse the rotated tree
        frontier = [(c, ordered)]
        while frontier:
            cc, tr = frontier.pop()
            for (o, g) in sk.symmetry_offsets:
                c2 = _rot_chunk(coll, cc, n, p, o, g)
                if c2 in done:
                    continue
                tr2 = [(rotate(u, o, g), rotate(v, o, g)) for (u, v) in tr]
                if all(e in lt.links for e in tr2):
                    trees[c2] = tr2
                    done.add(c2)
                    for e in tr2:
                        load[e] += lt.links[e].cost(chunk_mb)
                    frontier.append((c2, tr2))
    return trees


def order(lt: Topology, trees, chunk_mb, src_of, merge=True):
    """Stage 2 greedy (App. B.2) with the IB contiguity stand-in (merge=False: one chunk per
    transfer, the input of the Stage-3 MILP, milp.py): returns scheduled transfers
    [(start, end, chunks, u, v)]."""
    link_t = {l: 0.0 for l in lt.links}
    send_port = {u: 0.0 for u in range(lt.n)}
    recv_port = {u: 0.0 for u in range(lt.n)}
    switched = set()
    for sw in lt.switches:
        for a in sw:
            for b in sw:
                if a != b:
                    switched.add((a, b))
    avail = {(c, src_of[c]): 0.0 for c in trees}
    children = {}
    for c, tr in trees.items():
        for (u, v) in tr:
            children.setdefault((c, u), []).append(v)
    memo = {}

    def remaining(c, v):  # longest remaining path (latency) below v in c's tree
        if (c, v) not in memo:
            memo[(c, v)] = max([lt.links[(v, w)].cost(chunk_mb) + remaining(c, w)
                                for w in children.get((c, v), [])] or [0.0])
        return memo[(c, v)]

    traversed = {(c, src_of[c]): 0.0 for c in trees}
    pending = {(c, u, v) for c, tr in trees.items() for (u, v) in tr}
    out = []

    def key_of(c, u, v):
        l = (u, v)
        start = max(link_t[l], avail[(c, u)])
        if l in switched:
            start = max(start, send_port[u], recv_port[v])
        return (start, -(lt.links[l].cost(chunk_mb) + remaining(c, v)), traversed[(c, u)], c, v)

    while pending:
        ready = [(key_of(c, u, v), c, u, v) for (c, u, v) in pending if (c, u) in avail]
        (start, *_), c, u, v = min(ready)
        link = lt.links[(u, v)]
        group = [(c, u, v)]
        if merge and link.kind == "ib":
            # contiguity: everything else waiting for this link that is already available
            # at u by `start` goes in the same transfer (one alpha)
            more = sorted(k for k in ready if k[2] == u and k[3] == v and k[1] != c and avail[(k[1], u)] <= start)
            group += [(k[1], k[2], k[3]) for k in more]
        end = start + link.cost(chunk_mb, len(group))
        link_t[(u, v)] = end
        if (u, v) in switched:
            send_port[u] = end
            recv_port[v] = end
        for (cc, _, _) in group:
            avail[(cc, v)] = end
            traversed[(cc, v)] = traversed[(cc, u)] + link.cost(chunk_mb)
            pending.remove((cc, u, v))
        out.append((start, end, tuple(sorted(g[0] for g in group)), u, v))
    return out


def schedule_time(transfers):
    return max(t.arrive_time for t in transfers) if transfers else 0.0


def synthesize(coll, nranks, chunks=1, policy="uc-max", topology=None, sketch=None, size=None,
               _reverse=False, **_):
    """Greedy AG / A2A (and AR = inverse-AG ++ AG). `topology`: a Topology, "nvswitch"
    (default) or "2xK" for the emulated two-node sketch (inter-node GPU i <-> GPU i)."""
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
            sk.internode_conn = {i: [i] for i in range(k)}  # dgx2-sk-2 style
    else:
        topo = topology
    if topo.n != nranks:
        raise ValueError("topology size != nranks")
    if coll == "allreduce":
        # RS = inverse of an Allgather synthesized on the reversed logical topology, so the
        # reduce-scatter flows the same way as the Allgather that follows (a uc-min ring
        # stays one ring)
        ag = synthesize("allgather", nranks, chunks, policy, topo, sk, size)
        ag_rev = synthesize("allgather", nranks, chunks, policy, topo, sk, size, _reverse=True)
        return templates.allreduce(templates.invert_allgather(ag_rev), ag, f"ar_greedy_{sk.policy}_n{nranks}_p{chunks}")
    if coll == "reducescatter":
        ag_rev = synthesize("allgather", nranks, chunks, policy, topo, sk, size, _reverse=True)
        return templates.invert_allgather(ag_rev, f"rs_greedy_{sk.policy}_n{nranks}_p{chunks}", coll="reducescatter")
    lt = apply_sketch(topo, sk)
    if _reverse:
        lt.links = {(v, u): l for (u, v), l in lt.links.items()}
    # chunk size in MB for the cost model: input_size is the per-rank input buffer
    per_chunk = sk.input_size / (chunks if coll == "allgather" else chunks * nranks)
    mb = per_chunk / (1 << 20)
    cl = _chunks(coll, nranks, chunks)
    trees = route(coll, lt, sk, cl, mb)
    src_of = {c: s for c, s, _ in cl}
    merged = order(lt, trees, mb, src_of)
    alg = Algorithm(f"{'ag' if coll == 'allgather' else 'a2a'}_greedy_{sk.policy}_n{nranks}_p{chunks}", coll, nranks, chunks)
    for (s, e, cs, u, v) in sorted(merged):
        alg.add(cs, u, v, s, arrive=e)
    return alg
