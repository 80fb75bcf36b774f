"""Template algorithms: ring, direct (all-pairs), hierarchical 2 x k, and combining.

* ring — NCCL's template: "identifies rings in the target topology", n-1 link transfer
  steps per chunk; the uc-min outcome on a switch.
* direct — all-pairs point-to-point, NCCL's Alltoall and the uc-max
  outcome on a switch.
* hier — the dgx2-sk-2 structure: inter-node sends only between GPUs
  with the same local index, overlapped with an intra-node all-pairs Allgather of local
  chunks, then an intra-node all-pairs Allgather of the chunks that arrived from the other
  node; Alltoall coalesces all chunks for the other node over that one link
   and relays them.
* reduce-scatter as the inverse of an Allgather (also the standalone ReduceScatter
  collective), Allreduce as reduce-scatter followed by
  Allgather with per-chunk chaining.
Times are abstract (unit per hop; `inter_lat` for emulated inter-node hops).
"""
from __future__ import annotations

from .algorithm import Algorithm, a2a_chunk, ag_chunk


# ------------------------------------------------------------------------------ allgather

def ring_allgather(n, p=1):
    alg = Algorithm(f"ag_ring_n{n}_p{p}", "allgather", n, p)
    for h in range(n - 1):
        for s in range(n):
            for k in range(p):
                alg.add(ag_chunk(s, k, p), (s + h) % n, (s + h + 1) % n, h * p + k)
    return alg


def direct_allgather(n, p=1):
    alg = Algorithm(f"ag_direct_n{n}_p{p}", "allgather", n, p)
    for s in range(n):
        for off in range(1, n):      # rotational symmetry
            for k in range(p):
                alg.add(ag_chunk(s, k, p), s, (s + off) % n, k)
    return alg


def hier_allgather(nodes_k, p=1, inter_lat=3.0):
    """2 nodes x k GPUs; rank = node*k + i; inter-node partner (1-node)*k + i."""
    k = nodes_k
    n = 2 * k
    alg = Algorithm(f"ag_hier_2x{k}_p{p}", "allgather", n, p)
    for s in range(n):
        node, i = divmod(s, k)
        partner = (1 - node) * k + i
        for q in range(p):
            c = ag_chunk(s, q, p)
            alg.add(c, s, partner, q, lat=inter_lat)
            for j in range(k):
                if j != i:
                    alg.add(c, s, node * k + j, q)
            # the partner forwards it inside its node once it arrives
            for j in range(k):
                if j != i:
                    alg.add(c, partner, (1 - node) * k + j, q + inter_lat)
    return alg


# ------------------------------------------------------------------------------ alltoall

def direct_alltoall(n, p=1):
    alg = Algorithm(f"a2a_direct_n{n}_p{p}", "alltoall", n, p)
    for s in range(n):
        for off in range(1, n):
            d = (s + off) % n
            for k in range(p):
                alg.add(a2a_chunk(s, d, k, n, p), s, d, k)
    return alg


def hier_alltoall(nodes_k, p=1, inter_lat=3.0):
    """Intra-node chunks go direct; all chunks for the other node cross once, coalesced, to
    the partner with the same local index, which relays each to its destination."""
    k = nodes_k
    n = 2 * k
    alg = Algorithm(f"a2a_hier_2x{k}_p{p}", "alltoall", n, p)
    for s in range(n):
        node, i = divmod(s, k)
        partner = (1 - node) * k + i
        for j in range(k):
            d = node * k + j
            if d != s:
                for q in range(p):
                    alg.add(a2a_chunk(s, d, q, n, p), s, d, q)
        remote = [a2a_chunk(s, (1 - node) * k + j, q, n, p) for j in range(k) for q in range(p)]
        alg.add(tuple(remote), s, partner, 0, lat=inter_lat)
        for j in range(k):
            d = (1 - node) * k + j
            if d != partner:
                alg.add(tuple(a2a_chunk(s, d, q, n, p) for q in range(p)), partner, d, inter_lat)
    return alg


# ------------------------------------------------------------------------------ combining

def invert_allgather(ag: Algorithm, name=None, coll="allreduce") -> Algorithm:
    """ReduceScatter from an Allgather: every send (c, u->v) becomes a
    reduce-receive (c, v->u) and time runs backwards, so contributions flow toward the
    chunk's owner along the reversed multicast tree. coll="allreduce" gives the first phase
    of an Allreduce; coll="reducescatter" the standalone collective (owner keeps its part)."""
    T = max((t.arrive_time for t in ag.transfers), default=0.0)
    rs = Algorithm(name or ag.name.replace("ag_", "rs_"), coll, ag.nranks, ag.chunks_per_rank)
    for t in sorted(ag.transfers, key=lambda t: (-t.arrive_time, t.src, t.dst)):
        rs.add(t.chunks, t.dst, t.src, T - t.arrive_time, reduce=True, arrive=T - t.send_time)
    return rs


def allreduce(rs: Algorithm, ag: Algorithm, name) -> Algorithm:
    """Allreduce = ReduceScatter ++ Allgather; AR chunk k is AG chunk k (owner
    k // p). The Allgather phase is shifted after the last reduce so each chunk's phase-2
    sends follow its reduction (per-chunk chaining via lowering's dependencies)."""
    T = max((t.arrive_time for t in rs.transfers), default=0.0)
    ar = Algorithm(name, "allreduce", rs.nranks, rs.chunks_per_rank)
    ar.transfers = list(rs.transfers)
    for t in ag.transfers:
        ar.add(t.chunks, t.src, t.dst, t.send_time + T, arrive=t.arrive_time + T)
    return ar


def ring_reducescatter(n, p=1):
    return invert_allgather(ring_allgather(n, p), coll="reducescatter")


def direct_reducescatter(n, p=1):
    return invert_allgather(direct_allgather(n, p), coll="reducescatter")


def oneshot_allreduce(n, p=1):
    """Latency-optimal Allreduce for small buffers: every rank sends its whole input to every
    other rank, which reduces all n contributions locally — one link hop instead of the
    2(n-1) (ring) or 2 (direct RS+AG) hops of the combining construction,
    at (n-1)x the link bytes. The paper keeps size-specialised algorithms and picks the best
    per size; this one is meant for the small-size range."""
    alg = Algorithm(f"ar_oneshot_n{n}_p{p}", "allreduce", n, p)
    allc = tuple(range(n * p))
    for s in range(n):
        for off in range(1, n):
            alg.add(allc, s, (s + off) % n, 0, reduce=True)
    return alg


def ring_allreduce(n, p=1):
    return allreduce(invert_allgather(ring_allgather(n, p)), ring_allgather(n, p),
                     f"ar_ring_n{n}_p{p}")


def direct_allreduce(n, p=1):
    return allreduce(invert_allgather(direct_allgather(n, p)), direct_allgather(n, p),
                     f"ar_direct_n{n}_p{p}")


def nvls_text(coll, n, p=1, instances=1, min_bytes=0, max_bytes=float("inf"), dtypes=None):
    """EF v1 text of the Allreduce through the switch (NVLink SHARP; reading N1):
    rank r, one threadblock (its peer is the switch), ONE multicast-reduce step (`mr`) over its
    own p chunks r*p .. r*p+p-1 — multimem.ld_reduce sums the n copies in the NVSwitch,
    multimem.st writes the result to every rank. Per GPU the links carry ~S out and ~S in
    (1/n of it as the reduced result) instead of RS ++ AG's 2(n-1)/n S each way (PAPER.md:
    720-728). There are no point-to-point transfers, so nothing is lowered."""
    if coll != "allreduce":
        raise ValueError("nvls: allreduce only")
    mx = "inf" if max_bytes == float("inf") else str(int(max_bytes))
    out = [f'<algo name="ar_nvls_n{n}_p{p}_m{instances}" coll="allreduce" nranks="{n}" chunks_per_rank="{p}" '
           f'instances="{instances}" minBytes="{int(min_bytes)}" maxBytes="{mx}" inplace="0"'
           + (f' dtypes="{",".join(dtypes)}"' if dtypes else "") + '>']
    for r in range(n):
        out.append(f' <gpu id="{r}" i_chunks="{n * p}" o_chunks="{n * p}" s_chunks="0">')
        out.append('  <tb id="0" send="-1" recv="-1" chan="0">')
        out.append(f'   <step s="0" type="mr" srcbuf="i" srcoff="{r * p}" dstbuf="o" dstoff="{r * p}" cnt="{p}" deps=""/>')
        out.append('  </tb>')
        out.append(' </gpu>')
    out.append('</algo>')
    return "\n".join(out) + "\n"


def direct_ring_allreduce(n, p=1):
    """All-pairs reduce-scatter (every partial sum travels one hop: no fp32 partial hops for
    bf16, reading R6) followed by a ring Allgather (one connection per GPU: the connection-count
    sweep measured 10% more per-GPU egress over one connection than over three at n=4,
    profiles/r02_nvlink_probe.jsonl) — PAPER.md:728's combination with mixed templates. Registered as "dring"."""
    return allreduce(invert_allgather(direct_allgather(n, p)), ring_allgather(n, p), f"ar_direct_ring_n{n}_p{p}")


# ------------------------------------------------------------------------------ registry

TEMPLATES = {
    ("allgather", "ring"): ring_allgather,
    ("allgather", "direct"): direct_allgather,
    ("alltoall", "direct"): direct_alltoall,
    ("allreduce", "ring"): ring_allreduce,
    ("allreduce", "direct"): direct_allreduce,
    ("allreduce", "dring"): direct_ring_allreduce,
    ("allreduce", "oneshot"): oneshot_allreduce,
    ("reducescatter", "ring"): ring_reducescatter,
    ("reducescatter", "direct"): direct_reducescatter,
}
