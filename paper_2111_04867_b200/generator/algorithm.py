"""Abstract algorithms: timed chunk transfers before lowering (§5.1).

An abstract algorithm is what the paper's synthesizer hands to lowering:
for every transfer, which chunk(s) move over which link, when, and — for combining
collectives — whether the receiver reduces. Chunk ids follow the
collective's layout (docs/SCHEDULE.md): AG `src*p + k`, A2A `(src*n + dst)*p + k`,
AR `k` (owner `k // p` after the reduce-scatter phase).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Transfer:
    chunks: tuple          # chunk ids sent together as one contiguous transfer
    src: int
    dst: int
    send_time: float       # when the sender issues it (greedy / template clock)
    arrive_time: float     # when it is available at dst
    reduce: bool = False   # receiver reduces into its copy (recvReduceCopy)


@dataclass
class Algorithm:
    name: str
    coll: str              # allgather | alltoall | allreduce
    nranks: int
    chunks_per_rank: int   # p ("chunk partitioning")
    transfers: list = field(default_factory=list)

    def add(self, chunks, src, dst, t, lat=1.0, reduce=False, arrive=None):
        """`arrive` (default t + lat) must equal the send_time of any later forward of the
        same chunk exactly: lowering orders a rank's events by these times."""
        if isinstance(chunks, int):
            chunks = (chunks,)
        a = float(t) + lat if arrive is None else float(arrive)
        self.transfers.append(Transfer(tuple(chunks), src, dst, float(t), a, reduce))


# ---- chunk-id helpers --------------------------------------------------

def ag_chunk(src, k, p):
    return src * p + k


def a2a_chunk(src, dst, k, n, p):
    return (src * n + dst) * p + k


def a2a_parts(c, n, p):
    """chunk id -> (src, dst, k)"""
    k = c % p
    sd = c // p
    return sd // n, sd % n, k
