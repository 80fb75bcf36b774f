"""Offline CPU schedule generator: template, greedy and MILP algorithms lowered
to EF v1 text (docs/SCHEDULE.md). Not on the timed path."""
from .algorithm import Algorithm, Transfer  # noqa: F401
from .lowering import LoweringError, lower  # noqa: F401
from . import templates  # noqa: F401
from .tuned import default_schedules  # noqa: F401


def generate(coll, algo, nranks, chunks=1, instances=1, min_bytes=0, max_bytes=float("inf"), pair=True, merge=True,
             dtypes=None, overlap=False, **kw):
    """EF v1 text for (collective, algorithm) — the one-call entry the CLI and tests use.
    pair=False lowers sends and receives into separate threadblocks; pair="peer" pairs only by
    peer (no relay-first threadblocks, lowering.py); merge=False keeps every transfer its own
    step (no contiguity coalescing, lowering.coalesce); overlap=True adds the overlap="1"
    execution hint (warp-specialised send + receive-reduce pairs, docs/SCHEDULE.md)."""
    if algo == "nvls":  # multicast reduce through the switch: written directly (templates.nvls_text)
        return templates.nvls_text(coll, nranks, chunks, instances, min_bytes, max_bytes, dtypes)
    if algo == "rounds":  # all-pairs in rounds (A/B experiment, DESIGN.md §6 merged threadblocks)
        return _rounds(generate(coll, "direct", nranks, chunks, instances, min_bytes, max_bytes, pair=False,
                                merge=merge, dtypes=dtypes), nranks)
    if algo == "hier":
        if nranks % 2:
            raise ValueError("hier needs 2 x k ranks")
        fn = {"allgather": templates.hier_allgather, "alltoall": templates.hier_alltoall}[coll]
        alg = fn(nranks // 2, chunks, **kw)
    elif algo == "greedy":
        from .greedy import synthesize
        alg = synthesize(coll, nranks, chunks, **kw)
    elif algo == "milp":  # the paper's three-stage synthesizer (HiGHS MILPs, milp.py)
        from .milp import synthesize
        alg = synthesize(coll, nranks, chunks, **kw)
    else:
        alg = templates.TEMPLATES[(coll, algo)](nranks, chunks)
    name = f"{alg.name}_m{instances}"
    if not pair:
        name += "_split"
    elif pair == "peer":
        name += "_peer"
    if not merge:
        name += "_nomerge"
    if overlap:
        name += "_ovl"
    return lower(alg, instances=instances, min_bytes=min_bytes, max_bytes=max_bytes, name=name, pair=pair,
                 merge=merge, dtypes=dtypes, overlap=overlap)


def _rounds(text, n):
    """The split all-pairs schedule with round order: the send to rank r + d waits for the
    receive from rank r - (d - 1) (round d - 1 landed), so with merged threadblocks every round
    is one permutation of peers, flow-controlled by the previous round's arrival."""
    import re
    out, pos = [], 0
    for m in re.finditer(r'<gpu id="(\d+)".*?</gpu>', text, re.S):
        r = int(m.group(1))
        body = m.group(0)
        recv_tb = {int(b): int(a) for a, b in re.findall(r'<tb id="(\d+)" send="-1" recv="(\d+)"', body)}

        def dep(mt):
            t, peer = int(mt.group(1)), int(mt.group(2))
            d = (peer - r) % n
            if d < 2:
                return mt.group(0)
            prev = recv_tb[(r - (d - 1)) % n]
            return mt.group(0).replace('deps=""', f'deps="{prev}:0"', 1)
        body = re.sub(r'<tb id="(\d+)" send="(\d+)" recv="-1"[^>]*>\s*<step s="0" type="s"[^/]*/>', dep, body)
        out.append(text[pos:m.start()] + body)
        pos = m.end()
    out.append(text[pos:])
    return "".join(out).replace('_split"', '_rounds"', 1)
