"""Offline CPU schedule generator: template, greedy and MILP algorithms lowered
to EF v1 text (docs/SCHEDULE.md). Not on the timed path."""
from .algorithm import Algorithm, Transfer  # noqa: F401
from .lowering import LoweringError, lower  # noqa: F401
from . import templates  # noqa: F401
from .tuned import default_schedules  # noqa: F401


def generate(coll, algo, nranks, chunks=1, instances=1, min_bytes=0, max_bytes=float("inf"), pair=True, merge=True,
             dtypes=None, **kw):
    """EF v1 text for (collective, algorithm) — the one-call entry the CLI and tests use.
    pair=False lowers sends and receives into separate threadblocks; pair="peer" pairs only by
    peer (no relay-first threadblocks, lowering.py); merge=False keeps every transfer its own
    step (no contiguity coalescing, lowering.coalesce)."""
    if algo == "nvls":  # multicast reduce through the switch: written directly (templates.nvls_text)
        return templates.nvls_text(coll, nranks, chunks, instances, min_bytes, max_bytes, dtypes)
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
    return lower(alg, instances=instances, min_bytes=min_bytes, max_bytes=max_bytes, name=name, pair=pair,
                 merge=merge, dtypes=dtypes)
