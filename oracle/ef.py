"""EF v1 parser for the oracle (test infrastructure; see oracle/__init__.py).

Follows the TACCL-EF description, PAPER.md:741–752 (§6.1): "three buffers: input, output
and scratch", per-buffer chunk counts with "all chunks equal size", GPU programs made of
threadblocks, each "a series of steps that are executed sequentially", instructions
"sends, receives (with optional reduction), and local copies", "each threadblock can send
to and receive from at most one GPU", and dependencies between steps.
The concrete syntax is repo-defined (docs/SCHEDULE.md). This parser uses the standard
library XML reader; the product's C++ loader has its own hand-written parser.
"""
from __future__ import annotations

import math
import xml.etree.ElementTree as ET
from dataclasses import dataclass, field


class ScheduleError(Exception):
    """A schedule failed a check. `kind` is one of the classes in docs/SCHEDULE.md."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg


COLLS = ("allgather", "alltoall", "allreduce", "reducescatter")
STEP_TYPES = ("s", "r", "rrc", "cpy", "nop", "mr")
BUFS = ("i", "o", "s")


@dataclass
class Step:
    s: int
    type: str
    srcbuf: str | None = None
    srcoff: int = 0
    dstbuf: str | None = None
    dstoff: int = 0
    cnt: int = 0
    deps: list = field(default_factory=list)  # list of (tb, step) on the same rank


@dataclass
class TB:
    id: int
    send: int
    recv: int
    chan: int
    steps: list = field(default_factory=list)


@dataclass
class Gpu:
    id: int
    i_chunks: int
    o_chunks: int
    s_chunks: int
    tbs: list = field(default_factory=list)

    def nchunks(self, buf: str) -> int:
        return {"i": self.i_chunks, "o": self.o_chunks, "s": self.s_chunks}[buf]


@dataclass
class Program:
    name: str
    coll: str
    nranks: int
    chunks_per_rank: int
    instances: int
    min_bytes: float
    max_bytes: float
    inplace: int
    gpus: list = field(default_factory=list)
    # set by instances.expand_instances: chunk k' of the expanded program is subchunk k' % m of
    # the original chunk k' // m (reading G3's floor split); 1 = ordinary equal chunks
    subchunks: int = 1


def _int(el, key, lo=None):
    v = el.get(key)
    if v is None:
        raise ScheduleError("syntax", f"<{el.tag}> missing attribute {key}")
    try:
        x = int(v)
    except ValueError:
        raise ScheduleError("syntax", f"<{el.tag}> attribute {key}={v!r} is not an integer")
    if lo is not None and x < lo:
        raise ScheduleError("syntax", f"<{el.tag}> attribute {key}={x} < {lo}")
    return x


def _bytes(el, key):
    v = el.get(key)
    if v is None:
        raise ScheduleError("syntax", f"<algo> missing attribute {key}")
    if v == "inf":
        return math.inf
    try:
        x = int(v)
    except ValueError:
        raise ScheduleError("syntax", f"<algo> attribute {key}={v!r} is not an integer or inf")
    if x < 0:
        raise ScheduleError("syntax", f"<algo> attribute {key} is negative")
    return x


def _deps(text: str):
    out = []
    text = text.strip()
    if not text:
        return out
    for item in text.split(","):
        parts = item.strip().split(":")
        if len(parts) != 2:
            raise ScheduleError("syntax", f"bad dependency {item!r} (want tb:step)")
        try:
            t, k = int(parts[0]), int(parts[1])
        except ValueError:
            raise ScheduleError("syntax", f"bad dependency {item!r} (want tb:step)")
        if t < 0 or k < 0:
            raise ScheduleError("syntax", f"bad dependency {item!r} (negative)")
        out.append((t, k))
    return out


def _buf(el, key):
    v = el.get(key)
    if v not in BUFS:
        raise ScheduleError("syntax", f"<step> {key}={v!r} is not one of i/o/s")
    return v


def parse(text: str) -> Program:
    """Parse EF v1 text into a Program. Raises ScheduleError('syntax', ...)."""
    try:
        root = ET.fromstring(text)
    except ET.ParseError as e:
        raise ScheduleError("syntax", f"not well-formed: {e}")
    if root.tag != "algo":
        raise ScheduleError("syntax", "root element must be <algo>")
    coll = root.get("coll")
    if coll not in COLLS:
        raise ScheduleError("syntax", f"coll={coll!r} unsupported")
    prog = Program(
        name=root.get("name", ""),
        coll=coll,
        nranks=_int(root, "nranks", 1),
        chunks_per_rank=_int(root, "chunks_per_rank", 1),
        instances=_int(root, "instances", 1),
        min_bytes=_bytes(root, "minBytes"),
        max_bytes=_bytes(root, "maxBytes"),
        inplace=_int(root, "inplace", 0),
    )
    if prog.inplace != 0:
        raise ScheduleError("syntax", "inplace=1 is not supported (reading G10)")
    # optional dtypes="...": which element types a runtime may select the algorithm for (a
    # selection attribute only; it changes nothing the program computes)
    for d in filter(None, (root.get("dtypes") or "").split(",")):
        if d not in ("int32", "float32", "bfloat16"):
            raise ScheduleError("syntax", f"dtypes: unknown element type {d!r}")
    # optional overlap="0|1": an execution hint for a runtime (warp-specialised send + reduce
    # pairs); like dtypes it changes nothing the program computes
    if (root.get("overlap") or "0") not in ("0", "1"):
        raise ScheduleError("syntax", "overlap must be 0 or 1")
    gpus = [g for g in root if g.tag == "gpu"]
    if any(g.tag != "gpu" for g in root):
        raise ScheduleError("syntax", "<algo> may only contain <gpu>")
    if len(gpus) != prog.nranks:
        raise ScheduleError("syntax", f"{len(gpus)} <gpu> elements for nranks={prog.nranks}")
    for r, g in enumerate(gpus):
        gid = _int(g, "id", 0)
        if gid != r:
            raise ScheduleError("syntax", f"<gpu> #{r} has id={gid}")
        gpu = Gpu(gid, _int(g, "i_chunks", 0), _int(g, "o_chunks", 0), _int(g, "s_chunks", 0))
        for t, tbel in enumerate(g):
            if tbel.tag != "tb":
                raise ScheduleError("syntax", "<gpu> may only contain <tb>")
            tid = _int(tbel, "id", 0)
            if tid != t:
                raise ScheduleError("syntax", f"rank {r}: <tb> #{t} has id={tid}")
            tb = TB(tid, _int(tbel, "send", -1), _int(tbel, "recv", -1), _int(tbel, "chan", 0))
            for k, st in enumerate(tbel):
                if st.tag != "step":
                    raise ScheduleError("syntax", "<tb> may only contain <step>")
                sid = _int(st, "s", 0)
                if sid != k:
                    raise ScheduleError("syntax", f"rank {r} tb {t}: <step> #{k} has s={sid}")
                typ = st.get("type")
                if typ not in STEP_TYPES:
                    raise ScheduleError("syntax", f"rank {r} tb {t} step {k}: type={typ!r}")
                step = Step(sid, typ, deps=_deps(st.get("deps", "")))
                if typ in ("s", "rrc", "cpy", "mr"):
                    step.srcbuf = _buf(st, "srcbuf")
                    step.srcoff = _int(st, "srcoff", 0)
                if typ in ("r", "rrc", "cpy", "mr"):
                    step.dstbuf = _buf(st, "dstbuf")
                    step.dstoff = _int(st, "dstoff", 0)
                if typ != "nop":
                    step.cnt = _int(st, "cnt", 1)
                tb.steps.append(step)
            gpu.tbs.append(tb)
        prog.gpus.append(gpu)
    return prog


def serialize(prog: Program) -> str:
    """Write a Program back to EF v1 text (used for instance-expanded programs)."""
    mx = "inf" if prog.max_bytes == math.inf else str(int(prog.max_bytes))
    lines = [
        f'<algo name="{prog.name}" coll="{prog.coll}" nranks="{prog.nranks}" '
        f'chunks_per_rank="{prog.chunks_per_rank}" instances="{prog.instances}" '
        f'minBytes="{int(prog.min_bytes)}" maxBytes="{mx}" inplace="{prog.inplace}">'
    ]
    for g in prog.gpus:
        lines.append(f' <gpu id="{g.id}" i_chunks="{g.i_chunks}" o_chunks="{g.o_chunks}" '
                     f's_chunks="{g.s_chunks}">')
        for tb in g.tbs:
            lines.append(f'  <tb id="{tb.id}" send="{tb.send}" recv="{tb.recv}" chan="{tb.chan}">')
            for st in tb.steps:
                a = [f's="{st.s}"', f'type="{st.type}"']
                if st.srcbuf is not None:
                    a += [f'srcbuf="{st.srcbuf}"', f'srcoff="{st.srcoff}"']
                if st.dstbuf is not None:
                    a += [f'dstbuf="{st.dstbuf}"', f'dstoff="{st.dstoff}"']
                if st.type != "nop":
                    a.append(f'cnt="{st.cnt}"')
                a.append('deps="' + ",".join(f"{t}:{k}" for t, k in st.deps) + '"')
                lines.append("   <step " + " ".join(a) + "/>")
            lines.append("  </tb>")
        lines.append(" </gpu>")
    lines.append("</algo>")
    return "\n".join(lines) + "\n"
