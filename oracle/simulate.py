"""Schedule execution on host buffers (test infrastructure; see oracle/__init__.py).

Executes a TACCL-EF program the way PAPER.md:741–752 describes it: every rank runs its
threadblocks' steps in order, a step waits for its dependencies, a send's chunks reach the
matched receive on the peer, a receive "with optional reduction" combines them with a local
source (sum; readings G4/G5), and a copy moves chunks locally
(PAPER.md:768–769). The engine walks one topological order of the happens-before DAG
(default: deterministic Kahn; tests pass every linear extension of tiny programs).

Two value domains share the engine:
* symbolic — AG/A2A tokens are chunk ids, AR tokens are (chunk index, contribution count
  per rank); scratch and output start as BOTTOM; reading BOTTOM is an `uninit` error; the
  final state is checked against the postcondition (App. B);
* numeric — NumPy arrays, `c_e` elements per chunk; scratch and output
  start poisoned with 0xA5 bytes (reading G11); sums: int32 wraps mod 2^32 (G13), float32 is
  one IEEE binary32 round-to-nearest-even add, bfloat16 is the correctly rounded bf16 sum of
  two bf16 values computed as fp32 add + RNE to bf16 (G6; pinned in tests against exact
  rational arithmetic).
"""
from __future__ import annotations

from collections import deque

import numpy as np

from .collectives import DTYPES, chunk_elems, postcondition, precondition
from .ef import Program, ScheduleError
from .validate import build_graph, check_structure, topo_order

BOTTOM = None


def _steps(prog: Program, graph, order):
    for v in order:
        r, t, k = graph.nodes[v]
        tb = prog.gpus[r].tbs[t]
        yield v, r, tb, tb.steps[k]


def _execute(prog: Program, graph, order, bufs, read, write, reduce, mreduce=None):
    """Shared engine. bufs[r][buf] is a rank's buffer; read/write move cnt chunks."""
    queues = {key: deque() for key in graph.conns}
    for v, r, tb, st in _steps(prog, graph, order):
        where = (r, tb.id, st.s)
        if st.type == "mr":  # multicast reduce: sum over every rank's src, to every rank's dst
            vals = [read(bufs[q][st.srcbuf], st.srcoff, st.cnt, where) for q in range(prog.nranks)]
            out = mreduce(vals, where)
            for q in range(prog.nranks):
                write(bufs[q][st.dstbuf], st.dstoff, st.cnt, out)
            continue
        if st.type == "cpy":
            write(bufs[r][st.dstbuf], st.dstoff, st.cnt, read(bufs[r][st.srcbuf], st.srcoff, st.cnt, where))
        elif st.type == "s":
            queues[(r, tb.send, tb.chan)].append(read(bufs[r][st.srcbuf], st.srcoff, st.cnt, where))
        elif st.type == "r":
            write(bufs[r][st.dstbuf], st.dstoff, st.cnt, queues[(tb.recv, r, tb.chan)].popleft())
        elif st.type == "rrc":
            got = queues[(tb.recv, r, tb.chan)].popleft()
            mine = read(bufs[r][st.srcbuf], st.srcoff, st.cnt, where)
            write(bufs[r][st.dstbuf], st.dstoff, st.cnt, reduce(mine, got, where))
        # nop: nothing moves


def _prepare(prog, graph, order):
    if graph is None:
        errs = check_structure(prog)
        if errs:
            raise ScheduleError("structure", errs[0])
        graph = build_graph(prog)
    if order is None:
        order = topo_order(graph)
    return graph, order


# ------------------------------------------------------------------------------ symbolic

def run_symbolic(prog: Program, graph=None, order=None, check=True):
    """Execute on chunk tokens; return per-rank output token lists. With check=True raise
    ScheduleError('uninit' | 'postcondition') like the validator."""
    graph, order = _prepare(prog, graph, order)
    n, p = prog.nranks, prog.chunks_per_rank
    pre = precondition(prog.coll, n, p)
    bufs = []
    for g in prog.gpus:
        b = {"i": [BOTTOM] * g.i_chunks, "o": [BOTTOM] * g.o_chunks, "s": [BOTTOM] * g.s_chunks}
        for k, tok in pre[g.id].items():
            b["i"][k] = tok
        bufs.append(b)

    def read(buf, off, cnt, where):
        vals = buf[off:off + cnt]
        for q, x in enumerate(vals):
            if x is BOTTOM:
                raise ScheduleError("uninit", "rank %d tb%d:s%d reads chunk %d before any write"
                                    % (where + (off + q,)))
        return list(vals)

    def write(buf, off, cnt, vals):
        buf[off:off + cnt] = vals

    def reduce(mine, got, where):
        if prog.coll not in ("allreduce", "reducescatter"):
            raise ScheduleError("structure", "rank %d tb%d:s%d reduces in a non-reducing "
                                             "collective" % where)
        out = []
        for a, b in zip(mine, got):
            if a[0] != b[0]:
                raise ScheduleError("postcondition", "rank %d tb%d:s%d reduces chunk %d with "
                                                     "chunk %d" % (where + (a[0], b[0])))
            out.append((a[0], tuple(x + y for x, y in zip(a[1], b[1]))))
        return out

    def mreduce(vals, where):
        out = vals[0]
        for x in vals[1:]:
            out = reduce(out, x, where)
        return out

    _execute(prog, graph, order, bufs, read, write, reduce, mreduce)
    outs = [b["o"] for b in bufs]
    if check:
        post = postcondition(prog.coll, n, p)
        for r in range(n):
            for k, want in sorted(post[r].items()):
                got = outs[r][k]
                if got != want:
                    raise ScheduleError("postcondition", _post_msg(prog.coll, r, k, want, got))
    return outs


def _post_msg(coll, r, k, want, got):
    if coll not in ("allreduce", "reducescatter"):
        return f"(chunk {want}, rank {r}) missing: o[{k}] holds {got!r}"
    if got is BOTTOM:
        return f"(chunk {k}, rank {r}) missing: o[{k}] never written"
    missing = [s for s, c in enumerate(got[1]) if c == 0]
    extra = [s for s, c in enumerate(got[1]) if c > 1]
    return (f"(chunk {k}, rank {r}) reduction wrong: chunk {got[0]}, missing contributions "
            f"from ranks {missing}, repeated from ranks {extra}")


# ------------------------------------------------------------------------------ numeric

def bf16_round(f32: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bits, round to nearest even; NaN stays a quiet NaN."""
    bits = np.ascontiguousarray(f32, dtype=np.float32).view(np.uint32)
    rounded = ((bits.astype(np.uint64) + 0x7FFF + ((bits >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(f32)
    if nan.any():
        rounded[nan] = ((bits[nan] >> 16) | 0x0040).astype(np.uint16)
    return rounded


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def add(a: np.ndarray, b: np.ndarray, dtype: str) -> np.ndarray:
    """One reduction step dst = src + received in the schedule's dtype."""
    if dtype == "int32":
        return (a.view(np.uint32) + b.view(np.uint32)).view(np.int32)
    if dtype == "float32":
        with np.errstate(over="ignore", invalid="ignore"):
            return (a + b).astype(np.float32)
    if dtype == "bfloat16":
        with np.errstate(over="ignore", invalid="ignore"):
            return bf16_round(bf16_to_f32(a) + bf16_to_f32(b))
    raise ValueError(dtype)


class _Val:
    """bf16 partials mode: a range's bits plus its fp32 partials (None unless every chunk of
    the range holds one) — what a read returns and a send carries."""
    __slots__ = ("bits", "part")

    def __init__(self, bits, part):
        self.bits, self.part = bits, part


class _Reduced(_Val):
    """The result of an rrc in bf16 partials mode: bits = RNE(acc), part = acc (fp32)."""


def run(prog: Program, inputs, dtype: str, graph=None, order=None, bf16: str = "partials"):
    """Numeric execution. inputs: one 1-D array per rank (dtype storage per DTYPES, bf16 as
    uint16 bits). Returns the per-rank output arrays.

    bf16 selects the bfloat16 reduction semantics (reading G6, DESIGN.md §2 R6); int32 and
    float32 are unaffected (a float32 partial is the float32 value itself):
    * "partials" (the executor's): every chunk an `rrc` writes keeps its fp32 accumulator as a
      partial next to the RNE-rounded bf16 bits. An operand of a later `rrc` — its local
      source, or the message of a send — is read as those fp32 partials when every chunk of
      its range holds one, else as the bf16 bits widened (exactly). `r` and `cpy` write bf16
      bits and drop the destination's partials (so a value that leaves a reduction chain
      through a receive or a copy is rounded once, there). The rrc adds in fp32 (RNE).
      Consequence: a chain of rrcs — on one rank or hop to hop across ranks — sums in fp32
      in chain order and rounds once per value anyone reads as bf16.
    * "per_step": every rrc rounds to bf16 (correctly rounded bf16 addition of two bf16 values).
    """
    graph, order = _prepare(prog, graph, order)
    n, p, m = prog.nranks, prog.chunks_per_rank, prog.subchunks
    np_dt, _ = DTYPES[dtype]
    e_in = inputs[0].size
    count = e_in // n if prog.coll in ("alltoall", "reducescatter") else e_in
    # chunk q of an instance-expanded program (m > 1) is subchunk q % m of the original chunk
    # q // m: elements [floor(j*c_e/m), floor((j+1)*c_e/m)) of it (reading G3)
    ce = chunk_elems(prog.coll, n, p // m, count)
    if bf16 not in ("partials", "per_step"):
        raise ValueError(bf16)
    partials = dtype == "bfloat16" and bf16 == "partials"

    def span(q):
        if m == 1:
            return q * ce, (q + 1) * ce
        k, j = divmod(q, m)
        return k * ce + (j * ce) // m, k * ce + ((j + 1) * ce) // m
    bufs = []
    for g in prog.gpus:
        x = np.ascontiguousarray(inputs[g.id], dtype=np_dt)
        if x.size != g.i_chunks // m * ce:
            raise ValueError(f"rank {g.id}: input has {x.size} elements, want {g.i_chunks // m * ce}")
        o = np.full(g.o_chunks // m * ce * x.itemsize, 0xA5, np.uint8).view(np_dt)
        s = np.full(g.s_chunks // m * ce * x.itemsize, 0xA5, np.uint8).view(np_dt)
        bufs.append({"i": x, "o": o, "s": s})
    part = {}  # partials mode: id(buffer array) -> {chunk: fp32 partial of that chunk}

    def read_bits(buf, off, cnt):
        return np.concatenate([buf[slice(*span(q))] for q in range(off, off + cnt)])

    def read(buf, off, cnt, where):
        bits = read_bits(buf, off, cnt)
        if not partials:
            return bits
        have = part.get(id(buf), {})
        if all(q in have for q in range(off, off + cnt)):
            return _Val(bits, np.concatenate([have[q] for q in range(off, off + cnt)]))
        return _Val(bits, None)

    def write(buf, off, cnt, vals):
        bits = vals.bits if partials else vals
        at = 0
        for q in range(off, off + cnt):
            a, b = span(q)
            buf[a:b] = bits[at:at + b - a]
            if partials:
                have = part.setdefault(id(buf), {})
                if isinstance(vals, _Reduced):  # an rrc's result: keep its fp32 accumulator
                    have[q] = vals.part[at:at + b - a].copy()
                else:  # r / cpy: bf16 bits only
                    have.pop(q, None)
            at += b - a

    def reduce(mine, got, where):
        if not partials:
            return add(mine, got, dtype)
        a = mine.part if mine.part is not None else bf16_to_f32(mine.bits)
        b = got.part if got.part is not None else bf16_to_f32(got.bits)
        with np.errstate(over="ignore", invalid="ignore"):
            acc = (a + b).astype(np.float32)  # one IEEE binary32 add, RNE
        return _Reduced(bf16_round(acc), acc)

    def mreduce(vals, where):
        """mr (reading N1): the switch sums every rank's bits in one reduction —
        int32 wraps, float32 adds (rank order), bfloat16 accumulates in fp32 (rank order) and
        rounds once (multimem.ld_reduce .acc::f32). Partials are not visible to the switch:
        it reads and writes bf16 bits only."""
        bits = [x.bits if partials else x for x in vals]
        if dtype == "int32":
            acc = np.zeros(bits[0].size, np.uint32)
            for x in bits:
                acc = acc + x.view(np.uint32)
            res = acc.view(np.int32)
        elif dtype == "float32":
            acc = bits[0].astype(np.float32).copy()
            with np.errstate(over="ignore", invalid="ignore"):
                for x in bits[1:]:
                    acc = (acc + x).astype(np.float32)
            res = acc
        else:
            acc = bf16_to_f32(bits[0]).copy()
            with np.errstate(over="ignore", invalid="ignore"):
                for x in bits[1:]:
                    acc = (acc + bf16_to_f32(x)).astype(np.float32)
            res = bf16_round(acc)
        return _Val(res, None) if partials else res

    _execute(prog, graph, order, bufs, read, write, reduce, mreduce)
    return [b["o"] for b in bufs]
