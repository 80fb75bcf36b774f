"""Literal instance expansion (test infrastructure; see oracle/__init__.py).

PAPER.md:785–789 (§6.2, "Instances"): "subdividing each chunk into n subchunks that follow
the same path as the parent chunk. All groups of instructions and their threadblocks are
duplicated n times and executed in parallel."

Reading G3: subchunk j of chunk k is the element range [floor(j*c_e/m), floor((j+1)*c_e/m))
of chunk k (c_e need not be a multiple of m: the subchunks then differ by one element) and
becomes chunk k*m + j of the expanded program (chunks_per_rank p*m, so the collective's
chunk-id layout is preserved; `Program.subchunks = m` tells `simulate.run` that chunk k' names
that element range of the original chunk k' // m rather than an equal m-th); a `cnt=q` step becomes q single-chunk steps
(instance j of its q chunks are strided, so one contiguous range cannot name them);
instance j of tb t is tb t*m + j on channel chan*m + j, and a dependency on step k of tb t
becomes a dependency on the last expanded step of k in the same instance.
The invariant test: the expanded program's outputs equal the original's, bit for bit.
"""
from __future__ import annotations

import copy

from .ef import TB, Gpu, Program, Step


def expand_instances(prog: Program) -> Program:
    m = prog.instances
    if m == 1:
        return copy.deepcopy(prog)
    out = Program(prog.name + f"_x{m}", prog.coll, prog.nranks, prog.chunks_per_rank * m, 1,
                  prog.min_bytes, prog.max_bytes, prog.inplace, subchunks=prog.subchunks * m)
    if prog.subchunks != 1:
        raise ValueError("expand_instances: the program is already expanded")
    for g in prog.gpus:
        ng = Gpu(g.id, g.i_chunks * m, g.o_chunks * m, g.s_chunks * m)
        # last expanded index of every original step
        last = {}
        for tb in g.tbs:
            k2 = -1
            for st in tb.steps:
                k2 += max(1, st.cnt) if st.type != "nop" else 1
                last[(tb.id, st.s)] = k2
        tbs = {}
        for tb in g.tbs:
            for j in range(m):
                ntb = TB(tb.id * m + j, tb.send, tb.recv, tb.chan * m + j)
                for st in tb.steps:
                    deps = [(t * m + j, last[(t, k)]) for (t, k) in st.deps]
                    if st.type == "nop":
                        ntb.steps.append(Step(len(ntb.steps), "nop", deps=deps))
                        continue
                    for q in range(st.cnt):
                        ns = Step(len(ntb.steps), st.type, cnt=1, deps=deps if q == 0 else [])
                        if st.srcbuf is not None:
                            ns.srcbuf, ns.srcoff = st.srcbuf, (st.srcoff + q) * m + j
                        if st.dstbuf is not None:
                            ns.dstbuf, ns.dstoff = st.dstbuf, (st.dstoff + q) * m + j
                        ntb.steps.append(ns)
                tbs[ntb.id] = ntb
        ng.tbs = [tbs[t] for t in sorted(tbs)]
        out.gpus.append(ng)
    return out
