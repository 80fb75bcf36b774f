"""Mutation operators for schedule-checker tests (tests/golden/mutations.txt)."""
import copy



def _renumber(tb):
    for k, st in enumerate(tb.steps):
        st.s = k


def apply(prog, op):
    """Return a mutated deep copy of an oracle Program. `op` is a mutations.txt op string."""
    p = copy.deepcopy(prog)
    w = op.split()
    if w[0] == "delete":
        r, t, k = map(int, w[1:4])
        g = p.gpus[r]
        del g.tbs[t].steps[k]
        for tb in g.tbs:
            for st in tb.steps:
                nd = []
                for (dt, dk) in st.deps:
                    if dt == t and dk == k:
                        continue
                    nd.append((dt, dk - 1 if (dt == t and dk > k) else dk))
                st.deps = nd
        _renumber(g.tbs[t])
    elif w[0] == "swap":
        r, t, a, b = map(int, w[1:5])
        steps = p.gpus[r].tbs[t].steps
        steps[a], steps[b] = steps[b], steps[a]
        _renumber(p.gpus[r].tbs[t])
    elif w[0] == "set":
        r, t, k = map(int, w[1:4])
        attr, val = w[4], w[5]
        st = p.gpus[r].tbs[t].steps[k]
        if attr == "deps":
            st.deps = [] if val == "-" else [tuple(map(int, x.split(":"))) for x in val.split(",")]
        elif attr == "type":
            st.type = val
            if val in ("r",):
                st.srcbuf = None
            if val in ("s",):
                st.dstbuf = None
        elif attr in ("srcbuf", "dstbuf"):
            setattr(st, attr, val)
        else:
            setattr(st, attr, int(val))
    elif w[0] == "settb":
        r, t = map(int, w[1:3])
        setattr(p.gpus[r].tbs[t], w[3], int(w[4]))
    else:
        raise ValueError(op)
    return p


def load_mutations(text):
    out = []
    for line in text.splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f, op, sem, direct, cite = [x.strip() for x in line.split("|")]
        out.append((f, op, sem, direct, cite))
    return out
