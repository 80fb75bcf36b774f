"""CLI: python -m paper_2111_04867_b200.generator --coll allgather --algo ring --nranks 8
   --chunks 2 --instances 4 [-o out.xml]  (flag names mirror the sketch hyperparameters,
   PAPER.md:1311-1314)."""
import argparse
import sys

from . import generate


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--coll", required=True, choices=["allgather", "alltoall", "allreduce", "reducescatter"])
    ap.add_argument("--algo", default="direct", choices=["ring", "direct", "hier", "greedy", "milp", "oneshot"])
    ap.add_argument("--nranks", type=int, required=True)
    ap.add_argument("--chunks", type=int, default=1, help="input_chunkup p")
    ap.add_argument("--instances", type=int, default=1)
    ap.add_argument("--policy", default=None, choices=[None, "uc-max", "uc-min"])
    ap.add_argument("--topology", default=None, help="greedy/milp: nvswitch (default) or 2xK")
    ap.add_argument("--size", type=int, default=None, help="greedy/milp: input_size bytes for the cost model")
    ap.add_argument("--min-bytes", type=int, default=0)
    ap.add_argument("--max-bytes", type=float, default=float("inf"))
    ap.add_argument("-o", "--out", default="-")
    a = ap.parse_args(argv)
    kw = {"policy": a.policy} if a.policy else {}
    if a.topology:
        kw["topology"] = a.topology
    if a.size:
        kw["size"] = a.size
    text = generate(a.coll, a.algo, a.nranks, a.chunks, a.instances, a.min_bytes, a.max_bytes, **kw)
    (sys.stdout if a.out == "-" else open(a.out, "w")).write(text)


if __name__ == "__main__":
    main()
