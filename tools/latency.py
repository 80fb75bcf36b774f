#!/usr/bin/env python
"""Per-call device time of tiny collectives under CUDA-graph replay (no host overhead):
n=1 copy path and emulated n-rank schedules on cuda:0, plus an empty torch kernel for scale."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402


def graph_time(fn, iters=200):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters):
            fn(s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


x = torch.zeros(256, device="cuda")
print(f"torch add_ (1 small kernel): {graph_time(lambda s: x.add_(1)):.2f} us")
for coll, algo, n in (("allgather", "direct", 1), ("allgather", "direct", 2), ("allreduce", "direct", 2),
                      ("allgather", "direct", 4), ("allreduce", "direct", 4)):
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=16 << 20)
    comm.load(generate(coll, algo, n, 1, 1))
    count = 512 if coll == "allreduce" else 512 // n
    ins = [torch.zeros(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    outs = [torch.zeros(count * (n if coll == "allgather" else 1), dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    t = graph_time(lambda s: comm.run_emulated(coll, outs, ins, stream=s))
    print(f"{coll} {algo} n={n} (emulated, 1 KB): {t:.2f} us  plan={comm.plan_info(coll, count, taccl.BFLOAT16)}")
    comm.destroy()
