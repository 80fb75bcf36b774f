#!/usr/bin/env python
"""Time one schedule with all ranks emulated on cuda:0 (one launch per call).
  python tools/emu_time.py --coll allreduce --algo ring --n 4 --bytes 268435456 [--iters 20] [--overlap] [--split]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--coll", default="allreduce")
ap.add_argument("--algo", default="ring")
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--chunks", type=int, default=1)
ap.add_argument("--instances", type=int, default=1)
ap.add_argument("--bytes", type=int, default=1 << 28)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--overlap", action="store_true", help='the overlap="1" hint (warp-specialised pairs)')
ap.add_argument("--split", action="store_true", help="sends and receives in separate threadblocks")
a = ap.parse_args()
n = a.n
comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=2 * a.bytes + (64 << 20))
comm.load(generate(a.coll, a.algo, n, a.chunks, a.instances, pair=not a.split, overlap=a.overlap))
es = 2
count = a.bytes // es // (1 if a.coll == "allreduce" else n)
e_in = n * count if a.coll in ("alltoall", "reducescatter") else count
e_out = count if a.coll in ("allreduce", "reducescatter") else n * count
ins = [torch.randint(-8, 8, (e_in,), device="cuda").to(torch.bfloat16) for _ in range(n)]
outs = [torch.empty(e_out, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
for _ in range(3):
    comm.run_emulated(a.coll, outs, ins)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    comm.run_emulated(a.coll, outs, ins)
e1.record()
torch.cuda.synchronize()
comm.check()
print(f"{a.coll} {a.algo} n={n} bytes={a.bytes} us/call={e0.elapsed_time(e1) * 1e3 / a.iters:.1f} plan={comm.plan_info(a.coll, count, taccl.BFLOAT16)}")
comm.destroy()
