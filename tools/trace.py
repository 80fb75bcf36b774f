#!/usr/bin/env python
"""Per-step device timeline of one collective call (taccl_trace; SURVEY.md §5 tracing).

  python tools/trace.py --coll allgather --algo direct --n 2 --bytes 1024 [--emulated]
  torchrun --nproc-per-node 2 tools/trace.py --coll allreduce --bytes 1024

Runs a few warm calls, then one traced call, and prints for every CTA (first piece) the
%globaltimer stamps relative to the earliest kernel entry over all ranks: prologue end, and
per step start / waits satisfied / done, and exit (microseconds)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--coll", default="allgather")
ap.add_argument("--algo", default="direct")
ap.add_argument("--n", type=int, default=2)
ap.add_argument("--chunks", type=int, default=1)
ap.add_argument("--bytes", type=int, default=1024)
ap.add_argument("--emulated", action="store_true")
ap.add_argument("--calls", type=int, default=1, help="traced back-to-back calls (last one shown)")
ap.add_argument("--pair", default="1", help="1 (default pairing), peer, or split (sends and receives in separate tbs)")
ap.add_argument("--summary", action="store_true", help="per (rank, tb): median of every stamp instead of every CTA")
ap.add_argument("--overlap", action="store_true", help='the overlap="1" hint (warp-specialised pairs)')
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
n = a.n if a.emulated or world == 1 else world
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
emu = world == 1
comm = taccl.Comm(rank=rank, nranks=n, device=torch.cuda.current_device(), emulated=emu, scratch_bytes=64 << 20)
comm.load(generate(a.coll, a.algo, n, a.chunks, 1, pair={"1": True, "peer": "peer", "split": False}[a.pair],
                   overlap=a.overlap))
es = 2
S = a.bytes
count = {"allgather": S // es // n, "alltoall": S // es // n, "allreduce": S // es,
         "reducescatter": S // es // n}[a.coll]
e_in = n * count if a.coll in ("alltoall", "reducescatter") else count
e_out = n * count if a.coll in ("allgather", "alltoall") else count
nl = n if emu else 1
ins = [torch.ones(e_in, dtype=torch.bfloat16, device="cuda") for _ in range(nl)]
outs = [torch.empty(e_out, dtype=torch.bfloat16, device="cuda") for _ in range(nl)]
if not emu:  # registration is explicit and collective
    comm.register(outs[0])
    comm.register(ins[0])


def call():
    if emu:
        comm.run_emulated(a.coll, outs, ins)
    else:
        comm.run(a.coll, outs[0], ins[0])


for _ in range(5):
    call()
torch.cuda.synchronize()
buf = torch.zeros(4096 * taccl.TRACE_SLOTS, dtype=torch.int64, device="cuda")
if world > 1:
    dist.barrier()
comm.trace(buf)
for _ in range(a.calls):
    call()
torch.cuda.synchronize()
comm.trace(None)
comm.check()
info = comm.plan_info(a.coll, count, taccl.BFLOAT16)
grid = info["ctas"]  # emulated: already every rank's CTAs
T = buf[:grid * taccl.TRACE_SLOTS].view(grid, taccl.TRACE_SLOTS).cpu()
if world > 1:
    allT = [None] * world
    dist.all_gather_object(allT, T)
    T = torch.cat(allT)
T = T[T[:, 0] > 0]
# %globaltimer is per GPU: stamps are shown relative to the earliest entry on the same rank
ranks_of = (T[:, -2] >> 32)
t0s = {int(r): int(T[ranks_of == r, 0].min()) for r in ranks_of.unique()}
nsteps = (taccl.TRACE_SLOTS - 4) // 4
if rank == 0:
    print(f"{a.coll} {a.algo} n={n} S={S} B plan={info} (us from the earliest entry)")
    rows = T.tolist()
    if a.summary:  # one line per (rank, tb): the median over its CTAs of every stamp
        groups = {}
        for row in rows:
            groups.setdefault((row[-2] >> 32, (row[-2] >> 16) & 0xFFFF), []).append(row)
        rows = []
        for (r, tb), g in sorted(groups.items()):
            med = torch.tensor(g, dtype=torch.float64).median(dim=0).values.long().tolist()
            med[-2] = (r << 32) | (tb << 16) | 0xFFFF
            rows.append(med)
    for row in rows:
        ident = row[-2]
        r, tb, j = ident >> 32, (ident >> 16) & 0xFFFF, ident & 0xFFFF
        t0 = t0s[r]

        def us(x):
            return f"{(x - t0) / 1e3:6.2f}" if x else "   -  "
        steps = []
        for k in range(nsteps):
            s0, s1, s2, s3 = row[2 + 4 * k], row[3 + 4 * k], row[4 + 4 * k], row[5 + 4 * k]
            if not s0:
                break
            steps.append(f"s{k}[{us(s0)} w{us(s1)}" + (f" x{us(s2)}" if s2 else "") + f" d{us(s3)}]")
        jj = "med" if j == 0xFFFF else f"j{j}"
        print(f"r{r} tb{tb} {jj}: entry {us(row[0])} pro {us(row[1])} " + " ".join(steps) + f" exit {us(row[-1])}")
comm.destroy()
if world > 1:
    dist.destroy_process_group()
