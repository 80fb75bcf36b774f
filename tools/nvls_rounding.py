#!/usr/bin/env python
"""Which rounding does the NVSwitch's bf16 multimem.ld_reduce (.acc::f32) use when it converts
its fp32 sum back to bf16? Runs hand-picked 2-rank sums through the multicast-reduce step and
prints, per case, the observed bits next to the candidates (RNE, round-to-odd, toward zero).
torchrun --nproc-per-node 2 tools/nvls_rounding.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402

CASES = [  # (rank-0 bits, rank-1 bits, note)
    (0x3F80, 0x3B00, "1 + 2^-9: nearest below (even)"),
    (0x3F80, 0x3BC0, "1 + 1.5*2^-8: nearest above (odd)"),
    (0x3F80, 0x3B80, "1 + 2^-8: tie, even below"),
    (0x3F81, 0x3B80, "(1+2^-7) + 2^-8: tie, even above"),
    (0xBF80, 0xBB00, "-1 - 2^-9"),
    (0xBF80, 0xBB80, "-1 - 2^-8: tie"),
    (0x3F80, 0x3A80, "1 + 2^-10"),
    (0x3F81, 0x3A80, "(1+2^-7) + 2^-10"),
    (0x4000, 0x3F81, "2 + (1+2^-7) = 3 + 2^-7: below half ulp of 3"),
    (0x3F80, 0x3F80, "exact"),
]


def rne(f):
    b = np.float32(f).view(np.uint32)
    return int((b + 0x7FFF + ((b >> 16) & 1)) >> 16)


def rto(f):  # round to odd: truncate, set the last bit if inexact
    b = int(np.float32(f).view(np.uint32))
    t = b >> 16
    return t | 1 if b & 0xFFFF else t


def rtz(f):
    return int(np.float32(f).view(np.uint32)) >> 16


def main():
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    comm = taccl.Comm(rank=rank, nranks=n, device=rank, scratch_bytes=16 << 20)
    comm.create_pool(64 << 20)
    comm.load(generate("allreduce", "nvls", n, 1, 1))
    k = 8 * n * 8  # 16-byte chunks
    vals = np.zeros(k, np.uint16)
    for i, (a, b, _) in enumerate(CASES):
        vals[i] = a if rank == 0 else (b if rank == 1 else 0)
    x = comm.pool_tensor(k, torch.bfloat16)
    out = comm.pool_tensor(k, torch.bfloat16)
    x.view(torch.int16).copy_(torch.from_numpy(vals.view(np.int16)))
    comm.run("allreduce", out, x)
    torch.cuda.synchronize()
    comm.check()
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    # random U[1,2) bf16 on every rank: which rule explains every element?
    from paper_2111_04867_b200.inputs import allreduce_input
    kk = 8 * n * 4096
    ins = [allreduce_input(kk, "bfloat16", "uniform", 23, r) for r in range(n)]
    x2 = comm.pool_tensor(kk, torch.bfloat16)
    o2 = comm.pool_tensor(kk, torch.bfloat16)
    x2.view(torch.int16).copy_(torch.from_numpy(ins[rank].view(np.int16)))
    torch.cuda.synchronize()
    dist.barrier()
    comm.run("allreduce", o2, x2)
    torch.cuda.synchronize()
    g2 = o2.view(torch.int16).cpu().numpy().view(np.uint16)
    if rank == 0:
        f32 = [(v.astype(np.uint32) << 16).view(np.float32) for v in ins]
        acc = f32[0].copy()
        for v in f32[1:]:
            acc = (acc + v).astype(np.float32)
        exact = sum(v.astype(np.float64) for v in f32)
        b = acc.view(np.uint32)
        r_ne = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
        r_tz = (b >> 16).astype(np.uint16)
        r_to = np.where(b & 0xFFFF, (b >> 16) | 1, b >> 16).astype(np.uint16)
        print(f"n={n} random U[1,2): fp32 sum exact {np.mean(acc.astype(np.float64) == exact):.3f}; "
              f"got==rne {np.mean(g2 == r_ne):.4f} ==rtz {np.mean(g2 == r_tz):.4f} ==rto {np.mean(g2 == r_to):.4f}")
        bad = np.nonzero(g2 != r_tz)[0]
        for i in bad[:6]:
            print("  not rtz:", [hex(v[i]) for v in ins], "sum", exact[i], "got", hex(g2[i]), "rtz", hex(r_tz[i]), "rne", hex(r_ne[i]))
    if rank == 0:
        for i, (a, b, note) in enumerate(CASES):
            f = float((np.array([a], np.uint32) << 16).view(np.float32)[0]) + float((np.array([b], np.uint32) << 16).view(np.float32)[0])
            print(f"{note:40s} got {got[i]:04x}  rne {rne(f):04x}  rto {rto(f):04x}  rtz {rtz(f):04x}")
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
