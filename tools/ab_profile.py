#!/usr/bin/env python
"""The paper's alpha-beta profiler on B200 NVLink 5, through this executor (SURVEY.md §8(f)
row 3; §4.1):

  torchrun --nproc-per-node 2 tools/ab_profile.py [--out profiles/r02_alphabeta.json]
           [--probe profiles/r02_nvlink_probe.jsonl]

For k in {2, 4, 8} chunks of s bytes (s = 1 KiB .. 64 MiB): a 2-rank Allgather with k chunks
per rank whose chunks travel one after another (k send steps: generate(..., merge=False)) and
all at once (one k-chunk step: the default lowering's contiguity), graph-replayed, max over
ranks. The executor picks its protocol by message size (LL lines up to 2 MiB of output, the
zero-copy kernel above), so alpha and beta are fitted per protocol with
generator.profiler.solve_alpha_beta. With --probe, the connection-count sweep of
tools/nvlink_probe.cu (fig:multiconnection) is summarised alongside.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402
from paper_2111_04867_b200.generator.profiler import connection_table, solve_alpha_beta  # noqa: E402
from sweep import timeit_graph  # noqa: E402

LL_MAX = 2 << 20  # TACCL_STAGED_MAX default for Allgather (runtime.cpp geometry)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "alphabeta.json"))
    ap.add_argument("--probe", default=None, help="nvlink_probe JSON lines to summarise")
    ap.add_argument("--lo", type=int, default=10)
    ap.add_argument("--hi", type=int, default=26)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == 2, "one link: 2 ranks"
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kmax, smax = 8, 1 << a.hi
    comm = taccl.Comm(rank=rank, nranks=2, device=local, scratch_bytes=64 << 20)
    inp = torch.empty(kmax * smax // 2, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(2 * kmax * smax // 2, dtype=torch.bfloat16, device="cuda")
    comm.register(out)
    comm.register(inp)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    meas = []
    for k in (2, 4, 8):
        texts = {"seq": generate("allgather", "direct", 2, k, 1, merge=False),
                 "tog": generate("allgather", "direct", 2, k, 1)}
        for e in range(a.lo, a.hi + 1):
            s = 1 << e
            count = k * s // 2
            x, y = inp[:count], out[:2 * count]
            for mode, text in texts.items():
                h = comm.load(text)
                ms, _ = timeit_graph(lambda: comm.run("allgather", y, x, stream), stream, world)
                comm.free(h)
                proto = "ll" if 2 * count * 2 <= LL_MAX else "direct"
                meas.append({"mode": mode, "k": k, "chunk_bytes": s, "us": round(ms * 1e3, 3), "protocol": proto})
                if rank == 0:
                    print(json.dumps(meas[-1]), flush=True)
    comm.check()
    if rank == 0:
        fits = {}
        for proto in ("ll", "direct"):
            pts = [(m["mode"], m["k"], m["chunk_bytes"] / (1 << 20), m["us"]) for m in meas if m["protocol"] == proto]
            if len(pts) >= 3:
                fits[proto] = solve_alpha_beta(pts)
        res = {"what": "alpha-beta of one NVLink 5 connection through this executor (2 ranks, both directions "
                       "busy), PAPER.md:540-546 method: k chunks one after another vs all at once",
               "fits": fits, "measurements": meas}
        if a.probe and os.path.exists(a.probe):
            rows = [json.loads(l) for l in open(a.probe) if l.strip().startswith("{")]
            res["direction"] = [r for r in rows if r.get("probe") == "direction"]
            res["connections"] = connection_table(rows)
            res["connections_small"] = connection_table(rows, volume=min(r["volume_bytes"] for r in rows
                                                                          if r.get("probe") == "connections"))
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(fits))
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
