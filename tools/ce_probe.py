#!/usr/bin/env python
"""Copy-engine peer bandwidth probe (one process, all visible GPUs): every GPU copies S bytes
to each of its n-1 peers at once with cudaMemcpyPeerAsync (one stream per peer), for comparison
with the SM-store connection sweep (tools/nvlink_probe.cu). Prints per-GPU egress GB/s."""
import json
import sys

import torch

n = torch.cuda.device_count()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 256 << 20
for i in range(n):
    for j in range(n):
        if i != j:
            torch.cuda.set_device(i)
            assert torch.cuda.can_device_access_peer(i, j)
src = [torch.empty(S, dtype=torch.uint8, device=f"cuda:{i}") for i in range(n)]
dst = [[torch.empty(S, dtype=torch.uint8, device=f"cuda:{j}") for j in range(n)] for _ in range(n)]
streams = [[torch.cuda.Stream(device=i) for _ in range(n)] for i in range(n)]


def run(peers):
    for i in range(n):
        for k, j in enumerate(peers(i)):
            with torch.cuda.stream(streams[i][k]):
                dst[i][j].copy_(src[i], non_blocking=True)


for conns in range(1, n):
    peers = lambda i: [(i + d) % n for d in range(1, conns + 1)]  # noqa: E731
    for _ in range(3):
        run(peers)
    for i in range(n):
        torch.cuda.synchronize(i)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    reps = 10
    for i in range(n):
        torch.cuda.set_device(i)
        ev[i][0].record(torch.cuda.current_stream(i))
        for s in streams[i]:
            s.wait_stream(torch.cuda.current_stream(i))
    for _ in range(reps):
        run(peers)
    for i in range(n):
        torch.cuda.set_device(i)
        for s in streams[i]:
            torch.cuda.current_stream(i).wait_stream(s)
        ev[i][1].record(torch.cuda.current_stream(i))
    for i in range(n):
        torch.cuda.synchronize(i)
    ms = max(ev[i][0].elapsed_time(ev[i][1]) for i in range(n)) / reps
    print(json.dumps({"probe": "copy_engine", "n_devices": n, "connections": conns, "bytes_per_connection": S,
                      "us": round(ms * 1e3, 1), "egress_GBps": round(conns * S / ms / 1e6, 1)}))
