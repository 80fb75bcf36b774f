#!/usr/bin/env python
"""Check the NVML NVLink counters against a known transfer: 8 x 1 GiB peer copies GPU0 -> GPU1
(expect ~8 GiB tx on GPU0 and rx on GPU1)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import nvlink_counters as nc

a = torch.empty(1 << 28, dtype=torch.int32, device="cuda:0")
b = torch.empty(1 << 28, dtype=torch.int32, device="cuda:1")
b.copy_(a)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
c0 = [nc.read(d) for d in range(2)]
for _ in range(8):
    b.copy_(a)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
c1 = [nc.read(d) for d in range(2)]
print("fields:", c0[0] and c0[0]["field"])
for d in range(2):
    if c0[d] and c1[d]:
        print(f"gpu{d}: tx {(c1[d]['tx'] - c0[d]['tx']) / 2**30:.3f} GiB  rx {(c1[d]['rx'] - c0[d]['rx']) / 2**30:.3f} GiB (expected 8 GiB one way)")
    else:
        print(f"gpu{d}: counters unavailable", c0[d], c1[d])
