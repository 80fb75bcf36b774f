#!/bin/bash
# LL latency evidence at n=2: per-step device timeline of AG/AR 1 KB (taccl_trace), the
# launch+prologue probe (TACCL_COPY_VARIANT=20) and an empty-kernel graph baseline.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29559"
for c in "allgather --algo direct" "allreduce --algo oneshot"; do
  timeout 120 $TR tools/trace.py --coll $c --bytes 1024 --calls 3 2>&1 | grep -v "^\*\|OMP\|NCCL\|^W1"
done
python - <<'PY'
import torch
x = torch.zeros(256, device="cuda"); s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): x.add_(1)
torch.cuda.synchronize(); g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(200): x.add_(1)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s); g.replay(); e1.record(s); torch.cuda.synchronize()
print(f"empty-ish kernel (torch add_ 256 elts) graph replay: {e0.elapsed_time(e1)*1e3/200:.2f} us/launch")
PY
TACCL_COPY_VARIANT=20 TACCL_TIMEOUT_S=3 timeout 300 $TR tools/sweep.py --graph --colls allgather --size-lo 10 --size-hi 10 --algos direct --no-nccl --out gpurun_out/llt_20.jsonl > /dev/null 2>&1
echo "variant 20 (launch + prologue + exit):"; python tools/show_sweep.py gpurun_out/llt_20.jsonl
