#!/bin/bash
# LL latency probes at n=2 (graph replay; timing-only variants, results invalid): default,
# 20 = launch + prologue + exit only, 21 = no arrival wait at exit, 22 = sends skip their
# source load. usage (under gpurun --gpus 2): bash tools/ll_probe.sh
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563"
for v in 0 20 21 22 0; do
  rm -f gpurun_out/llv_$v.jsonl
  TACCL_COPY_VARIANT=$v TACCL_TIMEOUT_S=3 timeout 300 $TR tools/sweep.py --graph --colls allgather,alltoall --size-lo 10 --size-hi 12 --algos direct --no-nccl --out gpurun_out/llv_$v.jsonl > /dev/null 2>&1
  echo "== variant $v"; python tools/show_sweep.py gpurun_out/llv_$v.jsonl | awk '{print $1, $2, $3, $4}'
done
