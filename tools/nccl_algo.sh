#!/bin/bash
# Which algorithm/protocol NCCL 2.28.9 picks for the comparator runs (pool buffers, n=4):
# NCCL_DEBUG=INFO COLL lines for 64 MiB and 1 GiB of each collective.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING,COLL timeout 600 $TR --master-port 29681 tools/sweep.py --pool --colls allreduce,allgather,alltoall,reducescatter \
  --size-lo 26 --size-hi 26 --algos auto --out gpurun_out/nccl_algo_tmp.jsonl > gpurun_out/nccl_algo_raw.log 2>&1
grep -iE "NVLS|algo|CollNet|nChannels" gpurun_out/nccl_algo_raw.log | grep -v "^\s*$" | sort | uniq -c | sort -rn | head -40
