#!/bin/bash
# C3 (BASELINE configs[2]) grid at n=4 (gpurun --gpus 4): Alltoall, chunk partitioning p in
# {1,2,4} x instances m in {1,4,8}, 1 KB - 1 GB, graph-replayed, with NCCL
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
tag=${1:-c3}
timeout 1500 $TR --master-port 29661 tools/sweep.py --graph --colls alltoall \
  --algos direct,direct_p2,direct_p4,direct_m4,direct_p2_m4,direct_p4_m4,direct_m8,direct_p2_m8,direct_p4_m8 \
  --out gpurun_out/c3_grid_n4_$tag.jsonl > /dev/null 2> gpurun_out/c3_grid_n4_$tag.err; echo "c3 rc=$?"
python tools/show_sweep.py gpurun_out/c3_grid_n4_$tag.jsonl
