#!/bin/bash
# A/B at n=2 (graph replay, LL sizes): HEAD library vs the working tree's library; then GPU tests
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558"
i=0
for lib in build/libtaccl_head.so "" build/libtaccl_head.so ""; do
  i=$((i+1)); rm -f gpurun_out/llr_$i.jsonl
  TACCL_LIB=$lib timeout 400 $TR tools/sweep.py --graph --colls allgather,allreduce,reducescatter --size-lo 10 --size-hi 21 --algos direct,auto --no-nccl --out gpurun_out/llr_$i.jsonl > gpurun_out/llr_$i.log 2>&1
  echo "== lib=$lib"; python tools/show_sweep.py gpurun_out/llr_$i.jsonl
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ll.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_ll.log
