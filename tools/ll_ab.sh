#!/bin/bash
# A/B at n=2 (graph replay): build/libtaccl_head.so (the last commit's library) vs the working
# tree's library, two interleaved reps each; sizes 2^LO..2^HI; then the GPU tests.
LO=${1:-10}; HI=${2:-21}; COLLS=${3:-allgather,allreduce,reducescatter}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558"
i=0
for lib in build/libtaccl_head.so "" build/libtaccl_head.so ""; do
  i=$((i+1)); rm -f gpurun_out/llr_$i.jsonl
  TACCL_LIB=$lib timeout 400 $TR tools/sweep.py --graph --colls $COLLS --size-lo $LO --size-hi $HI --algos direct,auto --no-nccl --out gpurun_out/llr_$i.jsonl > gpurun_out/llr_$i.log 2>&1
  echo "== lib=$lib"; python tools/show_sweep.py gpurun_out/llr_$i.jsonl
done
[ -n "$SKIP_TESTS" ] || { timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ll.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_ll.log; }
