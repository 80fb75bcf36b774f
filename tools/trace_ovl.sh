#!/bin/bash
# RS/AR n=4 device timelines, paired vs overlap="1" pairs (gpurun --gpus 4): BYTES, COLL
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29682"
mkdir -p gpurun_out
out=gpurun_out/trace_ovl_${1:-s}.txt; : > $out
for v in "" "--overlap"; do
  echo "== ${v:-paired}" >> $out
  timeout 300 $TR tools/trace.py --coll ${COLL:-reducescatter} --algo direct --bytes ${BYTES:-67108864} --summary --calls 3 $v 2>&1 \
    | grep -v "^\[W\|NCCL version\|OMP_NUM\|^\*\*\*" >> $out
done
cat $out
