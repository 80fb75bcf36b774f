#!/bin/bash
# RS 64 MiB n=4 device timelines (gpurun --gpus 4): paired vs split threadblocks x pieces per CTA
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29681"
mkdir -p gpurun_out
out=gpurun_out/trace_rs_${1:-s}.txt; : > $out
for cfg in "1 1" "split 1" "split 4" "1 2"; do
  set -- $cfg
  echo "== pair=$1 TACCL_PIECES_PER_CTA=$2" >> $out
  TACCL_PIECES_PER_CTA=$2 timeout 300 $TR tools/trace.py --coll ${COLL:-reducescatter} --algo direct --bytes ${BYTES:-67108864} --pair $1 --summary >> $out 2>&1
done
cat $out
