#!/bin/bash
# RS/AR n=4 device timelines (gpurun --gpus 4): CFGS = "pair,ENV=V,..." entries (pair: 1 | peer | split)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29681"
mkdir -p gpurun_out
out=gpurun_out/trace_rs_${1:-s}.txt; : > $out
for cfg in ${CFGS:-1 split}; do
  pair=${cfg%%,*}; envs=$( [ "$cfg" = "$pair" ] || echo ${cfg#*,} | tr , ' ')
  echo "== pair=$pair $envs" >> $out
  env X=1 $envs timeout 300 $TR tools/trace.py --coll ${COLL:-reducescatter} --algo direct --bytes ${BYTES:-67108864} \
    --pair $pair --summary --calls 3 2>&1 | grep -v "^\[W\|NCCL version\|OMP_NUM\|^\*\*\*" >> $out
done
cat $out
