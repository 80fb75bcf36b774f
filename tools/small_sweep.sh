#!/bin/bash
# small-size sweep at n GPUs (graph mode) for a few env settings: tools/small_sweep.sh N HI "ENV=a ENV2=b" "ENV=c" ...
n=$1; hi=$2; shift 2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555"
i=0
for e in "$@"; do
  i=$((i+1))
  rm -f gpurun_out/ss_$i.jsonl
  env $e timeout 600 $TR tools/sweep.py --graph --size-hi $hi --out gpurun_out/ss_$i.jsonl > gpurun_out/ss_$i.log 2>&1
  echo "== $e"; python tools/show_sweep.py gpurun_out/ss_$i.jsonl
done
