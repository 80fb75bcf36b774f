#!/bin/bash
# large-size env scan under gpurun: tools/envscan.sh N LO HI COLLS "ENV=a ENV2=b" "ENV=c" ...
n=$1; lo=$2; hi=$3; colls=$4; shift 4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29571"
i=0
for e in "$@"; do
  i=$((i+1))
  rm -f gpurun_out/es_$i.jsonl
  env $e timeout 900 $TR tools/sweep.py --graph --no-nccl --colls $colls --size-lo $lo --size-hi $hi --out gpurun_out/es_$i.jsonl > gpurun_out/es_$i.log 2>&1
  echo "== $e"; python tools/show_sweep.py gpurun_out/es_$i.jsonl | cut -c1-110
done
