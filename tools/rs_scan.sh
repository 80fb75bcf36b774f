#!/bin/bash
# ReduceScatter bf16 n=4 variants at 16 MiB - 1 GiB (gpurun --gpus 4): schedules x env knobs
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
out=gpurun_out/rs_scan_${1:-s}.txt; : > $out
for env in "base" "TACCL_PULL_KINDS=5" "TACCL_TARGET_CTAS=128" "TACCL_MIN_PIECE=262144" "TACCL_STRIPE=16384"; do
  e=$env; [ $e = base ] && e="X=1"
  env $e timeout 600 $TR --master-port 29651 tools/sweep.py --graph --colls reducescatter --size-lo 24 --size-hi 30 \
    $( [ $env = base ] || echo --no-nccl ) --algos direct,direct_split,direct_p2 --out gpurun_out/rs_scan_tmp.jsonl > /dev/null 2>&1
  echo "== $env" >> $out
  python tools/show_sweep.py gpurun_out/rs_scan_tmp.jsonl >> $out; rm -f gpurun_out/rs_scan_tmp.jsonl
done
cat $out
