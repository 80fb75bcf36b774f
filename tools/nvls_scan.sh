#!/bin/bash
# multicast-reduce knob scan at n=4 (gpurun --gpus 4): unroll, CTAs, min piece; AR bf16 16 MiB - 1 GiB
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
out=gpurun_out/nvls_scan_${1:-s}.txt; : > $out
for env in ${ENVS:-"base" "TACCL_NO_LEAN_MR=1" "TACCL_MR_CTAS_PER_SM=1" "TACCL_MR_CTAS_PER_SM=3" "TACCL_MR_CTAS_PER_SM=4"}; do
  e=$env; [ $e = base ] && e="X=1"
  env $e timeout 300 $TR --master-port 29641 tools/sweep.py --graph --pool --colls allreduce --size-lo ${LO:-20} --size-hi 30 $( [ $env = base ] || echo --no-nccl ) \
    --algos nvls --out gpurun_out/nvls_scan_tmp.jsonl > /dev/null 2>&1
  echo "== $env" >> $out
  python tools/show_sweep.py gpurun_out/nvls_scan_tmp.jsonl >> $out; rm -f gpurun_out/nvls_scan_tmp.jsonl
done
cat $out
