#!/bin/bash
# env-knob scan at n=4 (gpurun --gpus 4): COLLS, ALGOS, sizes LO..HI, ENVS list (A=1,B=2 sets two)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
out=gpurun_out/knob_scan_${1:-s}.txt; : > $out
for env in ${ENVS:-base}; do
  e=${env//,/ }; [ "$e" = base ] && e="X=1"
  env $e timeout 600 $TR --master-port 29671 tools/sweep.py --graph $POOL ${DTYPE:+--dtype $DTYPE} --colls ${COLLS:-reducescatter} --size-lo ${LO:-24} --size-hi ${HI:-28} ${SIZES:+--sizes $SIZES} \
    $( [ $env = base ] || echo --no-nccl ) --algos ${ALGOS:-direct} --out gpurun_out/knob_tmp.jsonl > /dev/null 2>&1
  echo "== $env" >> $out
  python tools/show_sweep.py gpurun_out/knob_tmp.jsonl >> $out; rm -f gpurun_out/knob_tmp.jsonl
done
cat $out
