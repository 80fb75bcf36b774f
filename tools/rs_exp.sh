#!/bin/bash
# RS large-message experiment at n GPUs (under gpurun --gpus n): paired vs split
# threadblocks, lanes (pieces per CTA), CTA targets. usage: bash tools/rs_exp.sh N TAG
n=$1; tag=${2:-rs}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541"
out=gpurun_out/rs_exp_n${n}_$tag.txt; : > $out
ENVS=${ENVS:-"base TACCL_LANES=256 TACCL_LANES=512 TACCL_TARGET_CTAS=148,TACCL_LANES=512"}
for envc in $ENVS; do
  env=$(echo $envc | tr ',' ' '); [ "$env" = base ] && env=""
  echo "== env: $env" >> $out
  rm -f gpurun_out/rs_tmp.jsonl
  env $env timeout 300 $TR tools/sweep.py --colls ${COLLS:-reducescatter} --size-lo ${SIZE_LO:-24} --size-hi ${SIZE_HI:-30} --graph --no-nccl \
     --algos ${ALGOS:-direct,direct_split} --out gpurun_out/rs_tmp.jsonl > gpurun_out/rs_tmp.log 2>&1 || tail -5 gpurun_out/rs_tmp.log >> $out
  python - >> $out <<'PY'
import json
for l in open("gpurun_out/rs_tmp.jsonl"):
    r = json.loads(l)
    print(r["coll"], r["S"], " ".join(f'{k[6:-6]}={v:.0f}' for k, v in r.items() if k.startswith("taccl_") and k.endswith("_busbw")),
          "us:", " ".join(f'{k[6:-3]}={v:.1f}' for k, v in r.items() if k.startswith("taccl_") and k.endswith("_us") and "best" not in k))
PY
done
cat $out
