#!/bin/bash
# Parameter scan helper (run under gpurun): env knob values x bench configs -> one line each.
# usage: tools/scan.sh KNOB "v1 v2 ..." NGPU [extra bench args]
knob=$1; vals=$2; n=$3; shift 3
for v in $vals; do
  if [ "$n" = "1" ]; then
    out=$(env $knob=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 1000 "$@" 2>&1 | tail -1)
  else
    out=$(env $knob=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $n --no-e2e --steps 500 "$@" 2>&1 | tail -1)
  fi
  echo "$knob=$v n=$n $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["plan"], d.get("busbw_per_gpu"))' 2>&1 | tail -1)"
done
