#!/bin/bash
# run tools/sweep.py under several env settings (under gpurun): tools/envsweep.sh N "ENV1=a ENV2=b;ENV1=c" [sweep args]
n=$1; sets=$2; shift 2
IFS=';' read -ra S <<< "$sets"
for e in "${S[@]}"; do
  rm -f gpurun_out/envsweep.jsonl
  env $e timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29516 tools/sweep.py --out gpurun_out/envsweep.jsonl --no-nccl "$@" > gpurun_out/envsweep.log 2>&1 || tail -5 gpurun_out/envsweep.log
  python - "$e" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("gpurun_out/envsweep.jsonl")]
print(sys.argv[1] or "default", " ".join(f"{r['coll'][:2]}{r['S']>>20}M:" + "/".join(str(r.get(f'taccl_{a}_us')) for a in ('direct', 'ring') if f'taccl_{a}_us' in r) for r in rows))
PY
done
