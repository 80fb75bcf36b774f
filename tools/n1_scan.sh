#!/bin/bash
# N=1 copy-path knob scan (gpurun, 1 GPU): bench value per env variant, interleaved twice
for rep in 1 2; do
for env in ${ENVS:-base TACCL_TARGET_CTAS=148 TACCL_STRIPE=131072 TACCL_STRIPE=262144 TACCL_TMA=0 TACCL_LEAN_MAX=4294967296 TACCL_MIN_PIECE=1048576}; do
  e=$(echo $env | tr '+' ' '); [ "$e" = base ] && e="X=1"
  v=$(env $e timeout 300 python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])")
  echo "$env $v"
done
done
