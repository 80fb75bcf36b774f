#!/bin/bash
# More 1-GPU ncu captures (emulated ranks on cuda:0; DRAM traffic of the local side):
# one large and one small size for Alltoall, Allreduce and ReduceScatter.
tag=${1:-r01}
mkdir -p gpurun_out
cap() {  # name, emu_time args
  local name=$1; shift
  python tools/emu_time.py "$@" --iters 5 > gpurun_out/plain_${name}_$tag.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_${name}_$tag python tools/emu_time.py "$@" --iters 5 > gpurun_out/ncu_${name}_$tag.log 2>&1
  echo "$name rc=$?"; cat gpurun_out/plain_${name}_$tag.log
}
cap a2a_big --coll alltoall --algo direct --n 4 --bytes 268435456
cap a2a_small --coll alltoall --algo direct --n 4 --bytes 65536
cap ar_small --coll allreduce --algo oneshot --n 4 --bytes 1024
cap rs_small --coll reducescatter --algo direct --n 4 --bytes 65536
