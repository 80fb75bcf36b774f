#!/bin/bash
# ncu of the warp-specialised pairs (overlap="1") vs the plain paired schedule: emulated RS n=4,
# 256 MiB per rank, one GPU. Plain runs first (&&), summaries via tools/ncu_summary.py.
tag=${1:-r02}
mkdir -p gpurun_out
for v in "" "--overlap"; do
  name=rs_plain; [ -n "$v" ] && name=rs_ovl
  C="python tools/emu_time.py --coll reducescatter --algo direct --n 4 --bytes 1073741824 --iters 3 $v"
  $C > gpurun_out/plain_${name}_$tag.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_${name}_$tag $C > gpurun_out/ncu_${name}_$tag.log 2>&1
  echo "$name rc=$?"; cat gpurun_out/plain_${name}_$tag.log
done
