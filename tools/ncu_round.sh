#!/bin/bash
# 1-GPU ncu evidence for the current kernels (under gpurun): launch list of the bench, full
# captures of the bench copy kernel, an emulated 4-rank Allreduce (reduce path) and an LL
# small Allgather. Each ncu run follows the same command's plain run (&&).
tag=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
AR="python tools/emu_time.py --coll allreduce --algo direct --n 4 --bytes 268435456 --iters 3"
LL="python tools/emu_time.py --coll allgather --algo direct --n 2 --bytes 65536 --iters 20"
$B > gpurun_out/plain_b_$tag.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$tag.csv $B > /dev/null 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_ -s 5 -c 1 -o gpurun_out/prof_copy_$tag $B > gpurun_out/ncu_copy_$tag.log 2>&1
echo "copy rc=$?"
$AR > gpurun_out/plain_ar_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_ar_$tag $AR > gpurun_out/ncu_ar_$tag.log 2>&1
echo "ar rc=$?"; cat gpurun_out/plain_ar_$tag.log
$LL > gpurun_out/plain_ll_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 10 -c 1 -o gpurun_out/prof_ll_$tag $LL > gpurun_out/ncu_ll_$tag.log 2>&1
echo "ll rc=$?"; cat gpurun_out/plain_ll_$tag.log
# ReduceScatter n=2 emulated, 256 MiB send bytes: pull mode (default for RS) and push mode —
# DRAM bytes per launch vs the algorithmic 1.5 S (pull) / 2.5 S (push) for both ranks
RS="python tools/emu_time.py --coll reducescatter --algo direct --n 2 --bytes 268435456 --iters 5"
$RS > gpurun_out/plain_rs_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_rs_pull_$tag $RS > gpurun_out/ncu_rs_pull_$tag.log 2>&1
echo "rs pull rc=$?"; cat gpurun_out/plain_rs_$tag.log
TACCL_PULL=0 $RS > gpurun_out/plain_rs0_$tag.log 2>&1 &&
TACCL_PULL=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_rs_push_$tag $RS > gpurun_out/ncu_rs_push_$tag.log 2>&1
echo "rs push rc=$?"; cat gpurun_out/plain_rs0_$tag.log
