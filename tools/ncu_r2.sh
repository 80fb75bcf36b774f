#!/bin/bash
# Round-2 ncu captures on one GPU (emulated ranks): the pulled-chain ReduceScatter plan (1 GiB,
# 4 ranks: 256 MiB chunks >= the 64 MiB threshold), the LL kernel's fp32-partials path (bf16
# ring Allreduce, 64 KiB, 4 ranks), and a 4-rank Alltoall 256 MiB per rank. Each ncu run
# follows the same command's plain run (&&); summaries go to profiles/ via tools/ncu_summary.py.
tag=${1:-r02}
mkdir -p gpurun_out
RS="python tools/emu_time.py --coll reducescatter --algo direct --n 4 --bytes 1073741824 --iters 3"
$RS > gpurun_out/plain_rs_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_rs_pc_$tag $RS > gpurun_out/ncu_rs_pc_$tag.log 2>&1
echo "rs rc=$?"; cat gpurun_out/plain_rs_$tag.log
LL="python tools/emu_time.py --coll allreduce --algo ring --n 4 --bytes 65536 --iters 20"
$LL > gpurun_out/plain_llring_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 10 -c 1 -o gpurun_out/prof_llring_$tag $LL > gpurun_out/ncu_llring_$tag.log 2>&1
echo "ll ring rc=$?"; cat gpurun_out/plain_llring_$tag.log
A2A="python tools/emu_time.py --coll alltoall --algo direct --n 4 --bytes 268435456 --iters 3"
$A2A > gpurun_out/plain_a2a_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_a2a_$tag $A2A > gpurun_out/ncu_a2a_$tag.log 2>&1
echo "a2a rc=$?"; cat gpurun_out/plain_a2a_$tag.log
