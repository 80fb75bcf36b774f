#!/bin/bash
# Round-2 measurements on a 4-GPU box (gpurun --gpus 4): NVLink probe (direction +
# connection count), the alpha-beta profiler through the executor (2 ranks), and the default
# set vs NCCL sweeps (graph-replayed and eager) with the CPU oracle timed per point.
mkdir -p gpurun_out
tag=${1:-r2m}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/nvlink_probe tools/nvlink_probe.cu && \
  timeout 600 /tmp/nvlink_probe > gpurun_out/nvlink_probe_$tag.jsonl 2> gpurun_out/nvlink_probe_$tag.err; echo "probe rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29611 tools/ab_profile.py \
  --out gpurun_out/alphabeta_$tag.json --probe gpurun_out/nvlink_probe_$tag.jsonl > gpurun_out/ab_profile_$tag.log 2>&1; echo "ab rc=$?"; tail -1 gpurun_out/ab_profile_$tag.log
for mode in graph eager; do
  flag=""; [ $mode = graph ] && flag="--graph"
  timeout 1500 $TR --nproc-per-node 4 --master-port 29612 tools/sweep.py $flag --algos auto --oracle-cap $((64<<20)) \
    --out gpurun_out/sweep_n4_${mode}_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n4_${mode}_$tag.err; echo "sweep n4 $mode rc=$?"
done
timeout 900 $TR --nproc-per-node 4 --master-port 29613 tools/sweep.py --graph --colls allreduce --dtype float32 \
  --size-lo 24 --size-hi 30 --algos direct,ring,ring_p2,auto --out gpurun_out/sweep_n4_fp32_ar_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n4_fp32_ar_$tag.err; echo "sweep fp32 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 $TR --nproc-per-node 2 --master-port 29614 tools/sweep.py --graph --algos auto --oracle-cap $((64<<20)) \
  --out gpurun_out/sweep_n2_graph_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n2_graph_$tag.err; echo "sweep n2 rc=$?"
python tools/show_sweep.py gpurun_out/sweep_n4_graph_$tag.jsonl | head -90
