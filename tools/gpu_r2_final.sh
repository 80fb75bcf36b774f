#!/bin/bash
# Round-2 evidence on a 4-GPU box (gpurun --gpus 4): smoke, every GPU test, bench N=1/2/4,
# ncu (bench launch list + copy capture; emulated bf16 ring Allreduce = the fp32-partials
# reduce path), sweeps vs NCCL with pool buffers (graph + eager, n=4; graph n=2) and the CPU
# oracle per point.
mkdir -p gpurun_out
tag=${1:-r2f}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nproc > gpurun_out/host_$tag.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host_$tag.txt; free -g >> gpurun_out/host_$tag.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; echo "bench1 rc=$?"
for n in 2 4; do
  timeout 600 $TR --nproc-per-node $n --master-port 2959$n bench.py --gpus $n > gpurun_out/bench_n${n}_$tag.json 2> gpurun_out/bench_n${n}_$tag.err; echo "bench$n rc=$?"
done
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
$B > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$tag.csv $B > /dev/null 2>&1; echo "ncu launches rc=$?"
$B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_ -s 5 -c 1 -o gpurun_out/prof_copy_$tag $B > gpurun_out/ncu_copy_$tag.log 2>&1; echo "ncu copy rc=$?"
AR="python tools/emu_time.py --coll allreduce --algo ring --n 4 --bytes 268435456 --iters 3"
$AR > gpurun_out/plain_arring_$tag.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_exec -s 3 -c 1 -o gpurun_out/prof_arring_$tag $AR > gpurun_out/ncu_arring_$tag.log 2>&1; echo "ncu ar ring rc=$?"; cat gpurun_out/plain_arring_$tag.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29612 tools/sweep.py --graph --pool --algos auto --oracle-cap $((64<<20)) \
  --out gpurun_out/sweep_n4_graph_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n4_graph_$tag.err; echo "sweep n4 graph rc=$?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29613 tools/sweep.py --pool --algos auto \
  --out gpurun_out/sweep_n4_eager_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n4_eager_$tag.err; echo "sweep n4 eager rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29614 tools/sweep.py --graph --pool --colls allreduce,reducescatter --dtype float32 --algos auto \
  --out gpurun_out/sweep_n4_fp32_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n4_fp32_$tag.err; echo "sweep n4 fp32 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 $TR --nproc-per-node 2 --master-port 29615 tools/sweep.py --graph --pool --algos auto --oracle-cap $((64<<20)) \
  --out gpurun_out/sweep_n2_graph_$tag.jsonl > /dev/null 2> gpurun_out/sweep_n2_graph_$tag.err; echo "sweep n2 rc=$?"
for f in gpurun_out/bench_n*_$tag.json; do tail -1 $f | cut -c1-250; done
python tools/show_sweep.py gpurun_out/sweep_n4_graph_$tag.jsonl | awk '{print $1,$2,$3,$4,$NF}' | head -90
