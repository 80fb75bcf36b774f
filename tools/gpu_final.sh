#!/bin/bash
# Round-end multi-GPU evidence (under gpurun --gpus N): GPU tests, bench line, graph sweep of
# every collective vs NCCL. usage: bash tools/gpu_final.sh N TAG
n=$1; tag=${2:-final}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29561"
if [ "$n" = 2 ]; then T="tests"; else T="tests/test_gpu_multiproc.py"; fi
timeout 1200 python -m pytest $T -m gpu -q > gpurun_out/pytest_gpu_n${n}_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_n${n}_$tag.log
timeout 600 $TR bench.py --gpus $n > gpurun_out/bench_n${n}_$tag.json 2> gpurun_out/bench_n${n}_$tag.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_n${n}_$tag.json
rm -f gpurun_out/sweepg_n${n}_$tag.jsonl
timeout 1500 $TR tools/sweep.py --graph --out gpurun_out/sweepg_n${n}_$tag.jsonl > gpurun_out/sweepg_n${n}_$tag.log 2>&1; echo "sweep rc=$?"
python tools/show_sweep.py gpurun_out/sweepg_n${n}_$tag.jsonl > gpurun_out/sweepg_n${n}_$tag.txt
grep -E " (1024|1048576|67108864|1073741824) " gpurun_out/sweepg_n${n}_$tag.txt
