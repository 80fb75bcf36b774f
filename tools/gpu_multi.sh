#!/bin/bash
# One multi-GPU call (under gpurun --gpus N): multi-process parity tests, bench line, sweeps vs NCCL.
# usage: bash tools/gpu_multi.sh N TAG
n=$1; tag=${2:-r01}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$tag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multiproc.py -m gpu -x -q > gpurun_out/pytest_multi_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi_$tag.log
tail -2 gpurun_out/pytest_multi_$tag.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $TR bench.py --gpus $n > gpurun_out/bench_n${n}_$tag.json 2> gpurun_out/bench_n${n}_$tag.err; echo "bench rc=$?"
cat gpurun_out/bench_n${n}_$tag.json
rm -f gpurun_out/sweep_n${n}_$tag.jsonl gpurun_out/sweepg_n${n}_$tag.jsonl
timeout 900 $TR tools/sweep.py --out gpurun_out/sweep_n${n}_$tag.jsonl > gpurun_out/sweep_n${n}_$tag.log 2>&1; echo "sweep rc=$?"
timeout 900 $TR tools/sweep.py --graph --out gpurun_out/sweepg_n${n}_$tag.jsonl > gpurun_out/sweepg_n${n}_$tag.log 2>&1; echo "sweep graph rc=$?"
