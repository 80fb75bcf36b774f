#!/bin/bash
# Quick validation of the current tree (under gpurun --gpus 2): smoke, every GPU test, the
# N=1 and N=2 bench lines.
mkdir -p gpurun_out
tag=${1:-check}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; echo "bench1 rc=$?"; cat gpurun_out/bench_n1_$tag.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 > gpurun_out/bench_n2_$tag.json 2> gpurun_out/bench_n2_$tag.err; echo "bench2 rc=$?"; tail -1 gpurun_out/bench_n2_$tag.json
