#!/bin/bash
# Round-end 1-GPU evidence: smoke, GPU tests, bench line (+ reference arm), n=1 sweep (copy
# path vs torch copy), launch list and ncu captures (tools/ncu_round.sh).
tag=${1:-final}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi_$tag.txt 2>&1
(nvidia-smi nvlink -s; nvidia-smi nvlink -gt d; nvidia-smi nvlink -h) > gpurun_out/nvlink_smi_$tag.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_n1_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_n1_$tag.log
timeout 600 python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; echo "bench rc=$?"; cat gpurun_out/bench_n1_$tag.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_n1_$tag.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_n1_$tag.json
rm -f gpurun_out/sweep_n1_$tag.jsonl
timeout 600 python tools/sweep.py --graph --colls allgather --out gpurun_out/sweep_n1_$tag.jsonl > gpurun_out/sweep_n1_$tag.log 2>&1; echo "sweep rc=$?"
bash tools/ncu_round.sh $tag
