#!/bin/bash
# One GPU call (1 GPU): parity tests, bench line, launch list + one full ncu capture.
# usage (under gpurun): bash tools/gpu_round.sh TAG
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; echo "bench rc=$?"
cat gpurun_out/bench_n1_$tag.json
C="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
timeout 300 $C > gpurun_out/plain_$tag.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$tag.csv $C > gpurun_out/ncu_launch_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_ -s 5 -c 1 -o gpurun_out/prof_$tag $C > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?"
