#!/bin/bash
# NVLink SHARP (multicast reduce) validation + Allreduce sweep with pool buffers (gpurun --gpus 4)
mkdir -p gpurun_out
tag=${1:-nv}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -k multicast -x > gpurun_out/pytest_nvls_$tag.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_nvls_$tag.log
timeout 900 $TR --nproc-per-node 4 --master-port 29621 tools/sweep.py --graph --pool --colls allreduce --size-lo 20 --size-hi 30 \
  --algos direct,nvls,auto --out gpurun_out/sweep_nvls_n4_$tag.jsonl > /dev/null 2> gpurun_out/sweep_nvls_n4_$tag.err; echo "sweep n4 rc=$?"
tail -3 gpurun_out/sweep_nvls_n4_$tag.err
python tools/show_sweep.py gpurun_out/sweep_nvls_n4_$tag.jsonl
timeout 900 $TR --nproc-per-node 4 --master-port 29622 tools/sweep.py --graph --pool --colls allreduce --dtype float32 --size-lo 20 --size-hi 30 \
  --algos ring,nvls,auto --out gpurun_out/sweep_nvls_fp32_n4_$tag.jsonl > /dev/null 2> gpurun_out/sweep_nvls_fp32_n4_$tag.err; echo "sweep fp32 rc=$?"
python tools/show_sweep.py gpurun_out/sweep_nvls_fp32_n4_$tag.jsonl
