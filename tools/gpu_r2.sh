#!/bin/bash
# Round-2 validation on a 4-GPU box: every GPU test (incl. the 2- and 4-rank multi-process
# ones), smoke, bench N=1/2/4, and an Allreduce bf16 A/B sweep of the ring lowering at n=4.
mkdir -p gpurun_out
tag=${1:-r2}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; echo "bench1 rc=$?"
for n in 2 4; do
  timeout 600 $TR --nproc-per-node $n --master-port 2959$n bench.py --gpus $n > gpurun_out/bench_n${n}_$tag.json 2> gpurun_out/bench_n${n}_$tag.err; echo "bench$n rc=$?"; tail -1 gpurun_out/bench_n${n}_$tag.json | cut -c1-300
done
timeout 900 $TR --nproc-per-node 4 --master-port 29601 tools/sweep.py --graph --colls allreduce --size-lo 20 --size-hi 30 --algos ring,ring_peer,direct,auto --out gpurun_out/sweep_ar_ring_ab_n4_$tag.jsonl > /dev/null 2> gpurun_out/sweep_ar_ring_ab_n4_$tag.err; echo "sweep rc=$?"
python tools/show_sweep.py gpurun_out/sweep_ar_ring_ab_n4_$tag.jsonl 2>/dev/null | head -30
