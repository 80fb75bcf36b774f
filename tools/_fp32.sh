mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "single_rank or lean" > gpurun_out/pytest_lean2.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_lean2.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29593"
rm -f gpurun_out/sweepg_n4_fp32.jsonl
timeout 900 $TR tools/sweep.py --graph --dtype float32 --colls allreduce,reducescatter --out gpurun_out/sweepg_n4_fp32.jsonl > gpurun_out/sweepg_n4_fp32.log 2>&1; echo "sweep rc=$?"
python tools/show_sweep.py gpurun_out/sweepg_n4_fp32.jsonl > gpurun_out/sweepg_n4_fp32.txt; python tools/results_table.py gpurun_out/sweepg_n4_fp32.jsonl
