# n=4: multi-process tests, RS/AR pull vs push, MILP/greedy schedules vs direct, bench
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551"
timeout 600 python -m pytest tests/test_gpu_multiproc.py -m gpu -q > gpurun_out/pytest_multi_n4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_multi_n4.log
COLLS=reducescatter ALGOS=direct,ring ENVS="TACCL_PULL=0 base" bash tools/rs_exp.sh 4 pull4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_pull4.txt
rm -f gpurun_out/sweep_milp_n4.jsonl
timeout 600 $TR tools/sweep.py --graph --colls allgather,alltoall --algos direct,greedy,milp,milp_p2 --size-lo 10 --size-hi 30 --out gpurun_out/sweep_milp_n4.jsonl > gpurun_out/sweep_milp_n4.log 2>&1; echo "milp sweep rc=$?"
python tools/show_sweep.py gpurun_out/sweep_milp_n4.jsonl 2>/dev/null | head -50
