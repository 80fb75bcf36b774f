mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_parity_g8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_parity_g8.log
COLLS=reducescatter,allreduce ALGOS=direct,ring ENVS="TACCL_PULL=0 base TACCL_PULL_KINDS=7 TACCL_PULL_KINDS=5" bash tools/rs_exp.sh 4 wide4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_wide4.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING,NVLS timeout 300 $TR tools/sweep.py --colls allreduce --algos direct --size-lo 26 --size-hi 26 --out gpurun_out/nccl_info.jsonl > gpurun_out/nccl_info_n4.log 2>&1
grep -iE "nvls|algorithm|Ring|Tree|CollNet|symmetric" gpurun_out/nccl_info_n4.log | sort | uniq -c | sort -rn | head -20
