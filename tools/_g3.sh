mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_pull.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_pull.log
COLLS=reducescatter,allreduce ALGOS=direct,ring ENVS="TACCL_PULL=0 base" bash tools/rs_exp.sh 2 pull1 > /dev/null 2>&1; cat gpurun_out/rs_exp_n2_pull1.txt
