mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_parity_g12.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_parity_g12.log
SIZE_LO=10 SIZE_HI=24 COLLS=reducescatter,allreduce ALGOS=direct,auto ENVS="TACCL_CHAIN_OLDDEPS=1 base TACCL_CHAIN_OLDDEPS=1 base" bash tools/rs_exp.sh 4 deps4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_deps4.txt
for b in 1024 65536 4194304; do timeout 120 python tools/trace.py --coll allgather --n 1 --bytes $b 2>&1 | grep -v "^\*" | head -20; done > gpurun_out/trace_n1.txt 2>&1; cat gpurun_out/trace_n1.txt | head -60
