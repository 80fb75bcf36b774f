mkdir -p gpurun_out
SIZE_LO=20 SIZE_HI=25 COLLS=allreduce,reducescatter,allgather,alltoall ALGOS=auto ENVS="base TACCL_STAGED_MAX=8388608 TACCL_STAGED_MAX=16777216 base" bash tools/rs_exp.sh 4 llth4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_llth4.txt
