mkdir -p gpurun_out
SIZE_LO=24 SIZE_HI=28 COLLS=allreduce ALGOS=direct,ring_p2 ENVS="base TACCL_CHAIN_SENDS=1 TACCL_PULL_KINDS=5 TACCL_CHAIN_SENDS=1,TACCL_PULL_KINDS=5 base" bash tools/rs_exp.sh 4 arx4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_arx4.txt
bash tools/gpu_final.sh 4 r01h
