mkdir -p gpurun_out
SIZE_LO=25 SIZE_HI=28 COLLS=allreduce ALGOS=direct,direct_split ENVS="base TACCL_LANES=96 TACCL_LANES=192 TACCL_LANES=384 TACCL_CHAIN_SENDS=1,TACCL_LANES=192" bash tools/rs_exp.sh 4 arsplit4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_arsplit4.txt
