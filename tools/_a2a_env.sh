mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SIZE_LO=26 SIZE_HI=30 COLLS=alltoall,allgather ALGOS=direct ENVS="base TACCL_TMA=2 TACCL_TARGET_CTAS=128 TACCL_COPY_VARIANT=2 TACCL_COPY_VARIANT=3 base" bash tools/rs_exp.sh 4 a2aenv4 > /dev/null 2>&1; cat gpurun_out/rs_exp_n4_a2aenv4.txt
