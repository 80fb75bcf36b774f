TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592"
for cfg in "base::" "t256_296:paper_2111_04867_b200/libtaccl_t256.so:296" "t256_256:paper_2111_04867_b200/libtaccl_t256.so:256"; do
  IFS=: read name lib ctas <<< "$cfg"
  rm -f gpurun_out/ab_$name.jsonl
  env ${lib:+TACCL_LIB=$PWD/$lib} ${ctas:+TACCL_TARGET_CTAS=$ctas} timeout 900 $TR tools/sweep.py --graph --no-nccl --colls allreduce,reducescatter,allgather --size-lo 26 --size-hi 30 --algos direct,ring,ring_p2 --out gpurun_out/ab_$name.jsonl > gpurun_out/ab_$name.log 2>&1
  echo "== $name"; python tools/show_sweep.py gpurun_out/ab_$name.jsonl | cut -c1-100
done
