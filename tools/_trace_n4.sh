mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581"
for c in allreduce alltoall; do
timeout 200 $TR tools/trace.py --coll $c --algo direct --bytes 67108864 2>&1 | grep -v "^\*\|OMP\|NCCL\|W1018\|warn" > gpurun_out/trace_n4_${c}_64M.txt
done
wc -l gpurun_out/trace_n4_*_64M.txt
