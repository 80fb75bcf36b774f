TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544"
for c in allgather allreduce; do
timeout 120 $TR tools/trace.py --coll $c --bytes 1024 2>&1 | grep -v "^\*\|OMP\|NCCL"
timeout 120 $TR tools/trace.py --coll $c --bytes 1024 --calls 2 2>&1 | grep -v "^\*\|OMP\|NCCL"
done
timeout 120 $TR tools/trace.py --coll allgather --bytes 1048576 2>&1 | grep -v "^\*\|OMP\|NCCL" | head -20
