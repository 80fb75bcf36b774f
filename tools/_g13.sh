mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_g13.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_g13.log
rm -f gpurun_out/sweep_n1_g13.jsonl
timeout 600 python tools/sweep.py --graph --colls allgather --out gpurun_out/sweep_n1_g13.jsonl > /dev/null 2>&1; echo "n1 sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/sweep_n1_g13.jsonl"):
    r = json.loads(l)
    print(r["S"], "ours us", r.get("taccl_direct_us"), "GB/s", r.get("taccl_direct_busbw"), "| torch copy us", r.get("torch_copy_us"), "GB/s", r.get("torch_copy_gbs"))
PY
bash tools/gpu_final.sh 2 r01h
