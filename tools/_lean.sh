mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_lean.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_lean.log
for e in "TACCL_NO_LEAN_COPY=1" "" "TACCL_NO_LEAN_COPY=1" ""; do
  env $e timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_lean.json 2>/dev/null; echo "[$e] $(python -c "import json;d=json.load(open('gpurun_out/bench_lean.json'));print(d['value'], d['roofline']['frac'], d['config']['plan'])")"
done
rm -f gpurun_out/sweep_n1_lean.jsonl
timeout 600 python tools/sweep.py --graph --colls allgather --out gpurun_out/sweep_n1_lean.jsonl > /dev/null 2>&1; echo "n1 sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/sweep_n1_lean.jsonl"):
    r = json.loads(l)
    print(r["S"], "ours us", r.get("taccl_direct_us"), "GB/s", r.get("taccl_direct_busbw"), "| torch us", r.get("torch_copy_us"), "GB/s", r.get("torch_copy_gbs"))
PY
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
$B > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_lean.csv $B > /dev/null 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:taccl_ -s 5 -c 1 -o gpurun_out/prof_copy_lean $B > gpurun_out/ncu_copy_lean.log 2>&1; echo "ncu rc=$?"
