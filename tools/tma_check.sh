timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
TACCL_TMA=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for t in 0 1; do for c in 128 148; do echo "TMA=$t CTAS=$c $(TACCL_TMA=$t TACCL_TARGET_CTAS=$c timeout 120 python bench.py --no-cpu --no-e2e --steps 2000 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["plan"])')"; done; done
