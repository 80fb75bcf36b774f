mkdir -p gpurun_out
timeout 120 python tools/nvlink_counters.py > gpurun_out/nvlink_counters.txt 2>&1; echo "counters rc=$?"; head -12 gpurun_out/nvlink_counters.txt
timeout 120 python tools/nvlink_probe_run.py > gpurun_out/nvlink_probe.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/nvlink_probe.txt
bash tools/gpu_final.sh 2 r01g
