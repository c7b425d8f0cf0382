set -x
mkdir -p gpurun_out
[ -n "$SKIPTEST" ] || timeout 420 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
timeout 150 python tools/quick_time.py 3 2>&1 | tail -6
timeout 150 python tools/quick_time.py 2 2>&1 | tail -3
timeout 150 python tools/quick_time.py 5 2>&1 | tail -3
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python tools/profile_step.py 3 > gpurun_out/ncu3.log 2>&1
python tools/launch_summary.py gpurun_out/launches3.csv 14
