mkdir -p gpurun_out
for c in 2 5 3 4; do timeout 300 python tools/quick_time.py $c 2>&1 | grep -E '^iter 3'; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not acceptance" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools/profile_step.py 2 > /dev/null 2>&1 && timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches2.csv python tools/profile_step.py 2 > gpurun_out/ncu2.log 2>&1
echo "ncu rc=$?"; python tools/launch_summary.py gpurun_out/launches2.csv 14
