mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for c in 3 2 5; do timeout 200 python tools/quick_time.py $c 2>&1 | grep -E "^iter 3|^sha|kernel_times" | cut -c1-1200; done
for c in 3 5 2; do
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches$c.csv python tools/profile_step.py $c > gpurun_out/ncu$c.log 2>&1
python tools/launch_summary.py gpurun_out/launches$c.csv 16
done
