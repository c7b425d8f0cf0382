mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for c in 5 2 3; do timeout 200 python tools/quick_time.py $c 2>&1 | grep -E "^iter 3|^sha|kernel_times" | cut -c1-700; done
for c in 5; do
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches$c.csv python tools/profile_step.py $c > gpurun_out/ncu$c.log 2>&1
python tools/launch_summary.py gpurun_out/launches$c.csv 10
done
