mkdir -p gpurun_out
for c in 3 2 5; do timeout 300 python tools/quick_time.py $c 2>&1 | grep -E '^iter 3|^sha'; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu.log
