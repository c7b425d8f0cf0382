mkdir -p gpurun_out
for c in 5 3 4 2; do timeout 300 python tools/quick_time.py $c 2>&1 | grep -E '^iter 3'; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not acceptance" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
