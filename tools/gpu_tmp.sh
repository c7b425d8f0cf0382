# scratch (under gpurun)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_kernels_api.py tests/test_multi_device.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
python tools/scratch_report.py 2>&1 | tee gpurun_out/scratch_small.txt | head -40
for c in 2 5 3; do timeout 300 python tools/quick_time.py $c 2>&1 | grep -v "^iter [012]" | cut -c1-1500; done
