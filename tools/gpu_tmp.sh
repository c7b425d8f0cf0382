mkdir -p gpurun_out
bash tools/run_variants.sh 5 msort64 c4t16
bash tools/run_variants.sh 2 msort64 c4t16
bash tools/run_variants.sh 3 msort64
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_kernels_api.py tests/test_multi_device.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_par.log
