mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multi_device.py tests/test_gpu_parity.py tests/test_python_api.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 200 python tools/quick_time.py 3 2>&1 | grep -E "^iter 3|^sha"
