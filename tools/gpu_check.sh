# usage (under gpurun): bash tools/gpu_check.sh [pytest-args...]
# GPU suite + quick timings of configs 3, 2, 5, 4; logs under gpurun_out/.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in 3 2 5 4; do timeout 300 python tools/quick_time.py $c 2>&1 | tail -3; done
