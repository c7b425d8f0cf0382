mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/run_variants.sh 3
bash tools/run_variants.sh 4 dl1 dl8
