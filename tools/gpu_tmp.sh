mkdir -p gpurun_out
bash tools/run_variants.sh 3 lanerow
bash tools/run_variants.sh 4 lanerow
export FGLT_LIB_OVERRIDE=$PWD/variants/lanerow/libfglt.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "forced or rmat or full_size or golden" > gpurun_out/pytest_lanerow.log 2>&1
echo "pytest lanerow rc=$?"; tail -3 gpurun_out/pytest_lanerow.log
