mkdir -p gpurun_out
bash tools/run_variants.sh 3 t104 t110
bash tools/run_variants.sh 4 t104 t110
