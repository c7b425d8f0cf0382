mkdir -p gpurun_out
bash tools/run_variants.sh 3 g1 g2 g4
bash tools/run_variants.sh 4 g2 g4
