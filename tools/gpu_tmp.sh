mkdir -p gpurun_out
bash tools/run_variants.sh 5 c4wlr
bash tools/run_variants.sh 3 c4wlr
bash tools/run_variants.sh 2 c4wlr
bash tools/run_variants.sh 4 c4wlr
