bash tools/run_variants.sh 3
bash tools/run_variants.sh 4
