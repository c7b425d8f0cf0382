bash tools/run_variants.sh 5
bash tools/run_variants.sh 2
