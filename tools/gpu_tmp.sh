bash tools/run_variants.sh 3 pin
bash tools/run_variants.sh 4 pin
