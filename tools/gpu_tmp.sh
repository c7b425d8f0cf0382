bash tools/run_variants.sh 3
bash tools/run_variants.sh 4 tps1280 tps1536
