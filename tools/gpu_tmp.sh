mkdir -p gpurun_out
bash tools/run_variants.sh 4 gb128 gb2k gb8k gbinf mgbinf m
