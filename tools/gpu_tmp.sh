mkdir -p gpurun_out
export FGLT_LIB_OVERRIDE=$PWD/variants/checked/libfglt.so
OUT=gpurun_out/bounds_checked_runs.txt
echo "# FGLT_DEBUG_BOUNDS build (tools/build_variant.sh checked -DFGLT_DEBUG_BOUNDS) of the final round-2 source: sanitize workload + full configs" > $OUT
run() { n=$1; shift; timeout 900 "$@" > gpurun_out/$n.log 2>&1; echo "== $n: $(grep -c 'FGLT bounds' gpurun_out/$n.log) bounds violations" >> $OUT; grep -v 'FGLT bounds' gpurun_out/$n.log | tail -3 >> $OUT; }
run bounds_cases python tools/sanitize_cases.py
run bounds_cfg3 python tools/run_case.py cfg 3
run bounds_cfg5 python tools/run_case.py cfg 5
run bounds_cfg2 python tools/run_case.py cfg 2
run bounds_cfg1 python tools/run_case.py cfg 1 check
run bounds_cfg4 python tools/run_case.py cfg 4
run bounds_rmat16_check python tools/run_case.py rmat 16 check
cat $OUT
