mkdir -p gpurun_out
./tools/mb_mixed > gpurun_out/mixed_atomics.log 2>&1; cat gpurun_out/mixed_atomics.log
export FGLT_LIB_OVERRIDE=$PWD/variants/checked/libfglt.so
timeout 900 python tools/sanitize_cases.py > gpurun_out/bounds_cases.log 2>&1; echo "checked cases rc=$?"; grep -c 'FGLT bounds' gpurun_out/bounds_cases.log; tail -2 gpurun_out/bounds_cases.log
for c in 3 5 2 4; do timeout 600 python tools/run_case.py cfg $c > gpurun_out/bounds_cfg$c.log 2>&1; echo "cfg $c rc=$? bounds-prints $(grep -c 'FGLT bounds' gpurun_out/bounds_cfg$c.log)"; done
unset FGLT_LIB_OVERRIDE
for c in 3 2; do timeout 300 python tools/quick_time.py $c 2>&1 | grep -E '^iter 3'; done
