# Round-end evidence refresh (run under gpurun): bench lines for every config,
# ncu launch lists (durations + DRAM bytes, warm cache) -> profiles summaries,
# the criterion-6 scratch report.
mkdir -p gpurun_out
for c in 3 2 5; do
  python tools/profile_step.py $c > /dev/null 2>&1 && \
  timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches$c.csv python tools/profile_step.py $c > gpurun_out/ncu$c.log 2>&1
  echo "ncu $c rc=$?"
  python tools/make_ncu_summary.py gpurun_out/launches$c.csv $c "ncu --nvtx --nvtx-include step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none of tools/profile_step.py $c"
done
timeout 600 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench3 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench4 rc=$?"
python tools/scratch_report.py > gpurun_out/scratch_small.txt 2>&1
python tools/scratch_report.py 3 > gpurun_out/scratch3.txt 2>&1
cp profiles/ncu_config*_summary.json gpurun_out/ 2>/dev/null
tail -c 600 gpurun_out/bench3.json
