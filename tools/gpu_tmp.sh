mkdir -p gpurun_out
python tools/scratch_report.py > gpurun_out/scratch_small.txt 2>&1; head -40 gpurun_out/scratch_small.txt
python tools/scratch_report.py 3 > gpurun_out/scratch3.txt 2>&1; head -30 gpurun_out/scratch3.txt
for c in 3 2 5; do timeout 300 python tools/quick_time.py $c 2>&1 | tail -3 | head -2; done
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench3.json; tail -3 gpurun_out/bench3.err
for c in 2 5 3; do
  python tools/profile_step.py $c > /dev/null 2>&1 && \
  timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches$c.csv python tools/profile_step.py $c > gpurun_out/ncu$c.log 2>&1
  echo "ncu $c rc=$?"; python tools/launch_summary.py gpurun_out/launches$c.csv 25
done
