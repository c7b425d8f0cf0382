# Round-end evidence refresh (run under gpurun): bench lines, reference arm,
# launch list with DRAM bytes, one --set full capture of the top kernel.
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench3 rc=$?"
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench5 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python tools/profile_step.py 3 > gpurun_out/ncu3.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --nvtx --nvtx-include "step/" -k regex:k_c4_dense -c 1 --set full --import-source on --clock-control none -o gpurun_out/full_top python tools/profile_step.py 3 > gpurun_out/full_top.log 2>&1; echo "ncu full rc=$?"
tail -c 400 gpurun_out/bench3.json
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench4 rc=$?"
ncu -i gpurun_out/full_top.ncu-rep --page details --csv > gpurun_out/full_top_details.csv 2>/dev/null
ncu -i gpurun_out/full_top.ncu-rep --page raw --csv > gpurun_out/full_top_raw.csv 2>/dev/null
ncu -i gpurun_out/full_top.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/full_top_src.csv 2>/dev/null
python tools/launch_summary.py gpurun_out/launches3.csv 20
