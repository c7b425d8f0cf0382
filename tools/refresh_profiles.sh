# Round-end evidence refresh (run under gpurun): the GPU test suite (which also
# runs the reference's acceptance harness and test_smoke.py), ncu launch lists
# (durations + DRAM bytes, warm cache) -> profiles summaries, one --set full
# capture of the dominant kernel -> on-chip digest, bench lines for every
# config, the reference arm on configs 3/2/5, scratch reports.
# Everything lands in gpurun_out/; copy what is judged into profiles/.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_lookup_hit.sum
M4=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum  # R-MAT 23: fewer replay passes
for c in 3 2 5 4; do
  MM=$M; [ $c = 4 ] && MM=$M4
  python tools/profile_step.py $c > /dev/null 2>&1 && \
  timeout 1500 ncu --nvtx --nvtx-include "step/" --metrics $MM --cache-control none --clock-control none --csv --log-file gpurun_out/launches$c.csv python tools/profile_step.py $c > gpurun_out/ncu$c.log 2>&1
  echo "ncu $c rc=$?"
  python tools/make_ncu_summary.py gpurun_out/launches$c.csv $c "ncu --nvtx --nvtx-include step/ --metrics $MM --cache-control none --clock-control none of tools/profile_step.py $c"
done
# dominant kernel: one --set full capture (after the plain run above exited 0)
bash tools/gpu_full.sh k_c4_dense 3 1 dense
ncu -i gpurun_out/full_dense.ncu-rep --page raw --csv > gpurun_out/full_dense_raw.csv 2>/dev/null
python tools/make_onchip_summary.py gpurun_out/full_dense_raw.csv 3 "ncu --nvtx --nvtx-include step/ -k regex:k_c4_dense -c 1 --set full --import-source on --clock-control none of tools/profile_step.py 3"
python tools/ncu_digest.py gpurun_out/full_dense.ncu-rep 25 > gpurun_out/digest_dense.txt 2>&1
cp profiles/ncu_config*_summary.json profiles/ncu_config3_dense_onchip.json gpurun_out/ 2>/dev/null
timeout 300 python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench1 rc=$?"
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench3 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref3.json 2> gpurun_out/bench_ref3.err; echo "ref3 rc=$?"
timeout 300 python bench.py --impl reference --config 1 > gpurun_out/bench_ref1.json 2> gpurun_out/bench_ref1.err; echo "ref1 rc=$?"
timeout 300 python bench.py --impl reference --config 2 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err; echo "ref2 rc=$?"
timeout 300 python bench.py --impl reference --config 5 > gpurun_out/bench_ref5.json 2> gpurun_out/bench_ref5.err; echo "ref5 rc=$?"
python tools/scratch_report.py > gpurun_out/scratch_small.txt 2>&1
python tools/scratch_report.py 3 > gpurun_out/scratch3.txt 2>&1
rm -f gpurun_out/full_dense.ncu-rep
tail -c 400 gpurun_out/bench3.json
