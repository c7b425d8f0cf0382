mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench3 rc=$?"
timeout 300 python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench1 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench4 rc=$?"
python -c "
import json
for c in (1,2,3,4,5):
    d=json.load(open('gpurun_out/bench%d.json'%c)); print(c, round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['roofline']['frac'])
"
