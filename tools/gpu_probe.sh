# usage (under gpurun): bash tools/gpu_probe.sh
# config-4 single-GPU timing + a --set full capture of the dense 4-cycle kernel
mkdir -p gpurun_out
timeout 400 python tools/quick_time.py 4 > gpurun_out/qt4.log 2>&1; echo "qt4 rc=$?"; tail -3 gpurun_out/qt4.log
bash tools/gpu_full.sh k_c4_dense 3 1 dense
ncu -i gpurun_out/full_dense.ncu-rep --page raw --csv > gpurun_out/full_dense_raw.csv 2>/dev/null
ncu -i gpurun_out/full_dense.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/full_dense_src.csv 2>/dev/null
python tools/ncu_raw.py gpurun_out/full_dense_raw.csv stall | sort -k3 -n -r | head -25
