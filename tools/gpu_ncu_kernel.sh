# usage (under gpurun): bash tools/gpu_ncu_kernel.sh <kernel-regex> <cfg> <count> <tag>
# --set full capture + raw and source pages, stall summary and hot lines
K=$1; CFG=$2; C=$3; TAG=$4
bash tools/gpu_full.sh "$K" $CFG $C $TAG
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/full_$TAG.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/full_${TAG}_src.csv 2>/dev/null
python tools/ncu_raw.py gpurun_out/full_${TAG}_raw.csv gpu__time_duration.sum launch__occupancy sm__warps_active.avg.pct launch__registers launch__grid_size launch__block_size
python tools/ncu_raw.py gpurun_out/full_${TAG}_raw.csv pcsamp_warps_issue_stalled | grep -v not_issued | sort -k3 -n -r | head -12
python tools/ncu_hot_lines.py gpurun_out/full_${TAG}_src.csv 25
