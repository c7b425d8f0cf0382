# usage: bash tools/gpu_full.sh <kernel-regex> <cfg> <count> <tag>
K=$1; CFG=$2; C=$3; TAG=$4
mkdir -p gpurun_out
timeout 150 python tools/profile_step.py $CFG || exit 1
timeout 900 ncu --nvtx --nvtx-include "step/" --kernel-name-base demangled -k regex:"$K" -c $C --set full --import-source on --clock-control none -o gpurun_out/full_$TAG python tools/profile_step.py $CFG > gpurun_out/full_$TAG.log 2>&1
tail -3 gpurun_out/full_$TAG.log
