#!/bin/bash
# ncu --set full of the second scan launch of tools/one_launch.py: tools/gpu_ncu_one.sh <tag> <kernel regex> <one_launch args...>
mkdir -p gpurun_out
TAG=$1; KREGEX=$2; shift; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 -f -o gpurun_out/prof_${TAG} \
   python tools/one_launch.py "$@" > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log | cut -c1-300
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_${TAG}_raw.csv
