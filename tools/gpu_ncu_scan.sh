#!/bin/bash
# ncu --set full capture of one scan kernel launch: tools/gpu_ncu_scan.sh <tag> <kernel regex> <bench args...>
mkdir -p gpurun_out
TAG=$1; KREGEX=$2; shift; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -f -o gpurun_out/prof_${TAG} \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records "$@" > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log | cut -c1-300
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv > gpurun_out/prof_${TAG}_source.csv 2>/dev/null
ls -la gpurun_out/prof_${TAG}*
