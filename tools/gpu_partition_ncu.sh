#!/bin/bash
# ncu --set full capture of the partition scan kernel (one launch), summaries as csv
mkdir -p gpurun_out
TAG=${1:-pt}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_partition -s 3 -c 1 -f -o gpurun_out/prof_${TAG} \
   python bench.py --steps 2 --warmup 3 --scan-mode partition --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv > gpurun_out/prof_${TAG}_source.csv 2>/dev/null
ls -la gpurun_out/prof_${TAG}*
