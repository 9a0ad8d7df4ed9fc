#!/bin/bash
# per-launch GPU times of a short bench run: tools/gpu_launchlist.sh <tag> [env assignments via env] [bench args]
mkdir -p gpurun_out
TAG=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records "$@" > gpurun_out/launches_${TAG}.log 2>&1
python - <<PY
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/launches_${TAG}.csv')) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4][:60]].append(float(r[-1].replace(',', '')))
for k, v in agg.items():
    print(f"{k:60s} n={len(v):3d} last={v[-1]:12.1f} mean={sum(v)/len(v):12.1f}")
PY
