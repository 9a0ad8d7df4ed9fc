#!/bin/bash
# after a change that touches the scan kernels only: parity tests of the scan, bench (all legs + reference arm), launch
# list and the full ncu capture of the flow-cache kernel -- the scan-related part of tools/gpu_profile_pass.sh
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_config3.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_flowcache -s 3 -c 1 -f -o gpurun_out/prof_scan_${TAG} \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_full.log 2>&1
timeout 1200 python tests/checks/contention.py > gpurun_out/config4_${TAG}.json 2> gpurun_out/config4.err; echo "contention exit $?" >> gpurun_out/config4.err
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; tail -n 2 gpurun_out/ncu_full.log; tail -n 2 gpurun_out/config4.err | cut -c1-200
python - <<PY
import json
d = json.load(open('gpurun_out/bench_${TAG}.json'))
print('value', round(d['value']), d['phase_ms'], d['gpu_launches'], d['roofline']['frac'], d['roofline'].get('frac_of_binding_ceiling'))
print('e2e', d['e2e']['value'], [(r['feeder_threads'], round(r['mpps'])) for r in d['e2e_dropin']['runs']], d['cpu_baseline']['value'], d['parity'])
d = json.load(open('gpurun_out/bench_${TAG}_config3.json')); print('config3', round(d['value']), d['phase_ms'])
PY
