#!/bin/bash
# default bench (all legs) + the reference arm: tools/gpu_bench.sh <tag> [bench args]
mkdir -p gpurun_out
TAG=${1:-x}; shift
timeout 900 python bench.py --steps 5 --warmup 3 "$@" > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench exit $?"
python - <<PY
import json
d = json.load(open('gpurun_out/bench_${TAG}.json'))
print('value', round(d['value']), 'phase', d['phase_ms'], 'launches', d['gpu_launches'])
print('roofline', {k: v for k, v in d['roofline'].items() if k not in ('l2_probe',)})
print('e2e', d.get('e2e'))
print('dropin', d.get('e2e_dropin'))
print('cpu', d.get('cpu_baseline'))
print('records', d.get('records_path'))
print('parity', d.get('parity'), d['clocks'], d['config']['scan_kernel_used'], d['config']['flow_cache'])
PY
tail -3 gpurun_out/bench_${TAG}.err
