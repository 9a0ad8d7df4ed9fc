#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['value'], d['phase_ms'], d['gpu_launches'], d['records_path']['device_resident_mpps'], d['parity'])"
DHSA_NO_GRAPH=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-probe --no-records > gpurun_out/b2.json 2> gpurun_out/b2.err
python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print('no graph', d['value'], d['phase_ms'], d['gpu_launches'])"
