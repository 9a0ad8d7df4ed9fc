#!/bin/bash
# quick GPU pass: selected parity tests (-k "$1") and the default bench (device legs only, records included)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_quick.log
tail -4 gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/quick.json 2> gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json')); print(round(d['value']), d['phase_ms'], d['parity'], d['records_path'])"
