#!/bin/bash
# flow-cache parity tests, then a table-size sweep of the device-resident bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow_cache or auto or update_batch_bits or ddos or contention" > gpurun_out/pytest_fc.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fc.log
tail -4 gpurun_out/pytest_fc.log
for mib in ${MIBS:-16 32 64 128}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --scan-mode flow_cache --flow-cache-mib $mib --no-e2e --no-cpu-baseline --no-records --no-probe > gpurun_out/fc_$mib.json 2> gpurun_out/fc_$mib.err
  python -c "
import json; d=json.load(open('gpurun_out/fc_$mib.json')); print($mib, round(d['value']), d['phase_ms'], d['parity']['bits_equal_oracle'], d['config'].get('flow_cache'))"
done
