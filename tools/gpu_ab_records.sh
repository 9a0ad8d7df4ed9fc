#!/bin/bash
# A/B of library variants on the raw-record path: tools/gpu_ab_records.sh <lib> ...
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename $lib .so)
  export DHSA_LIB=$PWD/$lib
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/abr_${name}_$rep.json 2> gpurun_out/abr_${name}_$rep.err
    python -c "
import json; d=json.load(open('gpurun_out/abr_${name}_$rep.json')); print('$name', $rep, round(d['value']), round(d['records_path']['device_resident_mpps']), d['records_path']['counts_match'], d['parity']['bits_equal_oracle'])"
  done
done
