#!/bin/bash
# A/B bench of library variants: tools/gpu_ab.sh <scan-mode> <lib or "default"> ...
mkdir -p gpurun_out
MODE=$1; shift
for lib in "$@"; do
  name=$(basename $lib .so)
  if [ "$lib" = "default" ]; then unset DHSA_LIB; else export DHSA_LIB=$PWD/$lib; fi
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --scan-mode $MODE --no-e2e --no-cpu-baseline --no-records --no-probe > gpurun_out/ab_${name}_$rep.json 2> gpurun_out/ab_${name}_$rep.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${name}_$rep.json')); print('$name', $rep, round(d['value']), d['phase_ms'], d['parity']['bits_equal_oracle'], d['config'].get('flow_cache'))"
  done
done
