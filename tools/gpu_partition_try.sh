#!/bin/bash
# quick GPU pass for scan mode 5 (partition): its parity tests under a timeout, bench legs, optional ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "partition" > gpurun_out/pytest_partition.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_partition.log
tail -5 gpurun_out/pytest_partition.log
for tpc in ${TPCS:-1 2 4}; do
  DHSA_PT_TPC=$tpc timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode partition --no-e2e --no-cpu-baseline --no-records --no-probe > gpurun_out/bench_partition_tpc$tpc.json 2> gpurun_out/bench_partition_tpc$tpc.err
  echo "tpc=$tpc exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_partition_tpc$tpc.json')); print(d['value'], d['phase_ms'], d['parity'], d.get('config',{}).get('partition'))"
done
if [ -n "$NCU_TAG" ]; then bash tools/gpu_partition_ncu.sh $NCU_TAG; fi
