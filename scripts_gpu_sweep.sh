#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "flow_cache" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for mib in 40 48 56 64 72 80 96; do
  timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode flow_cache --flow-cache-mib $mib --no-e2e --no-cpu-baseline --no-probe > gpurun_out/sweep_fc_$mib.json 2> gpurun_out/sweep_fc_$mib.err
  python - <<PY
import json
d=json.load(open("gpurun_out/sweep_fc_$mib.json"))
print("mib=$mib", "value Mpps", round(d["value"]), "scan ms", round(d["phase_ms"]["scan"],3), "readout ms", round(d["phase_ms"]["merge+estimate+restore+filter"],3), d["config"]["flow_cache"], d["parity"]["bits_equal_oracle"])
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_ -s 3 -c 1 -f -o gpurun_out/prof_scan_fc64 \
   python bench.py --steps 2 --warmup 3 --scan-mode flow_cache --flow-cache-mib 64 --no-e2e --no-cpu-baseline --no-parity --no-probe > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
