#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "flow_cache or auto or engine or records or 100m" 2>&1 | tail -3
for mib in 48 64 80; do
  timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode flow_cache --flow-cache-mib $mib --no-e2e --no-cpu-baseline --no-probe --no-records > gpurun_out/sweep_fc_$mib.json 2> gpurun_out/sweep_fc_$mib.err
  python - <<PY
import json
d=json.load(open("gpurun_out/sweep_fc_$mib.json"))
print("mib=$mib", "value Mpps", round(d["value"]), "scan ms", round(d["phase_ms"]["scan"],3), d["config"]["flow_cache"], d["parity"]["bits_equal_oracle"])
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_ -s 3 -c 1 -f -o gpurun_out/prof_scan_h32 \
   python bench.py --steps 2 --warmup 3 --scan-mode flow_cache --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
