#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "flow_cache or auto or engine or records" 2>&1 | tail -3
for mib in 32 40 48 56 64; do
  timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode flow_cache --flow-cache-mib $mib --no-e2e --no-cpu-baseline --no-probe --no-records > gpurun_out/sweep_fc_$mib.json 2> gpurun_out/sweep_fc_$mib.err
  python - <<PY
import json
d=json.load(open("gpurun_out/sweep_fc_$mib.json"))
print("mib=$mib", "value Mpps", round(d["value"]), "scan ms", round(d["phase_ms"]["scan"],3), d["config"]["flow_cache"], d["parity"]["bits_equal_oracle"])
PY
done
