#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3 4 5; do
  for mib in 56 64; do
  DHSA_FC_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode flow_cache --flow-cache-mib $mib --no-e2e --no-cpu-baseline --no-probe > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - <<PY
import json
d=json.load(open("gpurun_out/var_$v.json"))
print("variant=$v mib=$mib", "value Mpps", round(d["value"]), "scan ms", round(d["phase_ms"]["scan"],3), d["config"]["flow_cache"], d["parity"]["bits_equal_oracle"])
PY
  done
done
