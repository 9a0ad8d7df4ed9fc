#!/bin/bash
mkdir -p gpurun_out
DHSA_FC_VARIANT=1 timeout 600 python -m pytest tests -m gpu -x -q -k "flow_cache or auto or engine or records" 2>&1 | tail -3
for v in 0 1; do
  DHSA_FC_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode flow_cache --no-e2e --no-cpu-baseline --no-probe > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - <<PY
import json
d=json.load(open("gpurun_out/var_$v.json"))
print("variant=$v", "value Mpps", round(d["value"]), "scan ms", round(d["phase_ms"]["scan"],3), d["config"]["flow_cache"], d["parity"]["bits_equal_oracle"], "records", round(d["records_path"]["device_resident_mpps"]), d["records_path"]["counts_match"])
PY
done
DHSA_FC_VARIANT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_ -s 3 -c 1 -f -o gpurun_out/prof_scan_tma \
   python bench.py --steps 2 --warmup 3 --scan-mode flow_cache --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
