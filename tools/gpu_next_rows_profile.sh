#!/bin/bash
# ncu evidence for the rows either side of the hot path: launch lists of the record engine and of the
# evaluation tooling, and one full capture of the record-source scan kernel
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_records.csv \
   python tools/records_profile.py > gpurun_out/ncu_records.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_flowcache -s 4 -c 1 -f -o gpurun_out/prof_records \
   python tools/records_profile.py > gpurun_out/ncu_records_full.log 2>&1
ncu -i gpurun_out/prof_records.ncu-rep --page raw --csv > gpurun_out/prof_records_raw.csv 2>/dev/null
PYTHONPATH=. timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_tools.csv \
   python tools/tooling_timings.py > gpurun_out/ncu_tools.log 2>&1
timeout 300 python tools/records_profile.py | tail -1
tail -2 gpurun_out/ncu_records_full.log; python tools/ncu_summary.py gpurun_out/prof_records_raw.csv | head -30
