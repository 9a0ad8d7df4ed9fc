#!/bin/bash
# full GPU pass (run from the repo root: gpurun -- bash tools/gpu_profile_pass.sh r02): parity tests, smoke,
# bench (all scan modes + the reference arm + config 3), ncu launch list + full captures of the scan kernels,
# the config 3/4/5 checks, the host-feed and L2 probes.  tools/refresh_profiles.py turns gpurun_out/ into profiles/.
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2>> gpurun_out/bench_${TAG}.err
for mode in test_agg test red; do
  timeout 300 python bench.py --steps 5 --warmup 3 --scan-mode $mode --no-e2e --no-cpu-baseline --no-records > gpurun_out/bench_${TAG}_$mode.json 2>> gpurun_out/bench_${TAG}.err
done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_config3.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_ -s 3 -c 1 -f -o gpurun_out/prof_scan_${TAG} \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_vec4 -s 3 -c 1 -f -o gpurun_out/prof_vec4_${TAG} \
   python bench.py --steps 2 --warmup 3 --scan-mode test_agg --no-e2e --no-cpu-baseline --no-parity --no-probe --no-records > gpurun_out/ncu_full_vec4.log 2>&1
timeout 1200 python tests/checks/contention.py > gpurun_out/config4_${TAG}.json 2> gpurun_out/config4.err; echo "contention exit $?" >> gpurun_out/config4.err
timeout 900 python tools/accuracy_sweep.py > gpurun_out/config5_${TAG}.json 2> gpurun_out/config5.err
timeout 900 python tests/checks/config3_window.py > gpurun_out/config3_${TAG}.json 2> gpurun_out/config3.err
PYTHONPATH=. timeout 600 python tools/tooling_timings.py > gpurun_out/tools_${TAG}.json 2> gpurun_out/tools.err
timeout 600 python tools/host_feed_probe.py > gpurun_out/feed_probe_${TAG}.json 2> gpurun_out/feed_probe.err
timeout 300 python tools/l2_probe.py > gpurun_out/l2_probe_${TAG}.json 2> gpurun_out/l2_probe.err
timeout 600 python tests/checks/soak.py 120 > gpurun_out/soak_${TAG}.txt 2>&1
timeout 600 python tests/checks/soak_engine.py 90 >> gpurun_out/soak_${TAG}.txt 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; cat gpurun_out/bench_${TAG}.json gpurun_out/bench_${TAG}_reference.json | cut -c1-600; tail -n 2 gpurun_out/ncu_full.log
for f in gpurun_out/config3.err gpurun_out/config4.err gpurun_out/config5.err gpurun_out/tools.err gpurun_out/soak_${TAG}.txt; do tail -n 3 $f | cut -c1-300; done
