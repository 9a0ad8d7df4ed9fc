#!/bin/bash
# quick GPU pass: selected parity tests (-k "$1") and the default bench twice
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_quick.log
tail -4 gpurun_out/pytest_quick.log
bash tools/gpu_ab.sh auto default
