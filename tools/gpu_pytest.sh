#!/bin/bash
# GPU parity suite only: tools/gpu_pytest.sh [-k expr]
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 "$@" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -60 gpurun_out/pytest_gpu.log
