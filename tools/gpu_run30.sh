#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rmsprop_cm_gpu.py tests/test_drivers_gpu.py -q -k "rmsprop or centered" > gpurun_out/pytest_cm.log 2>&1
timeout 600 python tools/rms_cm_bench.py > gpurun_out/rms_cm_bench.txt 2>&1
