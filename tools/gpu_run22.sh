#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_drivers_gpu.py -q -k maml > gpurun_out/pytest_maml.log 2>&1
timeout 600 python bench.py --workload maml --steps 10 --warmup 3 > gpurun_out/bench_maml_gemm.json 2> gpurun_out/bench_maml_gemm.err
timeout 600 python bench.py --workload maml --steps 10 --warmup 3 --tasks 128 > gpurun_out/bench_maml_t128.json 2> gpurun_out/bench_maml_t128.err
timeout 600 python tools/maml_profile.py --net gemm > gpurun_out/maml_prof_gemm.txt 2>&1
