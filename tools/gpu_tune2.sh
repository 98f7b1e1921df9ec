#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
DIFFOPT_LIB=$PWD/tools/tune_build/lib_1-1-1-3-tma.so timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu_tma.log 2>&1
bash tools/tune_run.sh > gpurun_out/tune_summary.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload maml --steps 5 --warmup 3 > gpurun_out/bench_maml.json 2> gpurun_out/bench_maml.err
