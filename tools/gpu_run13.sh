#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
bash tools/tune_run.sh > gpurun_out/tune_summary.txt 2>&1
TUNE_ARGS=--bf16 bash tools/tune_run.sh > gpurun_out/tune_summary_bf16.txt 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --workload es --steps 20 --warmup 3 > gpurun_out/bench_es.json 2> gpurun_out/bench_es.err
timeout 900 python tools/c5_sweep.py --sizes 20,22,24,26,28,30 > gpurun_out/c5.log 2>&1
