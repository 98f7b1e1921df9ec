#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --workload es --steps 20 --warmup 3 > gpurun_out/bench_es.json 2> gpurun_out/bench_es.err
timeout 600 python bench.py --workload maml --steps 10 --warmup 3 > gpurun_out/bench_maml.json 2> gpurun_out/bench_maml.err
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
