#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for T in 32 16 8 4; do
timeout 600 python bench.py --workload maml --tasks $T --steps 10 --warmup 3 > gpurun_out/bench_maml_fused4_T$T.json 2> gpurun_out/bench_maml_fused4_T$T.err
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1
