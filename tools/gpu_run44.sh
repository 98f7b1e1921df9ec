#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mamlnet_gpu.py -q > gpurun_out/pytest_net4.log 2>&1
timeout 300 python tools/gemm_nt_bench.py > gpurun_out/gemm_nt_bench.jsonl 2>&1
for T in 32 4; do
timeout 600 python bench.py --workload maml --tasks $T --steps 10 --warmup 3 > gpurun_out/bench_maml_fused3_T$T.json 2> gpurun_out/bench_maml_fused3_T$T.err
done
