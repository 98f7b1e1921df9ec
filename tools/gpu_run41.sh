#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/maml_ops.py --tasks 32 > gpurun_out/maml_ops_32.txt 2>&1
for T in 4 8 16; do
timeout 600 python bench.py --workload maml --tasks $T --steps 10 --warmup 3 > gpurun_out/bench_maml_T$T.json 2> gpurun_out/bench_maml_T$T.err
done
