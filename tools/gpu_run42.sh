#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mamlnet_gpu.py tests/test_drivers_gpu.py -k "mamlnet or maml or bnpool or im2col or fused_network" -q -x > gpurun_out/pytest_net.log 2>&1
for T in 32 4; do
timeout 600 python bench.py --workload maml --maml-net fused --tasks $T --steps 10 --warmup 3 > gpurun_out/bench_maml_fused_T$T.json 2> gpurun_out/bench_maml_fused_T$T.err
done
timeout 600 python tools/maml_ops.py --tasks 32 --net fused > gpurun_out/maml_ops_fused_32.txt 2>&1
