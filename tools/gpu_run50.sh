#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mamlnet_gpu.py tests/test_drivers_gpu.py -k "mamlnet or maml or bnpool or im2col or fused_network or gemm_nt or task_conv" -q > gpurun_out/pytest_net6.log 2>&1
for T in 32 4; do
timeout 600 python bench.py --workload maml --tasks $T --steps 10 --warmup 3 > gpurun_out/bench_maml_w_T$T.json 2> gpurun_out/bench_maml_w_T$T.err
done
timeout 600 python tools/maml_profile.py --tasks 32 --net fused > gpurun_out/maml_prof_w_32.txt 2>&1
timeout 600 python tools/maml_profile.py --tasks 4 --net fused > gpurun_out/maml_prof_w_4.txt 2>&1
