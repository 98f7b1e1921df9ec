#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mamlnet_gpu.py tests/test_drivers_gpu.py tests/test_perf_gpu.py -k "mamlnet or maml or bnpool or im2col or fused_network or gemm_nt or task_conv or perf or stream or leaves" -q > gpurun_out/pytest_net7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_net7.log
for T in 32 4; do
timeout 600 python bench.py --workload maml --tasks $T --steps 10 --warmup 3 > gpurun_out/bench_maml_cb_T$T.json 2> gpurun_out/bench_maml_cb_T$T.err
done
timeout 600 python tools/maml_profile.py --tasks 32 --net fused > gpurun_out/maml_prof_cb_32.txt 2>&1
