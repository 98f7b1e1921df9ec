#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_drivers_gpu.py -q -k maml > gpurun_out/pytest_maml.log 2>&1
for net in gemm cudnn; do
  timeout 600 python bench.py --workload maml --steps 10 --warmup 3 --maml-net $net > gpurun_out/bench_maml_$net.json 2> gpurun_out/bench_maml_$net.err
done
timeout 600 python tools/maml_profile.py --net gemm > gpurun_out/maml_prof_gemm.txt 2>&1
