#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_drivers_gpu.py -q -k maml > gpurun_out/pytest_maml.log 2>&1
for impl in batched streams; do
  timeout 600 python bench.py --workload maml --steps 10 --warmup 3 --maml-impl $impl > gpurun_out/bench_maml_$impl.json 2> gpurun_out/bench_maml_$impl.err
done
timeout 600 python bench.py --workload maml --steps 10 --warmup 3 --tasks 128 > gpurun_out/bench_maml_t128.json 2> gpurun_out/bench_maml_t128.err
