#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/bench_c3_fused.json 2> gpurun_out/bench_c3_fused.err
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-fuse-glue > gpurun_out/bench_c3_unfused.json 2> gpurun_out/bench_c3_unfused.err
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --checkpoint-every 2 > gpurun_out/bench_c3_fused_ck2.json 2> gpurun_out/bench_c3_fused_ck2.err
