#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-maml > gpurun_out/all_c1.json 2>&1
timeout 300 python bench.py --bf16 --steps 200 --warmup 10 --no-maml --no-cpu-baseline > gpurun_out/all_c2_bf16.json 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/all_c3.json 2>&1
timeout 300 python bench.py --workload c5 --size 268435456 --steps 20 --warmup 3 --no-maml --no-cpu-baseline --quick > gpurun_out/all_c5_2e28.json 2>&1
timeout 300 python bench.py --workload es --steps 20 --warmup 3 > gpurun_out/all_es.json 2>&1
timeout 300 python bench.py --compute f64 --steps 100 --warmup 10 --no-maml --no-cpu-baseline --quick > gpurun_out/all_c2_f64.json 2>&1
