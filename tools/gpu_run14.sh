#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_drivers_gpu.py -m gpu -q > gpurun_out/pytest_drivers.log 2>&1
timeout 600 python tools/leaf_sweep.py > gpurun_out/leaf_sweep.log 2>&1
python bench.py --bf16 --no-cpu-baseline > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_uniform -s 6 -c 2 -o gpurun_out/prof_ldg python bench.py --steps 3 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_ldg.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"es_|cg_kernel|neumann" -c 6 -o gpurun_out/prof_next python -m pytest tests/test_es_gpu.py tests/test_implicit_gpu.py -m gpu -q -k "linear_objective or spd" > gpurun_out/ncu_next.log 2>&1
