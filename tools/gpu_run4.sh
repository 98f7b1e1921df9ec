#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
for v in tma256x1 tma512x1 tma256x2; do
DIFFOPT_LIB=$PWD/tools/tune_build/lib_1-1-1-3-$v.so timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "adam or tiny" > gpurun_out/pytest_gpu_$v.log 2>&1
done
bash tools/tune_run.sh > gpurun_out/tune_summary.txt 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python tools/c5_sweep.py > gpurun_out/c5.log 2>&1
DIFFOPT_LIB=$PWD/tools/tune_build/lib_1-1-1-3-tma256x1.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 6 -c 2 -o gpurun_out/prof_tma python bench.py --steps 3 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_tma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_uniform -s 6 -c 2 -o gpurun_out/prof_ldg python bench.py --steps 3 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_ldg.log 2>&1
