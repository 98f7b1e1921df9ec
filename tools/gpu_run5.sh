#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
DIFFOPT_LIB=$PWD/tools/tune_build/lib_1-1-1-3-pdl.so timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_drivers_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu_pdl.log 2>&1
bash tools/tune_run.sh > gpurun_out/tune_summary.txt 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --workload maml --steps 10 --warmup 3 > gpurun_out/bench_maml.json 2> gpurun_out/bench_maml.err
timeout 900 python bench.py --workload maml --steps 3 --warmup 2 --no-graph > gpurun_out/bench_maml_nograph.json 2> gpurun_out/bench_maml_nograph.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_bench.log 2>&1
