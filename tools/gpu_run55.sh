#!/bin/bash
# validation after the norm/pool slice cap: full GPU suite, smoke, default bench, maml T=32/4, ncu launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
for T in 32 4; do for i in 1 2; do timeout 300 python bench.py --workload maml --tasks $T --steps 10 --warmup 3 2>/dev/null | tail -1; done; done > gpurun_out/bench_maml_final.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 20 --warmup 3 --quick --no-cpu-baseline --no-maml > gpurun_out/ncu_bench_final.log 2>&1
