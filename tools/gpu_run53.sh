#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:'bnpool|im2col|col2im' --launch-skip 200 -c 60 --csv --log-file gpurun_out/net_kernels_T32.csv python bench.py --workload maml --tasks 32 --steps 2 --warmup 3 > gpurun_out/ncu_net.log 2>&1
