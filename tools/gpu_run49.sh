#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:'gemm_nt_partial|bnpool|im2col|col2im' --launch-skip 300 -c 40 -o gpurun_out/maml_net_T32 python bench.py --workload maml --tasks 32 --steps 2 --warmup 3 > gpurun_out/ncu_maml32.log 2>&1
ncu -i gpurun_out/maml_net_T32.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,launch__cluster_dim_x > gpurun_out/maml_net_T32.csv 2>&1
