#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:'gemm_nt_partial|bnpool_bwd_kernel|bnpool_bwd2|im2col_kernel|bnpool_fwd' -c 12 -o gpurun_out/maml_net_full python bench.py --workload maml --tasks 32 --steps 3 --warmup 3 --no-graph > gpurun_out/ncu_maml.log 2>&1
ncu -i gpurun_out/maml_net_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/maml_net_full.csv 2>&1
