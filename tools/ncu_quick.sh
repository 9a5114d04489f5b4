#!/bin/bash
# Quick per-kernel pipe/stall metrics of one library build on c2 (key by value):
#   tools/ncu_quick.sh <lib.so> <out.csv>
LIB=$1; OUT=$2
M=sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__inst_executed.sum,smsp__inst_executed_pipe_fmaheavy.sum,smsp__inst_executed_pipe_alu.sum,smsp__warps_active.avg.per_cycle_active,gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k regex:fill_kernel -s 2 -c 1 --csv --log-file $OUT python tools/variant_bench.py $LIB > /dev/null 2>&1
