#!/usr/bin/env bash
# Export the metrics DESIGN.md / profiles cite from an .ncu-rep (raw page, CSV) and the
# details page; the report itself stays on the box (too large to copy back).
rep=$1; out=$2
ncu -i "$rep" --page raw --csv --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_op_dmma.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,lts__t_bytes.sum > "$out.raw.csv" 2>&1
ncu -i "$rep" --page details --csv > "$out.details.csv" 2>&1
