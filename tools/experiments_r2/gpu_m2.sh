#!/bin/bash
# round 2, call m2: write ceilings, compressible vs incompressible data
O=gpurun_out/m2; mkdir -p $O
W=tools/experiments_r2/wprobe
$W 32 3 > $O/plain32.jsonl 2>&1
$W 4 3 > $O/plain4.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_write.sum --clock-control none --csv --log-file $O/kernels.csv $W 4 1 > $O/ncu_k.txt 2>&1
ncu --replay-mode app-range --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $O/memset_range.csv $W 4 1 range > $O/ncu_r.txt 2>&1
ls -la $O
