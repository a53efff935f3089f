#!/bin/bash
# round 2, call m3: write schedules for the generator's output (gen_sched.cu)
O=gpurun_out/m3; mkdir -p $O
G=tools/experiments_r2/gen_sched
$G 16777216 256 > $O/s24_t256.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:g1_persistent -c 2 --csv --log-file $O/ncu_g1.csv $G 16777216 256 g1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:g2_tile -c 40 --csv --log-file $O/ncu_g2.csv $G 16777216 256 g2 > /dev/null 2>&1
ls -la $O
