#!/bin/bash
O=gpurun_out/m5; mkdir -p $O
G=tools/experiments_r2/gen_sched
$G 16777216 256 > $O/s24_t256.jsonl 2>&1; exit 0
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_write.sum,lts__average_t_sector_hit_rate_realtime.pct --clock-control none -k regex:fill_persistent -c 20 --csv --log-file $O/ncu_fp.csv $G 16777216 32 fill_persistent > /dev/null 2>&1
