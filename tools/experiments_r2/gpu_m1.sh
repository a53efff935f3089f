#!/bin/bash
# round 2, call m1: what is the memset fill engine?  launch list + DRAM counters
O=gpurun_out/m1; mkdir -p $O
nvidia-smi -q -d CLOCK,POWER > $O/smi.txt 2>&1
python tools/experiments_r2/memset_probe.py $((32<<30)) 3 > $O/plain.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread --clock-control none --csv --log-file $O/launches.csv python tools/experiments_r2/memset_probe.py $((4<<30)) 1 > $O/ncu_stdout.txt 2>&1
ncu --set full --clock-control none -k regex:fill -c 1 -o $O/fill python tools/experiments_r2/memset_probe.py $((4<<30)) 1 > $O/ncu_full_stdout.txt 2>&1
ncu -i $O/fill.ncu-rep --page raw --csv > $O/fill_raw.csv 2>&1
ls -la $O
