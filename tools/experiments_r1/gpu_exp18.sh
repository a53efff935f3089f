#!/bin/bash
# exp18: is device-only throughput set by the number of concurrently written ring slots
# (slot = one iteration)?  Speed vs (slot size = numrn, R slots), both piece orders, and
# ncu DRAM bytes / DRAM activity spread for a few points.
OUT=gpurun_out/exp18
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
S="timeout 900 python tools/sweep.py --variants 0 --reps 5 --numiter 1000 --orders 0,1"
$S --numrn $((1 << 24)) --slots 16,32,64,128,256,512 >> $OUT/grid.jsonl 2>> $OUT/err.log
$S --numrn $((1 << 25)) --slots 16,64,128,256 >> $OUT/grid.jsonl 2>> $OUT/err.log
$S --numrn $((1 << 26)) --slots 16,32,64,128 >> $OUT/grid.jsonl 2>> $OUT/err.log
$S --numrn $((1 << 27)) --slots 16,32,64 >> $OUT/grid.jsonl 2>> $OUT/err.log
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.min.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed,lts__t_sectors_op_write.sum"
for cfg in "24 512 0" "24 64 0" "27 64 0" "27 64 1" "26 128 0"; do
  set -- $cfg
  PRNG_N=$((1 << $1)) PRNG_SLOTS=$2 PRNG_ORDER=$3 timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv \
     python tools/profile_step.py > $OUT/ncu_n$1_r$2_o$3.csv 2>> $OUT/err.log
done
ls -la $OUT
