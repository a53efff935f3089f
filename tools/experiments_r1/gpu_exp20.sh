#!/bin/bash
# exp20: cost of the epoch-major kernel vs E at the bench shape (all honest: E <= R = 512),
# and the large-numrn options: epoch kernel per variant vs a natural-order variant whose
# live set (R x warps x 8 KiB) exceeds L2 (v4n32s1), with ncu DRAM bytes.
OUT=gpurun_out/exp20
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
S="timeout 900 python tools/sweep.py --reps 5 --numiter 1000"
$S --variants 0 --numrn $((1 << 24)) --epochs -1,512,256,128,64,32 >> $OUT/e_2e24.jsonl 2>> $OUT/err.log
$S --variants 0,1,2,3 --numrn $((1 << 27)) --epochs 0,32 >> $OUT/e_2e27.jsonl 2>> $OUT/err.log
$S --variants 15,14,17 --numrn $((1 << 27)) --epochs -1 >> $OUT/e_2e27.jsonl 2>> $OUT/err.log
$S --variants 0,3 --numrn $((1 << 24)) --epochs -1,256 --warps 592,444 >> $OUT/e_2e24_w.jsonl 2>> $OUT/err.log
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.min.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed"
for cfg in "27 -1 15" "27 -1 17" "24 256 0" "24 -1 0"; do
  set -- $cfg
  PRNG_N=$((1 << $1)) PRNG_EPOCH=$2 PRNG_KERNEL=$3 timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv \
     python tools/profile_step.py > $OUT/ncu_n$1_e$2_k$3.csv 2>> $OUT/err.log
done
ls -la $OUT
