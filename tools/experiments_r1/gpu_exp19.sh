#!/bin/bash
# exp19: the epoch-major kernel.  Parity first, then device-only GB/s and ncu DRAM bytes
# per shape with the auto rule (epoch when R slots of live lines < 2x L2) vs epochs off.
OUT=gpurun_out/exp19
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "epoch or forced or wrapping or ring" > $OUT/pytest.log 2>&1
echo "rc=$?" >> $OUT/pytest.log
S="timeout 900 python tools/sweep.py --variants 0 --reps 5 --numiter 1000 --epochs 0,-1"
for n in 24 25 26 27 28; do
  $S --numrn $((1 << n)) >> $OUT/sizes.jsonl 2>> $OUT/err.log
done
$S --numrn $((1 << 24)) --slots 16,64 >> $OUT/small_rings.jsonl 2>> $OUT/err.log
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.min.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed,lts__t_sectors_op_write.sum"
for cfg in "25 0" "26 0" "27 0" "28 0" "27 -1"; do
  set -- $cfg
  PRNG_N=$((1 << $1)) PRNG_EPOCH=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv \
     python tools/profile_step.py > $OUT/ncu_n$1_e$2.csv 2>> $OUT/err.log
done
ls -la $OUT
