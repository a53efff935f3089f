#!/bin/bash
# exp22: anti-absorption rule (wide variant or epoch order when a device-only launch would
# rewrite L2-resident lines): parity, then GB/s and ncu DRAM bytes per numrn x 1000.
OUT=gpurun_out/exp22
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "epoch or absorption or forced or wrapping or ring or star or bench_shape" > $OUT/pytest.log 2>&1
echo "rc=$?" >> $OUT/pytest.log
S="timeout 900 python tools/sweep.py --reps 5 --numiter 1000 --variants 0"
for n in 24 25 26 27 28; do
  $S --numrn $((1 << n)) >> $OUT/sizes.jsonl 2>> $OUT/err.log
done
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed"
for n in 25 26 27 28; do
  PRNG_N=$((1 << n)) timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv \
     python tools/profile_step.py > $OUT/ncu_n$n.csv 2>> $OUT/err.log
done
ls -la $OUT
