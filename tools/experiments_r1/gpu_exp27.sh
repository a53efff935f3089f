#!/bin/bash
# exp27: epoch fallback on the widest variant (2^28 x 1000, 32 slots) + extended fuzz.
OUT=gpurun_out/exp27
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "randomised or absorption or epoch or auto or race or time_parallel or forced" > $OUT/pytest.log 2>&1
echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/sweep.py --reps 3 --numrn $((1 << 28)) --numiter 1000 --variants 0 >> $OUT/n28.jsonl 2>> $OUT/err.log
M="dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed"
PRNG_N=$((1 << 28)) timeout 600 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv \
     python tools/profile_step.py > $OUT/ncu_n28.csv 2>> $OUT/err.log
ls -la $OUT
