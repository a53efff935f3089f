#!/bin/bash
# exp24: per-DRAM-instance activity (is the min ~ half the mean structural?): the bench
# kernel vs the plain grid-stride store probe kernel, instance values.
OUT=gpurun_out/exp24
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
M="dram__cycles_active.sum,dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum"
timeout 600 ncu --metrics $M --print-metric-instances values --clock-control none -k regex:batch_kernel -c 1 --csv \
   python tools/profile_step.py > $OUT/inst_batch.csv 2> $OUT/err.log
cat > /tmp/probe_store.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch; torch.cuda.set_device(0)
import paper_1609_01257_b200 as P
print(P.prng_probe_store_gbs(16 << 30, 1))
PY
timeout 600 ncu --metrics $M --print-metric-instances values --clock-control none -c 3 --csv \
   python /tmp/probe_store.py > $OUT/inst_store.csv 2>> $OUT/err.log
ls -la $OUT
# default-variant decision: v4n4s1 (0) vs v4n8s1 (3) vs v4n16s1 (17) across numrn
S="timeout 900 python tools/sweep.py --reps 5 --variants 0,3,17"
$S --numrn $((1 << 18)) --numiter 10000 >> $OUT/sizes.jsonl 2>> $OUT/err.log
for n in 20 21 22 23 24; do
  $S --numrn $((1 << n)) --numiter 1000 >> $OUT/sizes.jsonl 2>> $OUT/err.log
done
$S --numrn $((1 << 25)) --numiter 100 >> $OUT/sizes.jsonl 2>> $OUT/err.log
$S --numrn $((1 << 24)) --numiter 1000 >> $OUT/sizes.jsonl 2>> $OUT/err.log
ls -la $OUT
