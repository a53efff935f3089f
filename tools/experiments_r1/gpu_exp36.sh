#!/bin/bash
# exp36: the "auto" threshold with the final variants: v4n4s1p (35) vs v4n8s1a (30) across numrn.
OUT=gpurun_out/exp36; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
S="timeout 900 python tools/sweep.py --reps 5 --variants 35,30"
for n in 16 18; do $S --numrn $((1 << n)) --numiter 10000 >> $OUT/sizes.jsonl 2>> $OUT/err.log; done
for n in 19 20 21 22 23 24; do $S --numrn $((1 << n)) --numiter 1000 >> $OUT/sizes.jsonl 2>> $OUT/err.log; done
$S --numrn $((1 << 20)) --numiter 10000 >> $OUT/sizes.jsonl 2>> $OUT/err.log
ls -la $OUT
