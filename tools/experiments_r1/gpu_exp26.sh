#!/bin/bash
# exp26: grid shape for the new default at the bench shape (2^24 x 1000, R = 512, honest):
# v4n8s1 (3) and v4n12s1 (16) over grid warps x warps per CTA; plus 2^18/2^19/2^20 x 10^4
# default vs v4n8s1 to locate the small-numrn cross-over.
OUT=gpurun_out/exp26
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
S="timeout 900 python tools/sweep.py --reps 5"
$S --variants 3,16 --numrn $((1 << 24)) --numiter 1000 --warps 444,512,592,740 --cta-warps 0 >> $OUT/grid.jsonl 2>> $OUT/err.log
$S --variants 3 --numrn $((1 << 24)) --numiter 1000 --warps 592,1184 --cta-warps 2,8 >> $OUT/grid.jsonl 2>> $OUT/err.log
$S --variants 0,3,28 --numrn $((1 << 24)) --numiter 1000 >> $OUT/grid.jsonl 2>> $OUT/err.log
for n in 18 19 20; do
  $S --variants 0,3,29 --numrn $((1 << n)) --numiter 10000 >> $OUT/small.jsonl 2>> $OUT/err.log
done
ls -la $OUT
