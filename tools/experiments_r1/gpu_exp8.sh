#!/bin/bash
OUT=gpurun_out/exp8; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
V=15,16,17,18
for L in 2 4 8; do
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --lag $L --reps 3 > $OUT/s24_l$L.jsonl 2>&1
done
timeout 600 python tools/sweep.py --variants $V --warps 592,1184 --lag 4 --numrn 1048576 --reps 3 > $OUT/s20.jsonl 2>&1
