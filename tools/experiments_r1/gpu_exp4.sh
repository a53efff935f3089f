#!/bin/bash
OUT=gpurun_out/exp4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/sweep.py --variants 2,8,9,10,11,12,1 --warps 592,1184 --reps 4 > $OUT/s24.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 2,8,9,11,12,1 --warps 592,1184 --numrn 1048576 --reps 3 > $OUT/s20.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 2,8,9,11,12,1 --warps 592,1184 --numrn 268435456 --numiter 100 --reps 3 > $OUT/s28.jsonl 2>&1
