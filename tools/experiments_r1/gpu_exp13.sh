#!/bin/bash
OUT=gpurun_out/exp13; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/sweep.py --variants 0,12 --warps 592,1184 --pads 0,32,512,8192,131072,262144,524288,1048576 --reps 3 > $OUT/pads.jsonl 2>&1
timeout 900 python tools/sweep.py --variants 0 --warps 296,444,592,740 --reps 3 > $OUT/warps.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,1 --warps 592,1184 --numrn 33554432 --numiter 500 --reps 3 > $OUT/s25.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,1 --warps 592,1184 --numrn 67108864 --numiter 250 --reps 3 > $OUT/s26.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,1 --warps 592,1184 --numrn 8388608 --numiter 1000 --reps 3 > $OUT/s23.jsonl 2>&1
