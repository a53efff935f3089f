#!/bin/bash
OUT=gpurun_out/exp3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/sweep.py --variants 0,1,2,3,4,7 --warps 444,592,740,888,1036,1184 --reps 4 > $OUT/sweep_warps.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,2,7 --warps 592 --slots 8,16,32,64 --reps 4 > $OUT/sweep_slots.jsonl 2>&1
timeout 300 python tools/sweep.py --variants 2 --warps 592 --numrn 268435456 --numiter 100 --reps 3 > $OUT/sweep_big.jsonl 2>&1
timeout 300 python tools/sweep.py --variants 2 --warps 592 --numrn 1048576 --numiter 1000 --reps 3 > $OUT/sweep_small.jsonl 2>&1
