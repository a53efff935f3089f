#!/bin/bash
OUT=gpurun_out/exp5; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/sweep.py --variants 8,12,11 --warps 592,1184 --numrn 1048576 --pads 0,512,524288,1048576,3145728,15728640 --reps 3 > $OUT/s20pad.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 8,12,11 --warps 592,1184 --numrn 268435456 --numiter 100 --slots 2,4,8 --reps 3 > $OUT/s28slots.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 8,12,11 --warps 592,1184 --numrn 4194304 --reps 3 > $OUT/s22.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 8,12,11 --warps 592,1184 --numrn 67108864 --numiter 250 --reps 3 > $OUT/s26.jsonl 2>&1
