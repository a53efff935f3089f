#!/bin/bash
OUT=gpurun_out/exp2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/sweep.py --variants 0,1,2,3 --warps 296,592,888,1184,1480,1776 --reps 4 > $OUT/sweep_warps.jsonl 2>&1
timeout 600 python tools/sweep.py --variants 0,1 --warps 0,1184 --slots 16 --pads 0,32,512,4096,65536 --reps 4 > $OUT/sweep_pad.jsonl 2>&1
